// CUDA-core fp32 GEMM tile engine used for the strict-parity precision mode
// and for the small layers of the image MLP.  C[M,N] = A[M,K] . B[K,N] with
// operand loaders that gather rows and apply PReLU on the fly, so no gathered
// or activated copy of an operand is ever materialized.
#pragma once
#include "common.cuh"

namespace dicm {
namespace simt {

constexpr int BM = 64, BN = 64, BK = 16, THREADS = 256;

template <typename T>
__device__ __forceinline__ float4 load4(const T* p);
template <>
__device__ __forceinline__ float4 load4<float>(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
template <>
__device__ __forceinline__ float4 load4<__nv_bfloat16>(const __nv_bfloat16* p) {
  const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
  __nv_bfloat162 lo = *reinterpret_cast<const __nv_bfloat162*>(&u.x);
  __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
  float2 a = __bfloat1622float2(lo), b = __bfloat1622float2(hi);
  return make_float4(a.x, a.y, b.x, b.y);
}

// A(m,k) = act(src[row(m)*ld + k]); K-contiguous.  row(m) = idx ? idx[m] : m
template <typename T>
struct LoadA_Rows {
  const T* src;
  int64_t ld;
  const int32_t* idx;
  const float* alpha;  // PReLU prologue on column k (nullptr = none)
  __device__ void operator()(float (*As)[BM + 4], int m0, int k0, int Mr, int Ke) const {
    const int t = threadIdx.x, m = t >> 2, kq = (t & 3) * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const int gm = m0 + m, gk = k0 + kq;
    if (gm < Mr && gk < Ke) {  // K is a multiple of 4 for every caller
      const int64_t r = idx ? (int64_t)idx[gm] : (int64_t)gm;
      v = load4<T>(src + r * ld + gk);
      if (alpha) {
        v.x = prelu(v.x, alpha[gk]);
        v.y = prelu(v.y, alpha[gk + 1]);
        v.z = prelu(v.z, alpha[gk + 2]);
        v.w = prelu(v.w, alpha[gk + 3]);
      }
    }
    As[kq][m] = v.x;
    As[kq + 1][m] = v.y;
    As[kq + 2][m] = v.z;
    As[kq + 3][m] = v.w;
  }
};

// A(m,k) = src[k*ld + m]  (A stored transposed, M-contiguous)
struct LoadA_Cols {
  const float* src;
  int64_t ld;
  __device__ void operator()(float (*As)[BM + 4], int m0, int k0, int Mr, int Ke) const {
    const int t = threadIdx.x, k = t >> 4, mq = (t & 15) * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const int gk = k0 + k, gm = m0 + mq;
    if (gk < Ke && gm < Mr) v = __ldg(reinterpret_cast<const float4*>(src + (int64_t)gk * ld + gm));
    *reinterpret_cast<float4*>(&As[k][mq]) = v;
  }
};

// B(k,n) = W[n*ld + k]  (weights [N,K] row-major, the reference's [out,in])
struct LoadB_WT {
  const float* w;
  int64_t ld;
  __device__ void operator()(float (*Bs)[BN + 4], int k0, int n0, int Ke, int N) const {
    const int t = threadIdx.x, n = t >> 2, kq = (t & 3) * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const int gn = n0 + n, gk = k0 + kq;
    if (gn < N && gk < Ke) v = __ldg(reinterpret_cast<const float4*>(w + (int64_t)gn * ld + gk));
    Bs[kq][n] = v.x;
    Bs[kq + 1][n] = v.y;
    Bs[kq + 2][n] = v.z;
    Bs[kq + 3][n] = v.w;
  }
};

// B(k,n) = act(src[row(k)*ld + n])  (N-contiguous rows, optional gather/PReLU)
template <typename T>
struct LoadB_Rows {
  const T* src;
  int64_t ld;
  const int32_t* idx;
  const float* alpha;
  __device__ void operator()(float (*Bs)[BN + 4], int k0, int n0, int Ke, int N) const {
    const int t = threadIdx.x, k = t >> 4, nq = (t & 15) * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const int gk = k0 + k, gn = n0 + nq;
    if (gk < Ke && gn < N) {
      const int64_t r = idx ? (int64_t)idx[gk] : (int64_t)gk;
      v = load4<T>(src + r * ld + gn);
      if (alpha) {
        v.x = prelu(v.x, alpha[gn]);
        v.y = prelu(v.y, alpha[gn + 1]);
        v.z = prelu(v.z, alpha[gn + 2]);
        v.w = prelu(v.w, alpha[gn + 3]);
      }
    }
    *reinterpret_cast<float4*>(&Bs[k][nq]) = v;
  }
};

// out[m*ld+n] = acc + bias[n]
struct EpBias {
  float* out;
  int64_t ld;
  const float* bias;
  __device__ void operator()(float (&acc)[4][4], int m, int n, int Mr, int N, int split) const {
    for (int i = 0; i < 4; ++i) {
      if (m + i >= Mr) break;
      for (int j = 0; j < 4; ++j)
        if (n + j < N) out[(int64_t)(m + i) * ld + n + j] = acc[i][j] + (bias ? bias[n + j] : 0.f);
    }
  }
};

// out[split][m][n] = acc  (split-K partials, all M x N entries written)
struct EpPartial {
  float* out;
  int M, Nn;
  __device__ void operator()(float (&acc)[4][4], int m, int n, int Mr, int N, int split) const {
    float* base = out + (int64_t)split * M * Nn;
    for (int i = 0; i < 4; ++i) {
      if (m + i >= M) break;
      for (int j = 0; j < 4; ++j)
        if (n + j < N) base[(int64_t)(m + i) * Nn + n + j] = acc[i][j];
    }
  }
};

template <class LA, class LB, class EP>
__global__ void __launch_bounds__(THREADS)
k_gemm(LA la, LB lb, EP ep, int M, int N, int K, const int32_t* Mdev, const int32_t* Kdev, int ksplit) {
  const int Mr = Mdev ? min(M, (int)*Mdev) : M;
  const int Kr = Kdev ? min(K, (int)*Kdev) : K;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= Mr) return;
  const int kchunk = (((Kr + ksplit - 1) / ksplit) + BK - 1) / BK * BK;
  const int kb = blockIdx.z * kchunk;
  const int ke = min(Kr, kb + kchunk);
  __shared__ __align__(16) float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][BN + 4];
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int k0 = kb; k0 < ke; k0 += BK) {
    la(As, m0, k0, Mr, ke);
    lb(Bs, k0, n0, ke, N);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      const float4 a = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  ep(acc, m0 + ty * 4, n0 + tx * 4, Mr, N, blockIdx.z);
}

template <class LA, class LB, class EP>
inline void gemm(cudaStream_t st, LA la, LB lb, EP ep, int M, int N, int K, const int32_t* Mdev,
                 const int32_t* Kdev, int ksplit) {
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, ksplit);
  k_gemm<LA, LB, EP><<<grid, THREADS, 0, st>>>(la, lb, ep, M, N, K, Mdev, Kdev, ksplit);
}

}  // namespace simt
}  // namespace dicm
