// Probe of tcgen05 MN-major operand layouts (one MMA, one CTA).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 scripts/umma_probe.cu -o build/umma_probe
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_bf16.h>
#include "../paper_1711_06505_b200/csrc/tc_ptx.cuh"

using namespace dicm::tc;

// element (mn, k) byte offset inside the operand tile
// mode 0: SW128 16B chunks ^ (k&7), 8-row groups (1024 B)
// mode 1: SW128 32B granules ^ (k&3), 4-row groups (512 B)
// mode 2: 32B granules ^ ((k>>1)&3), 8-row groups (1024 B)
__device__ __host__ inline uint32_t off(int mode, int esz, int mn, int k, int lbo) {
  int epb = 128 / esz;
  int atom = mn / epb, inrow = (mn % epb) * esz;
  uint32_t rowoff = 0;
  if (mode == 0) {
    int c = inrow >> 4, lo = inrow & 15;
    rowoff = (((c ^ (k & 7)) << 4) | lo);
  } else if (mode == 1) {
    int g = inrow >> 5, lo = inrow & 31;
    rowoff = (((g ^ (k & 3)) << 5) | lo);
  } else {
    int g = inrow >> 5, lo = inrow & 31;
    rowoff = (((g ^ ((k >> 1) & 3)) << 5) | lo);
  }
  return atom * lbo + k * 128 + rowoff;
}

template <int KIND>
__global__ void probe(const float* A, const float* B, float* D, int M, int N, int K, int mode, uint32_t layout,
                      uint32_t sbo, int amn, int bmn) {
  __shared__ __align__(1024) uint8_t sa[16384];
  __shared__ __align__(1024) uint8_t sb[16384];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int esz = KIND == 0 ? 4 : 2;
  const int lboA = K * 128, lboB = K * 128;  // atom stride along MN (K rows of 128 B)
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) {
    ((uint32_t*)sa)[i] = 0;
    ((uint32_t*)sb)[i] = 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < M * K; i += blockDim.x) {
    int m = i / K, k = i % K;
    uint32_t o = amn ? off(mode, esz, m, k, lboA) : (uint32_t)(m * 128 + ((((k * esz) >> 4) ^ (m & 7)) << 4) + ((k * esz) & 15));
    if (KIND == 0) *(float*)(sa + o) = A[i]; else *(__nv_bfloat16*)(sa + o) = __float2bfloat16(A[i]);
  }
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    int n = i / K, k = i % K;
    uint32_t o = bmn ? off(mode, esz, n, k, lboB) : (uint32_t)(n * 128 + ((((k * esz) >> 4) ^ (n & 7)) << 4) + ((k * esz) & 15));
    if (KIND == 0) *(float*)(sb + o) = B[i]; else *(__nv_bfloat16*)(sb + o) = __float2bfloat16(B[i]);
  }
  fence_proxy_async();
  __syncthreads();
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc(smem_u32(&slot), 256); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    uint32_t idesc = instr_desc(KIND == 0 ? 2 : 1, M, N, amn, bmn);
    uint64_t ad = amn ? smem_desc(smem_u32(sa), lboA, sbo, layout) : smem_desc(smem_u32(sa), 16, 1024, 2);
    uint64_t bd = bmn ? smem_desc(smem_u32(sb), lboB, sbo, layout) : smem_desc(smem_u32(sb), 16, 1024, 2);
    mma<KIND>(tmem, ad, bd, idesc, 0);
    mma_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  if (warp < 4) {
    for (int cb = 0; cb < N / 32; ++cb) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + cb * 32, v);
      int row = warp * 32 + threadIdx.x % 32;
      if (row < M)
        for (int j = 0; j < 32; ++j) D[row * N + cb * 32 + j] = v[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

int main() {
  const int M = 128, N = 64;
  for (int kind = 0; kind < 2; ++kind) {
    const int K = kind == 0 ? 8 : 16;
    std::vector<float> A(M * K), B(N * K), D(M * N), R(M * N, 0.f);
    srand(1);
    for (auto& x : A) x = (rand() % 17 - 8) / 8.0f;
    for (auto& x : B) x = (rand() % 17 - 8) / 8.0f;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) R[m * N + n] += A[m * K + k] * B[n * K + k];
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    struct V { int mode; uint32_t layout, sbo; int amn, bmn; const char* name; } vs[] = {
        {0, 2, 1024, 0, 0, "K-major control"},
        {0, 2, 1024, 1, 1, "MN SW128 16B, sbo 1024"},
        {1, 1, 512, 1, 1, "MN BASE32B 32B^k&3, sbo 512"},
        {2, 1, 1024, 1, 1, "MN BASE32B 32B^(k>>1)&3, sbo 1024"},
        {1, 1, 1024, 1, 1, "MN BASE32B 32B^k&3, sbo 1024"},
        {1, 2, 512, 1, 1, "MN layout2 32B^k&3 sbo 512"},
        {0, 2, 1024, 1, 0, "A MN SW128 / B K"},
        {1, 1, 512, 1, 0, "A MN BASE32B / B K"},
        {0, 2, 1024, 0, 1, "A K / B MN SW128"},
        {1, 1, 512, 0, 1, "A K / B MN BASE32B"},
    };
    for (auto& v : vs) {
      cudaMemset(dD, 0, D.size() * 4);
      if (kind == 0)
        probe<0><<<1, 128>>>(dA, dB, dD, M, N, K, v.mode, v.layout, v.sbo, v.amn, v.bmn);
      else
        probe<1><<<1, 128>>>(dA, dB, dD, M, N, K, v.mode, v.layout, v.sbo, v.amn, v.bmn);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      double err = 0, nrm = 0;
      for (int i = 0; i < M * N; ++i) { err = fmax(err, fabs(D[i] - R[i])); nrm = fmax(nrm, fabs(R[i])); }
      printf("%s %-36s err %.3g (|ref| %.3g) %s\n", kind == 0 ? "tf32" : "bf16", v.name, err, nrm,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
    }
  }
  return 0;
}
