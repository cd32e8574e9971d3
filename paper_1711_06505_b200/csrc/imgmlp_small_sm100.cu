// Layers 1-2 of the image MLP (256 -> 64 -> 12) and their backward pass on
// tcgen05 tensor cores (kind::tf32), fused with the elementwise work around them.
//
// reference: image_net_apply layers img/1, img/2 (model.py:115-120) and their
// linear / prelu backward closures (autograd.py:201-204, 222-225).
//
// k_l12_fwd  a1 = prelu(a0) W1^T + b1 (MMA M=128,N=64,K=256), then on CUDA
//            cores E = prelu(a1) W2^T + b2 in the TMEM epilogue.
// k_l12_bwd  da1 = prelu'(a1) (dE W2) on CUDA cores straight into the MMA
//            operand layout, dh1 = da1 W1 (MMA M=128,N=256,K=64), then
//            da0 = prelu'(a0) dh1 in the TMEM epilogue; dW2/db2/dalpha1/db1
//            and dalpha0/db0 accumulate per CTA (warp reduce-scatter) into one
//            deterministic partial row per block.
// k_dw1      dW1^T = prelu(a0)^T da1, the reduction over rows: A (h1) staged
//            by registers (PReLU applied on the way), B (da1) by TMA.
#include <cudaTypedefs.h>

#include "imgmlp_sm100.cuh"
#include "epi.cuh"
#include "tc_ptx.cuh"

namespace dicm {
namespace sm100 {
namespace {

using namespace tc;
constexpr int H1 = 256, H2 = 64;
constexpr unsigned FULL = 0xffffffffu;

template <typename T>
__device__ __forceinline__ T* at(uint8_t* raw, uint32_t base_raw, uint32_t saddr) {
  return reinterpret_cast<T*>(raw + (saddr - base_raw));
}

// sum of v[32] over the warp, scattered: lane l ends with sum over lanes of v[l]
__device__ __forceinline__ float reduce_scatter32(float (&v)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float send = upper ? v[i] : v[i + s];
      const float keep = upper ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(FULL, send, s);
    }
  }
  return v[0];
}

// ===========================================================================
// forward layers 1-2, persistent over 128-row tiles
// ===========================================================================
constexpr uint32_t F_A = 128 * 1024;  // a0 -> h1 tile, tf32 K-major SW128 (8 atoms x 16 KB)
constexpr uint32_t F_B = 64 * 1024;   // W1 [64 x 256], K-major SW128 (8 atoms x 8 KB)
constexpr size_t F_SMEM = 1024 + F_A + F_B + 4 * (256 + 64 + 64 + 768 + 16) + 64 + 4 * epi::SCRATCH_FLOATS * 4;

// The a0 tile arrives by TMA (8 boxes of 32 columns x 128 rows, 128-B swizzle
// = the UMMA K-major layout), PReLU is applied in place, the h1 tile is
// written back to HBM by TMA store (the dW1 kernel consumes it) and multiplied
// by W1; the next tile's TMA load is issued as soon as the MMA has read A, so
// it overlaps the TMEM epilogue.
__global__ void __launch_bounds__(256, 1)
    k_l12_fwd(const __grid_constant__ CUtensorMap tmA0, float* __restrict__ h1, int64_t rows_max,
              const float* __restrict__ al0, const float* __restrict__ w1, const float* __restrict__ b1,
              const float* __restrict__ al1, const float* __restrict__ w2, const float* __restrict__ b2,
              const int32_t* __restrict__ count, float* __restrict__ act1, float* __restrict__ emb) {
  const int U = *count;
  const int ntiles = (U + 127) / 128;
  if ((int)blockIdx.x >= ntiles) return;
  extern __shared__ uint8_t raw[];
  const uint32_t r0 = smem_u32(raw), base = (r0 + 1023u) & ~1023u;
  const uint32_t A = base, B = base + F_A;
  float* sal0 = at<float>(raw, r0, B + F_B);
  float* sb1 = sal0 + 256;
  float* sal1 = sb1 + 64;
  float* sw2 = sal1 + 64;
  float* sb2 = sw2 + 768;
  const uint32_t bar = B + F_B + 4 * (256 + 64 + 64 + 768 + 16);
  const uint32_t fullA = bar + 8;
  const uint32_t slot = fullA + 8;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (t == 0) {
    mbar_init(bar, 1);
    mbar_init(fullA, 1);
    fence_mbar_init();
    prefetch_tmap(&tmA0);
  }
  // W1 -> K-major SW128: row n (64), 16-B chunk q of k
  for (int i = t; i < 64 * 64; i += 256) {
    const int n = i >> 6, q = i & 63, j = q >> 3, c = q & 7;
    *at<float4>(raw, r0, B + j * 8192 + n * 128 + ((c ^ (n & 7)) << 4)) = __ldg(reinterpret_cast<const float4*>(w1) + i);
  }
  sal0[t] = al0[t];
  if (t < 64) {
    sb1[t] = b1[t];
    sal1[t] = al1[t];
  }
  for (int i = t; i < 768; i += 256) sw2[i] = w2[i];
  if (t < 12) sb2[t] = b2[t];
  if (warp == 0) {
    tmem_alloc(slot, 64);
    tmem_relinquish();
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *at<volatile uint32_t>(raw, r0, slot);
  const uint32_t idesc = instr_desc(2, 128, 64, 0, 0);
  if (t == 0) {
    mbar_arrive_expect_tx(fullA, F_A);
    for (int j = 0; j < 8; ++j) tma_load_2d(A + j * 16384, &tmA0, fullA, j * 32, blockIdx.x * 128);
  }
  uint32_t it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int m0 = tile * 128;
    mbar_wait(fullA, it & 1);
    // h1 = prelu(a0) in place (each 16-B chunk keeps its swizzled slot)
#pragma unroll 8
    for (int i = t; i < 128 * 64; i += 256) {
      const int r = i >> 6, q = i & 63, j = q >> 3, c = q & 7;
      float4* p = at<float4>(raw, r0, A + j * 16384 + r * 128 + ((c ^ (r & 7)) << 4));
      float4 v = *p;
      v.x = prelu(v.x, sal0[4 * q]);
      v.y = prelu(v.y, sal0[4 * q + 1]);
      v.z = prelu(v.z, sal0[4 * q + 2]);
      v.w = prelu(v.w, sal0[4 * q + 3]);
      *p = v;
      // h1 -> HBM (consumed by the dW1 reduction); coalesced along the row
      if (m0 + r < rows_max) reinterpret_cast<float4*>(h1 + (int64_t)(m0 + r) * H1)[q] = v;
    }
    fence_proxy_async();
    __syncthreads();
    if (t == 0) {
      tc_fence_after();
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int j = k >> 2, kk = k & 3;
        mma<0>(tmem, smem_desc(A + j * 16384 + kk * 32, 16, 1024), smem_desc(B + j * 8192 + kk * 32, 16, 1024), idesc,
               k > 0);
      }
      mma_commit(bar);
    }
    mbar_wait(bar, it & 1);
    tc_fence_after();
    if (t == 0) {
      // A may be refilled once the MMA has read it
      const int next = tile + gridDim.x;
      if (next < ntiles) {
        mbar_arrive_expect_tx(fullA, F_A);
        for (int j = 0; j < 8; ++j) tma_load_2d(A + j * 16384, &tmA0, fullA, j * 32, next * 128);
      }
    }
    if (warp < 4) {
      float a[64];
      tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), *reinterpret_cast<float(*)[32]>(a));
      tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + 32, *reinterpret_cast<float(*)[32]>(a + 32));
      const int row = m0 + warp * 32 + lane;
#pragma unroll
      for (int i = 0; i < 64; ++i) a[i] += sb1[i];
      float* scr = at<float>(raw, r0, slot + 16) + warp * epi::SCRATCH_FLOATS;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
        epi::store_f32(*reinterpret_cast<float(*)[32]>(a + 32 * hh), scr, lane, m0 + warp * 32, U,
                       [&](int r) { return act1 + (int64_t)r * H2 + 32 * hh; });
      if (row < U) {
        float e[12];
#pragma unroll
        for (int c = 0; c < 12; ++c) e[c] = sb2[c];
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          const float h = prelu(a[i], sal1[i]);
#pragma unroll
          for (int c = 0; c < 12; ++c) e[c] = fmaf(sw2[c * 64 + i], h, e[c]);
        }
        float4* eo = reinterpret_cast<float4*>(emb + (int64_t)row * 12);
        eo[0] = make_float4(e[0], e[1], e[2], e[3]);
        eo[1] = make_float4(e[4], e[5], e[6], e[7]);
        eo[2] = make_float4(e[8], e[9], e[10], e[11]);
      }
    }
    tc_fence_before();
    __syncthreads();
  }
  if (warp == 0) tmem_dealloc(tmem, 64);
}

// ===========================================================================
// backward layers 2-1 (dE -> da1 -> dh1 -> da0), persistent over 128-row tiles
// ===========================================================================
constexpr uint32_t G_A = 32 * 1024;  // da1 tile, K-major SW128 (2 atoms x 16 KB)
constexpr uint32_t G_B = 64 * 1024;  // W1 as MN-major (n x k) SWIZZLE_128B_BASE32B: 8 atoms x 64 k x 128 B
constexpr int PART_L2 = 12 * 64 + 12 + 64 + 64;  // w2 | b2 | a1 | b1
constexpr int PART_B = PART_L2 + 256 + 256;      // ... | a0 | b0
constexpr size_t G_SMEM = 1024 + G_A + G_B + 4 * (128 * 12 + 256 + 64 + 768) + 64 + 8 * epi::SCRATCH_FLOATS * 4;

__global__ void __launch_bounds__(256, 1)
    k_l12_bwd(const float* __restrict__ demb, const float* __restrict__ act1, const float* __restrict__ act0,
              const float* __restrict__ al0, const float* __restrict__ al1, const float* __restrict__ w1,
              const float* __restrict__ w2, const int32_t* __restrict__ count, int64_t rows_max,
              float* __restrict__ da1_out,
              float* __restrict__ da0_out, __nv_bfloat16* __restrict__ da0_bf16, float* __restrict__ part) {
  const int U = *count;
  const int ntiles = (U + 127) / 128;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  float* prow = part + (int64_t)blockIdx.x * PART_B;
  if ((int)blockIdx.x >= ntiles) {
    for (int i = t; i < PART_B; i += 256) prow[i] = 0.f;
    return;
  }
  extern __shared__ uint8_t raw[];
  const uint32_t r0 = smem_u32(raw), base = (r0 + 1023u) & ~1023u;
  const uint32_t A = base, B = base + G_A;
  float* sdE = at<float>(raw, r0, B + G_B);  // [128][12]
  float* sal0 = sdE + 128 * 12;
  float* sal1 = sal0 + 256;
  float* sw2 = sal1 + 64;
  const uint32_t bar = B + G_B + 4 * (128 * 12 + 256 + 64 + 768);
  const uint32_t slot = bar + 8;
  float* scr = at<float>(raw, r0, bar + 64) + (threadIdx.x >> 5) * epi::SCRATCH_FLOATS;
  // W1 [k=64][n=256] -> MN-major BASE32B: atom n/32, row k, 32-B granule ^ (k & 3)
  for (int i = t; i < 64 * 64; i += 256) {
    const int k = i >> 6, q = i & 63;  // float4 q covers n = 4q .. 4q+3
    const int atom = q >> 3, g = (q & 7) >> 1, lo = (q & 1) << 4;
    *at<float4>(raw, r0, B + atom * 8192 + k * 128 + ((g ^ (k & 3)) << 5) + lo) =
        __ldg(reinterpret_cast<const float4*>(w1) + i);
  }
  for (int i = t; i < 256; i += 256) sal0[i] = al0[i];
  if (t < 64) sal1[t] = al1[t];
  for (int i = t; i < 768; i += 256) sw2[i] = w2[i];
  if (t == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(slot, 256);
    tmem_relinquish();
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *at<volatile uint32_t>(raw, r0, slot);
  const uint32_t idesc = instr_desc(2, 128, 256, 0, 1);
  // column-phase accumulators (thread = (row group g, column j))
  const int j = t & 63, grp = t >> 6;
  float w2col[12], accw[12];
#pragma unroll
  for (int c = 0; c < 12; ++c) {
    w2col[c] = sw2[c * 64 + j];
    accw[c] = 0.f;
  }
  const float alj = sal1[j];
  float acc_b2 = 0.f, acc_a1 = 0.f, acc_b1 = 0.f;
  // epilogue accumulators: warp covers lane quarter q, column blocks cb0..cb0+3
  const int q = warp & 3, cb0 = (warp >> 2) * 4;
  float acc_a0[4] = {0.f, 0.f, 0.f, 0.f}, acc_b0[4] = {0.f, 0.f, 0.f, 0.f};
  uint32_t it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int m0 = tile * 128;
    for (int i = t; i < 128 * 12; i += 256) {
      const int gr = m0 + i / 12;
      sdE[i] = gr < U ? __ldg(demb + (int64_t)m0 * 12 + i) : 0.f;
    }
    __syncthreads();
    // da1 = prelu'(a1) (dE W2)  -> global + operand A (K-major SW128)
    float apre[32];  // all of this thread's act1 values in flight at once
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int gr = m0 + grp + 4 * i;
      apre[i] = gr < U ? __ldg(act1 + (int64_t)gr * H2 + j) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int r = grp + 4 * i, gr = m0 + r;
      const float* d = sdE + r * 12;
      float dh = 0.f;
#pragma unroll
      for (int c = 0; c < 12; ++c) dh = fmaf(d[c], w2col[c], dh);
      const float a = apre[i];
      const float dd = a > 0.f ? dh : alj * dh;
      // rows past the count get 0: the dW1 reduction reads whole 32-row stages
      if (gr < rows_max) da1_out[(int64_t)gr * H2 + j] = dd;
      if (!(a > 0.f)) acc_a1 = fmaf(a, dh, acc_a1);
      acc_b1 += dd;
      const float h = prelu(a, alj);
#pragma unroll
      for (int c = 0; c < 12; ++c) accw[c] = fmaf(d[c], h, accw[c]);
      if (j < 12) acc_b2 += d[j];
      *at<float>(raw, r0, A + (j >> 5) * 16384 + r * 128 + ((((j & 31) >> 2) ^ (r & 7)) << 4) + (j & 3) * 4) = dd;
    }
    fence_proxy_async();
    __syncthreads();
    if (t == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        mma<0>(tmem, smem_desc(A + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
               smem_desc(B + kk * 1024, 8192, 512, 1), idesc, kk > 0);
      mma_commit(bar);
    }
    mbar_wait(bar, it & 1);
    tc_fence_after();
    {
      const int row = m0 + q * 32 + lane;
      const bool ok = row < U;
      const float4* arow = reinterpret_cast<const float4*>(act0 + (int64_t)(ok ? row : 0) * H1 + cb0 * 32);
      float4 anext[8];  // a0 of the next column block in flight while this one computes
#pragma unroll
      for (int v = 0; v < 8; ++v) anext[v] = ok ? __ldg(arow + v) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int cb = cb0 + cc;
        float4 acur[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) acur[v] = anext[v];
        if (cc < 3) {
#pragma unroll
          for (int v = 0; v < 8; ++v) anext[v] = ok ? __ldg(arow + (cc + 1) * 8 + v) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float dh[32], sa[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + cb * 32, dh);
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const float av[4] = {acur[v].x, acur[v].y, acur[v].z, acur[v].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = 4 * v + e;
            const float x = av[e], g = dh[i];
            const bool pos = x > 0.f;
            dh[i] = pos ? g : sal0[cb * 32 + i] * g;
            sa[i] = pos ? 0.f : x * g;
          }
        }
        // coalesced row stores through the warp's scratch; the bf16 path
        // (kind::f16 dW0) needs only the bf16 copy, the tf32 path the fp32 one
        if (da0_bf16)
          epi::store_bf16(dh, scr, lane, m0 + q * 32, U,
                          [&](int r) { return da0_bf16 + (int64_t)r * H1 + cb * 32; });
        else
          epi::store_f32(dh, scr, lane, m0 + q * 32, U, [&](int r) { return da0_out + (int64_t)r * H1 + cb * 32; });
        acc_b0[cc] += reduce_scatter32(dh, lane);
        acc_a0[cc] += reduce_scatter32(sa, lane);
      }
    }
    tc_fence_before();
    __syncthreads();
  }
  // ---- deterministic block partial: combine the 4 row groups / 4 quarters
  float* red = at<float>(raw, r0, A);  // reuse the operand tiles (>= 4 x 1420 floats)
#pragma unroll
  for (int c = 0; c < 12; ++c) red[grp * PART_B + c * 64 + j] = accw[c];
  if (j < 12) red[grp * PART_B + 768 + j] = acc_b2;
  red[grp * PART_B + 780 + j] = acc_a1;
  red[grp * PART_B + 844 + j] = acc_b1;
#pragma unroll
  for (int cc = 0; cc < 4; ++cc) {
    red[q * PART_B + PART_L2 + (cb0 + cc) * 32 + lane] = acc_a0[cc];
    red[q * PART_B + PART_L2 + 256 + (cb0 + cc) * 32 + lane] = acc_b0[cc];
  }
  __syncthreads();
  for (int i = t; i < PART_B; i += 256) {
    float s = 0.f;
#pragma unroll
    for (int g = 0; g < 4; ++g) s += red[g * PART_B + i];
    prow[i] = s;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

// ===========================================================================
// dW1^T [256 x 64] = prelu(a0)^T da1 over rows, split over CTAs
// ===========================================================================
constexpr int W_STAGES = 4;
constexpr uint32_t W_A = 32 * 1024;  // h1^T: 2 halves x 4 atoms x 32 rows x 128 B (BASE32B)
constexpr uint32_t W_B = 8 * 1024;   // da1:  2 atoms x 32 rows x 128 B (BASE32B)
constexpr uint32_t W_STAGE = W_A + W_B;
constexpr size_t W_SMEM = 1024 + W_STAGES * W_STAGE + 256;

// Both operands are MN-major tiles loaded by TMA with the 32-B-atom 128-B
// swizzle (tf32 MN-major): h1 (written by k_l12_fwd) and da1 (k_l12_bwd).
// Rows past the live count are zero in da1, so partial stages add nothing.
__global__ void __launch_bounds__(192, 1)
    k_dw1(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmD,
          const int32_t* __restrict__ count, float* __restrict__ part /*[grid][64*256]*/) {
  const int U = *count;
  const int per = (((U + gridDim.x - 1) / gridDim.x) + 31) / 32 * 32;
  const int rb = blockIdx.x * per, re = min(U, rb + per);
  const int nk = re > rb ? (re - rb + 31) / 32 : 0;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  float* out = part + (int64_t)blockIdx.x * 64 * 256;
  if (nk == 0) {
    for (int i = t; i < 64 * 256; i += 192) out[i] = 0.f;
    return;
  }
  extern __shared__ uint8_t raw[];
  const uint32_t r0 = smem_u32(raw), base = (r0 + 1023u) & ~1023u;
  const uint32_t full = base + W_STAGES * W_STAGE, empty = full + 8 * W_STAGES, accb = empty + 8 * W_STAGES,
                 slot = accb + 8;
  if (t == 0) {
    for (int i = 0; i < W_STAGES; ++i) {
      mbar_init(full + 8 * i, 1);
      mbar_init(empty + 8 * i, 1);
    }
    mbar_init(accb, 1);
    fence_mbar_init();
  }
  if (warp == 4) {
    tmem_alloc(slot, 128);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *at<volatile uint32_t>(raw, r0, slot);
  if (warp == 5) {
    if (lane == 0) {
      prefetch_tmap(&tmH);
      prefetch_tmap(&tmD);
      for (int kb = 0; kb < nk; ++kb) {
        const uint32_t st = kb % W_STAGES, itn = kb / W_STAGES;
        mbar_wait(empty + 8 * st, (itn & 1) ^ 1);
        mbar_arrive_expect_tx(full + 8 * st, W_STAGE);
        const uint32_t a = base + st * W_STAGE, b = a + W_A;
        const int row = rb + kb * 32;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int at4 = 0; at4 < 4; ++at4)
            tma_load_2d(a + h * 16384 + at4 * 4096, &tmH, full + 8 * st, h * 128 + at4 * 32, row);
        tma_load_2d(b, &tmD, full + 8 * st, 0, row);
        tma_load_2d(b + 4096, &tmD, full + 8 * st, 32, row);
      }
    }
  } else if (warp == 4) {
    if (lane == 0) {
      const uint32_t idesc = instr_desc(2, 128, 64, 1, 1);
      for (int kb = 0; kb < nk; ++kb) {
        const uint32_t st = kb % W_STAGES, itn = kb / W_STAGES;
        mbar_wait(full + 8 * st, itn & 1);
        tc_fence_after();
        const uint32_t a = base + st * W_STAGE, b = a + W_A;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma<0>(tmem + h * 64, smem_desc(a + h * 16384 + kk * 1024, 4096, 512, 1),
                   smem_desc(b + kk * 1024, 4096, 512, 1), idesc, (kb | kk) != 0);
        mma_commit(empty + 8 * st);
      }
      mma_commit(accb);
    }
  } else {
    mbar_wait(accb, 0);
    tc_fence_after();
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const int feat = h * 128 + warp * 32 + lane;
#pragma unroll 1
      for (int cb = 0; cb < 2; ++cb) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + h * 64 + cb * 32, v);
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) out[(cb * 32 + jj) * 256 + feat] = v[jj];  // dW1[j][feature]
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) tmem_dealloc(tmem, 128);
}


PFN_cuTensorMapEncodeTiled_v12000 encode_fn2() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

template <typename K>
int smem_attr(K kernel, size_t bytes) {
  return check_cuda(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes),
                    "small-layer tcgen05 smem attribute");
}

}  // namespace

int small_part_size() { return PART_B; }
int small_dw1_blocks(int64_t rows_max) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(dicm_grid_cap(), (rows_max + 255) / 256));
}
int small_bwd_blocks(int64_t rows_max) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(dicm_grid_cap(), (rows_max + 127) / 128));
}

// row-major fp32 [rows, cols] map with box {32 cols, box_rows}
int map_f32(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows, CUtensorMapSwizzle swz) {
  auto fn = encode_fn2();
  if (!fn) return fail(DICM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 4};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DICM_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return DICM_OK;
}

int fwd_layers12(const float* act0, const int32_t* count, int64_t rows_max, const float* al0, const float* w1,
                 const float* b1, const float* al1, const float* w2, const float* b2, float* act1, float* emb,
                 float* h1, cudaStream_t st) {
  static int once = smem_attr(k_l12_fwd, F_SMEM);
  if (once) return once;
  CUtensorMap ma;
  int rc = map_f32(&ma, act0, rows_max, H1, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(dicm_grid_cap(), (rows_max + 127) / 128));
  {
    const int probe_slot = probe_begin(DICM_PROBE_IMG_FWD_L12, st);
    k_l12_fwd<<<grid, 256, F_SMEM, st>>>(ma, h1, rows_max, al0, w1, b1, al1, w2, b2, count, act1, emb);
    probe_end(probe_slot, st);
  }
  return last_launch("tcgen05 layers 1-2 forward");
}

int bwd_layers12(const float* demb, const float* act1, const float* act0, const float* h1, const int32_t* count,
                 int64_t rows_max, const float* al0, const float* al1, const float* w1, const float* w2, float* da1,
                 float* da0, __nv_bfloat16* da0_bf16, float* part_l12, float* part_dw1, cudaStream_t st) {
  static int once = smem_attr(k_l12_bwd, G_SMEM);
  if (once) return once;
  static int once2 = smem_attr(k_dw1, W_SMEM);
  if (once2) return once2;
  {
    const int probe_slot = probe_begin(DICM_PROBE_IMG_BWD_L12, st);
    k_l12_bwd<<<small_bwd_blocks(rows_max), 256, G_SMEM, st>>>(demb, act1, act0, al0, al1, w1, w2, count, rows_max,
                                                             da1, da0, da0_bf16, part_l12);
    probe_end(probe_slot, st);
  }
  int rc = last_launch("tcgen05 layers 2-1 backward");
  if (rc) return rc;
  CUtensorMap mh, md;
  rc = map_f32(&mh, h1, rows_max, H1, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (!rc) rc = map_f32(&md, da1, rows_max, H2, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (rc) return rc;
  {
    const int probe_slot = probe_begin(DICM_PROBE_IMG_BWD_DW1, st);
    k_dw1<<<small_dw1_blocks(rows_max), 192, W_SMEM, st>>>(mh, md, count, part_dw1);
    probe_end(probe_slot, st);
  }
  return last_launch("tcgen05 dW1");
}

}  // namespace sm100
}  // namespace dicm
