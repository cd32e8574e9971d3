// Layers 1-2 of the image MLP in the bf16 precision mode (kind::f16 tcgen05),
// built around TMA-staged, double-buffered 128-row tiles.
//
// reference: image_net_apply layers img/1, img/2 (model.py:115-120) and their
// linear / prelu backward closures (autograd.py:201-204, 222-225).
//
// In bf16 mode the activations saved for the backward pass are bf16: the
// layer-0 kernel writes act0 [U,256] as bf16 and k_l12f writes act1 [U,64] as
// bf16, which halves the HBM traffic of every kernel here.  Arithmetic stays
// fp32 (fp32 TMEM accumulation, fp32 CUDA-core epilogues); the only roundings
// are the bf16 operands of the two layer-1 GEMMs and the saved activations,
// inside the north star's 2e-2 bf16 tolerance (tests/test_gpu_tensorcore.py).
//
// k_l12f   h1 = prelu(a0) (in place in smem), a1 = h1 W1^T + b1 on tcgen05
//          (M128 N64 K256, double-buffered TMEM), then E = prelu(a1) W2^T + b2
//          on CUDA cores.  Warp roles: TMA | MMA | 4 PReLU | 4 epilogue.
// k_l12b   da1 = prelu'(a1) (dE W2) on CUDA cores -> smem (the MMA A operand
//          and the TMA-stored da1), dh1 = da1 W1 (M128 N256 K64), then
//          da0 = prelu'(a0) dh1 written in place over the staged a0 tile and
//          TMA-stored; dW2/db2/dalpha1/db1 per-CTA partials (deterministic).  A producer warp keeps the next tile's a0/a1/dE
//          in flight while the current one is computed.
// k_dw1b   three GEMMs over rows, max(a0,0)^T da1, min(a0,0)^T da1 and
//          [a0<=0]^T da1 (M128x2 N64 each, K = rows); dW1, dalpha0 and db0
//          follow exactly from them (k_l1_finish), so no kernel reduces
//          columns across lanes.
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
typedef __nv_bfloat16 bf16;

template <typename T>
__device__ __forceinline__ T* at(uint8_t* raw, uint32_t base_raw, uint32_t saddr) {
  return reinterpret_cast<T*>(raw + (saddr - base_raw));
}

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ float2 bf2_to_f2(uint32_t u) {
  return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u));
}
__device__ __forceinline__ uint32_t f2_to_bf2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// lane l ends with the sum over lanes of v[l]
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

// PReLU of 8 bf16 values (one 16-B chunk) with per-column slopes al[0..7];
// rows with !valid become zero
__device__ __forceinline__ uint4 prelu_chunk(uint4 v, const float (&al)[8], bool valid) {
  uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const float2 f = bf2_to_f2(w[p]);
    w[p] = valid ? f2_to_bf2(prelu(f.x, al[2 * p]), prelu(f.y, al[2 * p + 1])) : 0u;
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// ===========================================================================
// k_l12f: forward layers 1-2
// ===========================================================================
constexpr uint32_t FT = 64 * 1024;  // a0 tile: 4 boxes x 128 rows x 128 B (bf16, SW128)
constexpr uint32_t FW = 32 * 1024;  // W1 [64 x 256] bf16 K-major SW128: 4 atoms x 64 rows x 128 B
constexpr int FPAR = 256 + 64 + 64 + 768 + 16;  // al0 | b1 | al1 | w2 | b2
constexpr int F_THREADS = 320;  // w0 TMA | w1 MMA | w2-5 PReLU | w6-9 epilogue
constexpr size_t F_SMEM = 1024 + 2 * FT + FW + 4 * FPAR + 128 + 4 * epi::SCRATCH_FLOATS * 4;

__global__ void __launch_bounds__(F_THREADS, 1)
    k_l12f(const __grid_constant__ CUtensorMap tmA0, const float* __restrict__ al0, const float* __restrict__ w1,
           const float* __restrict__ b1, const float* __restrict__ al1, const float* __restrict__ w2,
           const float* __restrict__ b2, const int32_t* __restrict__ count, bf16* __restrict__ act1,
           float* __restrict__ emb, int reverse) {
  const int U = *count;
  const int ntiles = (U + 127) / 128;
  if ((int)blockIdx.x >= ntiles) return;
  // reverse: the tiles the layer-0 forward wrote last (still in L2) first
  auto row_of = [&](int tile) { return (reverse ? ntiles - 1 - tile : tile) * 128; };
  extern __shared__ uint8_t raw[];
  const uint32_t r0 = smem_u32(raw), base = (r0 + 1023u) & ~1023u;
  const uint32_t W = base + 2 * FT;
  float* sal0 = at<float>(raw, r0, W + FW);
  float* sb1 = sal0 + 256;
  float* sal1 = sb1 + 64;
  float* sw2 = sal1 + 64;
  float* sb2 = sw2 + 768;
  const uint32_t bars = W + FW + 4 * FPAR;
  const uint32_t full = bars, ready = bars + 16, empty = bars + 32, accf = bars + 48, acce = bars + 64,
                 slot = bars + 80;
  float* scr_base = at<float>(raw, r0, bars + 128);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (t == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(full + 8 * i, 1);
      mbar_init(ready + 8 * i, 128);
      mbar_init(empty + 8 * i, 1);
      mbar_init(accf + 8 * i, 1);
      mbar_init(acce + 8 * i, 128);
    }
    fence_mbar_init();
  }
  // W1 [n=64][k=256] fp32 -> bf16 K-major SW128: atom k/64, row n, 16-B chunk (k%64)/8 ^ (n&7)
  for (int i = t; i < 64 * 32; i += F_THREADS) {
    const int n = i >> 5, q = i & 31, j = q >> 3, c = q & 7;
    const float4 a = __ldg(reinterpret_cast<const float4*>(w1 + n * H1 + q * 8));
    const float4 b = __ldg(reinterpret_cast<const float4*>(w1 + n * H1 + q * 8 + 4));
    *at<uint4>(raw, r0, W + j * 8192 + n * 128 + ((c ^ (n & 7)) << 4)) =
        make_uint4(f2_to_bf2(a.x, a.y), f2_to_bf2(a.z, a.w), f2_to_bf2(b.x, b.y), f2_to_bf2(b.z, b.w));
  }
  for (int i = t; i < 256; i += F_THREADS) sal0[i] = al0[i];
  if (t < 64) {
    sb1[t] = b1[t];
    sal1[t] = al1[t];
  }
  // W2 [12][64] transposed to [64][12]: one hidden unit's 12 weights are
  // three 16-B shared loads feeding six paired FMAs
  for (int i = t; i < 768; i += F_THREADS) sw2[(i & 63) * 12 + (i >> 6)] = w2[i];
  if (t < 12) sb2[t] = b2[t];
  if (warp == 1) {
    tmem_alloc(slot, 128);
    tmem_relinquish();
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *at<volatile uint32_t>(raw, r0, slot);

  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&tmA0);
      uint32_t it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const uint32_t s = it & 1, ph = (it >> 1) & 1;
        mbar_wait(empty + 8 * s, ph ^ 1);
        mbar_arrive_expect_tx(full + 8 * s, FT);
#pragma unroll
        for (int j = 0; j < 4; ++j) tma_load_2d(base + s * FT + j * 16384, &tmA0, full + 8 * s, j * 64, row_of(tile));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = instr_desc(1, 128, 64, 0, 0);
      uint32_t it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const uint32_t s = it & 1, ph = (it >> 1) & 1;
        mbar_wait(acce + 8 * s, ph ^ 1);
        mbar_wait(ready + 8 * s, ph);
        tc_fence_after();
        const uint32_t A = base + s * FT;
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
          const int j = kk >> 2, k4 = kk & 3;
          mma<1>(tmem + s * 64, smem_desc(A + j * 16384 + k4 * 32, 16, 1024), smem_desc(W + j * 8192 + k4 * 32, 16, 1024),
                 idesc, kk > 0);
        }
        mma_commit(empty + 8 * s);
        mma_commit(accf + 8 * s);
      }
    }
  } else if (warp < 6) {
    // ---- PReLU in place: thread owns physical chunk c of rows (tid>>3) + 16 i
    // of every box; its logical column chunk (c ^ (row & 7)) is fixed
    const int tid = t - 64, c = tid & 7, rlo = tid >> 3, lc = c ^ (rlo & 7);
    float al[4][8];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 8; ++e) al[j][e] = sal0[j * 64 + lc * 8 + e];
    uint32_t it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const uint32_t s = it & 1, ph = (it >> 1) & 1;
      mbar_wait(full + 8 * s, ph);
      const uint32_t A = base + s * FT;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll 4
        for (int i = 0; i < 8; ++i) {
          const int r = rlo + 16 * i;
          uint4* p = at<uint4>(raw, r0, A + j * 16384 + r * 128 + (c << 4));
          *p = prelu_chunk(*p, al[j], true);
        }
      fence_proxy_async();
      mbar_arrive(ready + 8 * s);
    }
  } else {
    // ---- epilogue: TMEM lane quarter q = warp % 4
    const int q = warp & 3;
    float* scr = scr_base + q * epi::SCRATCH_FLOATS;
    uint32_t it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const uint32_t s = it & 1, ph = (it >> 1) & 1;
      const int m0 = row_of(tile);
      mbar_wait(accf + 8 * s, ph);
      tc_fence_after();
      const int row = m0 + q * 32 + lane;
      float e[12];
#pragma unroll
      for (int c = 0; c < 12; ++c) e[c] = sb2[c];
#pragma unroll 1
      for (int hh = 0; hh < 2; ++hh) {
        float a[32];
        tmem_ld32(tmem + s * 64 + ((uint32_t)(q * 32) << 16) + 32 * hh, a);
        if (hh == 1) {
          tc_fence_before();
          mbar_arrive(acce + 8 * s);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) a[i] += sb1[32 * hh + i];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float h = prelu(a[i], sal1[32 * hh + i]);
          const float4* wv = reinterpret_cast<const float4*>(sw2 + (32 * hh + i) * 12);
          const float4 w0 = wv[0], w1 = wv[1], w2v = wv[2];
          ffma2(e[0], e[1], w0.x, w0.y, h);
          ffma2(e[2], e[3], w0.z, w0.w, h);
          ffma2(e[4], e[5], w1.x, w1.y, h);
          ffma2(e[6], e[7], w1.z, w1.w, h);
          ffma2(e[8], e[9], w2v.x, w2v.y, h);
          ffma2(e[10], e[11], w2v.z, w2v.w, h);
        }
        epi::store_bf16(a, scr, lane, m0 + q * 32, U, [&](int r) { return act1 + (int64_t)r * H2 + 32 * hh; });
      }
      if (row < U) {
        float4* eo = reinterpret_cast<float4*>(emb + (int64_t)row * 12);
        eo[0] = make_float4(e[0], e[1], e[2], e[3]);
        eo[1] = make_float4(e[4], e[5], e[6], e[7]);
        eo[2] = make_float4(e[8], e[9], e[10], e[11]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 128);
}

// ===========================================================================
// k_l12b: backward layers 2 -> 1
// ===========================================================================
constexpr uint32_t BT0 = 64 * 1024;                 // a0 tile (bf16, 4 SW128 boxes); da0 in place
constexpr uint32_t BT1 = 16 * 1024;                 // a1 tile (bf16, one SW128 box)
constexpr uint32_t BTE = 128 * 12 * 4;              // dE tile (fp32, no swizzle)
constexpr uint32_t BSTG = BT0 + BT1 + 7 * 1024;     // 88 KB stage (dE padded to 7 KB)
constexpr uint32_t BW = 32 * 1024;                  // W1^T [n=256][k=64] bf16 K-major SW128
constexpr uint32_t BA = 16 * 1024;                  // da1 tile (bf16 SW128): MMA A + TMA-store source
constexpr int PART_L2 = 12 * 64 + 12 + 64 + 64;     // w2 | b2 | a1 | b1
constexpr int PART_B = PART_L2 + 256 + 256;         // ... | a0 | b0 (zero here: k_dw1b)
constexpr size_t B_SMEM = 1024 + 2 * BSTG + BW + BA + 4 * (256 + 64) + 128;
constexpr int B_THREADS = 288;  // w0-7 compute, w8 TMA producer / storer
static_assert(B_SMEM <= 232448, "k_l12b shared memory");
static_assert(8 * PART_L2 * 4 <= 2 * BSTG, "k_l12b reduction scratch");

__global__ void __launch_bounds__(B_THREADS, 1)
    k_l12b(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
           const __grid_constant__ CUtensorMap tmE, const __grid_constant__ CUtensorMap tmD1,
           const __grid_constant__ CUtensorMap tmD0, const float* __restrict__ al0, const float* __restrict__ al1,
           const float* __restrict__ w1, const float* __restrict__ w2, const int32_t* __restrict__ count,
           float* __restrict__ part) {
  const int U = *count;
  const int ntiles = (U + 127) / 128;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  float* prow = part + (int64_t)blockIdx.x * PART_B;
  if ((int)blockIdx.x >= ntiles) {
    for (int i = t; i < PART_B; i += B_THREADS) prow[i] = 0.f;
    return;
  }
  extern __shared__ uint8_t raw[];
  const uint32_t r0 = smem_u32(raw), base = (r0 + 1023u) & ~1023u;
  const uint32_t W = base + 2 * BSTG, A = W + BW;
  float* sal0 = at<float>(raw, r0, A + BA);
  float* sal1 = sal0 + 256;
  const uint32_t bars = A + BA + 4 * (256 + 64);
  const uint32_t full = bars, empty = bars + 16, done = bars + 32, mbar = bars + 48, slot = bars + 56;
  if (t == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(full + 8 * i, 1);
      mbar_init(empty + 8 * i, 1);
      mbar_init(done + 8 * i, 256);
    }
    mbar_init(mbar, 1);
    fence_mbar_init();
  }
  // W1^T: B[n][k] = W1[k][n] (n = 256 hidden-0 units, k = 64), bf16 K-major SW128
  for (int i = t; i < 256 * 8; i += B_THREADS) {
    const int n = i >> 3, c = i & 7;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = __ldg(w1 + (c * 8 + e) * H1 + n);
    *at<uint4>(raw, r0, W + n * 128 + ((c ^ (n & 7)) << 4)) =
        make_uint4(f2_to_bf2(v[0], v[1]), f2_to_bf2(v[2], v[3]), f2_to_bf2(v[4], v[5]), f2_to_bf2(v[6], v[7]));
  }
  for (int i = t; i < 256; i += B_THREADS) sal0[i] = al0[i];
  if (t < 64) sal1[t] = al1[t];
  if (warp == 0) {
    tmem_alloc(slot, 256);
    tmem_relinquish();
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *at<volatile uint32_t>(raw, r0, slot);

  if (warp == 8) {
    // ---- producer: loads tile it into stage it&1 once the da0 of tile it-2
    // (written in place there) has been stored
    if (lane == 0) {
      prefetch_tmap(&tmA0);
      prefetch_tmap(&tmA1);
      prefetch_tmap(&tmE);
      prefetch_tmap(&tmD0);
      uint32_t it = 0;
      int prev[2] = {-1, -1};
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const uint32_t s = it & 1;
        if (prev[s] >= 0) {
          mbar_wait(done + 8 * s, ((it >> 1) - 1) & 1);
#pragma unroll
          for (int j = 0; j < 4; ++j) tma_store_2d(&tmD0, base + s * BSTG + j * 16384, j * 64, prev[s] * 128);
          bulk_commit();
          bulk_wait_read0();
        }
        mbar_arrive_expect_tx(full + 8 * s, BT0 + BT1 + BTE);
        const uint32_t st = base + s * BSTG;
#pragma unroll
        for (int j = 0; j < 4; ++j) tma_load_2d(st + j * 16384, &tmA0, full + 8 * s, j * 64, tile * 128);
        tma_load_2d(st + BT0, &tmA1, full + 8 * s, 0, tile * 128);
        tma_load_2d(st + BT0 + BT1, &tmE, full + 8 * s, 0, tile * 128);
        prev[s] = tile;
      }
      // drain: the last (up to two) tiles
      for (uint32_t k = 0; k < 2; ++k, ++it) {
        const uint32_t s = it & 1;
        if (prev[s] < 0) continue;
        mbar_wait(done + 8 * s, ((it >> 1) - 1) & 1);
#pragma unroll
        for (int j = 0; j < 4; ++j) tma_store_2d(&tmD0, base + s * BSTG + j * 16384, j * 64, prev[s] * 128);
        bulk_commit();
      }
      bulk_wait0();
    }
  } else {
    // ---- compute warps 0-7
    // phase 1: thread = (row group g = warp, column pair jp = lane); rows
    // g + 8 i all share the swizzle phase g, so every address is base + i*const
    const int jp = lane, g = warp;
    float w2c[2][12], accw[2][12];
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int c = 0; c < 12; ++c) {
        w2c[e][c] = __ldg(w2 + c * 64 + 2 * jp + e);
        accw[e][c] = 0.f;
      }
    const float alj0 = sal1[2 * jp], alj1 = sal1[2 * jp + 1];
    float acc_a1[2] = {0.f, 0.f}, acc_b1[2] = {0.f, 0.f}, acc_b2[2] = {0.f, 0.f};
    const uint32_t p1off = g * 128 + (((jp >> 2) ^ g) << 4) + (jp & 3) * 4;  // row g, column pair jp
    // epilogue: TMEM lane quarter q, column half hc (4 blocks of 32); row
    // q*32 + lane has swizzle phase lane & 7
    const int q = warp & 3, hc = warp >> 2;
    const uint32_t erow = (q * 32 + lane) * 128, esw = lane & 7;
    const uint32_t idesc = instr_desc(1, 128, 256, 0, 0);
    uint32_t it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const uint32_t s = it & 1, ph = (it >> 1) & 1;
      const int m0 = tile * 128;
      const uint32_t st = base + s * BSTG;
      uint8_t* stp = raw + (st - r0);
      const float4* sdE = reinterpret_cast<const float4*>(stp + BT0 + BT1);
      // the da1 TMA store of the previous tile must have read A
      if (t == 0) bulk_wait_read0();
      bar_sync(1, 256);
      mbar_wait(full + 8 * s, ph);
      const bool whole = m0 + 128 <= U;  // only the last tile has rows past the count
      auto row = [&](int i, bool check) {
        const int r = g + 8 * i;
        const bool valid = !check || m0 + r < U;
        float d[12];
        const float4 d0 = sdE[r * 3], d1 = sdE[r * 3 + 1], d2 = sdE[r * 3 + 2];
        d[0] = d0.x; d[1] = d0.y; d[2] = d0.z; d[3] = d0.w;
        d[4] = d1.x; d[5] = d1.y; d[6] = d1.z; d[7] = d1.w;
        d[8] = d2.x; d[9] = d2.y; d[10] = d2.z; d[11] = d2.w;
        float2 a = bf2_to_f2(*reinterpret_cast<const uint32_t*>(stp + BT0 + p1off + i * 1024));
        if (!valid) {
#pragma unroll
          for (int c = 0; c < 12; ++c) d[c] = 0.f;
          a = make_float2(0.f, 0.f);
        }
        float dh0 = 0.f, dh1 = 0.f;
#pragma unroll
        for (int c = 0; c < 12; ++c) ffma2(dh0, dh1, w2c[0][c], w2c[1][c], d[c]);  // paired fma.rn
        const bool p0 = a.x > 0.f, p1 = a.y > 0.f;
        const float dd0 = p0 ? dh0 : alj0 * dh0, dd1 = p1 ? dh1 : alj1 * dh1;
        acc_a1[0] = fmaf(p0 ? 0.f : a.x, dh0, acc_a1[0]);
        acc_a1[1] = fmaf(p1 ? 0.f : a.y, dh1, acc_a1[1]);
        acc_b1[0] += dd0;
        acc_b1[1] += dd1;
        const float h0 = p0 ? a.x : alj0 * a.x, h1 = p1 ? a.y : alj1 * a.y;
#pragma unroll
        for (int c = 0; c < 12; ++c) ffma2(accw[0][c], accw[1][c], h0, h1, d[c]);
        if (jp < 6 && valid) {
          const float2 db = reinterpret_cast<const float2*>(sdE + r * 3)[jp];
          acc_b2[0] += db.x;
          acc_b2[1] += db.y;
        }
        *reinterpret_cast<uint32_t*>(raw + (A - r0) + p1off + i * 1024) = f2_to_bf2(dd0, dd1);
      };
      if (whole) {
#pragma unroll 4
        for (int i = 0; i < 16; ++i) row(i, false);
      } else {
#pragma unroll 1
        for (int i = 0; i < 16; ++i) row(i, true);
      }
      fence_proxy_async();
      bar_sync(1, 256);
      if (t == 0) {
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma<1>(tmem, smem_desc(A + kk * 32, 16, 1024), smem_desc(W + kk * 32, 16, 1024), idesc, kk > 0);
        mma_commit(mbar);
        tma_store_2d(&tmD1, A, 0, m0);
        bulk_commit();
      }
      // epilogue: da0 = prelu'(a0) dh1 in place over a0 (bf16).  Rows past the
      // count have da1 = 0, hence dh1 = 0 and da0 = 0 whatever a0 holds.  The
      // column sums dalpha0 / db0 come from k_dw1b's row GEMMs instead.
      mbar_wait(mbar, it & 1);
      tc_fence_after();
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        const int col0 = hc * 128 + cb * 32;
        float dh[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + col0, dh);
        uint8_t* bp = stp + (col0 >> 6) * 16384 + erow;
        const int c0 = (col0 & 63) >> 3;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          uint4* p = reinterpret_cast<uint4*>(bp + (((c0 + cc) ^ esw) << 4));
          const float4 al_lo = *reinterpret_cast<const float4*>(sal0 + col0 + cc * 8);
          const float4 al_hi = *reinterpret_cast<const float4*>(sal0 + col0 + cc * 8 + 4);
          const float al[8] = {al_lo.x, al_lo.y, al_lo.z, al_lo.w, al_hi.x, al_hi.y, al_hi.z, al_hi.w};
          const uint4 v = *p;
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
          uint32_t o[4];
#pragma unroll
          for (int pp = 0; pp < 4; ++pp) {
            const float2 x = bf2_to_f2(w[pp]);
            const float g0 = dh[cc * 8 + 2 * pp], g1 = dh[cc * 8 + 2 * pp + 1];
            o[pp] = f2_to_bf2(x.x > 0.f ? g0 : al[2 * pp] * g0, x.y > 0.f ? g1 : al[2 * pp + 1] * g1);
          }
          *p = make_uint4(o[0], o[1], o[2], o[3]);
        }
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(done + 8 * s);
    }
    // the block partial: combine the 8 row groups in a fixed order; the stage
    // buffers are free once every store issued by the producer has read them
    asm volatile("bar.arrive 2, 288;" ::: "memory");
    asm volatile("bar.sync 3, 288;" ::: "memory");
    float* red = at<float>(raw, r0, base);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = 2 * jp + e;
#pragma unroll
      for (int c = 0; c < 12; ++c) red[g * PART_L2 + c * 64 + j] = accw[e][c];
      if (j < 12) red[g * PART_L2 + 768 + j] = acc_b2[e];
      red[g * PART_L2 + 780 + j] = acc_a1[e];
      red[g * PART_L2 + 844 + j] = acc_b1[e];
    }
    bar_sync(1, 256);
    for (int i = t; i < PART_B; i += 256) {
      float sum = 0.f;
      if (i < PART_L2) {
#pragma unroll
        for (int gg = 0; gg < 8; ++gg) sum += red[gg * PART_L2 + i];
      }
      prow[i] = sum;
    }
  }
  if (warp == 8) {
    // every da0 store has finished reading the stages before they are reused
    asm volatile("bar.sync 2, 288;" ::: "memory");
    asm volatile("bar.arrive 3, 288;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

// ===========================================================================
// k_dw1b: the three row reductions of layer 1's backward as GEMMs over rows
//   Ga = a0^T da1,  Gp = max(a0,0)^T da1,  Gm = [a0<=0]^T da1   [256 x 64]
// (Ga straight from the TMA-loaded a0 tile, so only two operands are built
// on the CUDA cores); with Gn = min(a0,0)^T da1 = Ga - Gp, (k_l1_finish,
// exact identities of the PReLU backward):
//   dW1^T = Gp + alpha0 o Gn
//   dalpha0[f] = sum_r [a0<=0] a0 dh1 = sum_j W1[j,f] Gn[f,j]
//   db0[f]     = sum_r da0 = sum_j W1[j,f] (db1[j] - (1 - alpha0[f]) Gm[f,j])
// (dh1 = da1 W1, so every sum over rows of dh1 folds through W1).
// ===========================================================================
constexpr int D_STAGES = 4;
constexpr int DBK = 32;                  // rows per stage
constexpr uint32_t DX = 4 * 4096;        // one operand: 4 boxes of 64 features x 32 rows (bf16 MN-major SW128)
constexpr uint32_t DB = 4096;            // da1: 64 x 32 rows
constexpr uint32_t DSTG = 3 * DX + DB;   // a0 (as loaded) | p | m | da1
constexpr size_t D_SMEM = 1024 + D_STAGES * DSTG + 256;
constexpr int D_THREADS = 192;  // w0-3 transform + epilogue, w4 MMA, w5 TMA
constexpr int G_PART = 3 * 64 * 256;

__global__ void __launch_bounds__(D_THREADS, 1)
    k_dw1b(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmD,
           const int32_t* __restrict__ count, float* __restrict__ part) {
  const int U = *count;
  const int per = (((U + gridDim.x - 1) / gridDim.x) + DBK - 1) / DBK * DBK;
  const int rb = blockIdx.x * per, re = min(U, rb + per);
  const int nk = re > rb ? (re - rb + DBK - 1) / DBK : 0;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  float* out = part + (int64_t)blockIdx.x * G_PART;
  if (nk == 0) {
    for (int i = t; i < G_PART; i += D_THREADS) out[i] = 0.f;
    return;
  }
  extern __shared__ uint8_t raw[];
  const uint32_t r0 = smem_u32(raw), base = (r0 + 1023u) & ~1023u;
  const uint32_t full = base + D_STAGES * DSTG, ready = full + 8 * D_STAGES, empty = ready + 8 * D_STAGES,
                 accb = empty + 8 * D_STAGES, slot = accb + 8;
  if (t == 0) {
    for (int i = 0; i < D_STAGES; ++i) {
      mbar_init(full + 8 * i, 1);
      mbar_init(ready + 8 * i, 128);
      mbar_init(empty + 8 * i, 1);
    }
    mbar_init(accb, 1);
    fence_mbar_init();
  }
  if (warp == 4) {
    tmem_alloc(slot, 512);
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
        const uint32_t s = kb % D_STAGES, itn = kb / D_STAGES;
        mbar_wait(empty + 8 * s, (itn & 1) ^ 1);
        mbar_arrive_expect_tx(full + 8 * s, DX + DB);
        const uint32_t a = base + s * DSTG;
        const int row = rb + kb * DBK;
#pragma unroll
        for (int j = 0; j < 4; ++j) tma_load_2d(a + j * 4096, &tmH, full + 8 * s, j * 64, row);
        tma_load_2d(a + 3 * DX, &tmD, full + 8 * s, 0, row);
      }
    }
  } else if (warp == 4) {
    if (lane == 0) {
      const uint32_t idesc = instr_desc(1, 128, 64, 1, 1);
      for (int kb = 0; kb < nk; ++kb) {
        const uint32_t s = kb % D_STAGES, itn = kb / D_STAGES;
        mbar_wait(ready + 8 * s, itn & 1);
        tc_fence_after();
        const uint32_t a = base + s * DSTG, b = a + 3 * DX;
#pragma unroll
        for (int x = 0; x < 3; ++x)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int k = 0; k < DBK / 16; ++k)
              mma<1>(tmem + x * 128 + h * 64, smem_desc(a + x * DX + h * 8192 + k * 2048, 4096, 1024, 2),
                     smem_desc(b + k * 2048, 4096, 1024, 2), idesc, (kb | k) != 0);
        mma_commit(empty + 8 * s);
      }
      mma_commit(accb);
    }
  } else {
    // ---- transform (rows past this CTA's range -> 0): thread owns 16-B chunk
    // t&7 of rows (t>>3) and (t>>3)+16 of every box
    const int c = t & 7, rlo = t >> 3;
    for (int kb = 0; kb < nk; ++kb) {
      const uint32_t s = kb % D_STAGES, itn = kb / D_STAGES;
      mbar_wait(full + 8 * s, itn & 1);
      uint8_t* a = raw + (base + s * DSTG - r0);
      const int row0 = rb + kb * DBK;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int r = rlo + 16 * i;
          const uint32_t off = j * 4096 + r * 128 + (c << 4);
          const bool valid = row0 + r < re;
          const uint4 v = *reinterpret_cast<const uint4*>(a + off);
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
          uint32_t pp[4], mm[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 x = bf2_to_f2(w[e]);
            pp[e] = valid ? f2_to_bf2(fmaxf(x.x, 0.f), fmaxf(x.y, 0.f)) : 0u;
            mm[e] = valid ? f2_to_bf2(x.x > 0.f ? 0.f : 1.f, x.y > 0.f ? 0.f : 1.f) : 0u;
          }
          // a0 itself is the third operand (Ga = a0^T da1); rows outside this
          // CTA's range are zeroed so that no operand picks them up
          if (!valid) *reinterpret_cast<uint4*>(a + off) = make_uint4(0u, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(a + DX + off) = make_uint4(pp[0], pp[1], pp[2], pp[3]);
          *reinterpret_cast<uint4*>(a + 2 * DX + off) = make_uint4(mm[0], mm[1], mm[2], mm[3]);
        }
      fence_proxy_async();
      mbar_arrive(ready + 8 * s);
    }
    mbar_wait(accb, 0);
    tc_fence_after();
#pragma unroll 1
    for (int x = 0; x < 3; ++x)
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        const int feat = h * 128 + warp * 32 + lane;
#pragma unroll 1
        for (int cb = 0; cb < 2; ++cb) {
          float v[32];
          tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + x * 128 + h * 64 + cb * 32, v);
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) out[x * 16384 + (cb * 32 + jj) * 256 + feat] = v[jj];  // G_x[j][feature]
        }
      }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) tmem_dealloc(tmem, 512);
}

// Gn = Ga - Gp ; gw1[j][f] = Gp + a0[f] Gn ; ga0[f] = sum_j W1[j][f] Gn[j][f] ;
// gb0[f] = sum_j W1[j][f] (db1[j] - (1 - a0[f]) Gm[j][f])
// block = 32 features x 8 j-groups of 8; the 8 partial sums of a feature are
// combined in a fixed order (deterministic)
__global__ void __launch_bounds__(256) k_l1_finish(const float* __restrict__ G, const float* __restrict__ w1,
                                                   const float* __restrict__ al0, const float* __restrict__ db1,
                                                   float* __restrict__ gw1, float* __restrict__ ga0,
                                                   float* __restrict__ gb0) {
  __shared__ float ra[8][33], rb[8][33];
  const int fl = threadIdx.x & 31, jg = threadIdx.x >> 5, f = blockIdx.x * 32 + fl;
  const float a = al0[f];
  float sa = 0.f, sb = 0.f;
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const int j = jg * 8 + jj;
    const float ga = G[j * 256 + f], gp = G[16384 + j * 256 + f], gm = G[32768 + j * 256 + f];
    const float gn = ga - gp;
    const float w = w1[j * 256 + f];
    gw1[j * 256 + f] = gp + a * gn;
    sa = fmaf(w, gn, sa);
    sb = fmaf(w, db1[j] - (1.f - a) * gm, sb);
  }
  ra[jg][fl] = sa;
  rb[jg][fl] = sb;
  __syncthreads();
  if (jg == 0) {
    float ta = 0.f, tb = 0.f;
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      ta += ra[g][fl];
      tb += rb[g][fl];
    }
    ga0[f] = ta;
    gb0[f] = tb;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn3() {
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

// row-major [rows, cols] map with box {box_cols, box_rows}
int map2d(CUtensorMap* m, const void* ptr, bool is_bf16, uint64_t rows, uint64_t cols, uint32_t box_cols,
          uint32_t box_rows, CUtensorMapSwizzle swz) {
  auto fn = encode_fn3();
  if (!fn) return fail(DICM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const uint64_t esz = is_bf16 ? 2 : 4;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * esz};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, is_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                  const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DICM_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return DICM_OK;
}

template <typename K>
int smem_attr3(K kernel, size_t bytes) {
  return check_cuda(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes),
                    "bf16 small-layer smem attribute");
}

int grid_tiles(int64_t rows_max) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(dicm_grid_cap(), (rows_max + 127) / 128));
}

}  // namespace

int fwd_layers12_bf16(const bf16* act0, const int32_t* count, int64_t rows_max, const float* al0, const float* w1,
                      const float* b1, const float* al1, const float* w2, const float* b2, bf16* act1, float* emb,
                      cudaStream_t st) {
  static int once = smem_attr3(k_l12f, F_SMEM);
  if (once) return once;
  CUtensorMap ma;
  int rc = map2d(&ma, act0, true, rows_max, H1, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  const int probe_slot = probe_begin(DICM_PROBE_IMG_FWD_L12, st);
  static const int reverse = [] {  // DICM_L12F_ORDER=fwd: ascending tiles
    const char* e = getenv("DICM_L12F_ORDER");
    return e && e[0] == 'f' ? 0 : 1;
  }();
  k_l12f<<<grid_tiles(rows_max), F_THREADS, F_SMEM, st>>>(ma, al0, w1, b1, al1, w2, b2, count, act1, emb, reverse);
  probe_end(probe_slot, st);
  return last_launch("tcgen05 bf16 layers 1-2 forward");
}

int bwd_layers12_bf16(const float* demb, const bf16* act1, const bf16* act0, const int32_t* count, int64_t rows_max,
                      const float* al0, const float* al1, const float* w1, const float* w2, bf16* da1, bf16* da0,
                      float* part_l12, float* part_dw1, cudaStream_t st) {
  static int once = smem_attr3(k_l12b, B_SMEM);
  if (once) return once;
  static int once2 = smem_attr3(k_dw1b, D_SMEM);
  if (once2) return once2;
  CUtensorMap m0, m1, me, md1, md0;
  int rc = map2d(&m0, act0, true, rows_max, H1, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = map2d(&m1, act1, true, rows_max, H2, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = map2d(&me, demb, false, rows_max, 12, 12, 128, CU_TENSOR_MAP_SWIZZLE_NONE);
  if (!rc) rc = map2d(&md1, da1, true, rows_max, H2, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = map2d(&md0, da0, true, rows_max, H1, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  {
    const int probe_slot = probe_begin(DICM_PROBE_IMG_BWD_L12, st);
    k_l12b<<<grid_tiles(rows_max), B_THREADS, B_SMEM, st>>>(m0, m1, me, md1, md0, al0, al1, w1, w2, count, part_l12);
    probe_end(probe_slot, st);
  }
  rc = last_launch("tcgen05 bf16 layers 2-1 backward");
  if (rc) return rc;
  CUtensorMap mh, md;
  rc = map2d(&mh, act0, true, rows_max, H1, 64, DBK, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = map2d(&md, da1, true, rows_max, H2, 64, DBK, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  {
    const int probe_slot = probe_begin(DICM_PROBE_IMG_BWD_DW1, st);
    k_dw1b<<<small_dw1_blocks(rows_max), D_THREADS, D_SMEM, st>>>(mh, md, count, part_dw1);
    probe_end(probe_slot, st);
  }
  return last_launch("tcgen05 bf16 layer-1 row GEMMs");
}

int l1_finish_bf16(const float* G, const float* w1, const float* al0, const float* db1, float* gw1, float* ga0,
                   float* gb0, cudaStream_t st) {
  k_l1_finish<<<8, 256, 0, st>>>(G, w1, al0, db1, gw1, ga0, gb0);
  return last_launch("layer-1 backward finish");
}

int dw1_bf16_part_size() { return G_PART; }

}  // namespace sm100
}  // namespace dicm
