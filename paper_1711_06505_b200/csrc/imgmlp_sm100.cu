// Layer 0 of the image MLP on the 5th-generation tensor cores (tcgen05).
//
// Forward  act0[U,256] = X[rows] . W0^T + b0      (reference model.py:115-120,
//                                                  autograd.py:199)
// Backward dW0[256,d_raw] = da0^T . X[rows]       (autograd.py:202)
//
// Both kernels keep a 256 x 256 fp32 accumulator tile in TMEM (two M=128
// halves, all 512 columns) fed by a 3-stage shared-memory ring:
//   * the dense operand (W0 forward, da0 backward) arrives by TMA tile loads
//     (128-B swizzle) signalled through mbarrier transaction counts;
//   * the gathered operand -- pool rows picked by the dedup's unique ids --
//     arrives by 16-byte cp.async (LDGSTS) gathers written straight into the
//     same swizzled layout (no gathered copy of X is ever formed); each
//     gather thread signals the stage with cp.async.mbarrier.arrive, so the
//     producers never block on their own loads;
//   * one elected thread issues tcgen05.mma (kind::tf32 on an fp32 pool,
//     kind::f16 on a bf16 pool) and releases stages with tcgen05.commit;
//   * tcgen05.ld drains TMEM in the epilogue.
// The forward kernel is persistent (one CTA per SM looping over 256-row
// tiles) with dedicated epilogue warps, so the gather of tile i+1 overlaps
// the drain of tile i.  The backward reduction over rows is split into
// nsplit chunks per 256-feature tile and finished by a deterministic reduce.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "imgmlp_sm100.cuh"
#include "epi.cuh"
#include "tc_ptx.cuh"

namespace dicm {
namespace sm100 {
namespace {

using namespace tc;

constexpr int STAGES = 3;
constexpr uint32_t OPB = 256 * 128;  // bytes per operand per stage (256 x 128 B)
constexpr uint32_t STAGE_BYTES = 2 * OPB;
constexpr size_t SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ +
                              4 * epi::SCRATCH_FLOATS * 4 /*epilogue transpose*/;
constexpr int THREADS_F = 320;  // fwd: warps 0-3 gather, 4 MMA, 5 TMA, 6-9 epilogue
constexpr int THREADS_B = 192;  // bwd: warps 0-3 gather + epilogue, 4 MMA, 5 TMA
constexpr unsigned FULL = 0xffffffffu;

template <int KIND>
using Elem = typename std::conditional<KIND == 0, float, __nv_bfloat16>::type;

struct Smem {
  uint32_t base, full, empty, acc_full, acc_empty, slot;
  uint32_t* slot_ptr;
};

__device__ __forceinline__ Smem carve(uint8_t* raw) {
  Smem s;
  const uint32_t r = smem_u32(raw);
  s.base = (r + 1023u) & ~1023u;
  s.full = s.base + STAGES * STAGE_BYTES;
  s.empty = s.full + 8 * STAGES;
  s.acc_full = s.empty + 8 * STAGES;
  s.acc_empty = s.acc_full + 8;
  s.slot = s.acc_empty + 8;
  s.slot_ptr = reinterpret_cast<uint32_t*>(raw + (s.slot - r));
  return s;
}

__device__ __forceinline__ uint32_t setup(const Smem& s, int warp, uint32_t acc_empty_count) {
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(s.full + 8 * i, 128 + 1);  // 128 gather threads (cp.async arrive) + TMA expect_tx
      mbar_init(s.empty + 8 * i, 1);       // tcgen05.commit
    }
    mbar_init(s.acc_full, 1);
    mbar_init(s.acc_empty, acc_empty_count);
    fence_mbar_init();
  }
  if (warp == 4) {
    tmem_alloc(s.slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  return *reinterpret_cast<volatile uint32_t*>(s.slot_ptr);
}

__device__ __forceinline__ void wait_stage(uint32_t bar, uint32_t g, bool producer) {
  const uint32_t it = g / STAGES;
  mbar_wait(bar + 8 * (g % STAGES), producer ? ((it & 1) ^ 1) : (it & 1));
}

// ---------------------------------------------------------------------------
// forward: act0 = X[rows] W0^T + b0, persistent over 256-row tiles
// ---------------------------------------------------------------------------
template <int KIND>
__global__ void __launch_bounds__(THREADS_F, 1)
    k_fwd(const __grid_constant__ CUtensorMap tmW, const void* __restrict__ pool_, int d_raw,
          const int32_t* __restrict__ rows, const int32_t* __restrict__ count, const float* __restrict__ bias,
          void* __restrict__ act0_) {
  using T = Elem<KIND>;
  constexpr int EPB = 128 / sizeof(T);  // elements per 128-byte row slice
  const int U = *count;
  const int ntiles = (U + 255) / 256;
  if ((int)blockIdx.x >= ntiles) return;
  extern __shared__ uint8_t smem_raw[];
  const Smem s = carve(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t tmem = setup(s, warp, 128);
  const int nk = d_raw / EPB;
  const T* pool = reinterpret_cast<const T*>(pool_);

  if (warp < 4) {
    // ---- gather producer: 16 rows x one 16-B chunk per thread and stage
    const int t = threadIdx.x, c = t & 7, rb = t >> 3;
    const uint32_t dst0 = (uint32_t)(rb * 128 + ((c ^ (rb & 7)) << 4));  // (rb + 16 i) & 7 == rb & 7
    uint32_t g = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int m0 = tile * 256;
      const T* src[16];
      uint32_t ok[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int gr = m0 + rb + 16 * i;
        const bool v = gr < U;
        src[i] = pool + (int64_t)(v ? __ldg(rows + gr) : 0) * d_raw + c * (16 / sizeof(T));
        ok[i] = v ? 16u : 0u;
      }
      for (int kb = 0; kb < nk; ++kb, ++g) {
        wait_stage(s.empty, g, true);
        const uint32_t a = s.base + (g % STAGES) * STAGE_BYTES + dst0;
#pragma unroll
        for (int i = 0; i < 16; ++i) cp_async16(a + i * 16 * 128, src[i] + (int64_t)kb * EPB, ok[i]);
        cp_async_arrive_noinc(s.full + 8 * (g % STAGES));
      }
    }
    cp_async_wait<0>();
  } else if (warp == 5) {
    if (lane == 0) {
      // ---- TMA producer for W0 [256, d_raw] (K-major, 128-B swizzle)
      prefetch_tmap(&tmW);
      uint32_t g = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
        for (int kb = 0; kb < nk; ++kb, ++g) {
          wait_stage(s.empty, g, true);
          const uint32_t st = g % STAGES;
          mbar_arrive_expect_tx(s.full + 8 * st, OPB);
          tma_load_2d(s.base + st * STAGE_BYTES + OPB, &tmW, s.full + 8 * st, kb * EPB, 0);
        }
    }
  } else if (warp == 4) {
    if (lane == 0) {
      // ---- MMA issuer: 2 halves (rows 0-127, 128-255) x 4 k-steps of 32 B
      const uint32_t idesc = instr_desc(KIND == 0 ? 2u : 1u, 128, 256, 0, 0);
      uint32_t g = 0, tl = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tl) {
        mbar_wait(s.acc_empty, (tl & 1) ^ 1);  // epilogue drained the previous tile
        tc_fence_after();
        for (int kb = 0; kb < nk; ++kb, ++g) {
          wait_stage(s.full, g, false);
          tc_fence_after();
          fence_proxy_async();
          const uint32_t a = s.base + (g % STAGES) * STAGE_BYTES, b = a + OPB;
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma<KIND>(tmem + h * 256, smem_desc(a + h * 16384 + k * 32, 16, 1024), smem_desc(b + k * 32, 16, 1024),
                        idesc, (kb | k) != 0);
          mma_commit(s.empty + 8 * (g % STAGES));
        }
        mma_commit(s.acc_full);
      }
    }
  } else {
    // ---- epilogue warps 6-9: TMEM lane quarter = warp % 4
    const int q = warp & 3;
    float* scr = reinterpret_cast<float*>(smem_raw + (s.slot + 16 - smem_u32(smem_raw))) + q * epi::SCRATCH_FLOATS;
    uint32_t tl = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tl) {
      mbar_wait(s.acc_full, tl & 1);
      tc_fence_after();
      const int m0 = tile * 256;
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
#pragma unroll 1
        for (int cb = 0; cb < 8; ++cb) {
          float v[32];
          tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + h * 256 + cb * 32, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] += __ldg(bias + cb * 32 + j);
          // bf16 mode saves act0 as bf16 (the layer-1 operand precision)
          if constexpr (KIND == 1)
            epi::store_bf16(v, scr, lane, m0 + h * 128 + q * 32, U, [&](int r) {
              return reinterpret_cast<__nv_bfloat16*>(act0_) + (int64_t)r * 256 + cb * 32;
            });
          else
            epi::store_f32(v, scr, lane, m0 + h * 128 + q * 32, U,
                           [&](int r) { return reinterpret_cast<float*>(act0_) + (int64_t)r * 256 + cb * 32; });
        }
      }
      tc_fence_before();
      mbar_arrive(s.acc_empty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------
// forward on CTA pairs (cta_group::2): a cluster of two CTAs computes a
// 256-row tile with one M256 x N256 MMA per k-step.  Each CTA gathers its own
// 128 rows and TMA-loads its half of W0 (128 of the 256 output features), so
// per SM the MMA reads half the B operand from shared memory, and the
// accumulator (128 lanes x 256 columns per CTA) is double-buffered in TMEM:
// the epilogue of tile i overlaps the MMAs of tile i+1.  The peer CTA's
// stage completion is relayed to the leader's barrier by one peer thread.
// ---------------------------------------------------------------------------
constexpr uint32_t OPB2 = 128 * 128;  // 16 KB: one CTA's operand half per k-block
__host__ __device__ constexpr size_t smem2(int sa, int sb) {
  return (size_t)(sa + sb) * OPB2 + 1024 + 256 + 4 * epi::SCRATCH_FLOATS * 4;
}

// SA2 gathered-row slots (HBM latency), SB2 W0 slots (L2-resident)
template <int KIND, int SA2, int SB2>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS_F, 1)
    k_fwd2(const __grid_constant__ CUtensorMap tmW, const void* __restrict__ pool_, int d_raw,
           const int32_t* __restrict__ rows, const int32_t* __restrict__ count, const float* __restrict__ bias,
           void* __restrict__ act0_) {
  using T = Elem<KIND>;
  constexpr int EPB = 128 / sizeof(T);
  const int U = *count;
  const int ntiles = (U + 255) / 256;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  if (pair >= ntiles) return;  // uniform across the pair
  extern __shared__ uint8_t smem_raw[];
  const uint32_t r0s = smem_u32(smem_raw);
  const uint32_t base = (r0s + 1023u) & ~1023u, bbase = base + SA2 * OPB2;
  const uint32_t fullA = bbase + SB2 * OPB2, emptyA = fullA + 8 * SA2, fullB = emptyA + 8 * SA2,
                 emptyB = fullB + 8 * SB2, accf = emptyB + 8 * SB2, acce = accf + 16, slot = acce + 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < SA2; ++i) {
      mbar_init(fullA + 8 * i, 128 + (rank == 0 ? 1 : 0));  // gathers (+ the peer's relay)
      mbar_init(emptyA + 8 * i, 1);                         // pair MMA commit (multicast)
    }
    for (int i = 0; i < SB2; ++i) {
      mbar_init(fullB + 8 * i, 1);
      mbar_init(emptyB + 8 * i, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(accf + 8 * b, 1);
      mbar_init(acce + 8 * b, 8);  // both CTAs' 4 epilogue warps (leader's copy is used)
    }
    fence_mbar_init();
  }
  if (warp == 4) {
    tmem_alloc2(slot, 512);
    tmem_relinquish2();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem_raw + (slot - r0s));
  const int nk = d_raw / EPB;
  const T* pool = reinterpret_cast<const T*>(pool_);

  if (warp < 4) {
    // ---- gather producer: 8 rows x one 16-B chunk per thread and stage
    const int t = threadIdx.x, c = t & 7, rb = t >> 3;
    const uint32_t dst0 = (uint32_t)(rb * 128 + ((c ^ (rb & 7)) << 4));
    uint32_t g = 0;
    for (int tile = pair; tile < ntiles; tile += npairs) {
      const int m0 = tile * 256 + (int)rank * 128;
      const T* src[8];
      uint32_t ok[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int gr = m0 + rb + 16 * i;
        const bool v = gr < U;
        src[i] = pool + (int64_t)(v ? __ldg(rows + gr) : 0) * d_raw + c * (16 / sizeof(T));
        ok[i] = v ? 16u : 0u;
      }
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const uint32_t st = g % SA2, it = g / SA2;
        mbar_wait(emptyA + 8 * st, (it & 1) ^ 1);
        const uint32_t a = base + st * OPB2 + dst0;
#pragma unroll
        for (int i = 0; i < 8; ++i) cp_async16(a + i * 16 * 128, src[i] + (int64_t)kb * EPB, ok[i]);
        cp_async_arrive_noinc(fullA + 8 * st);
      }
    }
    cp_async_wait<0>();
  } else if (warp == 5) {
    if (lane == 0) {
      // ---- TMA producer: this CTA's half of W0 (rows rank*128 .. +127)
      prefetch_tmap(&tmW);
      uint32_t g = 0;
      for (int tile = pair; tile < ntiles; tile += npairs)
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const uint32_t st = g % SB2, it = g / SB2;
          mbar_wait(emptyB + 8 * st, (it & 1) ^ 1);
          mbar_arrive_expect_tx(fullB + 8 * st, OPB2);
          tma_load_2d(bbase + st * OPB2, &tmW, fullB + 8 * st, kb * EPB, (int)rank * 128);
        }
    }
  } else if (warp == 4) {
    if (lane == 0) {
      if (rank == 0) {
        // ---- MMA issuer (leader): M256 x N256 per k-step into TMEM buffer tl&1
        const uint32_t idesc = instr_desc(KIND == 0 ? 2u : 1u, 256, 256, 0, 0);
        uint32_t g = 0, tl = 0;
        for (int tile = pair; tile < ntiles; tile += npairs, ++tl) {
          const uint32_t buf = tl & 1;
          mbar_wait(acce + 8 * buf, ((tl >> 1) & 1) ^ 1);
          tc_fence_after();
          for (int kb = 0; kb < nk; ++kb, ++g) {
            const uint32_t sa = g % SA2, sb = g % SB2;
            mbar_wait(fullA + 8 * sa, (g / SA2) & 1);
            mbar_wait(fullB + 8 * sb, (g / SB2) & 1);
            tc_fence_after();
            fence_proxy_async();
            const uint32_t a = base + sa * OPB2, b = bbase + sb * OPB2;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma2<KIND>(tmem + buf * 256, smem_desc(a + k * 32, 16, 1024), smem_desc(b + k * 32, 16, 1024), idesc,
                         (kb | k) != 0);
            mma_commit2(emptyA + 8 * sa, 0x3);
            mma_commit2(emptyB + 8 * sb, 0x3);
          }
          mma_commit2(accf + 8 * buf, 0x3);
        }
      } else {
        // ---- relay (peer): this CTA's stage landed -> the leader's full barrier
        const uint32_t lfull = mapa(fullA, 0);
        uint32_t g = 0;
        for (int tile = pair; tile < ntiles; tile += npairs)
          for (int kb = 0; kb < nk; ++kb, ++g) {
            const uint32_t sa = g % SA2;
            mbar_wait(fullA + 8 * sa, (g / SA2) & 1);
            mbar_wait(fullB + 8 * (g % SB2), (g / SB2) & 1);
            fence_proxy_async();
            mbar_arrive_cluster(lfull + 8 * sa);
          }
      }
    }
  } else {
    // ---- epilogue warps 6-9: this CTA's 128 rows, TMEM lane quarter = warp % 4
    const int q = warp & 3;
    float* scr = reinterpret_cast<float*>(smem_raw + (slot + 16 - r0s)) + q * epi::SCRATCH_FLOATS;
    const uint32_t lacce = mapa(acce, 0);
    uint32_t tl = 0;
    for (int tile = pair; tile < ntiles; tile += npairs, ++tl) {
      const uint32_t buf = tl & 1;
      mbar_wait(accf + 8 * buf, (tl >> 1) & 1);
      tc_fence_after();
      const int m0 = tile * 256 + (int)rank * 128 + q * 32;
#pragma unroll 1
      for (int cb = 0; cb < 8; ++cb) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + buf * 256 + cb * 32, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] += __ldg(bias + cb * 32 + j);
        if constexpr (KIND == 1)
          epi::store_bf16(v, scr, lane, m0, U, [&](int r) {
            return reinterpret_cast<__nv_bfloat16*>(act0_) + (int64_t)r * 256 + cb * 32;
          });
        else
          epi::store_f32(v, scr, lane, m0, U,
                         [&](int r) { return reinterpret_cast<float*>(act0_) + (int64_t)r * 256 + cb * 32; });
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(lacce + 8 * buf);
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 4) tmem_dealloc2(tmem, 512);
}

// ---------------------------------------------------------------------------
// forward, two sub-tiles per W0 pass: a pair tile is 512 rows = two 256-row
// pair MMAs that share every W0 stage.  Per CTA and stage: 32 KB of gathered
// rows (2 x 128 rows x 128 B) against 16 KB of W0, so the ring holds more
// gathered bytes in flight per byte of W0 and W0 is re-read from L2 half as
// often.  TMEM holds both sub-tile accumulators (2 x 256 columns), so the
// MMAs of tile i+1 wait for the epilogue of tile i; 8 epilogue warps (two
// per TMEM lane quarter, one per sub-tile) keep that drain short while the
// gather ring keeps filling.
// ---------------------------------------------------------------------------
constexpr int THREADS_F4 = 448;  // w0-3 gather, w4 MMA / relay, w5 TMA, w6-13 epilogue
constexpr uint32_t STG4 = 8 * 4096;  // EPI 2: one 32-row x 128-B TMA-store staging box per epilogue warp
__host__ __device__ constexpr size_t smem4(int sa, int sb, int epi_mode) {
  return (size_t)sa * 2 * OPB2 + (size_t)sb * OPB2 + 1024 + 256 +
         (epi_mode == 1 ? 8 * epi::SCRATCH_FLOATS * 4 : epi_mode == 2 ? STG4 : 0);
}

// EPI: how the epilogue writes act0.  1: each 32x32 block transposed through
// shared memory for whole-line stores; 0: every lane stores its own row;
// 2 (bf16): two blocks (64 columns) converted into a swizzled staging box and
// written by one TMA store (cp.async.bulk.tensor), so the drain issues no
// global stores of its own
template <int KIND, int SA, int SB, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS_F4, 1)
    k_fwd4(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmO,
           const void* __restrict__ pool_, int d_raw, const int32_t* __restrict__ rows,
           const int32_t* __restrict__ count, const float* __restrict__ bias, void* __restrict__ act0_) {
  constexpr bool SCR = EPI == 1;
  using T = Elem<KIND>;
  constexpr int EPB = 128 / sizeof(T);
  constexpr uint32_t ASTG = 2 * OPB2;  // two sub-tiles of 128 rows
  const int U = *count;
  const int ntiles = (U + 511) / 512;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  if (pair >= ntiles) return;  // uniform across the pair
  extern __shared__ uint8_t smem_raw[];
  const uint32_t r0s = smem_u32(smem_raw);
  const uint32_t base = (r0s + 1023u) & ~1023u, bbase = base + SA * ASTG;
  const uint32_t stg = bbase + SB * OPB2;  // EPI 2 staging (1024-B aligned)
  const uint32_t fullA = stg + (EPI == 2 ? STG4 : 0), emptyA = fullA + 8 * SA, fullB = emptyA + 8 * SA,
                 emptyB = fullB + 8 * SB, accf = emptyB + 8 * SB, acce = accf + 8, slot = acce + 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < SA; ++i) {
      mbar_init(fullA + 8 * i, 128 + (rank == 0 ? 1 : 0));  // gathers (+ the peer's relay)
      mbar_init(emptyA + 8 * i, 1);                         // pair MMA commit (multicast)
    }
    for (int i = 0; i < SB; ++i) {
      mbar_init(fullB + 8 * i, 1);
      mbar_init(emptyB + 8 * i, 1);
    }
    mbar_init(accf, 1);
    mbar_init(acce, 16);  // both CTAs' 8 epilogue warps (leader's copy is used)
    fence_mbar_init();
  }
  if (warp == 4) {
    tmem_alloc2(slot, 512);
    tmem_relinquish2();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem_raw + (slot - r0s));
  const int nk = d_raw / EPB;
  const T* pool = reinterpret_cast<const T*>(pool_);
  // this CTA's rows of sub-tile s of pair tile `tile`: tile*512 + s*256 + rank*128 + [0, 128)
  if (warp < 4) {
    // ---- gather producer: 16 rows x one 16-B chunk per thread and stage
    const int t = threadIdx.x, c = t & 7, rb = t >> 3;
    const uint32_t dst0 = (uint32_t)(rb * 128 + ((c ^ (rb & 7)) << 4));
    uint32_t g = 0;
    for (int tile = pair; tile < ntiles; tile += npairs) {
      const T* src[16];
      uint32_t ok[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int gr = tile * 512 + (i >> 3) * 256 + (int)rank * 128 + rb + 16 * (i & 7);
        const bool v = gr < U;
        src[i] = pool + (int64_t)(v ? __ldg(rows + gr) : 0) * d_raw + c * (16 / sizeof(T));
        ok[i] = v ? 16u : 0u;
      }
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const uint32_t st = g % SA, it = g / SA;
        mbar_wait(emptyA + 8 * st, (it & 1) ^ 1);
        const uint32_t a = base + st * ASTG + dst0;
#pragma unroll
        for (int i = 0; i < 16; ++i)
          cp_async16(a + (i >> 3) * OPB2 + (i & 7) * 16 * 128, src[i] + (int64_t)kb * EPB, ok[i]);
        cp_async_arrive_noinc(fullA + 8 * st);
      }
    }
    cp_async_wait<0>();
  } else if (warp == 5) {
    if (lane == 0) {
      // ---- TMA producer: this CTA's half of W0 (rows rank*128 .. +127)
      prefetch_tmap(&tmW);
      uint32_t g = 0;
      for (int tile = pair; tile < ntiles; tile += npairs)
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const uint32_t st = g % SB, it = g / SB;
          mbar_wait(emptyB + 8 * st, (it & 1) ^ 1);
          mbar_arrive_expect_tx(fullB + 8 * st, OPB2);
          tma_load_2d(bbase + st * OPB2, &tmW, fullB + 8 * st, kb * EPB, (int)rank * 128);
        }
    }
  } else if (warp == 4) {
    if (lane == 0) {
      if (rank == 0) {
        // ---- MMA issuer (leader): per k-step two M256 x N256 MMAs (sub-tiles) on one W0 stage
        const uint32_t idesc = instr_desc(KIND == 0 ? 2u : 1u, 256, 256, 0, 0);
        uint32_t g = 0, tl = 0;
        for (int tile = pair; tile < ntiles; tile += npairs, ++tl) {
          mbar_wait(acce, (tl & 1) ^ 1);  // the epilogue has drained both accumulators
          tc_fence_after();
          for (int kb = 0; kb < nk; ++kb, ++g) {
            const uint32_t sa = g % SA, sb = g % SB;
            mbar_wait(fullA + 8 * sa, (g / SA) & 1);
            mbar_wait(fullB + 8 * sb, (g / SB) & 1);
            tc_fence_after();
            fence_proxy_async();
            const uint32_t a = base + sa * ASTG, b = bbase + sb * OPB2;
#pragma unroll
            for (int sub = 0; sub < 2; ++sub)
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma2<KIND>(tmem + sub * 256, smem_desc(a + sub * OPB2 + k * 32, 16, 1024),
                           smem_desc(b + k * 32, 16, 1024), idesc, (kb | k) != 0);
            mma_commit2(emptyA + 8 * sa, 0x3);
            mma_commit2(emptyB + 8 * sb, 0x3);
          }
          mma_commit2(accf, 0x3);
        }
      } else {
        // ---- relay (peer): this CTA's stage landed -> the leader's full barrier
        const uint32_t lfull = mapa(fullA, 0);
        uint32_t g = 0;
        for (int tile = pair; tile < ntiles; tile += npairs)
          for (int kb = 0; kb < nk; ++kb, ++g) {
            const uint32_t sa = g % SA;
            mbar_wait(fullA + 8 * sa, (g / SA) & 1);
            mbar_wait(fullB + 8 * (g % SB), (g / SB) & 1);
            fence_proxy_async();
            mbar_arrive_cluster(lfull + 8 * sa);
          }
      }
    }
  } else {
    // ---- epilogue warps 6-13: sub-tile (warp - 6) / 4, TMEM lane quarter warp % 4
    const int q = warp & 3, sub = (warp - 6) >> 2;
    float* scr = reinterpret_cast<float*>(smem_raw + (slot + 8 - r0s)) + (warp - 6) * epi::SCRATCH_FLOATS;
    (void)scr;
    const uint32_t lacce = mapa(acce, 0);
    uint32_t tl = 0;
    for (int tile = pair; tile < ntiles; tile += npairs, ++tl) {
      mbar_wait(accf, tl & 1);
      tc_fence_after();
      const int m0 = tile * 512 + sub * 256 + (int)rank * 128 + q * 32;
      // one 32-column block: bias, then bf16/fp32 rows of act0
      auto emit = [&](int cb, uint32_t (&r)[32]) {
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) + __ldg(bias + cb * 32 + j);
#ifdef DICM_FWD4_NOSTORE  // measurement build only: the drain without its act0 stores
        float keep = 0.f;  // keeps the TMEM loads and bias adds live (no dynamic index: no local memory)
#pragma unroll
        for (int j = 0; j < 32; ++j) keep += v[j];
        if (keep == 12345.f) reinterpret_cast<float*>(act0_)[0] = keep;
        if (false)
#endif
        if constexpr (SCR) {
          if constexpr (KIND == 1)
            epi::store_bf16(v, scr, lane, m0, U, [&](int r) {
              return reinterpret_cast<__nv_bfloat16*>(act0_) + (int64_t)r * 256 + cb * 32;
            });
          else
            epi::store_f32(v, scr, lane, m0, U,
                           [&](int r) { return reinterpret_cast<float*>(act0_) + (int64_t)r * 256 + cb * 32; });
        } else if (m0 + lane < U) {
          if constexpr (KIND == 1) {
            uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(act0_) + (int64_t)(m0 + lane) * 256 +
                                                cb * 32);
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              uint32_t w[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                __nv_bfloat162 h = __floats2bfloat162_rn(v[8 * q4 + 2 * e], v[8 * q4 + 2 * e + 1]);
                w[e] = *reinterpret_cast<uint32_t*>(&h);
              }
              o[q4] = make_uint4(w[0], w[1], w[2], w[3]);
            }
          } else {
            float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(act0_) + (int64_t)(m0 + lane) * 256 + cb * 32);
#pragma unroll
            for (int q4 = 0; q4 < 8; ++q4) o[q4] = make_float4(v[4 * q4], v[4 * q4 + 1], v[4 * q4 + 2], v[4 * q4 + 3]);
          }
        }
      };
      const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + sub * 256;
      if constexpr (EPI == 2) {
        // per pair of blocks: both in registers, bias, bf16 into this warp's
        // staging box (row = lane, 16-B chunk c at c ^ (lane & 7): SWIZZLE_128B),
        // one TMA store of 32 rows x 64 columns (fp32: one box of 32 columns
        // per block); the accumulator is released once the last pair is in
        // registers
        const uint32_t box = stg + (uint32_t)(warp - 6) * 4096;
        uint32_t ra[32], rb[32];
#pragma unroll 1
        for (int cb = 0; cb < 8; cb += 2) {
          tmem_ld32_issue(tb + cb * 32, ra);
          tmem_ld32_issue(tb + (cb + 1) * 32, rb);
          tmem_ld_wait(ra);
          tmem_ld_wait(rb);
          if (cb == 6) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(lacce);
          }
          // a box reaching past the count (the last tile) is stored row by row
          // instead: rows >= U stay untouched
          const bool whole = m0 + 32 <= U;
          if constexpr (KIND == 0) {  // fp32 act0: one 32-column box per block
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (lane == 0) bulk_wait_read0();
              __syncwarp();
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + (cb + h) * 32 + 4 * c));
                const uint32_t(&r)[32] = h == 0 ? ra : rb;
                const float4 o = make_float4(__uint_as_float(r[4 * c]) + b4.x, __uint_as_float(r[4 * c + 1]) + b4.y,
                                             __uint_as_float(r[4 * c + 2]) + b4.z, __uint_as_float(r[4 * c + 3]) + b4.w);
                if (whole)
                  st_shared_v4(box + lane * 128 + ((c ^ (lane & 7)) << 4), __float_as_uint(o.x), __float_as_uint(o.y),
                               __float_as_uint(o.z), __float_as_uint(o.w));
                else if (m0 + lane < U)
                  reinterpret_cast<float4*>(reinterpret_cast<float*>(act0_) + (int64_t)(m0 + lane) * 256 +
                                            (cb + h) * 32)[c] = o;
              }
              if (whole) {
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                  tma_store_2d(&tmO, box, (cb + h) * 32, m0);
                  bulk_commit();
                }
              }
            }
            continue;
          }
          if (lane == 0) bulk_wait_read0();  // the previous store has read the box
          __syncwarp();
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            uint32_t w[4];
            // bias of the chunk's 8 columns: two 16-B uniform loads (b0 is 16-B aligned)
            const float4 bl = __ldg(reinterpret_cast<const float4*>(bias + cb * 32 + 8 * c));
            const float4 bh = __ldg(reinterpret_cast<const float4*>(bias + cb * 32 + 8 * c + 4));
            const float bv[8] = {bl.x, bl.y, bl.z, bl.w, bh.x, bh.y, bh.z, bh.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int j = (8 * c + 2 * e) & 31;  // column within its block
              const float x0 = __uint_as_float(c < 4 ? ra[j] : rb[j]) + bv[2 * e];
              const float x1 = __uint_as_float(c < 4 ? ra[j + 1] : rb[j + 1]) + bv[2 * e + 1];
              __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
              w[e] = *reinterpret_cast<uint32_t*>(&h);
            }
            if (whole)
              st_shared_v4(box + lane * 128 + ((c ^ (lane & 7)) << 4), w[0], w[1], w[2], w[3]);
            else if (m0 + lane < U)
              reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(act0_) + (int64_t)(m0 + lane) * 256 +
                                       cb * 32)[c] = make_uint4(w[0], w[1], w[2], w[3]);
          }
          if (whole) {
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmO, box, cb * 32, m0);
              bulk_commit();
            }
          }
        }
        continue;
      }
      // the TMEM loads are software-pipelined one block ahead of the
      // processing, and the accumulator is released (acce) as soon as its last
      // block is in registers, before that block is processed
      uint32_t ra[32], rb[32];
      tmem_ld32_issue(tb, ra);
      tmem_ld_wait(ra);
#pragma unroll 1
      for (int cb = 0; cb < 8; cb += 2) {
        tmem_ld32_issue(tb + (cb + 1) * 32, rb);
        emit(cb, ra);
        tmem_ld_wait(rb);
        if (cb + 2 < 8) {
          tmem_ld32_issue(tb + (cb + 2) * 32, ra);
          emit(cb + 1, rb);
          tmem_ld_wait(ra);
        } else {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(lacce);
          emit(cb + 1, rb);
        }
      }
    }
    if constexpr (EPI == 2)
      if (lane == 0) bulk_wait0();  // every act0 store of this warp has completed
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 4) tmem_dealloc2(tmem, 512);
}

// ---------------------------------------------------------------------------
// backward: part[split][256][d_raw] = da0[chunk]^T X[rows[chunk]]
// grid = (d_raw/256 feature tiles, nsplit row chunks).  BK rows of K per
// stage and NST stages: 32-row stages x 6 keep as many gathered bytes in
// flight as 64 x 3 but release each slot after half the MMAs, which
// shortens the slot turnaround the HBM gather is bound by.
// ---------------------------------------------------------------------------
template <int KIND, int BK, int NST>
__global__ void __launch_bounds__(THREADS_B, 1)
    k_dw0(const __grid_constant__ CUtensorMap tmA, const void* __restrict__ pool_, int d_raw,
          const int32_t* __restrict__ rows, const int32_t* __restrict__ count, float* __restrict__ part) {
  using T = Elem<KIND>;
  constexpr int EPB = 128 / sizeof(T);       // MN-atom width (elements)
  constexpr int KROWS = 32 / sizeof(T);      // rows per MMA: 8 (tf32) / 16 (bf16)
  constexpr int NA = 128 / EPB;              // MN atoms per 128-wide half
  constexpr int CPR = 256 * sizeof(T) / 16;  // 16-B chunks per row slice
  constexpr int RPI = 128 / CPR;             // rows covered per gather round
  constexpr int NI = BK / RPI;               // gather rounds per stage (<= 32)
  constexpr uint32_t OPB_ = 256u * BK * sizeof(T);  // one operand per stage
  constexpr uint32_t STG = 2 * OPB_;
  constexpr uint32_t HALF = NA * BK * 128;   // one 128-wide half of the A operand
  static_assert(NI <= 32, "row ids are shuffled from one warp");
  // MN-major layouts: tf32 -> SWIZZLE_128B_BASE32B (4-row k groups of 512 B),
  // bf16 -> SWIZZLE_128B (8-row groups of 1024 B)
  constexpr uint32_t MN_LAYOUT = KIND == 0 ? 1u : 2u;
  constexpr uint32_t MN_SBO = KIND == 0 ? 512u : 1024u;
  const int U = *count;
  const int f0 = blockIdx.x * 256, split = blockIdx.y, nsplit = gridDim.y;
  const int per = (((U + nsplit - 1) / nsplit) + BK - 1) / BK * BK;
  const int r0 = split * per;
  const int r1 = min(U, r0 + per);
  const int nk = r1 > r0 ? (r1 - r0 + BK - 1) / BK : 0;
  float* out = part + (int64_t)split * 256 * d_raw;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (nk == 0) {  // empty chunk: its partial is zero
    for (int i = threadIdx.x; i < 256 * 256; i += THREADS_B) out[(int64_t)(i >> 8) * d_raw + f0 + (i & 255)] = 0.f;
    return;
  }
  extern __shared__ uint8_t smem_raw[];
  const uint32_t rs = smem_u32(smem_raw);
  const uint32_t base = (rs + 1023u) & ~1023u;
  const uint32_t full = base + NST * STG, empty = full + 8 * NST, acc_full = empty + 8 * NST, slot = acc_full + 8;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(full + 8 * i, 128 + 1);  // 128 gather threads (cp.async arrive) + TMA expect_tx
      mbar_init(empty + 8 * i, 1);       // tcgen05.commit
    }
    mbar_init(acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 4) {
    tmem_alloc(slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem_raw + (slot - rs));
  const T* pool = reinterpret_cast<const T*>(pool_);

  if (warp < 4) {
    // ---- gather producer: X[rows] feature slice [f0, f0+256) of BK rows.
    // Thread t owns 16-B chunk c of rows kw + i*RPI (i < NI); lane i < NI of
    // the warp fetches row id i one stage ahead and the warp shuffles it.
    const int t = threadIdx.x, c = t % CPR, kw = t / CPR;
    const T* colbase = pool + f0 + c * (16 / sizeof(T));
    const uint32_t atom_off = (c >> 3) * (BK * 128);
    auto fetch = [&](int kb) {
      const int gr = r0 + kb * BK + lane * RPI + kw;
      return (lane < NI && kb < nk && gr < r1) ? __ldg(rows + gr) : -1;
    };
    int rid_next = fetch(0);
    for (int kb = 0; kb < nk; ++kb) {
      const int rid_cur = rid_next;
      rid_next = fetch(kb + 1);
      const uint32_t st = kb % NST, itn = kb / NST;
      mbar_wait(empty + 8 * st, (itn & 1) ^ 1);
      const uint32_t bb = base + st * STG + OPB_ + atom_off;
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int rid = __shfl_sync(FULL, rid_cur, i);
        const int k = i * RPI + kw;
        // tf32 MN-major operands need the 32-B-granule 128-B swizzle
        // (Swizzle<2,5,2>: granule ^= row & 3); bf16 uses the 16-B one
        const uint32_t sw = KIND == 0 ? ((((c & 7) >> 1) ^ (k & 3)) << 5) | ((c & 1) << 4)
                                      : (((c & 7) ^ (k & 7)) << 4);
        cp_async16(bb + k * 128 + sw, colbase + (int64_t)(rid < 0 ? 0 : rid) * d_raw, rid < 0 ? 0u : 16u);
      }
      cp_async_arrive_noinc(full + 8 * st);
    }
    cp_async_wait<0>();
  } else if (warp == 5) {
    if (lane == 0) {
      // ---- TMA producer: da0 [rows, 256] MN-major atoms (EPB hidden x BK rows)
      prefetch_tmap(&tmA);
      for (int kb = 0; kb < nk; ++kb) {
        const uint32_t st = kb % NST, itn = kb / NST;
        mbar_wait(empty + 8 * st, (itn & 1) ^ 1);
        mbar_arrive_expect_tx(full + 8 * st, OPB_);
        const uint32_t a = base + st * STG;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int j = 0; j < NA; ++j)
            tma_load_2d(a + h * HALF + j * (BK * 128), &tmA, full + 8 * st, h * 128 + j * EPB, r0 + kb * BK);
      }
    }
  } else {
    if (lane == 0) {
      const uint32_t idesc = instr_desc(KIND == 0 ? 2u : 1u, 128, 256, 1, 1);
      for (int kb = 0; kb < nk; ++kb) {
        const uint32_t st = kb % NST, itn = kb / NST;
        mbar_wait(full + 8 * st, itn & 1);
        tc_fence_after();
        fence_proxy_async();
        const uint32_t a = base + st * STG, bb = a + OPB_;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int k = 0; k < BK / KROWS; ++k)
            mma<KIND>(tmem + h * 256, smem_desc(a + h * HALF + k * KROWS * 128, BK * 128, MN_SBO, MN_LAYOUT),
                      smem_desc(bb + k * KROWS * 128, BK * 128, MN_SBO, MN_LAYOUT), idesc, (kb | k) != 0);
        mma_commit(empty + 8 * st);
      }
      mma_commit(acc_full);
    }
  }
  if (warp < 4) {
    mbar_wait(acc_full, 0);
    tc_fence_after();
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const int hid = h * 128 + warp * 32 + lane;
#pragma unroll 1
      for (int cb = 0; cb < 8; ++cb) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + h * 256 + cb * 32, v);
        float4* o = reinterpret_cast<float4*>(out + (int64_t)hid * d_raw + f0 + cb * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------
// backward on CTA pairs (bf16): a pair covers 512 features of dW0 for one row
// chunk.  M = 256 hidden units split over the pair (each CTA TMA-loads its 128
// columns of da0), N = 2 x 256 features (each CTA gathers its 2 x 128-feature
// halves of the X rows); both N halves accumulate in each CTA's 512 TMEM
// columns.  da0 is thereby read once per 512 features instead of once per
// 256.  The peer's stage completion is relayed to the leader's barrier, whose
// MMA commits multicast to both CTAs.
// ---------------------------------------------------------------------------
template <int BK, int NST>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS_B, 1)
    k_dw0p(const __grid_constant__ CUtensorMap tmA, const void* __restrict__ pool_, int d_raw,
           const int32_t* __restrict__ rows, const int32_t* __restrict__ count, float* __restrict__ part) {
  using T = __nv_bfloat16;
  constexpr int EPB = 64;    // MN-atom width (bf16 elements)
  constexpr int KROWS = 16;  // rows per MMA
  constexpr int CPR = 32;    // 16-B chunks per row: 2 segments x 128 features
  constexpr int RPI = 128 / CPR;
  constexpr int NI = BK / RPI;
  constexpr uint32_t OPA = 128u * BK * 2;  // this CTA's 128 hidden columns of da0
  constexpr uint32_t OPB_ = 256u * BK * 2;  // this CTA's 256 features of X
  constexpr uint32_t STG = OPA + OPB_;
  static_assert(NI <= 32, "row ids are shuffled from one warp");
  const int U = *count;
  const uint32_t rank = cluster_ctarank();
  const int F0 = (blockIdx.x >> 1) * 512, split = blockIdx.y, nsplit = gridDim.y;
  const int per = (((U + nsplit - 1) / nsplit) + BK - 1) / BK * BK;
  const int r0 = split * per;
  const int r1 = min(U, r0 + per);
  const int nk = r1 > r0 ? (r1 - r0 + BK - 1) / BK : 0;
  float* out = part + (int64_t)split * 256 * d_raw;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (nk == 0) {  // empty chunk (uniform across the pair): this CTA's partial rows are zero
    for (int i = threadIdx.x; i < 128 * 512; i += THREADS_B)
      out[(int64_t)(rank * 128 + (i >> 9)) * d_raw + F0 + (i & 511)] = 0.f;
    return;
  }
  extern __shared__ uint8_t smem_raw[];
  const uint32_t rs = smem_u32(smem_raw);
  const uint32_t base = (rs + 1023u) & ~1023u;
  const uint32_t full = base + NST * STG, empty = full + 8 * NST, acc_full = empty + 8 * NST, slot = acc_full + 8;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(full + 8 * i, 128 + 1 + (rank == 0 ? 1 : 0));  // gathers + TMA expect_tx (+ the peer's relay)
      mbar_init(empty + 8 * i, 1);                             // pair MMA commit (multicast)
    }
    mbar_init(acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 4) {
    tmem_alloc2(slot, 512);
    tmem_relinquish2();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem_raw + (slot - rs));
  const T* pool = reinterpret_cast<const T*>(pool_);

  if (warp < 4) {
    // ---- gather producer: X[rows] features F0 + j*256 + rank*128 + [0,128), j = 0, 1
    const int t = threadIdx.x, c = t % CPR, kw = t / CPR;
    const T* colbase = pool + F0 + (c >> 4) * 256 + (int)rank * 128 + (c & 15) * 8;
    const uint32_t atom_off = (c >> 3) * (BK * 128);
    auto fetch = [&](int kb) {
      const int gr = r0 + kb * BK + lane * RPI + kw;
      return (lane < NI && kb < nk && gr < r1) ? __ldg(rows + gr) : -1;
    };
    int rid_next = fetch(0);
    for (int kb = 0; kb < nk; ++kb) {
      const int rid_cur = rid_next;
      rid_next = fetch(kb + 1);
      const uint32_t st = kb % NST, itn = kb / NST;
      mbar_wait(empty + 8 * st, (itn & 1) ^ 1);
      const uint32_t bb = base + st * STG + OPA + atom_off;
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int rid = __shfl_sync(FULL, rid_cur, i);
        const int k = i * RPI + kw;
        const uint32_t sw = ((c & 7) ^ (k & 7)) << 4;
        cp_async16(bb + k * 128 + sw, colbase + (int64_t)(rid < 0 ? 0 : rid) * d_raw, rid < 0 ? 0u : 16u);
      }
      cp_async_arrive_noinc(full + 8 * st);
    }
    cp_async_wait<0>();
  } else if (warp == 5) {
    if (lane == 0) {
      // ---- TMA producer: da0 columns rank*128 .. +127 (two MN atoms of 64 hidden x BK rows)
      prefetch_tmap(&tmA);
      for (int kb = 0; kb < nk; ++kb) {
        const uint32_t st = kb % NST, itn = kb / NST;
        mbar_wait(empty + 8 * st, (itn & 1) ^ 1);
        mbar_arrive_expect_tx(full + 8 * st, OPA);
        const uint32_t a = base + st * STG;
#pragma unroll
        for (int j = 0; j < 2; ++j)
          tma_load_2d(a + j * (BK * 128), &tmA, full + 8 * st, (int)rank * 128 + j * EPB, r0 + kb * BK);
      }
    }
  } else {
    if (lane == 0) {
      if (rank == 0) {
        const uint32_t idesc = instr_desc(1u, 256, 256, 1, 1);
        for (int kb = 0; kb < nk; ++kb) {
          const uint32_t st = kb % NST, itn = kb / NST;
          mbar_wait(full + 8 * st, itn & 1);
          tc_fence_after();
          fence_proxy_async();
          const uint32_t a = base + st * STG, bb = a + OPA;
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int k = 0; k < BK / KROWS; ++k)
              mma2<1>(tmem + j * 256, smem_desc(a + k * KROWS * 128, BK * 128, 1024u, 2u),
                      smem_desc(bb + j * 2 * (BK * 128) + k * KROWS * 128, BK * 128, 1024u, 2u), idesc,
                      (kb | k) != 0);
          mma_commit2(empty + 8 * st, 0x3);
        }
        mma_commit2(acc_full, 0x3);
      } else {
        // ---- relay (peer): this CTA's stage landed -> the leader's full barrier
        const uint32_t lfull = mapa(full, 0);
        for (int kb = 0; kb < nk; ++kb) {
          const uint32_t st = kb % NST, itn = kb / NST;
          mbar_wait(full + 8 * st, itn & 1);
          fence_proxy_async();
          mbar_arrive_cluster(lfull + 8 * st);
        }
      }
    }
  }
  if (warp < 4) {
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const int hid = (int)rank * 128 + warp * 32 + lane;
#pragma unroll 1
    for (int j = 0; j < 2; ++j)
#pragma unroll 1
      for (int cb = 0; cb < 8; ++cb) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + j * 256 + cb * 32, v);
        float4* o = reinterpret_cast<float4*>(out + (int64_t)hid * d_raw + F0 + j * 256 + cb * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 4) tmem_dealloc2(tmem, 512);
}

template <int BK, int NST>
constexpr size_t dw0p_smem() {
  return (size_t)NST * (128u * BK * 2 + 256u * BK * 2) + 1024 + 256;
}

template <int KIND, int BK, int NST>
constexpr size_t dw0_smem() {
  return (size_t)NST * 2 * 256 * BK * (KIND == 0 ? 4 : 2) + 1024 + 256;
}

__global__ void k_sum_splits(const float* __restrict__ part, int nsplit, int64_t n, float* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n / 4; j += (int64_t)gridDim.x * blockDim.x) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < nsplit; ++s) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(part + (int64_t)s * n) + j);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    reinterpret_cast<float4*>(out)[j] = acc;
  }
}

__global__ void k_to_bf16(const float* __restrict__ in, const int32_t* __restrict__ count, int64_t row_width,
                          int64_t n_max, __nv_bfloat16* __restrict__ out) {
  int64_t n = n_max;
  if (count) n = min(n, (int64_t)*count * row_width);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n / 2; i += (int64_t)gridDim.x * blockDim.x) {
    const float2 v = reinterpret_cast<const float2*>(in)[i];
    reinterpret_cast<__nv_bfloat162*>(out)[i] = __floats2bfloat162_rn(v.x, v.y);
  }
}

// ---- host helpers -------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D row-major [rows, cols] map, box = [box_rows, 128 bytes], 128-B swizzle
int make_map(CUtensorMap* m, const void* ptr, bool bf16, uint64_t rows, uint64_t cols, uint32_t box_rows,
             CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto fn = encode_fn();
  if (!fn) return fail(DICM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const uint32_t esz = bf16 ? 2 : 4;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * esz};
  cuuint32_t box[2] = {128 / esz, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr),
                  dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DICM_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return DICM_OK;
}

int nsplit_for(int64_t rows_max, int d_raw) {
  const int tiles = d_raw / 256;
  const int64_t want = std::max<int64_t>(dicm_grid_cap() / tiles, 1);  // one wave of CTAs
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (rows_max + 255) / 256));
}

struct TcWs {
  __nv_bfloat16 *w0_bf16, *da0_bf16;
  float* part;
};

size_t carve_ws(int64_t rows_max, int d_raw, TcWs* w, char* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* p = base ? base + off : nullptr;
    off += (bytes + 1023) / 1024 * 1024;
    return p;
  };
  TcWs t;
  t.w0_bf16 = (__nv_bfloat16*)take((size_t)256 * d_raw * 2);
  t.da0_bf16 = (__nv_bfloat16*)take((size_t)std::max<int64_t>(rows_max, 1) * 256 * 2);
  t.part = (float*)take((size_t)nsplit_for(rows_max, d_raw) * 256 * d_raw * 4);
  if (w) *w = t;
  return off;
}

template <typename K>
int set_smem(K kernel) {
  return check_cuda(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES),
                    "tcgen05 kernel smem attribute");
}

}  // namespace

size_t workspace_bytes(int64_t rows_max, int d_raw) { return carve_ws(rows_max, d_raw, nullptr, nullptr); }

__nv_bfloat16* da0_bf16_ptr(void* ws, int64_t rows_max, int d_raw) {
  TcWs w;
  carve_ws(rows_max, d_raw, &w, (char*)ws);
  return w.da0_bf16;
}

int fwd_layer0(const void* pool, int pool_dtype, int d_raw, const int32_t* rows, const int32_t* count,
               int64_t rows_max, const float* w0, const float* b0, float* act0, int precision, void* ws,
               cudaStream_t st) {
  const bool bf16 = precision == DICM_PREC_BF16;
  if (bf16 != (pool_dtype == DICM_POOL_BF16))
    return fail(DICM_ERR_VALUE, "precision %s needs a %s pool", bf16 ? "bf16" : "tf32", bf16 ? "bf16" : "fp32");
  if (d_raw % 256) return fail(DICM_ERR_SHAPE, "tcgen05 layer 0: d_raw %d not a multiple of 256", d_raw);
  TcWs w;
  carve_ws(rows_max, d_raw, &w, (char*)ws);
  CUtensorMap map;
  int rc;
  const void* wsrc = w0;
  if (bf16) {
    k_to_bf16<<<dicm_grid(256 * d_raw / 2, 256, 148 * 4), 256, 0, st>>>(w0, nullptr, 0, (int64_t)256 * d_raw,
                                                                          w.w0_bf16);
    wsrc = w.w0_bf16;
  }
  static const bool pair = [] {
    const char* e = getenv("DICM_FWD_PAIR");
    return !(e && e[0] == '0');
  }();
  if (pair) {
    if ((rc = make_map(&map, wsrc, bf16, 256, d_raw, 128))) return rc;
    // persistent CTA pairs: <= 74 clusters of 2 (one CTA per SM)
    const int grid = 2 * (int)std::min<int64_t>(std::max<int64_t>(dicm_grid_cap() / 2, 1), (rows_max + 255) / 256);
    // ring depths: 6 gather slots and 6 W0 slots; deeper rings (8/5, 7/6)
    // measured no faster (the pipeline is not bound by stage turnaround)
    static int a66 = -1, t66 = -1;
    auto launch = [&](auto kern, size_t bytes, int& attr) -> int {
      if (attr < 0)
        attr = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes),
                          "k_fwd2 smem");
      if (attr) return attr;
      kern<<<grid, THREADS_F, bytes, st>>>(map, pool, d_raw, rows, count, b0, act0);
      return 0;
    };
    // default: 512-row pair tiles (k_fwd4); DICM_FWD4=0 selects the 256-row
    // tiles with double-buffered accumulators (k_fwd2)
    static const bool four = !(getenv("DICM_FWD4") && getenv("DICM_FWD4")[0] == '0');
    // DICM_FWD4_EPI: act0 epilogue mode (see k_fwd4): 2 (TMA store, default), 1, 0
    static const int epi_mode = [] {
      const char* e = getenv("DICM_FWD4_EPI");
      return e && (e[0] == '0' || e[0] == '1') ? e[0] - '0' : 2;
    }();
    static int a44 = -1, t44 = -1, a44n = -1, a44t = -1, t44t = -1;
    // the TMA-store epilogue reads the bias as float4: an unaligned b0 takes mode 1
    const int em = (epi_mode == 2 && ((uintptr_t)b0 & 15)) ? 1 : epi_mode;
    CUtensorMap omap{};
    if (em == 2 && (rc = make_map(&omap, act0, bf16, (uint64_t)rows_max, 256, 32))) return rc;
    auto launch4 = [&](auto kern, size_t bytes, int& attr) -> int {
      if (attr < 0)
        attr = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes),
                          "k_fwd4 smem");
      if (attr) return attr;
      const int grid4 = 2 * (int)std::min<int64_t>(std::max<int64_t>(dicm_grid_cap() / 2, 1), (rows_max + 511) / 512);
      kern<<<grid4, THREADS_F4, bytes, st>>>(map, omap, pool, d_raw, rows, count, b0, act0);
      return 0;
    };
    const int probe_slot = probe_begin(DICM_PROBE_IMG_FWD_L0, st);
    const int lrc = four ? (bf16 ? (em == 1   ? launch4(k_fwd4<1, 4, 4, 1>, smem4(4, 4, 1), a44)
                                    : em == 2 ? launch4(k_fwd4<1, 4, 4, 2>, smem4(4, 4, 2), a44t)
                                                    : launch4(k_fwd4<1, 4, 4, 0>, smem4(4, 4, 0), a44n))
                                 : (em == 2 ? launch4(k_fwd4<0, 4, 4, 2>, smem4(4, 4, 2), t44t)
                                            : launch4(k_fwd4<0, 4, 4, 1>, smem4(4, 4, 1), t44)))
                         : (bf16 ? launch(k_fwd2<1, 6, 6>, smem2(6, 6), a66) : launch(k_fwd2<0, 6, 6>, smem2(6, 6), t66));
    probe_end(probe_slot, st);
    if (lrc) return lrc;
    return last_launch("tcgen05 layer-0 forward (CTA pairs)");
  }
  if ((rc = make_map(&map, wsrc, bf16, 256, d_raw, 256))) return rc;
  const int grid = (int)std::min<int64_t>(dicm_grid_cap(), (rows_max + 255) / 256);  // persistent: <= one CTA per SM
  if (bf16) {
    static int once = set_smem(k_fwd<1>);
    if (once) return once;
    const int probe_slot = probe_begin(DICM_PROBE_IMG_FWD_L0, st);
    k_fwd<1><<<grid, THREADS_F, SMEM_BYTES, st>>>(map, pool, d_raw, rows, count, b0, act0);
    probe_end(probe_slot, st);
  } else {
    static int once = set_smem(k_fwd<0>);
    if (once) return once;
    const int probe_slot = probe_begin(DICM_PROBE_IMG_FWD_L0, st);
    k_fwd<0><<<grid, THREADS_F, SMEM_BYTES, st>>>(map, pool, d_raw, rows, count, b0, act0);
    probe_end(probe_slot, st);
  }
  return last_launch("tcgen05 layer-0 forward");
}

int bwd_dw0(const void* pool, int pool_dtype, int d_raw, const int32_t* rows, const int32_t* count,
            int64_t rows_max, const float* da0, float* gw0, int precision, void* ws, cudaStream_t st,
            bool da0_bf16_ready) {
  const bool bf16 = precision == DICM_PREC_BF16;
  if (bf16 != (pool_dtype == DICM_POOL_BF16))
    return fail(DICM_ERR_VALUE, "precision %s needs a %s pool", bf16 ? "bf16" : "tf32", bf16 ? "bf16" : "fp32");
  if (d_raw % 256) return fail(DICM_ERR_SHAPE, "tcgen05 layer 0: d_raw %d not a multiple of 256", d_raw);
  TcWs w;
  carve_ws(rows_max, d_raw, &w, (char*)ws);
  const void* asrc = da0;
  if (bf16) {
    if (!da0_bf16_ready)
      k_to_bf16<<<dicm_grid(rows_max * 128, 256, 148 * 8), 256, 0, st>>>(da0, count, 256, rows_max * 256, w.da0_bf16);
    asrc = w.da0_bf16;
  }
  CUtensorMap map;
  int rc;
  constexpr int BKB = 64, NSB = 3;  // bf16: 64-row stages x 3 (32 x 6 measured slower: 1.10 vs 0.89 ms)
  constexpr int BKT = 32, NST_ = 3;  // tf32: 32-row stages x 3 (32 KB + 32 KB each)
  const uint32_t box_rows = bf16 ? BKB : BKT;
  if ((rc = make_map(&map, asrc, bf16, (uint64_t)rows_max, 256, box_rows,
                     bf16 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)))
    return rc;
  const int nsplit = nsplit_for(rows_max, d_raw);
  dim3 grid(d_raw / 256, nsplit);
  static const bool pairs = !(getenv("DICM_DW0_PAIR") && getenv("DICM_DW0_PAIR")[0] == '0');
  if (bf16 && pairs && d_raw % 512 == 0) {
    constexpr int NSP = 4;  // 4 x 48 KB stages
    static int once = check_cuda(cudaFuncSetAttribute(k_dw0p<BKB, NSP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      (int)dw0p_smem<BKB, NSP>()), "k_dw0p smem");
    if (once) return once;
    const int probe_slot = probe_begin(DICM_PROBE_IMG_BWD_DW0, st);
    k_dw0p<BKB, NSP><<<grid, THREADS_B, dw0p_smem<BKB, NSP>(), st>>>(map, pool, d_raw, rows, count, w.part);
    probe_end(probe_slot, st);
  } else if (bf16) {
    static int once = check_cuda(cudaFuncSetAttribute(k_dw0<1, BKB, NSB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      (int)dw0_smem<1, BKB, NSB>()), "k_dw0 smem");
    if (once) return once;
    const int probe_slot = probe_begin(DICM_PROBE_IMG_BWD_DW0, st);
    k_dw0<1, BKB, NSB><<<grid, THREADS_B, dw0_smem<1, BKB, NSB>(), st>>>(map, pool, d_raw, rows, count, w.part);
    probe_end(probe_slot, st);
  } else {
    static int once = check_cuda(cudaFuncSetAttribute(k_dw0<0, BKT, NST_>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      (int)dw0_smem<0, BKT, NST_>()), "k_dw0 smem");
    if (once) return once;
    const int probe_slot = probe_begin(DICM_PROBE_IMG_BWD_DW0, st);
    k_dw0<0, BKT, NST_><<<grid, THREADS_B, dw0_smem<0, BKT, NST_>(), st>>>(map, pool, d_raw, rows, count, w.part);
    probe_end(probe_slot, st);
  }
  const int64_t n = (int64_t)256 * d_raw;
  k_sum_splits<<<dicm_grid(n / 4, 256, 148 * 8), 256, 0, st>>>(w.part, nsplit, n, gw0);
  return last_launch("tcgen05 layer-0 backward");
}

}  // namespace sm100
}  // namespace dicm
