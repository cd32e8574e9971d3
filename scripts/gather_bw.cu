// Microbenchmark: HBM bandwidth of the layer-0 row gather pattern.
// 148 persistent CTAs; a tile = 128 sorted-unique pool rows (bf16, 8 KB each);
// the tile is streamed k-block by k-block (CHUNK bytes of every row per
// stage) through a STAGES-deep cp.async ring with mbarrier arrivals -- the
// k_fwd access pattern without the MMA.  Prints GB/s per (CHUNK, STAGES).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 scripts/gather_bw.cu -o build/gather_bw
#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>
#include <cudaTypedefs.h>
#include "../paper_1711_06505_b200/csrc/tc_ptx.cuh"

using namespace dicm::tc;

template <int CHUNK, int STAGES, int WTMA>
__global__ void __launch_bounds__(192, 1) gather(const __grid_constant__ CUtensorMap tmW, const uint8_t* pool,
                                                 const int* rows, int U, int row_bytes, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  constexpr uint32_t SLOT = 128 * CHUNK + (WTMA ? 16384 : 0);
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const int ntiles = (U + 127) / 128, nk = row_bytes / CHUNK;
  const int t = threadIdx.x, warp = t >> 5;
  if (t == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(smem_u32(&full[i]), 128 + (WTMA ? 1 : 0));
      mbar_init(smem_u32(&empty[i]), 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp < 4) {
    constexpr int CPR = CHUNK / 16;      // 16-B pieces per row per stage
    constexpr int RPP = 128 / CPR;       // rows covered per pass of 128 threads
    const int c = t % CPR, rb = t / CPR;
    uint32_t g = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const uint32_t s = g % STAGES, it = g / STAGES;
        mbar_wait(smem_u32(&empty[s]), (it & 1) ^ 1);
        for (int r = rb; r < 128; r += RPP) {
          const int gr = tile * 128 + r;
          const bool v = gr < U;
          const uint8_t* src = pool + (size_t)(v ? rows[gr] : 0) * row_bytes + kb * CHUNK + c * 16;
          cp_async16(base + s * SLOT + r * CHUNK + c * 16, src, v ? 16u : 0u);
        }
        cp_async_arrive_noinc(smem_u32(&full[s]));
      }
    }
    cp_async_wait<0>();
  } else if (WTMA && t == 160) {
    uint32_t g = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const uint32_t s = g % STAGES, it = g / STAGES;
        mbar_wait(smem_u32(&empty[s]), (it & 1) ^ 1);
        mbar_arrive_expect_tx(smem_u32(&full[s]), 16384);
        tma_load_2d(base + s * SLOT + 128 * CHUNK, &tmW, smem_u32(&full[s]), (kb % 64) * 64, (blockIdx.x & 1) * 128);
      }
  } else if (t == 128) {
    uint32_t g = 0;
    unsigned long long acc = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const uint32_t s = g % STAGES, it = g / STAGES;
        mbar_wait(smem_u32(&full[s]), it & 1);
        acc += *reinterpret_cast<volatile uint32_t*>(smem + (base - smem_u32(smem)) + s * SLOT);
        if (WTMA == 2)
          mma_commit(smem_u32(&empty[s]));  // release through the tensor-core commit path
        else
          mbar_arrive(smem_u32(&empty[s]));
      }
    sink[blockIdx.x] = acc;
  }
}

CUtensorMap g_map, g_pool_map;

// the same k-block-by-k-block gather issued by ONE thread as TMA tile::gather4
// (4 rows x 128 B per instruction) into a STAGES-deep ring
template <int STAGES>
__global__ void __launch_bounds__(64, 1) gather_tma(const __grid_constant__ CUtensorMap pm, const int* rows, int U,
                                                   unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  __shared__ int rid[128];
  constexpr uint32_t SLOT = 128 * 128;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const int ntiles = (U + 127) / 128, nk = 64;
  const int t = threadIdx.x;
  if (t == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(smem_u32(&full[i]), 1);
      mbar_init(smem_u32(&empty[i]), 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (t < 32) {
    uint32_t g = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      for (int i = t; i < 128; i += 32) {
        const int gr = tile * 128 + i;
        rid[i] = gr < U ? rows[gr] : 0;
      }
      __syncwarp();
      if (t == 0) {
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const uint32_t s = g % STAGES, it = g / STAGES;
          mbar_wait(smem_u32(&empty[s]), (it & 1) ^ 1);
          mbar_arrive_expect_tx(smem_u32(&full[s]), SLOT);
          for (int q = 0; q < 32; ++q)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(base + s * SLOT + q * 512),
                "l"(&pm), "r"(kb * 64), "r"(rid[4 * q]), "r"(rid[4 * q + 1]), "r"(rid[4 * q + 2]),
                "r"(rid[4 * q + 3]), "r"(smem_u32(&full[s]))
                : "memory");
        }
      }
      __syncwarp();
    }
  } else if (t == 32) {
    uint32_t g = 0;
    unsigned long long acc = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const uint32_t s = g % STAGES, it = g / STAGES;
        mbar_wait(smem_u32(&full[s]), it & 1);
        acc += *reinterpret_cast<volatile uint32_t*>(smem + (base - smem_u32(smem)) + s * SLOT);
        mbar_arrive(smem_u32(&empty[s]));
      }
    sink[blockIdx.x] = acc;
  }
}

template <int STAGES>
void run_tma(const int* rows, int U, unsigned long long* sink) {
  const size_t smem = 1024 + (size_t)STAGES * 128 * 128;
  cudaFuncSetAttribute(gather_tma<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  gather_tma<STAGES><<<148, 64, smem>>>(g_pool_map, rows, U, sink);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) gather_tma<STAGES><<<148, 64, smem>>>(g_pool_map, rows, U, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("TMA gather4 128 B/row/stage, %2d stages: %7.1f GB/s  %s\n", STAGES, (double)U * 8192 * reps / (ms * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

template <int CHUNK, int STAGES, int WTMA = 0>
void run(const uint8_t* pool, const int* rows, int U, int row_bytes, unsigned long long* sink) {
  const size_t smem = 1024 + (size_t)STAGES * (128 * CHUNK + (WTMA ? 16384 : 0));
  cudaFuncSetAttribute(gather<CHUNK, STAGES, WTMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  gather<CHUNK, STAGES, WTMA><<<148, 192, smem>>>(g_map, pool, rows, U, row_bytes, sink);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) gather<CHUNK, STAGES, WTMA><<<148, 192, smem>>>(g_map, pool, rows, U, row_bytes, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)U * row_bytes * reps;
  printf("chunk %4d B/row/stage, %2d stages, W0 TMA %d (%3zu KB smem): %7.1f GB/s  %s\n", CHUNK, STAGES, WTMA, smem / 1024,
         bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int P = 1000000, row_bytes = 8192, U = 561000;
  uint8_t* pool;
  cudaMalloc(&pool, (size_t)P * row_bytes);
  cudaMemset(pool, 1, (size_t)P * row_bytes);
  std::vector<int> all(P);
  for (int i = 0; i < P; ++i) all[i] = i;
  std::mt19937 rng(1);
  std::shuffle(all.begin(), all.end(), rng);
  std::vector<int> h(all.begin(), all.begin() + U);
  std::sort(h.begin(), h.end());  // the dedup emits sorted unique ids
  int* rows;
  cudaMalloc(&rows, U * 4);
  cudaMemcpy(rows, h.data(), U * 4, cudaMemcpyHostToDevice);
  unsigned long long* sink;
  cudaMalloc(&sink, 148 * 8);
  {  // a 2 MB "W0" [256 x 4096] bf16, box 64 x 128, SW128
    void* w;
    cudaMalloc(&w, 256 * 4096 * 2);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    cuuint64_t dims[2] = {4096, 256}, strides[1] = {4096 * 2};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn)(&g_map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims,
        strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    cuuint64_t dims[2] = {4096, (cuuint64_t)P}, strides[1] = {4096 * 2};
    cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
    CUresult r = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn)(&g_pool_map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
        pool, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("pool map encode: %d\n", (int)r);
  }
  run_tma<6>(rows, U, sink);
  run_tma<8>(rows, U, sink);
  run_tma<12>(rows, U, sink);
  run<128, 6, 1>(pool, rows, U, row_bytes, sink);
  run<128, 6>(pool, rows, U, row_bytes, sink);
  run<128, 8>(pool, rows, U, row_bytes, sink);
  run<128, 12>(pool, rows, U, row_bytes, sink);
  run<256, 3>(pool, rows, U, row_bytes, sink);
  run<256, 6>(pool, rows, U, row_bytes, sink);
  run<512, 3>(pool, rows, U, row_bytes, sink);
  // a plain copy-rate reference: the same bytes read contiguously (rows 0..U-1)
  std::vector<int> seq(U);
  for (int i = 0; i < U; ++i) seq[i] = i;
  cudaMemcpy(rows, seq.data(), U * 4, cudaMemcpyHostToDevice);
  printf("-- contiguous rows --\n");
  run<128, 6>(pool, rows, U, row_bytes, sink);
  run<128, 12>(pool, rows, U, row_bytes, sink);
  run<512, 3>(pool, rows, U, row_bytes, sink);
  return 0;
}
