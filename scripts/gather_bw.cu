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

CUtensorMap g_map;

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
  run<128, 6, 1>(pool, rows, U, row_bytes, sink);
  run<128, 6, 2>(pool, rows, U, row_bytes, sink);
  run<128, 4, 2>(pool, rows, U, row_bytes, sink);
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
