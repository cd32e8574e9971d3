// Microbenchmark: sustained tcgen05.mma throughput per SM (kind::f16, bf16
// operands from shared memory, fp32 accumulate in TMEM), one CTA per SM,
// no global traffic.  Variants: K-major / MN-major operands, N = 64..256.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 scripts/mma_rate.cu -o build/mma_rate
#include <cstdio>
#include <cuda_bf16.h>
#include "../paper_1711_06505_b200/csrc/tc_ptx.cuh"

using namespace dicm::tc;

// smem: A 128 rows x 64 k (16 KB), B 256 rows x 64 k (32 KB), bf16 SW128
__device__ float g_src1[65536 * 4];
__device__ unsigned long long g_fill1;
__global__ void __launch_bounds__(256, 1) rate(int iters, int N, int mn, long long* cycles, int fill) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t A = base, B = base + 16384;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem + (base - smem_u32(smem)))[i] = 0x3f803f80u * ((i & 7) == 0);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) {
    tmem_alloc(smem_u32(&slot), 512);
    tmem_relinquish();
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  volatile int* stop1 = reinterpret_cast<volatile int*>(smem + (base - smem_u32(smem)) + 49152);
  if (threadIdx.x == 0) *stop1 = 0;
  __syncthreads();
  if (threadIdx.x >= 128 && fill) {
    const uint32_t dst = base + 49152 + 1024;
    const int i = threadIdx.x - 128;
    int k = 0;
    while (!*stop1) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        cp_async16(dst + (((i + j * 128) & 4095) << 4), g_src1 + (((size_t)(k * 2048 + i + j * 128)) & 65535) * 4, 16);
      cp_async_commit();
      cp_async_wait<4>();
      ++k;
    }
    cp_async_wait<0>();
    atomicAdd(&g_fill1, (unsigned long long)k * 16 * 16);
  }
  if (threadIdx.x == 0) {
    const uint32_t idesc = instr_desc(1, 128, N, mn, mn);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint64_t da, db;
        if (mn) {  // MN-major: 8-row k groups of 1024 B, atoms of 64 elements (LBO = atom stride)
          da = smem_desc(A + k * 2048, 8192, 1024, 2);
          db = smem_desc(B + k * 2048, 8192, 1024, 2);
        } else {
          da = smem_desc(A + k * 32, 16, 1024, 2);
          db = smem_desc(B + k * 32, 16, 1024, 2);
        }
        mma<1>(tmem + (it & 1) * 256, da, db, idesc, 1);
      }
    }
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    const long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
    *stop1 = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

__device__ float g_src[65536 * 4];  // 1 MB, L2-resident fill source
__device__ const float* g_big;     // 4 GB HBM fill source (fill == 3)
__device__ unsigned long long g_fill_bytes;

// pair (cta_group::2) MMA rate; `fill` warps stream STS.128 into a spare
// smem region meanwhile (simulated operand fills), `fill_bytes` per MMA slot
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    rate2(int iters, int N, int fill, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t A = base, B = base + 16384;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem + (base - smem_u32(smem)))[i] = 0x3f803f80u * ((i & 7) == 0);
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) {
    tmem_alloc2(smem_u32(&slot), 512);
    tmem_relinquish2();
  }
  fence_proxy_async();
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  volatile int* stop = reinterpret_cast<volatile int*>(smem + (base - smem_u32(smem)) + 65536);
  if (threadIdx.x == 0) *stop = 0;
  __syncthreads();
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t idesc = instr_desc(1, 256, N, 0, 0);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma2<1>(tmem + (it & 1) * 256, smem_desc(A + k * 32, 16, 1024), smem_desc(B + k * 32, 16, 1024), idesc, 1);
    }
    mma_commit2(smem_u32(&bar), 0x3);
    mbar_wait(smem_u32(&bar), 0);
    const long long t1 = clock64();
    cycles[blockIdx.x >> 1] = t1 - t0;
    *stop = 1;
  } else if (threadIdx.x == 0 && rank == 1) {
    mbar_wait(smem_u32(&bar), 0);
    *stop = 1;
  } else if (threadIdx.x >= 128 && fill == 1) {
    // 4 warps hammer a 64 KB smem region with 16-B stores until the MMAs finish
    uint4* p = reinterpret_cast<uint4*>(smem + (base - smem_u32(smem)) + 65536 + 1024);
    const uint4 v = make_uint4(1, 2, 3, 4);
    int i = threadIdx.x - 128;
    while (!*stop) {
#pragma unroll 8
      for (int j = 0; j < 64; ++j) p[(i + j * 128) & 4095] = v;
    }
  } else if (threadIdx.x >= 128 && fill >= 2) {
    // 4 warps stream cp.async (LDGSTS) 16-B copies from an L2-resident 1 MB
    // buffer into a 64 KB smem region: the operand-fill traffic of a GEMM
    const uint32_t dst = base + 65536 + 1024;
    const int i = threadIdx.x - 128;
    int k = 0;
    const float* src = fill == 3 ? g_big + (size_t)blockIdx.x * (1 << 22) : g_src;
    const size_t mask = fill == 3 ? ((size_t)1 << 22) / 4 - 1 : 65535;
    while (!*stop) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        cp_async16(dst + (((i + j * 128) & 4095) << 4), src + (((size_t)(k * 2048 + i + j * 128)) & mask) * 4, 16);
      cp_async_commit();
      cp_async_wait<4>();
      ++k;
    }
    cp_async_wait<0>();
    if (fill >= 2) atomicAdd(&g_fill_bytes, (unsigned long long)k * 16 * 16);
  }
  tc_fence_before();
  cluster_sync();
  if (threadIdx.x < 32) tmem_dealloc2(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  const int iters = 20000;
  for (int fill = 0; fill < 2; ++fill)
  for (int mn = 0; mn < 2; ++mn)
    for (int N : {256}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      rate<<<148, 256, 128 * 1024>>>(100, N, mn, d, fill);
      unsigned long long z1 = 0;
      cudaMemcpyToSymbol(g_fill1, &z1, sizeof(z1));
      cudaEventRecord(e0);
      rate<<<148, 256, 128 * 1024>>>(iters, N, mn, d, fill);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double cyc = 0;
      for (int i = 0; i < 148; ++i) cyc += h[i];
      cyc /= 148;
      const double n_mma = 4.0 * iters;
      const double flops = 2.0 * 128 * N * 16 * n_mma * 148;
      unsigned long long fb1 = 0;
      cudaMemcpyFromSymbol(&fb1, g_fill1, sizeof(fb1));
      printf("%s N=%3d fill=%d: %.1f cycles/MMA (floor %d), %.0f TFLOP/s (%.3f ms), fills %.1f B/clk/SM err=%s\n",
             mn ? "MN-major" : "K-major ", N, fill, cyc / n_mma, N / 2, flops / (ms * 1e-3) / 1e12, ms,
             fb1 / 148.0 / cyc, cudaGetErrorString(cudaGetLastError()));
    }
  cudaFuncSetAttribute(rate2, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  float* big;
  cudaMalloc(&big, (size_t)148 << 24);
  cudaMemset(big, 0, (size_t)148 << 24);
  cudaMemcpyToSymbol(g_big, &big, sizeof(big));
  for (int fill = 0; fill < 4; ++fill)
    for (int N : {128, 256}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      rate2<<<148, 256, 140 * 1024>>>(100, N, fill, d);
      cudaEventRecord(e0);
      rate2<<<148, 256, 140 * 1024>>>(iters, N, fill, d);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      long long h[74];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double cyc = 0;
      for (int i = 0; i < 74; ++i) cyc += h[i];
      cyc /= 74;
      const double n_mma = 4.0 * iters;
      const double flops = 2.0 * 256 * N * 16 * n_mma * 74;
      unsigned long long fb = 0;
      cudaMemcpyFromSymbol(&fb, g_fill_bytes, sizeof(fb));
      unsigned long long z = 0;
      cudaMemcpyToSymbol(g_fill_bytes, &z, sizeof(z));
      printf("pair M256 N=%3d fill=%d: %.1f cycles/MMA, %.0f TFLOP/s, fills %.1f B/clk/SM  err=%s\n", N, fill,
             cyc / n_mma, flops / (ms * 1e-3) / 1e12, fb / 2.0 / 148.0 / cyc, cudaGetErrorString(cudaGetLastError()));
    }
  // single-CTA with smem fill pressure for comparison
  return 0;
}
