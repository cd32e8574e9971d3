// Microbenchmark: does tcgen05.mma traffic slow TMA (bulk) or LDGSTS operand
// fills into shared memory?  One CTA per SM.  Thread 0 either issues
// M128xN256xK16 bf16 MMAs back to back (mma = 1) or idles for the same number
// of cycles (mma = 0); meanwhile warp 1 streams 16 KB bulk copies (fill = 1,
// cp.async.bulk from an L2-resident source) or 4 warps stream cp.async 16-B
// copies (fill = 2, HBM source), and the fill rate is reported in B/clk/SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 scripts/tma_vs_mma.cu -o build/tma_vs_mma
#include <cstdio>
#include <cuda_bf16.h>
#include "../paper_1711_06505_b200/csrc/tc_ptx.cuh"

using namespace dicm::tc;

__device__ float g_l2src[65536 * 4];  // 1 MB
__device__ const float* g_hbm;        // 148 x 16 MB
__device__ unsigned long long g_bytes;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__global__ void __launch_bounds__(256, 1) k(int iters, int use_mma, int fill, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, fb[4];
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t A = base, B = base + 16384, F = base + 49152;  // fills: 4 x 16 KB at F
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem + (base - smem_u32(smem)))[i] = 0x3f803f80u * ((i & 7) == 0);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&fb[i]), 1);
    fence_mbar_init();
    stop = 0;
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
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    if (use_mma) {
      const uint32_t idesc = instr_desc(1, 128, 256, 0, 0);
      for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma<1>(tmem + (it & 1) * 256, smem_desc(A + kk * 32, 16, 1024), smem_desc(B + kk * 32, 16, 1024), idesc, 1);
      mma_commit(smem_u32(&bar));
      mbar_wait(smem_u32(&bar), 0);
    } else {
      while (clock64() - t0 < (long long)iters * 512) {
      }
    }
    cycles[blockIdx.x] = clock64() - t0;
    stop = 1;
  } else if (fill == 1 && threadIdx.x == 32) {
    unsigned long long n = 0;
    uint32_t ph[4] = {0, 0, 0, 0};
    for (int i = 0; i < 4; ++i) {
      mbar_arrive_expect_tx(smem_u32(&fb[i]), 16384);
      bulk_g2s(F + i * 16384, g_l2src + (size_t)i * 4096, 16384, smem_u32(&fb[i]));
    }
    for (int j = 4; !stop; ++j) {
      const int i = j & 3;
      mbar_wait(smem_u32(&fb[i]), ph[i]);
      ph[i] ^= 1;
      n += 16384;
      mbar_arrive_expect_tx(smem_u32(&fb[i]), 16384);
      bulk_g2s(F + i * 16384, g_l2src + (size_t)(j & 63) * 4096, 16384, smem_u32(&fb[i]));
    }
    for (int i = 0; i < 4; ++i) mbar_wait(smem_u32(&fb[i]), ph[i]);
    atomicAdd(&g_bytes, n);
  } else if (fill == 2 && threadIdx.x >= 128) {
    const int i = threadIdx.x - 128;
    const float* src = g_hbm + (size_t)blockIdx.x * (1 << 22);
    int kk = 0;
    while (!stop) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        cp_async16(F + (((i + j * 128) & 4095) << 4), src + (((size_t)(kk * 2048 + i + j * 128)) & ((1 << 20) - 1)) * 4,
                   16);
      cp_async_commit();
      cp_async_wait<4>();
      ++kk;
    }
    cp_async_wait<0>();
    atomicAdd(&g_bytes, (unsigned long long)kk * 16 * 16);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  float* big;
  cudaMalloc(&big, (size_t)148 << 24);
  cudaMemset(big, 0, (size_t)148 << 24);
  cudaMemcpyToSymbol(g_hbm, &big, sizeof(big));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  const int iters = 20000;
  for (int fill = 1; fill <= 2; ++fill)
    for (int use_mma = 0; use_mma < 2; ++use_mma) {
      k<<<148, 256, 128 * 1024>>>(100, use_mma, fill, d);
      cudaDeviceSynchronize();
      unsigned long long z = 0;
      cudaMemcpyToSymbol(g_bytes, &z, sizeof(z));
      k<<<148, 256, 128 * 1024>>>(iters, use_mma, fill, d);
      cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double cyc = 0;
      for (int i = 0; i < 148; ++i) cyc += h[i];
      cyc /= 148;
      unsigned long long b = 0;
      cudaMemcpyFromSymbol(&b, g_bytes, sizeof(b));
      printf("fill=%s mma=%d: %.1f cycles per 4 MMA slots, fills %.1f B/clk/SM  err=%s\n",
             fill == 1 ? "bulk(L2)  " : "LDGSTS(HBM)", use_mma, cyc / iters, b / 148.0 / cyc,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
