// a3: the image pool, 4096-d feature rows resident in HBM.
#include "common.cuh"

namespace {

// rows[p][d] = tanh(sum_j latent[p][j] * proj[d][j]) in fp64 -> pool dtype.
// The frozen extractor of reference images.py:62-71; one block per pool row.
template <typename T>
__global__ void k_materialize(const float* __restrict__ latents, const double* __restrict__ proj,
                              int64_t rows, int d_raw, int k, T* __restrict__ out) {
  extern __shared__ double z[];
  for (int64_t p = blockIdx.x; p < rows; p += gridDim.x) {
    __syncthreads();
    for (int j = threadIdx.x; j < k; j += blockDim.x) z[j] = (double)latents[p * k + j];
    __syncthreads();
    for (int d = threadIdx.x; d < d_raw; d += blockDim.x) {
      const double* r = proj + (int64_t)d * k;
      double acc = 0.0;
      for (int j = 0; j < k; ++j) acc = fma(z[j], __ldg(r + j), acc);
      const double v = tanh(acc);
      if constexpr (sizeof(T) == 4)
        out[p * d_raw + d] = (float)v;
      else
        out[p * d_raw + d] = __float2bfloat16_rn((float)v);
    }
  }
}

template <typename T>
__global__ void k_gather(const T* __restrict__ pool, int d_raw, const int32_t* __restrict__ ids,
                         const int32_t* __restrict__ count, int64_t n_max, float* __restrict__ out) {
  const int64_t n = min((int64_t)*count, n_max);
  const int vec = d_raw / 4;
  for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
    const int64_t src = ids[r];
    if constexpr (sizeof(T) == 4) {
      const float4* s = reinterpret_cast<const float4*>(pool + src * d_raw);
      float4* d = reinterpret_cast<float4*>(out + r * d_raw);
      for (int c = threadIdx.x; c < vec; c += blockDim.x) d[c] = __ldg(s + c);
    } else {
      const __nv_bfloat162* s = reinterpret_cast<const __nv_bfloat162*>(pool + src * d_raw);
      float2* d = reinterpret_cast<float2*>(out + r * d_raw);
      for (int c = threadIdx.x; c < d_raw / 2; c += blockDim.x) d[c] = __bfloat1622float2(s[c]);
    }
  }
}

}  // namespace

extern "C" {

int dicm_pool_materialize(const float* latents, const double* proj, int64_t rows, int d_raw,
                          int latent_dim, void* pool, int pool_dtype, dicm_stream_t stream) {
  using namespace dicm;
  if (rows < 0 || d_raw < 1 || latent_dim < 1 || latent_dim > 4096)
    return fail(DICM_ERR_VALUE, "pool_materialize: bad sizes");
  if (rows == 0) return DICM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = (int)(rows < 148 * 64 ? rows : 148 * 64);
  const size_t smem = (size_t)latent_dim * sizeof(double);
  if (pool_dtype == DICM_POOL_F32)
    k_materialize<float><<<grid, 256, smem, st>>>(latents, proj, rows, d_raw, latent_dim, (float*)pool);
  else if (pool_dtype == DICM_POOL_BF16)
    k_materialize<__nv_bfloat16><<<grid, 256, smem, st>>>(latents, proj, rows, d_raw, latent_dim,
                                                          (__nv_bfloat16*)pool);
  else
    return fail(DICM_ERR_VALUE, "pool_materialize: unknown pool dtype %d", pool_dtype);
  return last_launch("dicm_pool_materialize");
}

int dicm_pool_gather(const void* pool, int pool_dtype, int d_raw, const int32_t* row_ids,
                     const int32_t* count_dev, int64_t n_max, float* out, dicm_stream_t stream) {
  using namespace dicm;
  if (d_raw % 4) return fail(DICM_ERR_SHAPE, "pool_gather: d_raw %d not a multiple of 4", d_raw);
  if (n_max <= 0) return DICM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = (int)(n_max < 148 * 32 ? n_max : 148 * 32);
  if (pool_dtype == DICM_POOL_F32)
    k_gather<float><<<grid, 256, 0, st>>>((const float*)pool, d_raw, row_ids, count_dev, n_max, out);
  else if (pool_dtype == DICM_POOL_BF16)
    k_gather<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)pool, d_raw, row_ids,
                                                   count_dev, n_max, out);
  else
    return fail(DICM_ERR_VALUE, "pool_gather: unknown pool dtype %d", pool_dtype);
  return last_launch("dicm_pool_gather");
}

}  // extern "C"
