// tcgen05 (5th-gen tensor core) kernels for layer 0 of the image MLP.
#pragma once
#include "common.cuh"

namespace dicm {
namespace sm100 {

size_t workspace_bytes(int64_t rows_max, int d_raw);

// act0[r, 0:256] = X[rows[r]] . W0^T + b0 for r < *count
int fwd_layer0(const void* pool, int pool_dtype, int d_raw, const int32_t* rows, const int32_t* count,
               int64_t rows_max, const float* w0, const float* b0, float* act0, int precision, void* ws,
               cudaStream_t st);

// gw0[256, d_raw] = da0^T . X[rows]  (overwrites)
int bwd_dw0(const void* pool, int pool_dtype, int d_raw, const int32_t* rows, const int32_t* count,
            int64_t rows_max, const float* da0, float* gw0, int precision, void* ws, cudaStream_t st);

}  // namespace sm100
}  // namespace dicm
