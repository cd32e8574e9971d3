// tcgen05 (5th-gen tensor core) kernels for layer 0 of the image MLP.
#pragma once
#include "common.cuh"

namespace dicm {
namespace sm100 {

size_t workspace_bytes(int64_t rows_max, int d_raw);

// act0[r, 0:256] = X[rows[r]] . W0^T + b0 for r < *count (bf16 in bf16 mode)
int fwd_layer0(const void* pool, int pool_dtype, int d_raw, const int32_t* rows, const int32_t* count,
               int64_t rows_max, const float* w0, const float* b0, float* act0, int precision, void* ws,
               cudaStream_t st);

// gw0[256, d_raw] = da0^T . X[rows]  (overwrites); a bf16 pool uses the bf16
// copy of da0 at da0_bf16_ptr(ws) when `da0_bf16_ready`, else converts it
int bwd_dw0(const void* pool, int pool_dtype, int d_raw, const int32_t* rows, const int32_t* count,
            int64_t rows_max, const float* da0, float* gw0, int precision, void* ws, cudaStream_t st,
            bool da0_bf16_ready = false);
__nv_bfloat16* da0_bf16_ptr(void* ws, int64_t rows_max, int d_raw);

// layers 1-2 on tcgen05 (kind::tf32), see imgmlp_small_sm100.cu
int small_part_size();
int small_dw1_blocks(int64_t rows_max);
int small_bwd_blocks(int64_t rows_max);
int fwd_layers12(const float* act0, const int32_t* count, int64_t rows_max, const float* al0, const float* w1,
                 const float* b1, const float* al1, const float* w2, const float* b2, float* act1, float* emb,
                 float* h1, cudaStream_t st);
int bwd_layers12(const float* demb, const float* act1, const float* act0, const float* h1, const int32_t* count,
                 int64_t rows_max, const float* al0, const float* al1, const float* w1, const float* w2, float* da1,
                 float* da0, __nv_bfloat16* da0_bf16, float* part_l12, float* part_dw1, cudaStream_t st);

// bf16 mode (imgmlp_bf16_sm100.cu): saved activations act0/act1 are bf16
int fwd_layers12_bf16(const __nv_bfloat16* act0, const int32_t* count, int64_t rows_max, const float* al0,
                      const float* w1, const float* b1, const float* al1, const float* w2, const float* b2,
                      __nv_bfloat16* act1, float* emb, cudaStream_t st);
int bwd_layers12_bf16(const float* demb, const __nv_bfloat16* act1, const __nv_bfloat16* act0, const int32_t* count,
                      int64_t rows_max, const float* al0, const float* al1, const float* w1, const float* w2,
                      __nv_bfloat16* da1, __nv_bfloat16* da0, float* part_l12, float* part_dw1, cudaStream_t st);
// dW1 / dalpha0 / db0 from the reduced row GEMMs G = [Gp | Gn | Gm] ([3][64][256])
int l1_finish_bf16(const float* G, const float* w1, const float* al0, const float* db1, float* gw1, float* ga0,
                   float* gb0, cudaStream_t st);
int dw1_bf16_part_size();  // floats per k_dw1b block partial

}  // namespace sm100
}  // namespace dicm
