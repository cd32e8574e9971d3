// tcgen05 layer-0 kernels (placeholder: filled in by the tensor-core build step).
#include "imgmlp_sm100.cuh"

namespace dicm {
namespace sm100 {

size_t workspace_bytes(int64_t rows_max, int d_raw) { return 0; }

int fwd_layer0(const void*, int, int, const int32_t*, const int32_t*, int64_t, const float*, const float*, float*,
               int precision, void*, cudaStream_t) {
  return fail(DICM_ERR_UNSUPPORTED, "image MLP precision %d: tensor-core path not built", precision);
}

int bwd_dw0(const void*, int, int, const int32_t*, const int32_t*, int64_t, const float*, float*, int precision,
            void*, cudaStream_t) {
  return fail(DICM_ERR_UNSUPPORTED, "image MLP precision %d: tensor-core path not built", precision);
}

}  // namespace sm100
}  // namespace dicm
