// Deterministic scatter-add support (a6 / a10 backward, np.add.at restated
// as per-key ordered sums).
//
// The reference accumulates every per-reference gradient row into the
// deduplicated rows it was gathered from with np.add.at (autograd.py:267-271),
// which sums in reference order; its runs are bit-reproducible
// (runtime.py:16-21).  Float atomics would make the sum order depend on
// scheduling.  Instead the dedup inverse inv[p] (reference p -> unique key)
// is transposed once per step -- a stable radix sort of (inv[p], p) gives,
// for every key, its references in ascending p -- and the backward reduces
// each key's references in that fixed order (sample.cu k_ref_reduce).  The
// transpose depends only on the batch, so the step runs it on a forked
// stream beside the image-MLP forward.
#include <cub/cub.cuh>

#include "common.cuh"

namespace {
using namespace dicm;

__global__ void k_iota(int32_t* __restrict__ v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

// start[k] = first position of key k in the sorted keys; start[last + 1] = n
__global__ void k_group_starts(const uint32_t* __restrict__ keys, int64_t n, int32_t* __restrict__ start) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = keys[i];
    if (i == 0 || keys[i - 1] != k) start[k] = (int32_t)i;
    if (i == n - 1) start[k + 1] = (int32_t)n;
  }
}

// seg[i] = b for off[b] <= i < off[b + 1]: warp per sample, coalesced stores
__global__ void k_csr_segments(const int32_t* __restrict__ off, int batch, int32_t* __restrict__ seg) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int b = w; b < batch; b += nw) {
    const int32_t i1 = off[b + 1];
    for (int32_t i = off[b] + lane; i < i1; i += 32) seg[i] = b;
  }
}

int key_bits(int64_t key_cap) {
  int b = 1;
  while (b < 31 && (int64_t(1) << b) < key_cap) ++b;
  return b;
}

size_t cub_temp(int64_t n, int bits) {
  size_t t = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t, (const uint32_t*)nullptr, (uint32_t*)nullptr, (const int32_t*)nullptr,
                                  (int32_t*)nullptr, (int)n, 0, bits);
  return t;
}

size_t align256(size_t b) { return (b + 255) / 256 * 256; }

}  // namespace

extern "C" {

size_t dicm_ref_transpose_workspace(int64_t n, int64_t key_cap) {
  if (n <= 0) return 256;
  return 2 * align256((size_t)n * 4) + align256(cub_temp(n, key_bits(key_cap)));
}

int dicm_ref_transpose(const int32_t* inv, int64_t n, int64_t key_cap, void* ws, size_t ws_bytes, int32_t* order,
                       int32_t* start, dicm_stream_t stream) {
  if (n <= 0) return DICM_OK;
  if (n >= INT32_MAX) return fail(DICM_ERR_VALUE, "ref_transpose: %lld references exceed int32", (long long)n);
  if (ws_bytes < dicm_ref_transpose_workspace(n, key_cap))
    return fail(DICM_ERR_VALUE, "ref_transpose: workspace %zu < %zu bytes", ws_bytes,
                dicm_ref_transpose_workspace(n, key_cap));
  cudaStream_t st = (cudaStream_t)stream;
  char* base = (char*)ws;
  uint32_t* keys_out = (uint32_t*)base;  // keys are non-negative: sorted as unsigned
  int32_t* iota = (int32_t*)(base + align256((size_t)n * 4));
  void* temp = base + 2 * align256((size_t)n * 4);
  const int bits = key_bits(key_cap);
  size_t temp_bytes = cub_temp(n, bits);
  k_iota<<<dicm_grid(n, 256, 148 * 8), 256, 0, st>>>(iota, n);
  // stable LSD radix sort: equal keys keep ascending positions
  if (check_cuda(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, reinterpret_cast<const uint32_t*>(inv), keys_out, iota,
                                                 order, (int)n, 0, bits, st),
                 "ref_transpose sort"))
    return DICM_ERR_CUDA;
  k_group_starts<<<dicm_grid(n, 256, 148 * 8), 256, 0, st>>>(keys_out, n, start);
  return last_launch("dicm_ref_transpose");
}

int dicm_csr_segments(const int32_t* off, int batch, int32_t* seg, dicm_stream_t stream) {
  if (batch <= 0) return DICM_OK;
  k_csr_segments<<<dicm_grid((int64_t)batch * 32, 256, 148 * 8), 256, 0, (cudaStream_t)stream>>>(off, batch, seg);
  return last_launch("dicm_csr_segments");
}

}  // extern "C"
