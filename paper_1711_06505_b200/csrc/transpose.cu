// Deterministic scatter-add support (a6 / a10 backward: np.add.at restated
// as per-key sums).
//
// The reference accumulates every per-reference gradient row into the
// deduplicated rows it was gathered from with np.add.at (autograd.py:267-271);
// its runs are bit-reproducible (runtime.py:16-21).  Float atomics would make
// each sum depend on the scheduling order.  Here the dedup inverse inv[p]
// (reference p -> unique key, keys dense in [0, K)) is transposed by a
// counting sort -- per-key counts (integer atomics, whose return values rank
// each reference inside its group), an exclusive scan, and an atomic-free
// fill -- so every key owns a contiguous group of its references.  The order inside a group is NOT fixed; the reduction over a
// group (sample.cu k_ref_reduce) restores determinism itself: a group of up
// to 16 references (nearly all of them) is sorted by position in registers
// and summed in reference order like np.add.at; a larger group is summed
// exactly in 64-bit fixed point (scale from the group's largest magnitude, an
// order-independent max), which does not depend on the order at all.  Three
// light passes over the references replace a three-pass radix sort (~0.14 ms
// per cfg2 step for the two lists).
#include <cub/cub.cuh>

#include "common.cuh"

namespace {
using namespace dicm;

constexpr unsigned FULL = 0xffffffffu;

// count[inv[p]] += 1 (one atomic per distinct key and warp); the value the
// atomic returns is this warp's place in the key's group, so every
// reference's slot in its group (rank[p]) falls out of the same pass
__global__ void k_count(const int32_t* __restrict__ inv, int64_t n, int32_t* __restrict__ count,
                        int32_t* __restrict__ rank) {
  const int lane = threadIdx.x & 31;
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ll; b < n;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = b + lane;
    const int32_t key = p < n ? __ldg(inv + p) : -1;
    const unsigned peers = __match_any_sync(FULL, key);
    const int leader = __ffs(peers) - 1;
    int32_t base = 0;
    if (key >= 0 && lane == leader) base = atomicAdd(count + key, __popc(peers));
    base = __shfl_sync(FULL, base, leader);
    if (key >= 0) rank[p] = base + __popc(peers & ((1u << lane) - 1));
  }
}

// order[start[inv[p]] + rank[p]] = p: no atomics
__global__ void k_fill(const int32_t* __restrict__ inv, const int32_t* __restrict__ rank, int64_t n,
                       const int32_t* __restrict__ start, int32_t* __restrict__ order) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    order[__ldg(start + __ldg(inv + p)) + __ldg(rank + p)] = (int32_t)p;
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

size_t scan_temp(int64_t n) {
  size_t t = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t, (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  return t;
}

size_t align256(size_t b) { return (b + 255) / 256 * 256; }

}  // namespace

extern "C" {

size_t dicm_ref_transpose_workspace(int64_t n, int64_t key_cap) {
  const int64_t k = std::max<int64_t>(key_cap, 1) + 1;
  return align256((size_t)k * 4) + align256((size_t)std::max<int64_t>(n, 1) * 4) + align256(scan_temp(k));
}

int dicm_ref_transpose(const int32_t* inv, int64_t n, int64_t key_cap, void* ws, size_t ws_bytes, int32_t* order,
                       int32_t* start, dicm_stream_t stream) {
  if (n <= 0) return DICM_OK;
  if (n >= INT32_MAX) return fail(DICM_ERR_VALUE, "ref_transpose: %lld references exceed int32", (long long)n);
  if (ws_bytes < dicm_ref_transpose_workspace(n, key_cap))
    return fail(DICM_ERR_VALUE, "ref_transpose: workspace %zu < %zu bytes", ws_bytes,
                dicm_ref_transpose_workspace(n, key_cap));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t k = std::max<int64_t>(key_cap, 1) + 1;
  char* base = (char*)ws;
  int32_t* count = (int32_t*)base;
  int32_t* rank = (int32_t*)(base + align256((size_t)k * 4));
  void* temp = base + align256((size_t)k * 4) + align256((size_t)n * 4);
  size_t temp_bytes = scan_temp(k);
  if (check_cuda(cudaMemsetAsync(count, 0, (size_t)k * 4, st), "ref_transpose clear")) return DICM_ERR_CUDA;
  const int grid = dicm_grid(n, 256, 148 * 8);
  k_count<<<grid, 256, 0, st>>>(inv, n, count, rank);
  // start[k] = references of the keys before k; start[K..key_cap] = n
  if (check_cuda(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, count, start, (int)k, st), "ref_transpose scan"))
    return DICM_ERR_CUDA;
  k_fill<<<grid, 256, 0, st>>>(inv, rank, n, start, order);
  return last_launch("dicm_ref_transpose");
}

int dicm_csr_segments(const int32_t* off, int batch, int32_t* seg, dicm_stream_t stream) {
  if (batch <= 0) return DICM_OK;
  k_csr_segments<<<dicm_grid((int64_t)batch * 32, 256, 148 * 8), 256, 0, (cudaStream_t)stream>>>(off, batch, seg);
  return last_launch("dicm_csr_segments");
}

}  // extern "C"
