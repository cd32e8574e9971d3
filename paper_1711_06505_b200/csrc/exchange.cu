// a16: AMS exchange helpers (reference Cluster._embed_plan / _key_plan,
// runtime.py:353-368, shard_of runtime.py:60-68).
//
// Keys are owned by rank = key % world and stored there at row key / world.
// Requests go out sorted within each destination (the reference sorts ids
// within a shard, runtime.py:353-358), so the stable partition below keeps
// the ascending order of the (already sorted) unique keys per owner.
#include "common.cuh"

namespace {
using namespace dicm;

constexpr int BLK = 1024;  // keys per block
constexpr int MAXW = 64;

__global__ void k_block_counts(const int32_t* __restrict__ keys, const int32_t* __restrict__ count, int64_t n_max,
                               int world, int32_t* __restrict__ blkcnt) {
  __shared__ int c[MAXW];
  if (threadIdx.x < world) c[threadIdx.x] = 0;
  __syncthreads();
  const int64_t n = min((int64_t)*count, n_max);
  const int64_t i = (int64_t)blockIdx.x * BLK + threadIdx.x;
  if (i < n) atomicAdd(&c[keys[i] % world], 1);
  __syncthreads();
  if (threadIdx.x < world) blkcnt[(int64_t)blockIdx.x * world + threadIdx.x] = c[threadIdx.x];
}

// per owner (block o): exclusive scan over the blocks' counts, relative to
// the owner's segment; send_counts[o] = its total
__global__ void __launch_bounds__(256) k_scan_counts(int32_t* __restrict__ blkcnt, int nblk, int world,
                                                     int32_t* __restrict__ send_counts) {
  __shared__ int wsum[8];
  const int o = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int carry = 0;
  for (int b0 = 0; b0 < nblk; b0 += 256) {
    const int b = b0 + threadIdx.x;
    const int v = b < nblk ? blkcnt[(int64_t)b * world + o] : 0;
    int x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    int before = carry;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    int tot = 0;
    for (int w = 0; w < 8; ++w) tot += wsum[w];
    if (b < nblk) blkcnt[(int64_t)b * world + o] = before + x - v;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) send_counts[o] = carry;
}

__global__ void k_place(const int32_t* __restrict__ keys, const int32_t* __restrict__ count, int64_t n_max, int world,
                        const int32_t* __restrict__ base, const int32_t* __restrict__ send_counts,
                        int32_t* __restrict__ send_keys, int32_t* __restrict__ perm,
                        int32_t* __restrict__ perm_inv) {
  __shared__ int warp_cnt[BLK / 32][MAXW];
  __shared__ int owner_base[MAXW];
  if (threadIdx.x == 0) {
    int run = 0;
    for (int o = 0; o < world; ++o) {
      owner_base[o] = run;
      run += send_counts[o];
    }
  }
  const int64_t n = min((int64_t)*count, n_max);
  const int64_t i = (int64_t)blockIdx.x * BLK + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool valid = i < n;
  const int32_t key = valid ? keys[i] : 0;
  const int own = valid ? key % world : -1;
  int rank = 0;
  for (int o = 0; o < world; ++o) {
    const unsigned mask = __ballot_sync(0xffffffffu, own == o);
    if (own == o) rank = __popc(mask & ((1u << lane) - 1u));
    if (lane == 0) warp_cnt[warp][o] = __popc(mask);
  }
  __syncthreads();
  if (valid) {
    int before = 0;
    for (int w = 0; w < warp; ++w) before += warp_cnt[w][own];
    const int pos = owner_base[own] + base[(int64_t)blockIdx.x * world + own] + before + rank;
    send_keys[pos] = key / world;
    perm[i] = pos;
    if (perm_inv) perm_inv[pos] = (int32_t)i;
  }
}

__global__ void k_permute12(const float* __restrict__ in, const int32_t* __restrict__ perm,
                            const int32_t* __restrict__ count, int64_t n_max, int scatter, float* __restrict__ out) {
  const int64_t n = min((int64_t)*count, n_max);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t src = scatter ? i : perm[i];
    const int64_t dst = scatter ? perm[i] : i;
    const float4* s = reinterpret_cast<const float4*>(in + src * DICM_D);
    float4* d = reinterpret_cast<float4*>(out + dst * DICM_D);
    d[0] = s[0];
    d[1] = s[1];
    d[2] = s[2];
  }
}

}  // namespace

extern "C" {

size_t dicm_bucket_workspace(int64_t n_max, int world) {
  const int64_t nblk = (n_max + BLK - 1) / BLK + 1;
  return (size_t)(nblk * world * 4 + 256);
}

int dicm_bucket_by_owner(const int32_t* keys, const int32_t* count_dev, int64_t n_max, int world, int32_t* send_keys,
                         int32_t* send_counts, int32_t* perm, int32_t* perm_inv, void* workspace,
                         size_t workspace_bytes, dicm_stream_t stream) {
  using namespace dicm;
  if (world < 1 || world > MAXW) return fail(DICM_ERR_VALUE, "bucket: world %d not in [1, %d]", world, MAXW);
  if (workspace_bytes < dicm_bucket_workspace(n_max, world)) return fail(DICM_ERR_VALUE, "bucket: workspace");
  cudaStream_t st = (cudaStream_t)stream;
  const int nblk = (int)((n_max + BLK - 1) / BLK);
  if (nblk == 0) {
    cudaMemsetAsync(send_counts, 0, world * 4, st);
    return last_launch("dicm_bucket_by_owner");
  }
  int32_t* blkcnt = (int32_t*)workspace;
  k_block_counts<<<nblk, BLK, 0, st>>>(keys, count_dev, n_max, world, blkcnt);
  k_scan_counts<<<world, 256, 0, st>>>(blkcnt, nblk, world, send_counts);
  k_place<<<nblk, BLK, 0, st>>>(keys, count_dev, n_max, world, blkcnt, send_counts, send_keys, perm, perm_inv);
  return last_launch("dicm_bucket_by_owner");
}

int dicm_permute_rows12(const float* in, const int32_t* perm, const int32_t* count_dev, int64_t n_max, int scatter,
                        float* out, dicm_stream_t stream) {
  if (n_max <= 0) return DICM_OK;
  k_permute12<<<dicm_grid(n_max, 256, 148 * 8), 256, 0, (cudaStream_t)stream>>>(in, perm, count_dev, n_max, scatter,
                                                                                out);
  return dicm::last_launch("dicm_permute_rows12");
}

}  // extern "C"

// ---------------------------------------------------------------------------
// rows of several tables addressed by combined keys (tables back to back in
// one key space, ascending bases): out[i] = table_f[key_i - base_f]
// ---------------------------------------------------------------------------
namespace {
struct TabRows {
  const float* t[DICM_MAX_FIELDS];
  int64_t base[DICM_MAX_FIELDS];
  int n;
};

__global__ void k_gather_keyed(const __grid_constant__ TabRows tb, const int32_t* __restrict__ keys,
                               const int32_t* __restrict__ count, int64_t n_max, float* __restrict__ out) {
  const int64_t n = count ? min((int64_t)*count, n_max) : n_max;
  const int lane = threadIdx.x & 31, part = lane % 3, slot = lane / 3;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w * 10 < n; w += warps) {
    const int64_t i = w * 10 + slot;
    if (slot >= 10 || i >= n) continue;
    const int64_t key = keys[i];
    int k = 0;
    while (k + 1 < tb.n && key >= tb.base[k + 1]) ++k;
    reinterpret_cast<float4*>(out + i * DICM_D)[part] =
        __ldg(reinterpret_cast<const float4*>(tb.t[k] + (key - tb.base[k]) * DICM_D) + part);
  }
}

// idx[s][inv[i]] = i for reference i of source segment s (offsets seg[s]..seg[s+1])
__global__ void k_scatter_index(const int32_t* __restrict__ inv, const int64_t* __restrict__ seg, int nsrc,
                                int64_t ucap, int32_t* __restrict__ idx) {
  const int64_t total = seg[nsrc];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int s = 0;
    while (s + 1 < nsrc && i >= seg[s + 1]) ++s;
    idx[(int64_t)s * ucap + inv[i]] = (int32_t)i;
  }
}

// out[u] = sum over sources s = 0..nsrc-1 (ascending, as the reference sums
// pushes in ascending worker order, runtime.py:177-185) of src[idx[s][u]]
__global__ void k_gather_sum12(const float* __restrict__ src, const int32_t* __restrict__ idx, int nsrc, int64_t ucap,
                               const int32_t* __restrict__ count, float* __restrict__ out) {
  const int64_t n = min((int64_t)*count, ucap);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n * 3; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = q / 3;
    const int part = (int)(q % 3);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < nsrc; ++s) {
      const int32_t i = idx[(int64_t)s * ucap + u];
      if (i < 0) continue;
      const float4 v = __ldg(reinterpret_cast<const float4*>(src + (int64_t)i * DICM_D) + part);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    reinterpret_cast<float4*>(out + u * DICM_D)[part] = acc;
  }
}
}  // namespace

extern "C" {

int dicm_gather_rows_by_key(const dicm_table_state_t* tabs, int ntab, const int32_t* keys, const int32_t* count_dev,
                            int64_t n_max, float* out, dicm_stream_t stream) {
  using namespace dicm;
  if (ntab < 1 || ntab > DICM_MAX_FIELDS) return fail(DICM_ERR_VALUE, "gather_rows_by_key: %d tables", ntab);
  if (n_max <= 0) return DICM_OK;
  TabRows tb{};
  tb.n = ntab;
  for (int i = 0; i < ntab; ++i) {
    tb.t[i] = tabs[i].table;
    tb.base[i] = tabs[i].base;
  }
  k_gather_keyed<<<dicm_grid((n_max + 9) / 10 * 32, 256, 148 * 8), 256, 0, (cudaStream_t)stream>>>(tb, keys, count_dev,
                                                                                                 n_max, out);
  return last_launch("dicm_gather_rows_by_key");
}

int dicm_owner_reduce_rows12(const float* recv, const int32_t* inv, const int64_t* seg_dev, int nsrc,
                             int64_t n_recv_max, const int32_t* count_dev, int64_t ucap, int32_t* idx_ws,
                             float* out, dicm_stream_t stream) {
  using namespace dicm;
  if (nsrc < 1) return fail(DICM_ERR_VALUE, "owner_reduce: nsrc %d", nsrc);
  cudaStream_t st = (cudaStream_t)stream;
  if (ucap <= 0) return DICM_OK;
  int rc = check_cuda(cudaMemsetAsync(idx_ws, 0xFF, (size_t)nsrc * ucap * 4, st), "owner_reduce memset");
  if (rc) return rc;
  if (n_recv_max > 0)
    k_scatter_index<<<dicm_grid(n_recv_max, 256, 148 * 8), 256, 0, st>>>(inv, seg_dev, nsrc, ucap, idx_ws);
  k_gather_sum12<<<dicm_grid(ucap * 3, 256, 148 * 8), 256, 0, st>>>(recv, idx_ws, nsrc, ucap, count_dev, out);
  return last_launch("dicm_owner_reduce_rows12");
}

}  // extern "C"
