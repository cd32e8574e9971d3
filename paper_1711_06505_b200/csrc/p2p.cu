// a16: the AMS exchanges over NVLink peer memory.
//
// Reference: Cluster._route (runtime.py:337-343) delivers EmbedRequest /
// EmbedResponse / IdParamPull / IdParamResponse / EmbedGradPush /
// IdParamPush messages between workers and servers (runtime.py:387-422).
// Here every rank is a worker and a server; the messages of one phase form an
// all-to-all-v that copy kernels write straight into the peers' receive
// buffers (CUDA IPC mappings of each rank's exchange region).  The counts of
// every pair travel the same way into a [world][world] matrix on every rank,
// so all placements are computed on the device: an iteration needs no host
// synchronisation and no collective library call for its sparse exchanges.
//
// Ordering: copies are plain stores to peer memory; a phase ends with
// dicm_p2p_barrier, whose release store (system scope) follows the copy
// kernel in stream order and whose acquire loads precede every consumer.
#include <algorithm>
#include <cstring>

#include "common.cuh"

namespace {
using namespace dicm;

struct Peers {
  int world, rank;
  uint8_t* region[DICM_MAX_PEERS];
};

Peers to_dev(const dicm_peers_t* p) {
  Peers q{};
  q.world = p->world;
  q.rank = p->rank;
  for (int i = 0; i < DICM_MAX_PEERS; ++i) q.region[i] = (uint8_t*)p->region[i];
  return q;
}

// epoch: the barrier's sequence number.  epoch == 0 takes it from (and
// advances) a counter at flags[63] of this rank's own region, so a captured
// CUDA graph replays with fresh epochs; every rank calls the same sequence.
__global__ void k_barrier(const __grid_constant__ Peers P, int64_t off, uint32_t epoch_in, int32_t* status) {
  const int t = threadIdx.x;
  __shared__ uint32_t ep;
  if (t == 0) {
    uint32_t* ctr = reinterpret_cast<uint32_t*>(P.region[P.rank] + off) + 63;
    ep = epoch_in ? epoch_in : *ctr + 1;
    if (!epoch_in) *ctr = ep;
  }
  __syncthreads();
  const uint32_t epoch = ep;
  if (t < P.world) {
    uint32_t* remote = reinterpret_cast<uint32_t*>(P.region[t] + off) + P.rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(remote), "r"(epoch) : "memory");
    const uint32_t* mine = reinterpret_cast<const uint32_t*>(P.region[P.rank] + off) + t;
    const long long t0 = clock64();
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
      if ((int32_t)(v - epoch) >= 0) break;  // a peer may already be one barrier ahead
      if (clock64() - t0 > 20000000000ll) {  // ~10 s: a peer is gone
        atomicExch(status + DICM_ST_P2P_TIMEOUT, 1);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
}

// my send counts [2][world] (image keys per owner, then ID keys per owner,
// as the two bucket passes write them) -> row [rank] of every peer's
// [world][world][2] count matrix
__global__ void k_counts(const __grid_constant__ Peers P, const int32_t* __restrict__ cnt, int64_t off) {
  const int W = P.world;
  for (int i = threadIdx.x; i < W * W * 2; i += blockDim.x) {
    const int p = i / (2 * W), e = i % (2 * W);
    reinterpret_cast<int32_t*>(P.region[p] + off)[P.rank * 2 * W + e] = cnt[(e & 1) * W + (e >> 1)];
  }
}

// plan[kind][0][d] my send offset for d      plan[kind][1][d] my position in d's receive buffer
// plan[kind][2][s] receive offset of source s plan[kind][3][s] where my rows for s go in s's buffer
__global__ void k_plan(const __grid_constant__ Peers P, int64_t off, int64_t* __restrict__ seg_img,
                       int64_t* __restrict__ seg_id, int32_t* __restrict__ cnt_dev, int64_t* __restrict__ plan) {
  const int W = P.world, r = P.rank, k = threadIdx.x;
  if (k >= 2) return;
  const int32_t* C = reinterpret_cast<const int32_t*>(P.region[r] + off);  // C[(s*W + d)*2 + k]
  auto c = [&](int s, int d) { return (int64_t)C[(s * W + d) * 2 + k]; };
  int64_t* pl = plan + (int64_t)k * 4 * (DICM_MAX_PEERS + 1);
  int64_t* seg = k == 0 ? seg_img : seg_id;
  int64_t a = 0, b = 0;
  for (int d = 0; d <= W; ++d) {
    pl[d] = a;                                 // my send offsets
    if (d < W) a += c(r, d);
    seg[d] = b;                                // receive segments by source
    pl[2 * (DICM_MAX_PEERS + 1) + d] = b;
    if (d < W) b += c(d, r);
  }
  for (int d = 0; d < W; ++d) {
    int64_t p = 0, q = 0;
    for (int s = 0; s < r; ++s) p += c(s, d);  // sources before me at destination d
    for (int e = 0; e < r; ++e) q += c(d, e);  // d's send offset for its rows owned by me
    pl[(DICM_MAX_PEERS + 1) + d] = p;
    pl[3 * (DICM_MAX_PEERS + 1) + d] = q;
  }
  cnt_dev[k] = (int32_t)b;      // n_recv
  cnt_dev[2 + k] = (int32_t)a;  // n_send
}

// blockIdx.y = peer; each block grid-strides over that peer's segment
__global__ void __launch_bounds__(256) k_scatter(const __grid_constant__ Peers P, const int64_t* __restrict__ plan,
                                                 int kind, int dir, const uint8_t* __restrict__ src, int row_bytes,
                                                 int64_t dst_off) {
  const int p = blockIdx.y;
  const int64_t* pl = plan + (int64_t)kind * 4 * (DICM_MAX_PEERS + 1);
  constexpr int S = DICM_MAX_PEERS + 1;
  int64_t s0, n, d0;
  if (dir == 0) {  // my rows for owner p
    s0 = pl[p];
    n = pl[p + 1] - pl[p];
    d0 = pl[S + p];
  } else {  // the rows of requester p's segment, back to p
    s0 = pl[2 * S + p];
    n = pl[2 * S + p + 1] - pl[2 * S + p];
    d0 = pl[3 * S + p];
  }
  uint8_t* dst = P.region[p] + dst_off;
  if (row_bytes % 16 == 0) {
    const int q = row_bytes / 16;
    const int4* s4 = reinterpret_cast<const int4*>(src + s0 * row_bytes);
    int4* d4 = reinterpret_cast<int4*>(dst + d0 * row_bytes);
    const int64_t m = n * q;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
      d4[i] = __ldg(s4 + i);
  } else {  // 4-byte rows (keys)
    const int32_t* s1 = reinterpret_cast<const int32_t*>(src) + s0;
    int32_t* d1 = reinterpret_cast<int32_t*>(dst) + d0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
      d1[i] = __ldg(s1 + i);
  }
}

// k_scatter with the row gather fused in (12-float rows): row j of the
// segment is rows[idx[s0 + j]] -- the owner's embedding of the j-th key a
// requester sent -- read locally and stored straight into the peer's buffer
// over NVLink (no staged copy in between)
__global__ void __launch_bounds__(256) k_gather_scatter12(const __grid_constant__ Peers P,
                                                          const int64_t* __restrict__ plan, int kind, int dir,
                                                          const float* __restrict__ rows,
                                                          const int32_t* __restrict__ idx, int64_t dst_off) {
  const int p = blockIdx.y;
  const int64_t* pl = plan + (int64_t)kind * 4 * (DICM_MAX_PEERS + 1);
  constexpr int S = DICM_MAX_PEERS + 1;
  const int64_t s0 = dir == 0 ? pl[p] : pl[2 * S + p];
  const int64_t n = dir == 0 ? pl[p + 1] - pl[p] : pl[2 * S + p + 1] - pl[2 * S + p];
  const int64_t d0 = dir == 0 ? pl[S + p] : pl[3 * S + p];
  int4* d4 = reinterpret_cast<int4*>(P.region[p] + dst_off) + d0 * 3;
  const int4* r4 = reinterpret_cast<const int4*>(rows);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * 3; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i / 3;
    const int q = (int)(i - j * 3);
    d4[i] = __ldg(r4 + (int64_t)__ldg(idx + s0 + j) * 3 + q);
  }
}

int check_peers(const dicm_peers_t* p) {
  if (!p || p->world < 1 || p->world > DICM_MAX_PEERS || p->rank < 0 || p->rank >= p->world)
    return fail(DICM_ERR_VALUE, "p2p: bad peer table");
  for (int i = 0; i < p->world; ++i)
    if (!p->region[i]) return fail(DICM_ERR_VALUE, "p2p: region of rank %d not mapped", i);
  return DICM_OK;
}

// one chunk of the all-reduce: this rank sums float4 i of every rank's staged
// buffer in rank order (the same order on every rank: bit-identical results)
// and writes the sum into every rank's result buffer over NVLink
__global__ void __launch_bounds__(256) k_allreduce_chunk(const __grid_constant__ Peers P, int64_t stage_off,
                                                         int64_t res_off, int64_t n4) {
  const int W = P.world;
  const int64_t per = (n4 + W - 1) / W, lo = per * P.rank, hi = min(n4, lo + per);
  for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
    float4 v[DICM_MAX_PEERS];
#pragma unroll
    for (int q = 0; q < DICM_MAX_PEERS; ++q)
      if (q < W) v[q] = __ldcv(reinterpret_cast<const float4*>(P.region[q] + stage_off) + i);
    float4 s = v[0];
#pragma unroll
    for (int q = 1; q < DICM_MAX_PEERS; ++q)
      if (q < W) {
        s.x += v[q].x;
        s.y += v[q].y;
        s.z += v[q].z;
        s.w += v[q].w;
      }
#pragma unroll
    for (int q = 0; q < DICM_MAX_PEERS; ++q)
      if (q < W) reinterpret_cast<float4*>(P.region[q] + res_off)[i] = s;
  }
}

}  // namespace

extern "C" {

int dicm_p2p_allreduce(const dicm_peers_t* peers, const float* src, int64_t n, int64_t stage_off, int64_t res_off,
                       int64_t flags_off, int32_t* status, float* dst, dicm_stream_t stream) {
  int rc = check_peers(peers);
  if (rc) return rc;
  if (n <= 0) return DICM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const Peers P = to_dev(peers);
  const int64_t n4 = (n + 3) / 4;  // the staged buffers are float4-padded (the pad holds zeros)
  rc = dicm::check_cuda(cudaMemcpyAsync(P.region[P.rank] + stage_off, src, n * sizeof(float),
                                        cudaMemcpyDeviceToDevice, st), "p2p allreduce stage");
  if (rc) return rc;
  k_barrier<<<1, 32, 0, st>>>(P, flags_off, 0, status);  // every rank's gradients are staged
  const int grid = (int)std::min<int64_t>(148 * 4, (n4 / P.world + 255) / 256 + 1);
  k_allreduce_chunk<<<grid, 256, 0, st>>>(P, stage_off, res_off, n4);
  k_barrier<<<1, 32, 0, st>>>(P, flags_off, 0, status);  // every chunk's sum has landed everywhere
  rc = dicm::check_cuda(cudaMemcpyAsync(dst, P.region[P.rank] + res_off, n * sizeof(float),
                                        cudaMemcpyDeviceToDevice, st), "p2p allreduce result");
  if (rc) return rc;
  return dicm::last_launch("dicm_p2p_allreduce");
}

int dicm_p2p_alloc(size_t bytes, void** out) {
  using namespace dicm;
  void* p = nullptr;
  int rc = check_cuda(cudaMalloc(&p, bytes), "p2p region cudaMalloc");
  if (rc) return rc;
  rc = check_cuda(cudaMemset(p, 0, bytes), "p2p region memset");
  if (rc) return rc;
  *out = p;
  return DICM_OK;
}

int dicm_p2p_free(void* ptr) { return dicm::check_cuda(cudaFree(ptr), "p2p region free"); }

int dicm_ipc_handle(const void* ptr, void* handle) {
  cudaIpcMemHandle_t h;
  int rc = dicm::check_cuda(cudaIpcGetMemHandle(&h, const_cast<void*>(ptr)), "cudaIpcGetMemHandle");
  if (rc) return rc;
  static_assert(sizeof(h) == 64, "IPC handle size");
  memcpy(handle, &h, sizeof(h));
  return DICM_OK;
}

int dicm_ipc_open(const void* handle, void** out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return dicm::check_cuda(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
}

int dicm_ipc_close(void* ptr) { return dicm::check_cuda(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle"); }

int dicm_p2p_barrier(const dicm_peers_t* peers, int64_t flags_off, uint32_t epoch, int32_t* status,
                     dicm_stream_t stream) {
  int rc = check_peers(peers);
  if (rc) return rc;
  k_barrier<<<1, 32, 0, (cudaStream_t)stream>>>(to_dev(peers), flags_off, epoch, status);
  return dicm::last_launch("dicm_p2p_barrier");
}

int dicm_p2p_counts(const dicm_peers_t* peers, const int32_t* send_counts, int64_t cmat_off, dicm_stream_t stream) {
  int rc = check_peers(peers);
  if (rc) return rc;
  k_counts<<<1, 128, 0, (cudaStream_t)stream>>>(to_dev(peers), send_counts, cmat_off);
  return dicm::last_launch("dicm_p2p_counts");
}

int dicm_p2p_plan(const dicm_peers_t* peers, int64_t cmat_off, int64_t* seg_img, int64_t* seg_id, int32_t* cnt_dev,
                  int64_t* plan, dicm_stream_t stream) {
  int rc = check_peers(peers);
  if (rc) return rc;
  k_plan<<<1, 32, 0, (cudaStream_t)stream>>>(to_dev(peers), cmat_off, seg_img, seg_id, cnt_dev, plan);
  return dicm::last_launch("dicm_p2p_plan");
}

int dicm_p2p_scatter(const dicm_peers_t* peers, const int64_t* plan, int kind, int dir, const void* src,
                     int row_bytes, int64_t dst_off, dicm_stream_t stream) {
  using namespace dicm;
  int rc = check_peers(peers);
  if (rc) return rc;
  if ((kind != 0 && kind != 1) || (dir != 0 && dir != 1) || (row_bytes != 4 && row_bytes % 16 != 0))
    return fail(DICM_ERR_VALUE, "p2p_scatter: kind %d dir %d row_bytes %d", kind, dir, row_bytes);
  // one wave: blocks per peer so that world * blocks ~ 4 per SM
  const int per = std::max(1, 148 * 4 / peers->world);
  k_scatter<<<dim3(per, peers->world), 256, 0, (cudaStream_t)stream>>>(to_dev(peers), plan, kind, dir,
                                                                      (const uint8_t*)src, row_bytes, dst_off);
  return last_launch("dicm_p2p_scatter");
}

int dicm_p2p_gather_scatter12(const dicm_peers_t* peers, const int64_t* plan, int kind, int dir, const float* rows,
                              const int32_t* idx, int64_t dst_off, dicm_stream_t stream) {
  using namespace dicm;
  int rc = check_peers(peers);
  if (rc) return rc;
  if ((kind != 0 && kind != 1) || (dir != 0 && dir != 1))
    return fail(DICM_ERR_VALUE, "p2p_gather_scatter12: kind %d dir %d", kind, dir);
  const int per = std::max(1, 148 * 4 / peers->world);
  k_gather_scatter12<<<dim3(per, peers->world), 256, 0, (cudaStream_t)stream>>>(to_dev(peers), plan, kind, dir, rows,
                                                                               idx, dst_off);
  return last_launch("dicm_p2p_gather_scatter12");
}

}  // extern "C"
