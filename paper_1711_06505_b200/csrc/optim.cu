// a14: Adam with the reference's semantics (reference optim.py).
//   dense (optim.py:44-63): per parameter span; an all-zero gradient skips the
//     span entirely (value, moments and step count untouched, optim.py:55-56);
//   rows  (optim.py:83-104): per-row step counter, zero rows skipped.
// Non-finite values anywhere in the step (loss or gradients, latched in the
// status words by earlier kernels) freeze every update, mirroring the
// reference raising before it touches a parameter (optim.py:53-54, 90-91).
#include <math.h>

#include "common.cuh"

namespace {
using namespace dicm;

constexpr int MAXSPANS = 64;

struct Spans {
  int64_t off[MAXSPANS + 1];
  int n;
};

__device__ __forceinline__ int span_of(const Spans& s, int64_t i) {
  int lo = 0, hi = s.n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s.off[mid] <= i)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

__global__ void k_dense_flags(const float* __restrict__ g, const __grid_constant__ Spans s, int32_t* __restrict__ nz,
                              int32_t* __restrict__ status) {
  // warp-aggregated: one flag update per (warp, span) instead of per element
  const int64_t total = s.off[s.n];
  const int lane = threadIdx.x & 31;
  bool bad = false;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < total; i0 += stride) {
    const int64_t i = i0 + lane;
    const float v = i < total ? g[i] : 0.f;
    bad |= !isfinite(v);
    const int k = span_of(s, i < total ? i : total - 1);
    const int k0 = __shfl_sync(0xffffffffu, k, 0);
    const bool nonzero = v != 0.f;
    if (__all_sync(0xffffffffu, k == k0)) {
      if (__any_sync(0xffffffffu, nonzero) && lane == 0 && !nz[k0]) atomicOr(&nz[k0], 1);
    } else if (nonzero && !nz[k]) {
      atomicOr(&nz[k], 1);
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&status[DICM_ST_NONFINITE], 2);
}

// bias corrections 1 / (1 - beta^t) = -1 / expm1(t ln beta): no cancellation
// at small t and no FP64 (which is a slow path on this part); ln beta is
// computed once on the host in double
__device__ __forceinline__ float inv_one_minus_pow(float ln_beta, int t) { return -1.f / expm1f((float)t * ln_beta); }

__global__ void k_dense_update(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                               float* __restrict__ v, const int32_t* __restrict__ t, const __grid_constant__ Spans s,
                               const int32_t* __restrict__ nz, const int32_t* __restrict__ status, float lr, float b1,
                               float b2, float eps, float ln_b1, float ln_b2) {
  if (status[DICM_ST_NONFINITE] || status[DICM_ST_KEY_FLAG] || status[DICM_ST_P2P_TIMEOUT]) return;
  const int64_t total = s.off[s.n];
  int cur = -1;
  float c1 = 0.f, c2 = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = span_of(s, i);
    if (!nz[k]) continue;
    if (k != cur) {
      cur = k;
      const int tt = t[k] + 1;
      c1 = inv_one_minus_pow(ln_b1, tt);
      c2 = inv_one_minus_pow(ln_b2, tt);
    }
    const float gi = g[i];
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p[i] -= lr * (mi * c1) / (sqrtf(vi * c2) + eps);
  }
}

__global__ void k_dense_steps(int32_t* __restrict__ t, const int32_t* __restrict__ nz, int n,
                              const int32_t* __restrict__ status) {
  if (status[DICM_ST_NONFINITE] || status[DICM_ST_KEY_FLAG] || status[DICM_ST_P2P_TIMEOUT]) return;
  const int k = threadIdx.x;
  if (k < n && nz[k]) t[k] += 1;
}

struct Tables {
  dicm_table_state_t t[DICM_MAX_FIELDS];
  int n;
};

// three lanes per row, one float4 (4 of the 12 columns) each: consecutive
// unique keys are ascending rows, so a warp's 10 rows stream contiguously
// through dense tables
__global__ void k_rows(const __grid_constant__ Tables tb, const int32_t* __restrict__ keys,
                       const int32_t* __restrict__ count, int64_t max_rows, const float* __restrict__ grads, float lr,
                       float b1, float b2, float eps, float ln_b1, float ln_b2, const int32_t* __restrict__ status) {
  if (status[DICM_ST_NONFINITE] || status[DICM_ST_KEY_FLAG] || status[DICM_ST_P2P_TIMEOUT]) return;
  const int64_t n = min((int64_t)*count, max_rows);
  const int lane = threadIdx.x & 31, part = lane % 3, slot = lane / 3;  // lanes 30, 31 idle
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w * 10 < n; w += warps) {
    const int64_t u = w * 10 + slot;
    const bool live = slot < 10 && u < n;
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t key = 0;
    if (live) {  // the gradient and the key in flight together
      g = __ldcg(reinterpret_cast<const float4*>(grads + u * DICM_D) + part);
      key = __ldg(keys + u);
    }
    const bool nz = g.x != 0.f || g.y != 0.f || g.z != 0.f || g.w != 0.f;
    const unsigned any = __ballot_sync(0xffffffffu, nz);
    const unsigned grp = 7u << (3 * (lane / 3));
    if (!live || !(any & grp)) continue;  // all-zero row: skipped (optim.py:93-94)
    int k = 0;
    while (k + 1 < tb.n && key >= tb.t[k + 1].base) ++k;
    const dicm_table_state_t& T = tb.t[k];
    const int64_t row = key - T.base;
    const int tt = T.t[row] + 1;
    const float c1 = inv_one_minus_pow(ln_b1, tt);
    const float c2 = inv_one_minus_pow(ln_b2, tt);
    float4* pm = reinterpret_cast<float4*>(T.m + row * DICM_D) + part;
    float4* pv = reinterpret_cast<float4*>(T.v + row * DICM_D) + part;
    float4* pp = reinterpret_cast<float4*>(T.table + row * DICM_D) + part;
    float4 m4 = *pm, v4 = *pv, p4 = *pp;
    const float gv[4] = {g.x, g.y, g.z, g.w};
    float mv[4] = {m4.x, m4.y, m4.z, m4.w}, vv[4] = {v4.x, v4.y, v4.z, v4.w}, pv4[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      mv[c] = b1 * mv[c] + (1.f - b1) * gv[c];
      vv[c] = b2 * vv[c] + (1.f - b2) * gv[c] * gv[c];
      pv4[c] -= lr * (mv[c] * c1) / (sqrtf(vv[c] * c2) + eps);
    }
    *pm = make_float4(mv[0], mv[1], mv[2], mv[3]);
    *pv = make_float4(vv[0], vv[1], vv[2], vv[3]);
    *pp = make_float4(pv4[0], pv4[1], pv4[2], pv4[3]);
    if (part == 0) T.t[row] = tt;
  }
}

}  // namespace

extern "C" {

size_t dicm_adam_dense_workspace(int nspans) { return (size_t)(nspans + 1) * 4 + 256; }

int dicm_adam_dense(float* param, const float* grad, float* m, float* v, int32_t* t, const dicm_span_t* spans,
                    int nspans, float lr, float beta1, float beta2, float eps, void* workspace,
                    size_t workspace_bytes, int32_t* status, dicm_stream_t stream) {
  using namespace dicm;
  if (nspans < 1 || nspans > MAXSPANS) return fail(DICM_ERR_VALUE, "adam_dense: %d spans (max %d)", nspans, MAXSPANS);
  if (workspace_bytes < dicm_adam_dense_workspace(nspans)) return fail(DICM_ERR_VALUE, "adam_dense: workspace");
  Spans s{};
  s.n = nspans;
  int64_t off = 0;
  for (int i = 0; i < nspans; ++i) {
    if (spans[i].offset != off) return fail(DICM_ERR_VALUE, "adam_dense: spans must tile the buffer contiguously");
    s.off[i] = off;
    off += spans[i].size;
  }
  s.off[nspans] = off;
  cudaStream_t st = (cudaStream_t)stream;
  int32_t* nz = (int32_t*)workspace;
  int rc = check_cuda(cudaMemsetAsync(nz, 0, nspans * 4, st), "adam_dense memset");
  if (rc) return rc;
  const int grid = dicm_grid(off, 256, 148 * 8);
  k_dense_flags<<<grid, 256, 0, st>>>(grad, s, nz, status);
  k_dense_update<<<grid, 256, 0, st>>>(param, grad, m, v, t, s, nz, status, lr, beta1, beta2, eps,
                                       (float)log((double)beta1), (float)log((double)beta2));
  k_dense_steps<<<1, MAXSPANS, 0, st>>>(t, nz, nspans, status);
  return last_launch("dicm_adam_dense");
}

int dicm_adam_rows(const dicm_table_state_t* tabs, int ntab, const int32_t* uniq_keys, const int32_t* count_dev,
                   int64_t max_rows, const float* grads, float lr, float beta1, float beta2, float eps,
                   int32_t* status, dicm_stream_t stream) {
  using namespace dicm;
  if (ntab < 1 || ntab > DICM_MAX_FIELDS) return fail(DICM_ERR_VALUE, "adam_rows: %d tables", ntab);
  if (max_rows <= 0) return DICM_OK;
  Tables tb{};
  tb.n = ntab;
  for (int i = 0; i < ntab; ++i) {
    tb.t[i] = tabs[i];
    if (i && tabs[i].base < tabs[i - 1].base + tabs[i - 1].vocab)
      return fail(DICM_ERR_VALUE, "adam_rows: table key ranges must be ascending and disjoint");
  }
  k_rows<<<dicm_grid((max_rows + 9) / 10 * 32, 256, 148 * 8), 256, 0, (cudaStream_t)stream>>>(tb, uniq_keys, count_dev, max_rows,
                                                                              grads, lr, beta1, beta2, eps,
                                                                              (float)log((double)beta1),
                                                                              (float)log((double)beta2), status);
  return last_launch("dicm_adam_rows");
}

}  // extern "C"
