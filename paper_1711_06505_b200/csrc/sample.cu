// a6-a10: per-sample gather and behavior aggregation, forward and backward.
//
// One warp owns one sample.  Forward builds the head input row
//   x[b] = [field vectors (schema order) | ad-image emb | pooled behaviors]
// (reference model.py:358-397) straight from the embedding tables and the
// deduplicated image embeddings E (gathered through the dedup inverse).
// Attentive pooling (model.py:206-215) is restructured so the per-reference
// cost is a 12->32 projection:  W0 [q || k] = Wq q + Wk k, with P = Wq q + b0
// formed once per sample; the segment softmax is computed online (running
// max / sum per lane, merged across the warp), and (max, sum) are kept for
// the backward pass together with the raw scores.
//
// Backward reverses the graph (segment_softmax bwd autograd.py:334-337,
// col_scale bwd 348-350, linear/prelu bwd 201-204/222-225).  The embedding and
// ID-row gradients (np.add.at into the deduplicated rows, autograd.py:267-271)
// are NOT scattered with float atomics: per-reference gradient rows that are
// not already a row of the head-input gradient (attention dk, max / concat
// routing) are written once per reference, per-sample query gradients once
// per sample, and k_ref_reduce then forms every unique row as the sum of its
// references in ascending reference order (the dedup inverse transposed by
// dicm_ref_transpose) -- bit-reproducible like the reference (runtime.py:16-21).
// Attention runs one kernel per channel, so each launch carries only the
// registers its own work needs; its parameter gradients are accumulated
// lane-per-hidden-unit and written as deterministic block partials.
//
// Every per-reference loop keeps several independent row loads in flight per
// lane (the index -> row gather chain is L2-latency bound otherwise).
#include <climits>
#include <stdlib.h>
#include <math.h>

#include "common.cuh"

namespace {
using namespace dicm;

constexpr unsigned FULL = 0xffffffffu;
constexpr int FWD_WARPS = 8;
constexpr int BWD_WARPS = 8;
constexpr int MAXQ = 2 * DICM_D;
constexpr int UNR = 4;  // rows in flight per lane in the gather loops

__device__ __forceinline__ void load12(const float* p, float (&v)[DICM_D]) {
  const Row12 r = load_row12(p);
#pragma unroll
  for (int c = 0; c < DICM_D; ++c) v[c] = r.v[c];
}

// acc += sum_{i in [i0, i1)} T[ids[i]]  (lane-strided, UNR rows in flight)
__device__ __forceinline__ void seg_sum(const int32_t* __restrict__ ids, int64_t i0, int64_t i1,
                                        const float* __restrict__ T, int lane, float (&acc)[DICM_D]) {
  for (int64_t b = i0 + lane; b < i1; b += 32 * UNR) {
    int id[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) id[u] = b + 32 * u < i1 ? __ldg(ids + b + 32 * u) : -1;
    Row12 r[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (id[u] >= 0) {
        r[u] = load_row12(T + (int64_t)id[u] * DICM_D);
      } else {
#pragma unroll
        for (int c = 0; c < DICM_D; ++c) r[u].v[c] = 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int c = 0; c < DICM_D; ++c) acc[c] += r[u].v[c];
  }
}

struct __align__(16) AttnSmem {
  float wq[DICM_ATT][MAXQ];
  float wk[DICM_ATT][DICM_D];
  float wkT[DICM_D][DICM_ATT];  // Wk transposed: 8 hidden units per two 16-B reads
  float b0[DICM_ATT], a0[DICM_ATT], w1[DICM_ATT];
  float b1;
};

struct Args {
  dicm_layout_t L;
  dicm_batch_view_t V;
  dicm_attn_params_t A[2];
  float* head_in;
  float* scores;
  float* stats;
  const float* d_head_in;
  float* d_emb;
  float* d_rows;
  float* attn_part;
};


__device__ void load_attn(AttnSmem& s, const dicm_attn_params_t& p, int dq) {
  const int in = dq + DICM_D;
  for (int i = threadIdx.x; i < DICM_ATT * in; i += blockDim.x) {
    const int j = i / in, t = i % in;
    const float v = p.w0[i];
    if (t < dq) {
      s.wq[j][t] = v;
    } else {
      s.wk[j][t - dq] = v;
      s.wkT[t - dq][j] = v;
    }
  }
  for (int j = threadIdx.x; j < DICM_ATT; j += blockDim.x) {
    s.b0[j] = p.b0[j];
    s.a0[j] = p.a0[j];
    s.w1[j] = p.w1[j];
  }
  if (threadIdx.x == 0) s.b1 = p.b1[0];
}

// the query of a channel, in every lane: ch 0 = ad-image embedding,
// ch 1 = hstack of the ID query fields (one-hot rows)
template <int DQ>
__device__ __forceinline__ void load_query(const Args& a, int ch, int b, float (&q)[DQ]) {
  if (ch == 0) {
    const Row12 r = load_row12(a.V.emb + (int64_t)a.V.ad_local[b] * DICM_D);
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) q[c] = r.v[c];
  } else {
#pragma unroll
    for (int f = 0; f < DQ / DICM_D; ++f) {
      const int fi = a.L.query_field[f];
      const Row12 r = load_row12(a.V.tables[fi] + (int64_t)a.V.field_inv[fi][b] * DICM_D);
#pragma unroll
      for (int c = 0; c < DICM_D; ++c) q[f * DICM_D + c] = r.v[c];
    }
  }
}

template <int DQ>
__device__ __forceinline__ float query_proj(const AttnSmem& s, const float (&q)[DQ], int j) {
  float p = s.b0[j];
#pragma unroll
  for (int t = 0; t < DQ; ++t) p = fmaf(s.wq[j][t], q[t], p);
  return p;
}

// score of one reference with its key projection recomputed from the 48-B
// row (no per-reference projection gather): pre_j = P_j + sum_c Wk[j][c] k_c
// in ascending c (the order the backward recomputes it in), eight hidden
// units at a time as paired FMAs from the transposed Wk
__device__ __forceinline__ float attn_score_rc(const AttnSmem& s, const float* P, const Row12& k) {
  float sc = s.b1;
#pragma unroll
  for (int g = 0; g < DICM_ATT / 8; ++g) {
    const float4 p0 = reinterpret_cast<const float4*>(P)[2 * g], p1 = reinterpret_cast<const float4*>(P)[2 * g + 1];
    float pre[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) {
      const float4* w = reinterpret_cast<const float4*>(&s.wkT[c][8 * g]);
      const float4 wa = w[0], wb = w[1];
      ffma2(pre[0], pre[1], wa.x, wa.y, k.v[c]);
      ffma2(pre[2], pre[3], wa.z, wa.w, k.v[c]);
      ffma2(pre[4], pre[5], wb.x, wb.y, k.v[c]);
      ffma2(pre[6], pre[7], wb.z, wb.w, k.v[c]);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) sc = fmaf(s.w1[8 * g + e], prelu(pre[e], s.a0[8 * g + e]), sc);
  }
  return sc;
}

// the scores of two references at once (each bit-identical to
// attn_score_rc's): every 16-B read of the transposed Wk feeds both, halving
// the shared-memory traffic per reference (the forward's limiter)
__device__ __forceinline__ void attn_score_rc2(const AttnSmem& s, const float* P, const Row12& ka, const Row12& kb,
                                               float& sa, float& sb) {
  sa = s.b1;
  sb = s.b1;
#pragma unroll
  for (int g = 0; g < DICM_ATT / 8; ++g) {
    const float4 p0 = reinterpret_cast<const float4*>(P)[2 * g], p1 = reinterpret_cast<const float4*>(P)[2 * g + 1];
    float pa[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
    float pb[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) {
      const float4* w = reinterpret_cast<const float4*>(&s.wkT[c][8 * g]);
      const float4 wa = w[0], wb = w[1];
      ffma2(pa[0], pa[1], wa.x, wa.y, ka.v[c]);
      ffma2(pa[2], pa[3], wa.z, wa.w, ka.v[c]);
      ffma2(pa[4], pa[5], wb.x, wb.y, ka.v[c]);
      ffma2(pa[6], pa[7], wb.z, wb.w, ka.v[c]);
      ffma2(pb[0], pb[1], wa.x, wa.y, kb.v[c]);
      ffma2(pb[2], pb[3], wa.z, wa.w, kb.v[c]);
      ffma2(pb[4], pb[5], wb.x, wb.y, kb.v[c]);
      ffma2(pb[6], pb[7], wb.z, wb.w, kb.v[c]);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float w1 = s.w1[8 * g + e], al = s.a0[8 * g + e];
      sa = fmaf(w1, prelu(pa[e], al), sa);
      sb = fmaf(w1, prelu(pb[e], al), sb);
    }
  }
}

// per-column max over a sample's behaviors and its FIRST argmax (the reference
// keeps the earliest row on ties); every lane ends with the warp result;
// am[c] = -1 for an empty segment
__device__ __forceinline__ void seg_max(const Args& a, int b, int lane, float (&m)[DICM_D], int (&am)[DICM_D]) {
  const int64_t i0 = a.V.beh_off[b], i1 = a.V.beh_off[b + 1];
#pragma unroll
  for (int c = 0; c < DICM_D; ++c) {
    m[c] = -INFINITY;
    am[c] = INT_MAX;
  }
  for (int64_t i = i0 + lane; i < i1; i += 32) {
    const Row12 r = load_row12(a.V.emb + (int64_t)__ldg(a.V.beh_local + i) * DICM_D);
#pragma unroll
    for (int c = 0; c < DICM_D; ++c)
      if (r.v[c] > m[c] || am[c] == INT_MAX) {  // first row of this lane, or strictly larger
        m[c] = r.v[c];
        am[c] = (int)(i - i0);
      }
  }
#pragma unroll
  for (int c = 0; c < DICM_D; ++c) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float mo = __shfl_xor_sync(FULL, m[c], o);
      const int ao = __shfl_xor_sync(FULL, am[c], o);
      if (ao != INT_MAX && (am[c] == INT_MAX || mo > m[c] || (mo == m[c] && ao < am[c]))) {
        m[c] = mo;
        am[c] = ao;
      }
    }
    if (am[c] == INT_MAX) am[c] = -1;
  }
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------

template <int DQ, bool PAIR>  // PAIR: two references per lane per pass (more registers, half the Wk reads)
__device__ void attn_fwd(const Args& a, const AttnSmem& s, int ch, int b, int lane, float* P) {
  {
    float q[DQ];
    load_query<DQ>(a, ch, b, q);
    const float pj = query_proj<DQ>(s, q, lane);
    __syncwarp();
    P[lane] = pj;
    __syncwarp();
  }
  const int64_t i0 = a.V.beh_off[b], i1 = a.V.beh_off[b + 1];
  float m = -INFINITY, ssum = 0.f, acc[DICM_D];
#pragma unroll
  for (int c = 0; c < DICM_D; ++c) acc[c] = 0.f;
  const bool norm = a.L.normalize != 0;
  auto take = [&](float sc, const Row12& k) {  // online segment softmax (or the raw weighted sum)
    if (norm) {
      const float mn = fmaxf(m, sc);
      const float scale = expf(m - mn);  // exp(-inf) = 0 on the first element
      const float e = expf(sc - mn);
      ssum = ssum * scale + e;
#pragma unroll
      for (int c = 0; c < DICM_D; ++c) acc[c] = fmaf(e, k.v[c], acc[c] * scale);
      m = mn;
    } else {
#pragma unroll
      for (int c = 0; c < DICM_D; ++c) acc[c] = fmaf(sc, k.v[c], acc[c]);
    }
  };
  auto row_of = [&](int64_t i) { return load_row12(a.V.emb + (int64_t)__ldg(a.V.beh_local + i) * DICM_D); };
  // chunks of 64 references (lane: references c0 + lane and c0 + 32 + lane,
  // scored together) while more than 32 remain, then one chunk of <= 32; the
  // next chunk's rows are in flight while this one is scored
  float* scores = a.scores + (int64_t)ch * a.V.refs;
  if (!PAIR) {
    // one reference per lane per pass; the next reference's row (and the one
    // after's index) are in flight while this one is scored
    Row12 k_n;
    int32_t u_nn = 0;
    {
      const int64_t i = i0 + lane;
      if (i < i1) k_n = load_row12(a.V.emb + (int64_t)__ldg(a.V.beh_local + i) * DICM_D);
      if (i + 32 < i1) u_nn = __ldg(a.V.beh_local + i + 32);
    }
    for (int64_t i = i0 + lane; i < i1; i += 32) {
      const Row12 k = k_n;
      if (i + 32 < i1) k_n = load_row12(a.V.emb + (int64_t)u_nn * DICM_D);
      if (i + 64 < i1) u_nn = __ldg(a.V.beh_local + i + 64);
      const float sc = attn_score_rc(s, P, k);
      scores[i] = sc;
      take(sc, k);
    }
  } else {
  Row12 ka, kb;
  if (i0 + lane < i1) ka = row_of(i0 + lane);
  if (i0 + 32 + lane < i1) kb = row_of(i0 + 32 + lane);
  for (int64_t c0 = i0; c0 < i1;) {
    const bool two = i1 - c0 > 32;  // warp-uniform
    const int64_t ia = c0 + lane, ib = ia + 32, n0 = c0 + (two ? 64 : 32);
    Row12 na, nb;
    if (n0 + lane < i1) na = row_of(n0 + lane);
    if (n0 + 32 + lane < i1) nb = row_of(n0 + 32 + lane);
    if (two) {
      float sa, sb;
      attn_score_rc2(s, P, ka, kb, sa, sb);
      scores[ia] = sa;
      take(sa, ka);
      if (ib < i1) {
        scores[ib] = sb;
        take(sb, kb);
      }
    } else if (ia < i1) {
      const float sa = attn_score_rc(s, P, ka);
      scores[ia] = sa;
      take(sa, ka);
    }
    ka = na;
    kb = nb;
    c0 = n0;
  }
  }
  float out[DICM_D];
  if (norm) {
    const float M = warp_max(m);
    const float f = (m == -INFINITY) ? 0.f : expf(m - M);
    const float S = warp_sum(ssum * f);
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) out[c] = warp_sum(acc[c] * f);
    const float inv = S > 0.f ? 1.f / S : 0.f;
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) out[c] *= inv;
    if (lane == 0) {
      a.stats[((int64_t)ch * a.V.batch + b) * 2] = M;
      a.stats[((int64_t)ch * a.V.batch + b) * 2 + 1] = S;
    }
  } else {
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) out[c] = warp_sum(acc[c]);
  }
  float* dst = a.head_in + (int64_t)b * a.L.width + a.L.pool_col + ch * DICM_D;
#pragma unroll
  for (int c = 0; c < DICM_D; ++c)
    if (lane == c) dst[c] = out[c];
}

// PART: 0 = the whole head input; 1 = the ID-field columns only; 2 = the
// image columns only (ad image, pooled behaviors).  The step runs part 1 on a
// forked stream as soon as the compact ID rows exist (beside the image-MLP
// forward) and part 2 on the main stream, each with only its own registers.
template <int MINB, int PART, int KIND = -1>  // MINB: resident blocks per SM the register budget is cut for;
                                             // KIND >= 0: only that aggregator's code (PART 2)
__global__ void __launch_bounds__(FWD_WARPS * 32, MINB) k_sample_fwd(const __grid_constant__ Args a) {
  __shared__ AttnSmem sa[PART == 1 ? 1 : 2];
  __shared__ __align__(16) float Pw[FWD_WARPS][DICM_ATT];  // per-warp query projection
  const bool att = PART != 1 && a.L.use_behavior_images && (a.L.kind == 1 || a.L.kind == 2);
  if constexpr (PART != 1) {
    if (att) {
      load_attn(sa[0], a.A[0], DICM_D);
      if (a.L.kind == 2) load_attn(sa[1], a.A[1], DICM_D * a.L.n_query);
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int b = blockIdx.x * FWD_WARPS + warp; b < a.V.batch; b += gridDim.x * FWD_WARPS) {
    float* row = a.head_in + (int64_t)b * a.L.width;
    // ID fields: one-hot rows and multi-hot sums
    for (int f = 0; PART != 2 && f < a.L.n_fields; ++f) {
      const float* T = a.V.tables[f];
      if (!a.L.field_multi[f]) {
        if (lane < DICM_D) row[a.L.field_col[f] + lane] = __ldg(T + (int64_t)a.V.field_inv[f][b] * DICM_D + lane);
      } else {
        const int32_t* off = a.V.field_off[f];
        float acc[DICM_D];
#pragma unroll
        for (int c = 0; c < DICM_D; ++c) acc[c] = 0.f;
        seg_sum(a.V.field_inv[f], off[b], off[b + 1], T, lane, acc);  // rows of the compact table
#pragma unroll
        for (int c = 0; c < DICM_D; ++c) acc[c] = warp_sum(acc[c]);
#pragma unroll
        for (int c = 0; c < DICM_D; ++c)
          if (lane == c) row[a.L.field_col[f] + c] = acc[c];
      }
    }
    if constexpr (PART == 1) continue;
    if (a.L.use_ad_image && lane < DICM_D)
      row[a.L.ad_col + lane] = __ldg(a.V.emb + (int64_t)a.V.ad_local[b] * DICM_D + lane);
    if (!a.L.use_behavior_images) continue;
    const int kind = KIND >= 0 ? KIND : a.L.kind;
    if (kind == 4) {  // concat (reference scatter_concat, autograd.py:370-385): slot j = j-th kept behavior
      const int64_t i0 = a.V.beh_off[b];
      const int len = (int)(a.V.beh_off[b + 1] - i0);
      const int n = a.L.width - a.L.pool_col;  // capacity * 12
      for (int e = lane; e < n; e += 32) {
        const int j = e / DICM_D;
        row[a.L.pool_col + e] = j < len ? __ldg(a.V.emb + (int64_t)__ldg(a.V.beh_local + i0 + j) * DICM_D + e % DICM_D)
                                        : 0.f;
      }
      continue;
    }
    if (kind == 3) {  // max pooling (reference segment_max, autograd.py:289-319)
      float m[DICM_D];
      int am[DICM_D];
      seg_max(a, b, lane, m, am);
#pragma unroll
      for (int c = 0; c < DICM_D; ++c)
        if (lane == c) row[a.L.pool_col + c] = am[c] < 0 ? 0.f : m[c];  // empty segment -> 0
      continue;
    }
    if (kind == 0) {
      float acc[DICM_D];
#pragma unroll
      for (int c = 0; c < DICM_D; ++c) acc[c] = 0.f;
      seg_sum(a.V.beh_local, a.V.beh_off[b], a.V.beh_off[b + 1], a.V.emb, lane, acc);
#pragma unroll
      for (int c = 0; c < DICM_D; ++c) acc[c] = warp_sum(acc[c]);
#pragma unroll
      for (int c = 0; c < DICM_D; ++c)
        if (lane == c) row[a.L.pool_col + c] = acc[c];
    } else {
      if constexpr (PART != 1) {
        attn_fwd<DICM_D, KIND == 1>(a, sa[0], 0, b, lane, Pw[warp]);
        if (kind == 2) {
          if (a.L.n_query == 2)
            attn_fwd<2 * DICM_D, false>(a, sa[1], 1, b, lane, Pw[warp]);
          else
            attn_fwd<DICM_D, false>(a, sa[1], 1, b, lane, Pw[warp]);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// backward
// ---------------------------------------------------------------------------

struct __align__(16) WarpScratch {
  float ds[32];
  float ks[32][DICM_D];
  float dp[32][DICM_ATT + 4];  // the chunk's key projections, overwritten by dpre (row = reference);
                               // stride 36: 16-B rows for cp.async, conflict-free column reads
  float wq[32][MAXQ + 1];      // lane j's dWq accumulators (kept out of registers)
};

__host__ __device__ constexpr int chan_part(int dq) { return 3 * DICM_ATT + 1 + DICM_ATT * (dq + DICM_D); }

// per-lane (= hidden unit j) accumulators of one channel
template <int DQ>
struct AttnAcc {
  float wq[DQ];
  float wk[DICM_D];
  float a0, b0, w1;
  float b1;  // lane-partial, warp-summed at the end
};

constexpr int QG_STRIDE = 3 * DICM_D;  // q_grad row: ad image (12) | ID query fields (<= 24)

template <int DQ>
__device__ void attn_bwd(const Args& a, const AttnSmem& s, WarpScratch& ws, int ch, int b, int lane,
                         AttnAcc<DQ>& acc, bool accumulate) {
  const int64_t i0 = a.V.beh_off[b], i1 = a.V.beh_off[b + 1];
  if (i1 <= i0) {  // empty segment: no references, a zero query gradient
    float* qg = a.V.q_grad + (int64_t)b * QG_STRIDE + (ch == 0 ? 0 : DICM_D);
    if (lane < DQ) qg[lane] = 0.f;
    return;
  }
  float Pj;
  {
    float q[DQ];  // reloaded at the end: not live across the reference loops
    load_query<DQ>(a, ch, b, q);
    Pj = query_proj<DQ>(s, q, lane);
  }
  const float w1j = s.w1[lane], a0j = s.a0[lane];
  float wkj[DICM_D];  // lane j's row of Wk: the key projection is recomputed per reference
#pragma unroll
  for (int c = 0; c < DICM_D; ++c) wkj[c] = s.wk[lane][c];
  float dout[DICM_D];
  const float* dsrc = a.d_head_in + (int64_t)b * a.L.width + a.L.pool_col + ch * DICM_D;
#pragma unroll
  for (int c = 0; c < DICM_D; ++c) dout[c] = __ldg(dsrc + c);
  const bool norm = a.L.normalize != 0;
  float M = 0.f, invS = 0.f;
  if (norm) {
    M = a.stats[((int64_t)ch * a.V.batch + b) * 2];
    const float S = a.stats[((int64_t)ch * a.V.batch + b) * 2 + 1];
    invS = S > 0.f ? 1.f / S : 0.f;
  }
  const float* sc = a.scores + (int64_t)ch * a.V.refs;
  // softmax backward (autograd.py:335-337) needs dot = sum_i w_i (dout . k_i)
  // = dout . (sum_i w_i k_i) = dout . out: the forward's pooled output, read
  // back from the head input instead of a second pass over the references
  float dot = 0.f;
  if (norm) {
    const float* outp = a.head_in + (int64_t)b * a.L.width + a.L.pool_col + ch * DICM_D;
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) dot = fmaf(dout[c], __ldg(outp + c), dot);
  }
  float dP = 0.f;
  // chunks of 32 references, lane r owns reference r of the chunk;
  // the next chunk's row and score are in flight while this one is processed
  int32_t row_n = i0 + lane < i1 ? __ldg(a.V.beh_local + i0 + lane) : 0;
  Row12 k_n;
  float sc_n = 0.f;
  if (i0 + lane < i1) {
    k_n = load_row12(a.V.emb + (int64_t)row_n * DICM_D);
    sc_n = sc[i0 + lane];
  }
  for (int64_t c0 = i0; c0 < i1; c0 += 32) {
    const int64_t i = c0 + lane;
    const bool valid = i < i1;
    Row12 k = k_n;
    const int32_t row = row_n;
    const float sci = sc_n;
    if (i + 32 < i1) {
      row_n = __ldg(a.V.beh_local + i + 32);
      k_n = load_row12(a.V.emb + (int64_t)row_n * DICM_D);
      sc_n = sc[i + 32];
    }
    float w = 0.f, ds = 0.f;
    if (valid) {
      float dw = 0.f;
#pragma unroll
      for (int c = 0; c < DICM_D; ++c) dw = fmaf(dout[c], k.v[c], dw);
      w = norm ? expf(sci - M) * invS : sci;
      ds = norm ? w * (dw - dot) : dw;
    } else {
#pragma unroll
      for (int c = 0; c < DICM_D; ++c) k.v[c] = 0.f;
    }
    ws.ds[lane] = ds;
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) ws.ks[lane][c] = k.v[c];
    acc.b1 += ds;
    __syncwarp();
    // lane j: hidden unit j across the chunk's references
    const int nr = (int)min((int64_t)32, i1 - c0);
    // per reference r (in order): the rest of hidden unit j's backward from its pre-activation
    auto unit = [&](int r, float pre, const float4& k0, const float4& k1, const float4& k2) {
      const float dsr = ws.ds[r];
      const float dh = dsr * w1j;
      const bool pos = pre > 0.f;
      const float dpre = pos ? dh : a0j * dh;
      acc.w1 = fmaf(dsr, pos ? pre : a0j * pre, acc.w1);
      if (!pos) acc.a0 = fmaf(pre, dh, acc.a0);
      acc.b0 += dpre;
      dP += dpre;
      // paired FMAs (FFMA2), same per-element fma.rn as before
      ffma2(acc.wk[0], acc.wk[1], k0.x, k0.y, dpre);
      ffma2(acc.wk[2], acc.wk[3], k0.z, k0.w, dpre);
      ffma2(acc.wk[4], acc.wk[5], k1.x, k1.y, dpre);
      ffma2(acc.wk[6], acc.wk[7], k1.z, k1.w, dpre);
      ffma2(acc.wk[8], acc.wk[9], k2.x, k2.y, dpre);
      ffma2(acc.wk[10], acc.wk[11], k2.z, k2.w, dpre);
      ws.dp[r][lane] = dpre;
    };
    // two references at a time: their pre-activations as paired FMAs (each
    // element the forward's chain pre = Pj, then fma(wk[c], k[c], pre) in c order)
    int r = 0;
#pragma unroll 2
    for (; r + 1 < nr; r += 2) {
      const float4* ka = reinterpret_cast<const float4*>(ws.ks[r]);
      const float4* kb = reinterpret_cast<const float4*>(ws.ks[r + 1]);
      const float4 a0 = ka[0], a1 = ka[1], a2 = ka[2], b0 = kb[0], b1 = kb[1], b2 = kb[2];
      float pa = Pj, pb = Pj;
      ffma2(pa, pb, a0.x, b0.x, wkj[0]);
      ffma2(pa, pb, a0.y, b0.y, wkj[1]);
      ffma2(pa, pb, a0.z, b0.z, wkj[2]);
      ffma2(pa, pb, a0.w, b0.w, wkj[3]);
      ffma2(pa, pb, a1.x, b1.x, wkj[4]);
      ffma2(pa, pb, a1.y, b1.y, wkj[5]);
      ffma2(pa, pb, a1.z, b1.z, wkj[6]);
      ffma2(pa, pb, a1.w, b1.w, wkj[7]);
      ffma2(pa, pb, a2.x, b2.x, wkj[8]);
      ffma2(pa, pb, a2.y, b2.y, wkj[9]);
      ffma2(pa, pb, a2.z, b2.z, wkj[10]);
      ffma2(pa, pb, a2.w, b2.w, wkj[11]);
      unit(r, pa, a0, a1, a2);
      unit(r + 1, pb, b0, b1, b2);
    }
    if (r < nr) {
      const float4* kr = reinterpret_cast<const float4*>(ws.ks[r]);
      const float4 k0 = kr[0], k1 = kr[1], k2 = kr[2];
      float pre = Pj;
      pre = fmaf(wkj[0], k0.x, pre);
      pre = fmaf(wkj[1], k0.y, pre);
      pre = fmaf(wkj[2], k0.z, pre);
      pre = fmaf(wkj[3], k0.w, pre);
      pre = fmaf(wkj[4], k1.x, pre);
      pre = fmaf(wkj[5], k1.y, pre);
      pre = fmaf(wkj[6], k1.z, pre);
      pre = fmaf(wkj[7], k1.w, pre);
      pre = fmaf(wkj[8], k2.x, pre);
      pre = fmaf(wkj[9], k2.y, pre);
      pre = fmaf(wkj[10], k2.z, pre);
      pre = fmaf(wkj[11], k2.w, pre);
      unit(r, pre, k0, k1, k2);
    }
    __syncwarp();
    if (valid) {
      float dk[DICM_D];
#pragma unroll
      for (int c = 0; c < DICM_D; ++c) dk[c] = w * dout[c];
      for (int q = 0; q < DICM_ATT / 4; ++q) {  // 16-B reads: conflict-free at stride 36
        const float4 d4 = reinterpret_cast<const float4*>(ws.dp[lane])[q];
        const float dq4[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float4* wr = reinterpret_cast<const float4*>(s.wk[4 * q + e]);
          const float4 w0 = wr[0], w1 = wr[1], w2 = wr[2];
          ffma2(dk[0], dk[1], w0.x, w0.y, dq4[e]);
          ffma2(dk[2], dk[3], w0.z, w0.w, dq4[e]);
          ffma2(dk[4], dk[5], w1.x, w1.y, dq4[e]);
          ffma2(dk[6], dk[7], w1.z, w1.w, dq4[e]);
          ffma2(dk[8], dk[9], w2.x, w2.y, dq4[e]);
          ffma2(dk[10], dk[11], w2.z, w2.w, dq4[e]);
        }
      }
      float4* g = reinterpret_cast<float4*>(a.V.ref_grad + i * DICM_D);
      if (accumulate) {  // the second channel adds to the first's row (fixed order)
        const Row12 o = load_row12_cg(a.V.ref_grad + i * DICM_D);
#pragma unroll
        for (int c = 0; c < DICM_D; ++c) dk[c] = o.v[c] + dk[c];
      }
      g[0] = make_float4(dk[0], dk[1], dk[2], dk[3]);
      g[1] = make_float4(dk[4], dk[5], dk[6], dk[7]);
      g[2] = make_float4(dk[8], dk[9], dk[10], dk[11]);
    }
    __syncwarp();
  }
  // query side: dWq[j] += dP_j q ; dq = Wq^T dP
  float q[DQ];
  load_query<DQ>(a, ch, b, q);
#pragma unroll
  for (int t = 0; t < DQ; ++t) ws.wq[lane][t] = fmaf(dP, q[t], ws.wq[lane][t]);
  // the query's gradient, once per sample: ad image (ch 0) at q_grad[b][0..12),
  // the ID query fields (ch 1) at q_grad[b][12..12+DQ)
  float* qg = a.V.q_grad + (int64_t)b * QG_STRIDE + (ch == 0 ? 0 : DICM_D);
#pragma unroll
  for (int t = 0; t < DQ; ++t) {
    const float v = warp_sum(s.wq[lane][t] * dP);
    if (lane == t) qg[t] = v;
  }
}

// writes a channel's accumulators into red[warp][...] in sorted-name order:
// 0/a [32], 0/b [32], 0/w [32 x (dq+12)], 1/b [1], 1/w [32]
template <int DQ>
__device__ void dump_acc(const AttnAcc<DQ>& acc, float* dst, int lane) {
  const int in = DQ + DICM_D;
  dst[lane] = acc.a0;
  dst[DICM_ATT + lane] = acc.b0;
  float* w = dst + 2 * DICM_ATT + lane * in;
#pragma unroll
  for (int t = 0; t < DQ; ++t) w[t] = acc.wq[t];
#pragma unroll
  for (int c = 0; c < DICM_D; ++c) w[DQ + c] = acc.wk[c];
  const float b1 = warp_sum(acc.b1);
  if (lane == 0) dst[2 * DICM_ATT + DICM_ATT * in] = b1;
  dst[2 * DICM_ATT + DICM_ATT * in + 1 + lane] = acc.w1;
}

template <int DQ>
__device__ void zero_acc(AttnAcc<DQ>& acc) {
#pragma unroll
  for (int t = 0; t < DQ; ++t) acc.wq[t] = 0.f;
#pragma unroll
  for (int c = 0; c < DICM_D; ++c) acc.wk[c] = 0.f;
  acc.a0 = acc.b0 = acc.w1 = acc.b1 = 0.f;
}

template <int DQ>
__device__ void attn_channel_bwd(const Args& a, const AttnSmem& s, WarpScratch& ws, int ch, int lane, int warp,
                                 float* red, float* part_base, bool accumulate) {
  AttnAcc<DQ> acc;
  zero_acc(acc);
#pragma unroll
  for (int t = 0; t < DQ; ++t) ws.wq[lane][t] = 0.f;
  for (int b = blockIdx.x * BWD_WARPS + warp; b < a.V.batch; b += gridDim.x * BWD_WARPS)
    attn_bwd<DQ>(a, s, ws, ch, b, lane, acc, accumulate);
#pragma unroll
  for (int t = 0; t < DQ; ++t) acc.wq[t] = ws.wq[lane][t];
  __syncthreads();  // scratch -> reduction buffer
  const int n = chan_part(DQ);
  dump_acc<DQ>(acc, red + warp * n, lane);
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    float t = 0.f;
    for (int w = 0; w < BWD_WARPS; ++w) t += red[w * n + i];
    part_base[i] = t;
  }
  __syncthreads();
}

// one attention channel per launch (its DQ fixed at compile time)
template <int DQ>
__global__ void __launch_bounds__(BWD_WARPS * 32, 2)
    k_attn_bwd(const __grid_constant__ Args a, int ch, int64_t part_stride, int64_t part_off, int accumulate) {
  __shared__ AttnSmem sa;
  extern __shared__ float dyn[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  load_attn(sa, a.A[ch], DQ);
  __syncthreads();
  WarpScratch& ws = reinterpret_cast<WarpScratch*>(dyn)[warp];
  attn_channel_bwd<DQ>(a, sa, ws, ch, lane, warp, dyn, a.attn_part + (int64_t)blockIdx.x * part_stride + part_off,
                       accumulate != 0);
}

// max / concat: the gradient of every behavior reference as its own row
// (ref_grad[i]): concat slot j of sample b carries dx[b][pool + 12 j ..];
// max routes each column's gradient to the column's first argmax row
// (segment_max bwd, autograd.py:307-315) and zero elsewhere
__global__ void __launch_bounds__(BWD_WARPS * 32) k_ref_rows(const __grid_constant__ Args a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int b = blockIdx.x * BWD_WARPS + warp; b < a.V.batch; b += gridDim.x * BWD_WARPS) {
    const float* dpool = a.d_head_in + (int64_t)b * a.L.width + a.L.pool_col;
    const int64_t i0 = a.V.beh_off[b], i1 = a.V.beh_off[b + 1];
    if (a.L.kind == 4) {
      const int n = (int)(i1 - i0) * DICM_D;  // <= width - pool_col (checked at upload)
      for (int e = lane; e < n; e += 32) a.V.ref_grad[i0 * DICM_D + e] = __ldg(dpool + e);
    } else {
      float m[DICM_D];
      int am[DICM_D];
      seg_max(a, b, lane, m, am);
      float dv[DICM_D];
      load12(dpool, dv);
      for (int64_t i = i0 + lane; i < i1; i += 32) {
        float r[DICM_D];
#pragma unroll
        for (int c = 0; c < DICM_D; ++c) r[c] = (am[c] == (int)(i - i0)) ? dv[c] : 0.f;
        float4* g = reinterpret_cast<float4*>(a.V.ref_grad + i * DICM_D);
        g[0] = make_float4(r[0], r[1], r[2], r[3]);
        g[1] = make_float4(r[4], r[5], r[6], r[7]);
        g[2] = make_float4(r[8], r[9], r[10], r[11]);
      }
    }
  }
}

// Where the gradient row of reference p of a reference list comes from:
// the list is a concatenation of segments (image list: ad images | behavior
// images; ID list: one segment per field in schema order).
//   mode 0: one reference per sample, b = p - begin: dx[b][col..] (+ the
//           attention query gradient q_grad[b][qcol..] when qgrad is set)
//   mode 1: CSR references, b = map[p - begin]: dx[b][col..] (sum pooling
//           and multi-hot sum fields: every reference gets the pooled row's
//           gradient, segment_sum bwd autograd.py:284-285)
//   mode 2: a row of its own, rows[p - begin] (attention dk, max, concat)
struct RefSeg {
  int64_t begin;
  const int32_t* map;
  const float* rows;
  const float* qgrad;
  int32_t mode, col, qcol, pad;
};

struct RefSrc {
  RefSeg s[DICM_MAX_FIELDS + 1];
  int32_t n, width;
  const float* dx;
};

__device__ __forceinline__ void ref_contrib(const RefSrc& S, int64_t p, float (&v)[DICM_D]) {
  int k = 0;
  while (k + 1 < S.n && S.s[k + 1].begin <= p) ++k;
  const RefSeg& g = S.s[k];
  const int64_t i = p - g.begin;
  if (g.mode == 2) {
    const Row12 r = load_row12_cg(g.rows + i * DICM_D);
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) v[c] = r.v[c];
    return;
  }
  const int64_t b = g.mode == 0 ? i : (int64_t)__ldg(g.map + i);
  const Row12 r = load_row12(S.dx + b * S.width + g.col);
#pragma unroll
  for (int c = 0; c < DICM_D; ++c) v[c] = r.v[c];
  if (g.qgrad) {
    const Row12 q = load_row12_cg(g.qgrad + b * QG_STRIDE + g.qcol);
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) v[c] += q.v[c];
  }
}

constexpr int HOT_REFS = 32;    // more references: one block per key (k_ref_reduce_hot)
constexpr int THREAD_REFS = 16;  // up to this many: one thread (sorting network); 17..32: one warp (k_ref_reduce_mid)

// ascending sort of N positions held in registers (bitonic network, every
// index a compile-time constant after unrolling)
template <int N>
__device__ __forceinline__ void sort_net(int32_t (&a)[N]) {
#pragma unroll
  for (int k = 2; k <= N; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int l = i ^ j;
        if (l > i) {
          const int32_t x = a[i], y = a[l];
          const bool sw = ((i & k) == 0) ? (x > y) : (x < y);
          a[i] = sw ? y : x;
          a[l] = sw ? x : y;
        }
      }
}

// a group of 3..N references by one thread: positions sorted in registers,
// rows fetched two at a time and summed in ascending reference order
template <int N>
__device__ __forceinline__ void thread_group(const RefSrc& S, const int32_t* __restrict__ order, int32_t s0, int cnt,
                                             float (&r)[DICM_D]) {
  int32_t p[N];
#pragma unroll
  for (int i = 0; i < N; ++i) p[i] = i < cnt ? __ldg(order + s0 + i) : INT_MAX;
  sort_net<N>(p);
  ref_contrib(S, p[0], r);
#pragma unroll
  for (int i = 1; i < N; i += 2) {
    if (i >= cnt) break;
    float v0[DICM_D], v1[DICM_D];
    ref_contrib(S, p[i], v0);
    const bool two = i + 1 < cnt;
    if (two) ref_contrib(S, p[i + 1], v1);
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) r[c] += v0[c];
    if (two)
#pragma unroll
      for (int c = 0; c < DICM_D; ++c) r[c] += v1[c];
  }
}

__device__ __forceinline__ void store_row12(float* p, const float (&v)[DICM_D]) {
  float4* q = reinterpret_cast<float4*>(p);
  q[0] = make_float4(v[0], v[1], v[2], v[3]);
  q[1] = make_float4(v[4], v[5], v[6], v[7]);
  q[2] = make_float4(v[8], v[9], v[10], v[11]);
}

// Exact, order-independent sums.  A key's references come in no particular
// order (the counting-sort transpose fills groups through atomic cursors), so
// each component is summed in 64-bit fixed point: scale 2^shift chosen from
// the group's largest finite |value| (max is order-independent) and count so
// that the integer sum cannot overflow; integer addition is associative, hence
// the same bits whatever the order (or however the group is split over
// threads and blocks), and the sum is exact up to the per-term rounding at
// 2^-shift (far below fp32's).  Non-finite components are tracked as flags:
// any nan, or both infinities -> nan, else the infinity's sign -- the outcome
// of the fp32 sum in every order.
constexpr int FL_POS = 16, FL_NEG = 32;  // flag bits: c nan, FL_POS + c +inf, FL_NEG + c -inf

__device__ __forceinline__ unsigned long long fx_flags(float v, int c) {
  if (isnan(v)) return 1ull << c;
  if (isinf(v)) return 1ull << ((v > 0.f ? FL_POS : FL_NEG) + c);
  return 0ull;
}

// max(|v|) over the finite values as float bits (non-negative floats order like their bits)
__device__ __forceinline__ unsigned fx_bits(float v) { return isfinite(v) ? __float_as_uint(fabsf(v)) : 0u; }

__device__ __forceinline__ int fx_shift(float mx, int n) {
  int e;
  frexpf(mx, &e);  // mx < 2^e
  const int lg = n > 1 ? 32 - __clz(n - 1) : 0;  // ceil(log2 n)
  return 62 - e - lg;
}

__device__ __forceinline__ long long fx_quant(float v, int shift) {
  return isfinite(v) ? __double2ll_rn(ldexp((double)v, shift)) : 0ll;
}

__device__ __forceinline__ float fx_result(long long q, int shift, float mx, unsigned long long fl, int c) {
  const bool nan = (fl >> c) & 1ull, pos = (fl >> (FL_POS + c)) & 1ull, neg = (fl >> (FL_NEG + c)) & 1ull;
  if (nan || (pos && neg)) return __int_as_float(0x7fffffff);
  if (pos) return __int_as_float(0x7f800000);
  if (neg) return __int_as_float(0xff800000);
  if (mx == 0.f) return 0.f;
  return (float)ldexp((double)q, -shift);  // exact scaling of the (53-bit rounded) sum, then fp32 rounding
}

// Keys with more than HOT_REFS references.  The first HOT_SLOTS listed keys
// get accumulators (dicm_batch_view_t.hot_acc) and are split into chunks of
// HOT_CHUNK references spread over every block: k_ref_mid_hot forms each
// key's maxima and flags, k_ref_reduce_hot its fixed-point sums (integer
// atomics: exact, so the split does not change a bit), and the last block to
// finish writes the rows.  Keys past HOT_SLOTS (or every key without
// accumulators) are summed one block each with the same arithmetic.
constexpr int HOT_SLOTS = 4096;
constexpr int HOT_CHUNK = 256;  // = block size: one reference per thread
struct HotEnt {
  int32_t u, s0, cnt, pad;
};
struct HotAcc {  // one key list's accumulators
  unsigned done, pad[3];
  HotEnt ent[HOT_SLOTS];
  unsigned mx[HOT_SLOTS][DICM_D];
  unsigned long long fl[HOT_SLOTS];
  long long q[HOT_SLOTS][DICM_D];
};

// out[u] = sum of the gradient rows of key u's references in ascending
// reference order (np.add.at's order).  Thread per key for up to 16
// references (positions sorted in registers); keys with 17..32 references
// are listed for mid_pass (a warp each), larger ones for the hot-key
// passes (exact fixed point).
template <int MINB>  // DICM_REDUCE_OCC: 2 or 3 (default) resident blocks per SM
__global__ void __launch_bounds__(256, MINB) k_ref_reduce(const __grid_constant__ RefSrc S,
                                                          const int32_t* __restrict__ order,
                                                          const int32_t* __restrict__ start,
                                                          const int32_t* __restrict__ n_keys, int64_t cap,
                                                          float* __restrict__ out, int32_t* __restrict__ counters,
                                                          int32_t* __restrict__ hot_list,
                                                          int32_t* __restrict__ mid_list, HotAcc* __restrict__ acc) {
  const int64_t n = min((int64_t)*n_keys, cap);
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s0 = __ldg(start + u), s1 = __ldg(start + u + 1);
    const int cnt = s1 - s0;
    if (cnt > HOT_REFS) {
      const int h = atomicAdd(counters, 1);
      hot_list[h] = (int32_t)u;
      if (acc && h < HOT_SLOTS) {  // this key's accumulator slot, cleared for the chunk passes
        acc->ent[h] = HotEnt{(int32_t)u, s0, cnt, 0};
#pragma unroll
        for (int c = 0; c < DICM_D; ++c) {
          acc->mx[h][c] = 0u;
          acc->q[h][c] = 0ll;
        }
        acc->fl[h] = 0ull;
      }
      continue;
    }
    if (cnt > THREAD_REFS) {
      mid_list[atomicAdd(counters + 1, 1)] = (int32_t)u;
      continue;
    }
    if (cnt > 2) {
      float r[DICM_D];
      if (cnt <= 4)
        thread_group<4>(S, order, s0, cnt, r);
      else if (cnt <= 8)
        thread_group<8>(S, order, s0, cnt, r);
      else
        thread_group<16>(S, order, s0, cnt, r);
      store_row12(out + u * DICM_D, r);
      continue;
    }
    int32_t p0 = __ldg(order + s0), p1 = cnt > 1 ? __ldg(order + s0 + 1) : INT_MAX;
    if (p1 < p0) {
      const int32_t x = p0;
      p0 = p1;
      p1 = x;
    }
    float r[DICM_D];
    ref_contrib(S, p0, r);
    if (cnt > 1) {
      float v[DICM_D];
      ref_contrib(S, p1, v);
#pragma unroll
      for (int c = 0; c < DICM_D; ++c) r[c] += v[c];
    }
    store_row12(out + u * DICM_D, r);
  }
}

// the keys with 17..32 references, a warp each: lane i takes reference i, its
// rank by position (a 32-way compare), the rows land in rank order in shared
// memory and lanes 0..11 sum their column in ascending reference order
__device__ __forceinline__ void mid_pass(const RefSrc& S, const int32_t* __restrict__ order,
                                         const int32_t* __restrict__ start, const int32_t* __restrict__ mid_count,
                                         const int32_t* __restrict__ mid_list, float* __restrict__ out) {
  __shared__ float slots[8][32][DICM_D + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nm = *mid_count;
  for (int w = blockIdx.x * 8 + warp; w < nm; w += gridDim.x * 8) {
    const int32_t u = __ldg(mid_list + w);
    const int32_t s0 = __ldg(start + u), cnt = __ldg(start + u + 1) - s0;
    const int32_t p = lane < cnt ? __ldg(order + s0 + lane) : INT_MAX;
    int rank = 0;
    for (int j = 0; j < cnt; ++j) rank += __shfl_sync(FULL, p, j) < p;
    if (lane < cnt) {
      float v[DICM_D];
      ref_contrib(S, p, v);
#pragma unroll
      for (int c = 0; c < DICM_D; ++c) slots[warp][rank][c] = v[c];
    }
    __syncwarp();
    if (lane < DICM_D) {
      float acc = slots[warp][0][lane];
      for (int i = 1; i < cnt; ++i) acc += slots[warp][i][lane];
      out[(int64_t)u * DICM_D + lane] = acc;
    }
    __syncwarp();
  }
}

// one hot key by one block (keys without an accumulator slot): per-thread
// partial maxima / flags / fixed-point sums over references t, t + 256, ...,
// combined in shared memory (integer sums associative, maxima and flags
// order-independent)
__device__ void hot_block(const RefSrc& S, const int32_t* __restrict__ order, int32_t u, int32_t s0, int32_t s1,
                          float* __restrict__ out) {
  __shared__ unsigned smx[8][DICM_D];
  __shared__ unsigned long long sfl[8];
  __shared__ long long sq[8][DICM_D];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  unsigned m[DICM_D];
  unsigned long long fl = 0;
#pragma unroll
  for (int c = 0; c < DICM_D; ++c) m[c] = 0u;
  for (int32_t j = s0 + t; j < s1; j += 256) {
    float v[DICM_D];
    ref_contrib(S, __ldg(order + j), v);
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) {
      m[c] = max(m[c], fx_bits(v[c]));
      fl |= fx_flags(v[c], c);
    }
  }
#pragma unroll
  for (int c = 0; c < DICM_D; ++c) m[c] = __reduce_max_sync(FULL, m[c]);
  fl = ((unsigned long long)__reduce_or_sync(FULL, (unsigned)(fl >> 32)) << 32) | __reduce_or_sync(FULL, (unsigned)fl);
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) smx[warp][c] = m[c];
    sfl[warp] = fl;
  }
  __syncthreads();
  int sh[DICM_D];
  long long q[DICM_D];
#pragma unroll
  for (int c = 0; c < DICM_D; ++c) {
    unsigned mm = 0u;
    for (int w = 0; w < 8; ++w) mm = max(mm, smx[w][c]);
    sh[c] = fx_shift(__uint_as_float(mm), s1 - s0);
    q[c] = 0;
  }
  fl = 0;
  for (int w = 0; w < 8; ++w) fl |= sfl[w];
  for (int32_t j = s0 + t; j < s1; j += 256) {
    float v[DICM_D];
    ref_contrib(S, __ldg(order + j), v);
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) q[c] += fx_quant(v[c], sh[c]);
  }
#pragma unroll
  for (int c = 0; c < DICM_D; ++c)
    for (int o = 16; o > 0; o >>= 1) q[c] += __shfl_down_sync(FULL, q[c], o);
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) sq[warp][c] = q[c];
  __syncthreads();
  if (t < DICM_D) {  // component t (register arrays stay compile-time indexed)
    long long tot = 0;
    unsigned mm = 0u;
    for (int w = 0; w < 8; ++w) {
      tot += sq[w][t];
      mm = max(mm, smx[w][t]);
    }
    const float mx = __uint_as_float(mm);
    out[(int64_t)u * DICM_D + t] = fx_result(tot, fx_shift(mx, s1 - s0), mx, fl, t);
  }
  __syncthreads();
}

// chunk offsets of the slotted hot keys (every block forms the same scan in
// shared memory); returns the number of chunks
__device__ int hot_chunks(const HotAcc* __restrict__ acc, int nh, int* off) {
  constexpr int PER = HOT_SLOTS / 256;
  __shared__ int part[256];
  const int t = threadIdx.x;
  int c[PER], sum = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int h = t * PER + k;
    c[k] = h < nh ? (acc->ent[h].cnt + HOT_CHUNK - 1) / HOT_CHUNK : 0;
    sum += c[k];
  }
  part[t] = sum;
  __syncthreads();
  for (int d = 1; d < 256; d <<= 1) {  // inclusive scan of the per-thread sums
    const int x = t >= d ? part[t - d] : 0;
    __syncthreads();
    part[t] += x;
    __syncthreads();
  }
  int run = part[t] - sum;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    off[t * PER + k] = run;
    run += c[k];
  }
  if (t == 255) off[HOT_SLOTS] = part[255];
  __syncthreads();
  return off[HOT_SLOTS];
}

// the slot owning chunk g: the last h with off[h] <= g
__device__ __forceinline__ int hot_slot_of(const int* off, int nh, int g) {
  int lo = 0, hi = nh - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= g)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// the keys with 17..32 references (mid_pass), then pass 1 over the hot-key
// chunks: each slot's maxima and non-finite flags.  counters: [hot, mid]
__global__ void __launch_bounds__(256) k_ref_mid_hot(const __grid_constant__ RefSrc S,
                                                     const int32_t* __restrict__ order,
                                                     const int32_t* __restrict__ start,
                                                     const int32_t* __restrict__ counters,
                                                     const int32_t* __restrict__ mid_list, float* __restrict__ out,
                                                     HotAcc* __restrict__ acc) {
  __shared__ int off[HOT_SLOTS + 1];
  mid_pass(S, order, start, counters + 1, mid_list, out);
  const int nh = acc ? min(counters[0], HOT_SLOTS) : 0;
  if (nh == 0) return;
  const int total = hot_chunks(acc, nh, off);
  const int t = threadIdx.x, lane = t & 31;
  for (int g = blockIdx.x; g < total; g += gridDim.x) {
    const int h = hot_slot_of(off, nh, g);
    const HotEnt e = acc->ent[h];
    const int32_t j = e.s0 + (g - off[h]) * HOT_CHUNK + t;
    unsigned m[DICM_D];
    unsigned long long fl = 0;
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) m[c] = 0u;
    if (j < e.s0 + e.cnt) {
      float v[DICM_D];
      ref_contrib(S, __ldg(order + j), v);
#pragma unroll
      for (int c = 0; c < DICM_D; ++c) {
        m[c] = fx_bits(v[c]);
        fl |= fx_flags(v[c], c);
      }
    }
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) m[c] = __reduce_max_sync(FULL, m[c]);
    fl = ((unsigned long long)__reduce_or_sync(FULL, (unsigned)(fl >> 32)) << 32) |
         __reduce_or_sync(FULL, (unsigned)fl);
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < DICM_D; ++c)
        if (m[c]) atomicMax(&acc->mx[h][c], m[c]);
      if (fl) atomicOr(&acc->fl[h], fl);
    }
  }
}

// pass 2: the keys without a slot one block each, then each slot's
// fixed-point sums over the chunks; the last block to finish writes the rows
// of the slotted keys and re-arms the done counter
__global__ void __launch_bounds__(256) k_ref_reduce_hot(const __grid_constant__ RefSrc S,
                                                        const int32_t* __restrict__ order,
                                                        const int32_t* __restrict__ start,
                                                        const int32_t* __restrict__ hot_count,
                                                        const int32_t* __restrict__ hot_list, HotAcc* __restrict__ acc,
                                                        float* __restrict__ out) {
  __shared__ int off[HOT_SLOTS + 1];
  __shared__ bool last;
  const int n_hot = *hot_count;
  const int first = acc ? min(n_hot, HOT_SLOTS) : 0;
  for (int h = first + blockIdx.x; h < n_hot; h += gridDim.x) {
    const int32_t u = hot_list[h];
    hot_block(S, order, u, start[u], start[u + 1], out);
  }
  const int nh = first;
  if (nh == 0) return;
  const int total = hot_chunks(acc, nh, off);
  const int t = threadIdx.x, lane = t & 31;
  for (int g = blockIdx.x; g < total; g += gridDim.x) {
    const int h = hot_slot_of(off, nh, g);
    const HotEnt e = acc->ent[h];
    const int32_t j = e.s0 + (g - off[h]) * HOT_CHUNK + t;
    long long q[DICM_D];
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) q[c] = 0;
    if (j < e.s0 + e.cnt) {
      float v[DICM_D];
      ref_contrib(S, __ldg(order + j), v);
#pragma unroll
      for (int c = 0; c < DICM_D; ++c) q[c] = fx_quant(v[c], fx_shift(__uint_as_float(__ldcg(&acc->mx[h][c])), e.cnt));
    }
#pragma unroll
    for (int c = 0; c < DICM_D; ++c)
      for (int o = 16; o > 0; o >>= 1) q[c] += __shfl_down_sync(FULL, q[c], o);
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < DICM_D; ++c)
        if (q[c]) atomicAdd(reinterpret_cast<unsigned long long*>(&acc->q[h][c]), (unsigned long long)q[c]);
  }
  __syncthreads();
  if (t == 0) {
    __threadfence();
    last = atomicAdd(&acc->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int i = t; i < nh * DICM_D; i += 256) {
    const int h = i / DICM_D, c = i % DICM_D;
    const HotEnt e = acc->ent[h];
    const float mx = __uint_as_float(__ldcg(&acc->mx[h][c]));
    out[(int64_t)e.u * DICM_D + c] =
        fx_result(__ldcg(&acc->q[h][c]), fx_shift(mx, e.cnt), mx, __ldcg(&acc->fl[h]), c);
  }
  if (t == 0) acc->done = 0;
}

int bwd_grid(int batch) {
  const int g = (batch + BWD_WARPS - 1) / BWD_WARPS;
  return g < 1 ? 1 : (g > 148 * 8 ? 148 * 8 : g);
}

template <typename K>
int dyn_smem_attr(K kernel, size_t bytes) {
  return check_cuda(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes),
                    "sample_bwd smem attribute");
}

size_t bwd_smem() {
  const size_t scratch = sizeof(WarpScratch) * BWD_WARPS;
  const size_t red = sizeof(float) * BWD_WARPS * chan_part(MAXQ);
  return scratch > red ? scratch : red;
}

int64_t part_size(const dicm_layout_t* L) {
  if (!L->use_behavior_images || L->kind == 0 || L->kind >= 3) return 0;
  int64_t n = chan_part(DICM_D);
  if (L->kind == 2) n += chan_part(DICM_D * L->n_query);
  return n;
}

int validate(const dicm_layout_t* L, const dicm_batch_view_t* V) {
  if (L->n_fields < 0 || L->n_fields > DICM_MAX_FIELDS) return fail(DICM_ERR_VALUE, "sample: %d fields (max 8)", L->n_fields);
  if (L->kind < 0 || L->kind > 4) return fail(DICM_ERR_UNSUPPORTED, "sample: aggregator kind %d", L->kind);
  if (L->kind == 4 && L->use_behavior_images && (L->width - L->pool_col) % DICM_D)
    return fail(DICM_ERR_VALUE, "concat: pooled width %d is not a multiple of 12", L->width - L->pool_col);
  if ((L->kind == 1 || L->kind == 2) && L->use_behavior_images && !L->use_ad_image)
    return fail(DICM_ERR_VALUE, "attentive aggregator needs the ad image as query");
  if (L->kind == 2 && (L->n_query < 1 || L->n_query > 2))
    return fail(DICM_ERR_VALUE, "multiquery-attn needs 1 or 2 one-hot query fields");
  if (L->kind == 2)
    for (int f = 0; f < L->n_query; ++f)
      if (L->query_field[f] < 0 || L->query_field[f] >= L->n_fields || L->field_multi[L->query_field[f]])
        return fail(DICM_ERR_UNSUPPORTED, "multiquery-attn: query fields must be one-hot fields");
  if (V->batch < 0) return fail(DICM_ERR_VALUE, "sample: negative batch");
  return DICM_OK;
}

Args make_args(const dicm_layout_t* L, const dicm_batch_view_t* V, const dicm_attn_params_t* A) {
  Args a{};
  a.L = *L;
  a.V = *V;
  if (A) {
    a.A[0] = A[0];
    a.A[1] = A[1];
  }
  return a;
}

}  // namespace

extern "C" {

int64_t dicm_attn_partial_size(const dicm_layout_t* layout) { return part_size(layout); }

int dicm_sample_blocks(int batch) { return bwd_grid(batch); }

static int sample_fwd_part(int part, const dicm_layout_t* layout, const dicm_batch_view_t* bv,
                           const dicm_attn_params_t* attn, float* head_in, float* scores, float* stats,
                           dicm_stream_t stream) {
  int rc = validate(layout, bv);
  if (rc) return rc;
  if (bv->batch == 0) return DICM_OK;
  Args a = make_args(layout, bv, attn);
  a.head_in = head_in;
  a.scores = scores;
  a.stats = stats;
  const int grid = (bv->batch + FWD_WARPS - 1) / FWD_WARPS;
  cudaStream_t st = (cudaStream_t)stream;
  // 2 blocks/SM at 128 registers; DICM_FWD_OCC=3 cuts the budget to 80
  // registers (spills in the whole-input variant: 0.127 vs 0.086 ms at cfg2, r2c)
  static const int occ = [] {
    const char* e = getenv("DICM_FWD_OCC");
    return e && e[0] == '3' ? 3 : 2;
  }();
  static const int occ_attn = [] {  // the single-head images kernel scores reference pairs: 128 registers
    const char* e = getenv("DICM_FWD_OCC");
    return e && e[0] == '3' ? 3 : 2;
  }();
  const int probe_slot = part == 1 ? -1 : probe_begin(DICM_PROBE_SAMPLE_FWD, st);
  if (part == 1)
    k_sample_fwd<3, 1><<<grid, FWD_WARPS * 32, 0, st>>>(a);
  else if (part == 2 && layout->kind == 1 && occ_attn == 3)  // single-head attention alone at 80 registers
    k_sample_fwd<3, 2, 1><<<grid, FWD_WARPS * 32, 0, st>>>(a);
  else if (part == 2 && layout->kind == 1)
    k_sample_fwd<2, 2, 1><<<grid, FWD_WARPS * 32, 0, st>>>(a);
  else if (part == 2)
    k_sample_fwd<2, 2><<<grid, FWD_WARPS * 32, 0, st>>>(a);
  else if (occ == 3)
    k_sample_fwd<3, 0><<<grid, FWD_WARPS * 32, 0, st>>>(a);
  else
    k_sample_fwd<2, 0><<<grid, FWD_WARPS * 32, 0, st>>>(a);
  probe_end(probe_slot, st);
  return last_launch("dicm_sample_fwd");
}

int dicm_sample_fwd(const dicm_layout_t* layout, const dicm_batch_view_t* bv, const dicm_attn_params_t* attn,
                    float* head_in, float* scores, float* stats, dicm_stream_t stream) {
  return sample_fwd_part(0, layout, bv, attn, head_in, scores, stats, stream);
}

int dicm_fields_fwd(const dicm_layout_t* layout, const dicm_batch_view_t* bv, float* head_in,
                    dicm_stream_t stream) {
  return sample_fwd_part(1, layout, bv, nullptr, head_in, nullptr, nullptr, stream);
}

int dicm_images_fwd(const dicm_layout_t* layout, const dicm_batch_view_t* bv, const dicm_attn_params_t* attn,
                    float* head_in, float* scores, float* stats, dicm_stream_t stream) {
  return sample_fwd_part(2, layout, bv, attn, head_in, scores, stats, stream);
}

// the reference lists of the image rows and the ID rows (see RefSeg)
static RefSrc image_src(const dicm_layout_t* L, const dicm_batch_view_t* V, const float* dx) {
  RefSrc S{};
  S.dx = dx;
  S.width = L->width;
  const bool attn = L->kind == 1 || L->kind == 2;
  int64_t pos = 0;
  if (L->use_ad_image) {
    RefSeg& g = S.s[S.n++];
    g.begin = 0;
    g.mode = 0;
    g.col = L->ad_col;
    g.qgrad = (attn && L->use_behavior_images) ? V->q_grad : nullptr;
    g.qcol = 0;
    pos = V->batch;
  }
  if (L->use_behavior_images) {
    RefSeg& g = S.s[S.n++];
    g.begin = pos;
    if (L->kind == 0) {
      g.mode = 1;
      g.map = V->beh_seg;
      g.col = L->pool_col;
    } else {
      g.mode = 2;
      g.rows = V->ref_grad;
    }
  }
  return S;
}

static RefSrc id_src(const dicm_layout_t* L, const dicm_batch_view_t* V, const float* dx) {
  RefSrc S{};
  S.dx = dx;
  S.width = L->width;
  for (int f = 0; f < L->n_fields; ++f) {
    RefSeg& g = S.s[S.n++];
    g.begin = V->field_ref_begin[f];
    g.col = L->field_col[f];
    if (L->field_multi[f]) {
      g.mode = 1;
      g.map = V->field_seg[f];
    } else {
      g.mode = 0;
      if (L->kind == 2 && L->use_behavior_images)
        for (int q = 0; q < L->n_query; ++q)
          if (L->query_field[q] == f) {
            g.qgrad = V->q_grad;
            g.qcol = DICM_D + DICM_D * q;
          }
    }
  }
  return S;
}

// counters: [hot, mid] of this list; the lists have room for every key;
// acc: this list's accumulators (or NULL)
static void ref_reduce(const RefSrc& S, const int32_t* order, const int32_t* start, const int32_t* n_keys, int64_t cap,
                       float* out, int32_t* counters, int32_t* hot_list, int32_t* mid_list, HotAcc* acc,
                       cudaStream_t st) {
  static const int occ = [] {
    const char* e = getenv("DICM_REDUCE_OCC");
    return e && e[0] == '2' ? 2 : 3;
  }();
  const int grid = dicm_grid(cap, 256, 148 * 16);
  if (occ == 2)
    k_ref_reduce<2><<<grid, 256, 0, st>>>(S, order, start, n_keys, cap, out, counters, hot_list, mid_list, acc);
  else
    k_ref_reduce<3><<<grid, 256, 0, st>>>(S, order, start, n_keys, cap, out, counters, hot_list, mid_list, acc);
  k_ref_mid_hot<<<148 * 4, 256, 0, st>>>(S, order, start, counters, mid_list, out, acc);
  k_ref_reduce_hot<<<148 * 4, 256, 0, st>>>(S, order, start, counters, hot_list, acc, out);
}

static HotAcc* hot_acc(const dicm_batch_view_t* bv, int list) {
  return bv->hot_acc ? reinterpret_cast<HotAcc*>(bv->hot_acc) + list : nullptr;
}

// every unique ID row's gradient (the ID list's counters bv->hot[2..3] must be
// zero: cleared by the calling entry point)
static void launch_id_reduce(const dicm_layout_t* layout, const dicm_batch_view_t* bv, const float* d_head_in,
                             float* d_rows, cudaStream_t st) {
  if (layout->n_fields <= 0) return;
  int32_t* lists = bv->hot + 4;
  const RefSrc S = id_src(layout, bv, d_head_in);
  ref_reduce(S, bv->id_order, bv->id_start, bv->n_id_keys, bv->id_cap, d_rows, bv->hot + 2,
             lists + 2 * bv->img_cap, lists + 2 * bv->img_cap + bv->id_cap, hot_acc(bv, 1), st);
}

size_t dicm_hot_acc_bytes(void) { return 2 * sizeof(HotAcc); }

int dicm_sample_bwd(const dicm_layout_t* layout, const dicm_batch_view_t* bv, const dicm_attn_params_t* attn,
                    const float* head_in, const float* d_head_in, const float* scores, const float* stats,
                    float* d_emb, float* d_rows, float* attn_partials, dicm_stream_t stream) {
  int rc = validate(layout, bv);
  if (rc) return rc;
  if (bv->batch == 0) {  // an empty slice: no rows to write, one all-zero attention partial block
    const int64_t n = part_size(layout);
    if (n > 0 && check_cuda(cudaMemsetAsync(attn_partials, 0, (size_t)n * bwd_grid(0) * sizeof(float),
                                            (cudaStream_t)stream), "sample_bwd empty batch"))
      return DICM_ERR_CUDA;
    return DICM_OK;
  }
  const bool attn_chan = layout->use_behavior_images && (layout->kind == 1 || layout->kind == 2);
  const bool own_rows = layout->use_behavior_images && layout->kind != 0;
  if ((own_rows && !bv->ref_grad) || (attn_chan && !bv->q_grad) || !bv->hot || !bv->img_order || !bv->id_order ||
      (layout->use_behavior_images && layout->kind == 0 && !bv->beh_seg))
    return fail(DICM_ERR_VALUE, "sample_bwd: the batch view lacks its backward buffers");
  Args a = make_args(layout, bv, attn);
  a.head_in = const_cast<float*>(head_in);
  a.d_head_in = d_head_in;
  a.scores = const_cast<float*>(scores);
  a.stats = const_cast<float*>(stats);
  a.d_emb = d_emb;
  a.d_rows = d_rows;
  a.attn_part = attn_partials;
  const size_t smem = bwd_smem();
  static int attr_rc = dyn_smem_attr(k_attn_bwd<DICM_D>, smem) | dyn_smem_attr(k_attn_bwd<2 * DICM_D>, smem);
  if (attr_rc) return attr_rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = bwd_grid(bv->batch);
  const int64_t stride = part_size(layout);
  const int probe_slot = probe_begin(DICM_PROBE_SAMPLE_BWD, st);
  // this call's list counters: the image list's, and the ID list's when it
  // sums the ID rows too (dicm_id_row_grads clears its own)
  if (check_cuda(cudaMemsetAsync(bv->hot, 0, (d_rows ? 4 : 2) * sizeof(int32_t), st), "sample_bwd list counters"))
    return DICM_ERR_CUDA;
  if (attn_chan) {
    // partial row layout in sorted names: attn/id/* before attn/img/*; the
    // id channel writes each reference's dk row, the img channel adds to it
    int64_t img_off = 0;
    if (layout->kind == 2) {
      img_off = chan_part(DICM_D * layout->n_query);
      if (layout->n_query == 2)
        k_attn_bwd<2 * DICM_D><<<grid, BWD_WARPS * 32, smem, st>>>(a, 1, stride, 0, 0);
      else
        k_attn_bwd<DICM_D><<<grid, BWD_WARPS * 32, smem, st>>>(a, 1, stride, 0, 0);
    }
    k_attn_bwd<DICM_D><<<grid, BWD_WARPS * 32, smem, st>>>(a, 0, stride, img_off, layout->kind == 2);
  } else if (own_rows) {
    k_ref_rows<<<grid, BWD_WARPS * 32, 0, st>>>(a);
  }
  // every unique image row and ID row: its references summed in order
  if (layout->use_ad_image || layout->use_behavior_images) {
    const RefSrc S = image_src(layout, bv, d_head_in);
    ref_reduce(S, bv->img_order, bv->img_start, bv->n_img_keys, bv->img_cap, d_emb, bv->hot, bv->hot + 4,
               bv->hot + 4 + bv->img_cap, hot_acc(bv, 0), st);
  }
  if (d_rows) launch_id_reduce(layout, bv, d_head_in, d_rows, st);
  probe_end(probe_slot, st);
  return last_launch("dicm_sample_bwd");
}

int dicm_id_row_grads(const dicm_layout_t* layout, const dicm_batch_view_t* bv, const float* d_head_in,
                      float* d_rows, dicm_stream_t stream) {
  int rc = validate(layout, bv);
  if (rc) return rc;
  if (bv->batch == 0) return DICM_OK;
  if (!bv->hot || !bv->id_order) return fail(DICM_ERR_VALUE, "id_row_grads: the batch view lacks its buffers");
  if (check_cuda(cudaMemsetAsync(bv->hot + 2, 0, 2 * sizeof(int32_t), (cudaStream_t)stream), "id_row_grads counters"))
    return DICM_ERR_CUDA;
  launch_id_reduce(layout, bv, d_head_in, d_rows, (cudaStream_t)stream);
  return last_launch("dicm_id_row_grads");
}

}  // extern "C"
