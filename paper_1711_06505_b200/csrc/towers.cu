// Two-tower pre-rank scoring and BCE, forward and backward fused per tile of
// 32 samples.
//
// Reference: PrerankModel (model.py:420-531).  tower_reps (model.py:508-520)
// hstacks each tower's inputs -- its ID-field vectors in the tower's order,
// then the sum-pooled behavior images (user tower) or the ad-image embedding
// (ad tower) -- and _tower (model.py:503-506) applies PReLU(x W0^T + b0)
// followed by a linear layer; logits_graph (model.py:522-526) scores by the
// row-wise inner product (autograd.py:388-398), and training applies the same
// sigmoid cross-entropy as the CTR head (autograd.py:230-246,
// training.py:39-42).
//
// The inputs are the head-input rows the per-sample kernel already wrote
// (fields in schema order, ad image, pooled behaviors), so each tower reads
// its blocks by column.  All per-sample state of both towers stays in shared
// memory (x^T, pre-activations and their PReLU, representations; [.][33] to keep the
// column-wise passes conflict-free); the weights are small and read through
// L1.  As in the head, dLoss/dz depends only on the sample, so forward, loss
// and backward run in one pass per tile, and weight gradients leave as one
// partial row per block (fixed order, deterministic).
#include <math.h>

#include "common.cuh"

namespace {
using namespace dicm;

constexpr int BT = 32;       // samples per block
constexpr int LD = BT + 1;   // padded row stride of the [.][BT] tiles
constexpr int THREADS = 256;
constexpr int PART = 12;     // width of one input block (d_id = d_img = 12)
constexpr int MAXW = 128;    // head-input width

struct Dims {
  int nin[2], H, R, W;
};

__host__ __device__ inline size_t smem_floats(const Dims& d) {
  return (size_t)LD * (d.nin[0] + d.nin[1] + 4 * d.H + 2 * d.R   // x^T, pre, PReLU(pre), rep of both towers
                       + d.R + d.H                               // dr, dh (one tower at a time)
                       + d.W)                                    // dx^T
         + 2 * BT;                                               // dz, loss
}

struct TowerPair {
  dicm_tower_t t[2];  // user, ad
};

__global__ void __launch_bounds__(THREADS) k_towers(const float* __restrict__ x, int B, Dims d,
                                                    const __grid_constant__ TowerPair tp,
                                                    const float* __restrict__ labels,
                                                    float inv_denom, float* __restrict__ logits,
                                                    float* __restrict__ dx, float* __restrict__ part,
                                                    int64_t pstride, float* __restrict__ loss_part) {
  extern __shared__ __align__(16) float sm[];
  const int t = threadIdx.x;
  const int b0 = blockIdx.x * BT;
  const int nb = min(BT, B - b0);
  const int H = d.H, R = d.R, W = d.W;
  float* xs[2];
  float* pre[2];
  float* hs[2];  // PReLU(pre), evaluated once
  float* rep[2];
  float* q = sm;
  for (int k = 0; k < 2; ++k) {
    xs[k] = q;
    q += LD * d.nin[k];
  }
  for (int k = 0; k < 2; ++k) {
    pre[k] = q;
    q += LD * H;
    hs[k] = q;
    q += LD * H;
  }
  for (int k = 0; k < 2; ++k) {
    rep[k] = q;
    q += LD * R;
  }
  float* dr = q;
  q += LD * R;
  float* dh = q;
  q += LD * H;
  float* dxs = q;
  q += LD * W;
  float* dz = q;
  float* ls = q + BT;
  const dicm_tower_t* tw = tp.t;

  // inputs: x^T of each tower, gathered by column blocks (row-major reads)
  for (int k = 0; k < 2; ++k) {
    const int nin = d.nin[k];
    for (int i = t; i < BT * nin; i += THREADS) {
      const int r = i / nin, c = i % nin;
      const int col = tw[k].part_col[c / PART] + c % PART;
      xs[k][c * LD + r] = r < nb ? x[(int64_t)(b0 + r) * W + col] : 0.f;
    }
  }
  if (labels)
    for (int i = t; i < W * LD; i += THREADS) dxs[i] = 0.f;
  __syncthreads();

  // layer 0 (PReLU applied on use): pre[j][r] = b0[j] + sum_k W0[j][k] x[k][r]
  for (int k = 0; k < 2; ++k) {
    const int nin = d.nin[k];
    const float* w0 = tw[k].w0;
    for (int i = t; i < H * BT; i += THREADS) {
      const int j = i / BT, r = i % BT;
      float acc = __ldg(tw[k].b0 + j);
      for (int c = 0; c < nin; ++c) acc = fmaf(__ldg(w0 + j * nin + c), xs[k][c * LD + r], acc);
      pre[k][j * LD + r] = acc;
      hs[k][j * LD + r] = prelu(acc, __ldg(tw[k].a0 + j));
    }
  }
  __syncthreads();
  // layer 1: rep[o][r] = b1[o] + sum_j W1[o][j] prelu(pre[j][r])
  for (int k = 0; k < 2; ++k) {
    const float* w1 = tw[k].w1;
    for (int i = t; i < R * BT; i += THREADS) {
      const int o = i / BT, r = i % BT;
      float acc = __ldg(tw[k].b1 + o);
      for (int j = 0; j < H; ++j) acc = fmaf(__ldg(w1 + o * H + j), hs[k][j * LD + r], acc);
      rep[k][o * LD + r] = acc;
    }
  }
  __syncthreads();
  // score = <user rep, ad rep>, BCE (same evaluation as the head, head.cu)
  if (t < BT) {
    float z = 0.f;
    for (int o = 0; o < R; ++o) z = fmaf(rep[0][o * LD + t], rep[1][o * LD + t], z);
    float l = 0.f, g = 0.f;
    if (t < nb && !labels) logits[b0 + t] = z;  // forward only
    if (t < nb && labels) {
      const float y = labels[b0 + t];
      l = fmaxf(z, 0.f) - z * y + log1pf(expf(-fabsf(z)));
      g = bce_grad(z, y, inv_denom);
      logits[b0 + t] = z;
    }
    dz[t] = g;
    ls[t] = l;
  }
  __syncthreads();
  if (!labels) return;
  float* out = part + (int64_t)blockIdx.x * pstride;
  if (t == 0) {
    float l = 0.f;
    for (int r = 0; r < BT; ++r) l += ls[r];
    loss_part[blockIdx.x] = l;
  }

  for (int k = 0; k < 2; ++k) {
    const dicm_tower_t& T = tw[k];
    const int nin = d.nin[k];
    const float* other = rep[1 - k];
    // rowwise_dot bwd: d rep_k = dz * rep_other
    for (int i = t; i < R * BT; i += THREADS) {
      const int o = i / BT, r = i % BT;
      dr[o * LD + r] = dz[r] * other[o * LD + r];
    }
    __syncthreads();
    // layer 1 weights: dW1[o][j] = sum_r dr[o][r] h[j][r]; db1[o] = sum_r dr[o][r]
    for (int i = t; i < R * H; i += THREADS) {
      const int o = i / H, j = i % H;
      float acc = 0.f;
#pragma unroll 8
      for (int r = 0; r < BT; ++r) acc = fmaf(dr[o * LD + r], hs[k][j * LD + r], acc);
      out[T.g_w1 + i] = acc;
    }
    for (int o = t; o < R; o += THREADS) {
      float acc = 0.f;
      for (int r = 0; r < BT; ++r) acc += dr[o * LD + r];
      out[T.g_b1 + o] = acc;
    }
    // dh[j][r] = sum_o W1[o][j] dr[o][r]
    for (int i = t; i < H * BT; i += THREADS) {
      const int j = i / BT, r = i % BT;
      float acc = 0.f;
      for (int o = 0; o < R; ++o) acc = fmaf(__ldg(T.w1 + o * H + j), dr[o * LD + r], acc);
      dh[j * LD + r] = acc;
    }
    __syncthreads();
    // PReLU bwd (autograd.py:222-225): da0, db0, dh -> d pre (in place)
    for (int j = t; j < H; j += THREADS) {
      const float al = __ldg(T.a0 + j);
      float sa = 0.f, sb = 0.f;
      for (int r = 0; r < BT; ++r) {
        const float p = pre[k][j * LD + r], g = dh[j * LD + r];
        const float dp = p > 0.f ? g : al * g;
        if (!(p > 0.f)) sa = fmaf(p, g, sa);
        sb += dp;
        dh[j * LD + r] = dp;
      }
      out[T.g_a0 + j] = sa;
      out[T.g_b0 + j] = sb;
    }
    __syncthreads();
    // dW0[j][c] = sum_r dpre[j][r] x[c][r]
    for (int i = t; i < H * nin; i += THREADS) {
      const int j = i / nin, c = i % nin;
      float acc = 0.f;
#pragma unroll 8
      for (int r = 0; r < BT; ++r) acc = fmaf(dh[j * LD + r], xs[k][c * LD + r], acc);
      out[T.g_w0 + i] = acc;
    }
    // dx[c][r] += sum_j W0[j][c] dpre[j][r] (a field in both towers gets both terms)
    for (int i = t; i < nin * BT; i += THREADS) {
      const int c = i / BT, r = i % BT;
      float acc = 0.f;
      for (int j = 0; j < H; ++j) acc = fmaf(__ldg(T.w0 + j * nin + c), dh[j * LD + r], acc);
      const int col = T.part_col[c / PART] + c % PART;
      dxs[col * LD + r] += acc;
    }
    __syncthreads();
  }
  for (int i = t; i < nb * W; i += THREADS) {
    const int r = i / W, c = i % W;
    dx[(int64_t)(b0 + r) * W + c] = dxs[c * LD + r];
  }
}

int check_args(int width, const dicm_tower_t* tw, int hidden, int rep, Dims* d) {
  if (width < 1 || width > MAXW) return fail(DICM_ERR_UNSUPPORTED, "towers: head width %d not in [1, %d]", width, MAXW);
  if (hidden < 1 || hidden > DICM_TOWER_MAX_HIDDEN)
    return fail(DICM_ERR_UNSUPPORTED, "towers: hidden width %d not in [1, %d]", hidden, DICM_TOWER_MAX_HIDDEN);
  if (rep < 1 || rep > DICM_TOWER_MAX_REP)
    return fail(DICM_ERR_UNSUPPORTED, "towers: representation width %d not in [1, %d]", rep, DICM_TOWER_MAX_REP);
  for (int k = 0; k < 2; ++k) {
    if (tw[k].n_parts < 1 || tw[k].n_parts > DICM_TOWER_MAX_PARTS)
      return fail(DICM_ERR_UNSUPPORTED, "towers: tower %d has %d input blocks (1..%d)", k, tw[k].n_parts,
                  DICM_TOWER_MAX_PARTS);
    for (int i = 0; i < tw[k].n_parts; ++i)
      if (tw[k].part_col[i] < 0 || tw[k].part_col[i] + PART > width)
        return fail(DICM_ERR_VALUE, "towers: block %d of tower %d outside the head input", i, k);
    d->nin[k] = PART * tw[k].n_parts;
  }
  d->H = hidden;
  d->R = rep;
  d->W = width;
  return DICM_OK;
}

int launch(const float* head_in, int batch, int width, const dicm_tower_t* tw, int hidden, int rep,
           const float* labels, float inv_denom, float* logits, float* dx, float* part, int64_t pstride,
           float* loss_part, cudaStream_t st, const char* where) {
  Dims d;
  if (int rc = check_args(width, tw, hidden, rep, &d)) return rc;
  if (batch <= 0) return DICM_OK;
  const size_t smem = smem_floats(d) * sizeof(float);
  static int attr = check_cuda(cudaFuncSetAttribute(k_towers, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    (int)(smem_floats(Dims{{12 * DICM_TOWER_MAX_PARTS,
                                                                            12 * DICM_TOWER_MAX_PARTS},
                                                                           DICM_TOWER_MAX_HIDDEN,
                                                                           DICM_TOWER_MAX_REP, MAXW}) *
                                                          sizeof(float))),
                               "towers smem attribute");
  if (attr) return attr;
  TowerPair tp;
  tp.t[0] = tw[0];
  tp.t[1] = tw[1];
  k_towers<<<(batch + BT - 1) / BT, THREADS, smem, st>>>(head_in, batch, d, tp, labels, inv_denom, logits,
                                                          dx, part, pstride, loss_part);
  return last_launch(where);
}

}  // namespace

extern "C" {

int dicm_towers_blocks(int batch) { return (batch + BT - 1) / BT; }

int dicm_towers_fwd_bwd(const float* head_in, int batch, int width, const dicm_tower_t* towers, int hidden, int rep,
                        const float* labels, float inv_denominator, float* logits, float* d_head_in,
                        float* partials, int64_t part_stride, float* loss_partials, dicm_stream_t stream) {
  if (!labels) return dicm::fail(DICM_ERR_VALUE, "dicm_towers_fwd_bwd: labels required");
  return launch(head_in, batch, width, towers, hidden, rep, labels, inv_denominator, logits, d_head_in, partials,
                part_stride, loss_partials, (cudaStream_t)stream, "dicm_towers_fwd_bwd");
}

int dicm_towers_fwd(const float* head_in, int batch, int width, const dicm_tower_t* towers, int hidden, int rep,
                    float* logits, dicm_stream_t stream) {
  return launch(head_in, batch, width, towers, hidden, rep, nullptr, 0.f, logits, nullptr, nullptr, 0, nullptr,
                (cudaStream_t)stream, "dicm_towers_fwd");
}

}  // extern "C"
