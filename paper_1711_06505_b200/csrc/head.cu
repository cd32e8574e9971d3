// a11-a12: the MLP head width -> 128 -> 64 -> 1 and the BCE loss, forward and
// backward fused per tile of 32 samples.
//
// Reference: logits_graph tail (model.py:397-401) = _layer x2 + linear,
// sigmoid_cross_entropy (autograd.py:230-246) summed and scaled by
// 1/denominator (training.py:39-42).  dLoss/dz = (sigmoid(z) - y)/denominator
// depends only on the sample itself, so the whole head -- forward, loss and
// backward down to dLoss/dx -- runs in one pass per tile without a grid-wide
// barrier.  Weight gradients are reduced over the tile in shared memory and
// written as one partial row per block (deterministic, fixed order).
#include <math.h>

#include "common.cuh"

namespace {
using namespace dicm;

constexpr int BT = 32;  // samples per block
constexpr int H0 = DICM_HEAD0, H1 = DICM_HEAD1;
constexpr int THREADS = 256;  // 8 warps: each phase splits its units or samples over two halves
constexpr int MAXW = 128;

__host__ __device__ inline int64_t part_size(int W) {
  return (int64_t)H0 + H0 + (int64_t)H0 * W + H1 + H1 + (int64_t)H1 * H0 + 1 + H1;
}

struct Smem {
  float w0[H0 * (MAXW + 1)];  // mlp/0/w [128][W] at an odd row stride (conflict-free column reads)
  float w1[H1 * H0];    // mlp/1/w [64][128]
  float xs[MAXW][BT];   // x^T
  float a0[H0][BT];     // layer-0 pre-activation^T
  float h0[H0][BT];     // PReLU(a0), evaluated once
  float a1[H1][BT];     // layer-1 pre-activation^T
  float da1[H1][BT];
  float da0[H0][BT];
  float dz[BT];
  float loss[BT];
  float red[4][3][H0];  // cross-half / cross-quarter partial sums (fixed order)
};

template <int N>
__device__ __forceinline__ void loadn(const float* p, float (&v)[N]) {
#pragma unroll
  for (int q = 0; q < N / 4; ++q) {
    const float4 t = *reinterpret_cast<const float4*>(p + 4 * q);
    v[4 * q] = t.x;
    v[4 * q + 1] = t.y;
    v[4 * q + 2] = t.z;
    v[4 * q + 3] = t.w;
  }
}

__device__ __forceinline__ void load32(const float* p, float (&v)[BT]) {
#pragma unroll
  for (int q = 0; q < BT / 4; ++q) {
    const float4 t = *reinterpret_cast<const float4*>(p + 4 * q);
    v[4 * q] = t.x;
    v[4 * q + 1] = t.y;
    v[4 * q + 2] = t.z;
    v[4 * q + 3] = t.w;
  }
}

__device__ __forceinline__ bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// n4 float4s of src handed to put(i, v), eight loads in flight per thread
template <typename F>
__device__ __forceinline__ void stage4(const float* __restrict__ src, int n4, F put) {
  const float4* g = reinterpret_cast<const float4*>(src);
  for (int base = threadIdx.x; base < n4; base += THREADS * 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (base + u * THREADS < n4) v[u] = __ldg(g + base + u * THREADS);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (base + u * THREADS < n4) put(base + u * THREADS, v[u]);
  }
}

// WIDE: the input is wider than the shared-memory-resident W0 allows (the
// concat aggregator); layer 0 then runs as separate GEMMs (k_sgemm below):
// ``x`` holds the layer-0 pre-activations [B][H0] on entry, and on exit
// ``dx`` receives da0 [B][H0] instead of dLoss/dx.  The partial row then
// omits the w0 block (o_w0 has zero length).
template <bool WIDE>
__global__ void __launch_bounds__(THREADS) k_head(const float* __restrict__ x, int B, int W,
                                                  const float* __restrict__ labels, float inv_denom,
                                                  dicm_head_params_t p, float* __restrict__ logits,
                                                  float* __restrict__ dx, float* __restrict__ part,
                                                  float* __restrict__ loss_part) {
  constexpr int HB = BT / 2, QB = BT / 4;  // samples per half / quarter
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int t = threadIdx.x;
  const int b0 = blockIdx.x * BT;
  const int nb = min(BT, B - b0);
  const int WS = W | 1;  // shared-memory row stride of w0: odd, so a warp reading one column hits 32 banks
  const bool vec = (W & 3) == 0 && aligned16(p.w0) && aligned16(p.w1) && aligned16(x);
  if (!WIDE && vec) {  // float4 loads, 8 in flight per thread
    const int W4 = W >> 2;
    stage4(p.w0, H0 * W4, [&](int i, float4 v) {
      const int r = i / W4, c = (i - r * W4) * 4;
      float* d = s.w0 + r * WS + c;
      d[0] = v.x, d[1] = v.y, d[2] = v.z, d[3] = v.w;
    });
    stage4(x + (int64_t)b0 * W, nb * W4, [&](int i, float4 v) {
      const int r = i / W4, c = (i - r * W4) * 4;
      s.xs[c][r] = v.x, s.xs[c + 1][r] = v.y, s.xs[c + 2][r] = v.z, s.xs[c + 3][r] = v.w;
    });
    for (int i = t; i < (BT - nb) * W; i += THREADS) s.xs[i % W][nb + i / W] = 0.f;  // a short last tile
  } else if (!WIDE) {
    for (int i = t; i < H0 * W; i += THREADS) s.w0[(i / W) * WS + i % W] = p.w0[i];
    for (int i = t; i < BT * W; i += THREADS) {
      const int r = i / W, c = i % W;
      s.xs[c][r] = r < nb ? x[(int64_t)(b0 + r) * W + c] : 0.f;
    }
  } else {
    for (int i = t; i < BT * H0; i += THREADS) {
      const int r = i / H0, j = i % H0;
      const float a = r < nb ? x[(int64_t)(b0 + r) * H0 + j] : 0.f;
      s.a0[j][r] = a;
      s.h0[j][r] = prelu(a, __ldg(p.a0 + j));
    }
  }
  if (vec)
    stage4(p.w1, H1 * H0 / 4, [&](int i, float4 v) { reinterpret_cast<float4*>(s.w1)[i] = v; });
  else
    for (int i = t; i < H1 * H0; i += THREADS) s.w1[i] = p.w1[i];
  __syncthreads();

  // layer 0: thread = (unit j, half of the tile)
  if (!WIDE) {
    const int j = t & (H0 - 1), h = t >> 7;
    float acc[HB];
    const float bj = p.b0[j];
#pragma unroll
    for (int r = 0; r < HB; ++r) acc[r] = bj;
    for (int k = 0; k < W; ++k) {
      const float w = s.w0[j * WS + k];
      float xv[HB];
      loadn<HB>(&s.xs[k][h * HB], xv);
#pragma unroll
      for (int r = 0; r < HB; ++r) acc[r] = fmaf(w, xv[r], acc[r]);
    }
    const float al = __ldg(p.a0 + j);
#pragma unroll
    for (int r = 0; r < HB; ++r) {
      s.a0[j][h * HB + r] = acc[r];
      s.h0[j][h * HB + r] = prelu(acc[r], al);
    }
  }
  __syncthreads();
  // layer 1: thread = (unit j, quarter of the tile)
  {
    const int j = t & (H1 - 1), q = t >> 6;
    float acc[QB];
    const float bj = p.b1[j];
#pragma unroll
    for (int r = 0; r < QB; ++r) acc[r] = bj;
    for (int k = 0; k < H0; ++k) {
      const float w = s.w1[j * H0 + k];
      float hv[QB];
      loadn<QB>(&s.h0[k][q * QB], hv);
#pragma unroll
      for (int r = 0; r < QB; ++r) acc[r] = fmaf(w, hv[r], acc[r]);
    }
#pragma unroll
    for (int r = 0; r < QB; ++r) s.a1[j][q * QB + r] = acc[r];
  }
  __syncthreads();
  // layer 2 + loss: thread = sample
  if (t < BT) {
    float z = p.b2[0];
    for (int j = 0; j < H1; ++j) z = fmaf(__ldg(p.w2 + j), prelu(s.a1[j][t], __ldg(p.a1 + j)), z);
    float l = 0.f, dz = 0.f;
    if (t < nb && !labels) logits[b0 + t] = z;  // forward only (inference)
    if (t < nb && labels) {
      const float y = labels[b0 + t];
      l = fmaxf(z, 0.f) - z * y + log1pf(expf(-fabsf(z)));
      dz = bce_grad(z, y, inv_denom);  // fp64, zero exactly where the reference's is
      logits[b0 + t] = z;
    }
    s.dz[t] = dz;
    s.loss[t] = l;
  }
  __syncthreads();
  if (!labels) return;  // forward only: no loss, no backward
  const int64_t w0len = WIDE ? 0 : (int64_t)H0 * W;
  float* out = part + (int64_t)blockIdx.x * (part_size(W) - (WIDE ? (int64_t)H0 * W : 0));
  const int64_t o_a0 = 0, o_b0 = H0, o_w0 = 2 * H0, o_a1 = o_w0 + w0len, o_b1 = o_a1 + H1,
                o_w1 = o_b1 + H1, o_b2 = o_w1 + (int64_t)H1 * H0, o_w2 = o_b2 + 1;
  if (t == 0) {
    float l = 0.f, d = 0.f;
    for (int r = 0; r < BT; ++r) {
      l += s.loss[r];
      d += s.dz[r];
    }
    loss_part[blockIdx.x] = l;
    out[o_b2] = d;
  }
  // layer 2 / PReLU 1 backward: thread = (unit j of layer 1, quarter)
  {
    const int j = t & (H1 - 1), q = t >> 6;
    const float al = __ldg(p.a1 + j), w2j = __ldg(p.w2 + j);
    float sw = 0.f, sa = 0.f, sb = 0.f;
#pragma unroll
    for (int rr = 0; rr < QB; ++rr) {
      const int r = q * QB + rr;
      const float a = s.a1[j][r], dz = s.dz[r];
      sw = fmaf(dz, prelu(a, al), sw);
      const float dh = dz * w2j;
      const float d = a > 0.f ? dh : al * dh;
      if (!(a > 0.f)) sa = fmaf(a, dh, sa);
      sb += d;
      s.da1[j][r] = d;
    }
    s.red[q][0][j] = sw;
    s.red[q][1][j] = sa;
    s.red[q][2][j] = sb;
  }
  __syncthreads();
  if (t < H1) {
    float v0 = 0.f, v1 = 0.f, v2 = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      v0 += s.red[q][0][t];
      v1 += s.red[q][1][t];
      v2 += s.red[q][2][t];
    }
    out[o_w2 + t] = v0;
    out[o_a1 + t] = v1;
    out[o_b1 + t] = v2;
  }
  // dW1[j][k] = sum_r da1[r][j] h0[r][k]: thread = (k, half of the j range);
  // then dh0 = da1 W1 and da0 = PReLU'(a0) dh0: thread = (k, half of the tile)
  {
    const int k = t & (H0 - 1), h = t >> 7;
    const float al = __ldg(p.a0 + k);
    {
      float hv[BT];
      load32(s.h0[k], hv);
      for (int j = h * (H1 / 2); j < (h + 1) * (H1 / 2); ++j) {
        float d[BT];
        load32(s.da1[j], d);
        float acc = 0.f;
#pragma unroll
        for (int r = 0; r < BT; ++r) acc = fmaf(d[r], hv[r], acc);
        out[o_w1 + (int64_t)j * H0 + k] = acc;
      }
    }
    float dh[HB];
#pragma unroll
    for (int r = 0; r < HB; ++r) dh[r] = 0.f;
    for (int j = 0; j < H1; ++j) {
      const float w = s.w1[j * H0 + k];
      float d[HB];
      loadn<HB>(&s.da1[j][h * HB], d);
#pragma unroll
      for (int r = 0; r < HB; ++r) dh[r] = fmaf(d[r], w, dh[r]);
    }
    float sa = 0.f, sb = 0.f;
    float av[HB];
    loadn<HB>(&s.a0[k][h * HB], av);
#pragma unroll
    for (int r = 0; r < HB; ++r) {
      const float a = av[r];
      const float d = a > 0.f ? dh[r] : al * dh[r];
      if (!(a > 0.f)) sa = fmaf(a, dh[r], sa);
      sb += d;
      dh[r] = d;
    }
    __syncthreads();  // every thread is done reading a0 / da1 for dW1 and dh0
#pragma unroll
    for (int r = 0; r < HB; ++r) s.da0[k][h * HB + r] = dh[r];
    s.red[h][0][k] = sa;
    s.red[h][1][k] = sb;
  }
  __syncthreads();
  if (t < H0) {
    out[o_a0 + t] = s.red[0][0][t] + s.red[1][0][t];
    out[o_b0 + t] = s.red[0][1][t] + s.red[1][1][t];
  }
  if (WIDE) {  // da0 rows for the dW0 / dx GEMMs
    for (int i = t; i < nb * H0; i += THREADS) {
      const int r = i / H0, j = i % H0;
      dx[(int64_t)(b0 + r) * H0 + j] = s.da0[j][r];
    }
    return;
  }
  // dW0[k][c] = sum_r da0[r][k] x[r][c]: thread = (column c, half of the k
  // range), so each k writes one coalesced partial row; da0[k] is a broadcast
  {
    const int per = (THREADS / 2 >= W) ? THREADS / 2 : THREADS;  // W <= 128: two k-halves
    const int c = t % per, h = t / per;
    if (c < W) {
      float xv[BT];
      load32(s.xs[c], xv);
      const int k0 = per == THREADS ? 0 : h * (H0 / 2), k1 = per == THREADS ? H0 : k0 + H0 / 2;
      for (int k = k0; k < k1; ++k) {
        float d[BT];
        load32(s.da0[k], d);
        float acc = 0.f;
#pragma unroll
        for (int r = 0; r < BT; ++r) acc = fmaf(d[r], xv[r], acc);
        out[o_w0 + (int64_t)k * W + c] = acc;
      }
    }
  }
  // dx[r][c] = sum_k da0[r][k] W0[k][c]: thread = (column c, half of the tile)
  {
    const int c = t & (H0 - 1), h = t >> 7;
    if (c < W) {
      float acc[HB];
#pragma unroll
      for (int r = 0; r < HB; ++r) acc[r] = 0.f;
      for (int k = 0; k < H0; ++k) {
        const float w = s.w0[k * WS + c];
        float d[HB];
        loadn<HB>(&s.da0[k][h * HB], d);
#pragma unroll
        for (int r = 0; r < HB; ++r) acc[r] = fmaf(d[r], w, acc[r]);
      }
      for (int r = 0; r < HB; ++r)
        if (h * HB + r < nb) dx[(int64_t)(b0 + h * HB + r) * W + c] = acc[r];
    }
  }
}

// ---------------------------------------------------------------------------
// wide head (concat aggregator): layer 0 as fp32 GEMMs on the CUDA cores.
// C[m][n] = sum_k A(m,k) B(k,n) (+ bias[n]) with A(m,k) = A[m*sam + k*sak],
// B(k,n) = B[k*sbk + n*sbn]: 64x64 tiles, 16-deep k slices staged in shared
// memory, 4x4 outputs per thread, every output summed in k order by one thread
// (deterministic).  Covers a0 = X W0^T + b0, dW0 = da0^T X and dX = da0 W0.
// ---------------------------------------------------------------------------
constexpr int GB = 64, GK = 16;

__global__ void __launch_bounds__(256) k_sgemm(int M, int N, int K, const float* __restrict__ A, int64_t sam,
                                               int64_t sak, const float* __restrict__ Bm, int64_t sbk, int64_t sbn,
                                               const float* __restrict__ bias, float* __restrict__ C, int64_t ldc) {
  __shared__ float As[GK][GB + 4], Bs[GK][GB + 4];
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const int m0 = blockIdx.y * GB, n0 = blockIdx.x * GB;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += GK) {
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int i = t + l * 256;
      // walk the unit-stride dimension with consecutive threads
      const int am = sak == 1 ? i / GK : i % GB, ak = sak == 1 ? i % GK : i / GB;
      const int bn = sbn == 1 ? i % GB : i / GK, bk = sbn == 1 ? i / GB : i % GK;
      const int gm = m0 + am, gk = k0 + ak;
      As[ak][am] = (gm < M && gk < K) ? __ldg(A + gm * sam + gk * sak) : 0.f;
      const int gn = n0 + bn, gk2 = k0 + bk;
      Bs[bk][bn] = (gn < N && gk2 < K) ? __ldg(Bm + gk2 * sbk + gn * sbn) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n < N) C[m * ldc + n] = acc[i][j] + (bias ? __ldg(bias + n) : 0.f);
    }
  }
}

void sgemm(cudaStream_t st, int M, int N, int K, const float* A, int64_t sam, int64_t sak, const float* Bm,
           int64_t sbk, int64_t sbn, const float* bias, float* C, int64_t ldc) {
  dim3 grid((N + GB - 1) / GB, (M + GB - 1) / GB);
  k_sgemm<<<grid, 256, 0, st>>>(M, N, K, A, sam, sak, Bm, sbk, sbn, bias, C, ldc);
}

// out[c] = sum over blocks (in order) of part[blk * stride + col0 + c]
__global__ void k_reduce_cols(const float* __restrict__ part, int nblk, int64_t stride, int64_t col0, int64_t n,
                              float* __restrict__ out) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int b = 0; b < nblk; ++b) acc += part[b * stride + col0 + c];
    out[c] = acc;
  }
}

struct WideWs {
  float *a0, *da0, *part;
  int64_t prow;
};

size_t wide_carve(int batch, int W, void* base, WideWs* w) {
  const int64_t B = batch > 0 ? batch : 1;
  const int nblk = (int)((B + BT - 1) / BT);
  const int64_t prow = part_size(W) - (int64_t)H0 * W;
  const size_t n_a = (size_t)B * H0 * sizeof(float);
  const size_t n_p = (size_t)nblk * prow * sizeof(float);
  if (w) {
    char* p = (char*)base;
    w->a0 = (float*)p;
    w->da0 = (float*)(p + n_a);
    w->part = (float*)(p + 2 * n_a);
    w->prow = prow;
  }
  return 2 * n_a + n_p;
}

__global__ void k_loss_finalize(const float* __restrict__ part, int n, float scale, float* __restrict__ out,
                                int32_t* __restrict__ status) {
  __shared__ float red[256];
  float s = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const float l = red[0] * scale;
    *out = l;
    if (!isfinite(l)) atomicOr(&status[DICM_ST_NONFINITE], 1);
  }
}

__global__ void k_check_finite(const float* __restrict__ x, int64_t n, const int32_t* __restrict__ count,
                               int row_width, int bit, int32_t* __restrict__ status) {
  if (count) n = min(n, (int64_t)*count * row_width);
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&status[DICM_ST_NONFINITE], bit);
}

}  // namespace

extern "C" {

int64_t dicm_head_partial_size(int width) { return part_size(width); }

int dicm_head_blocks(int batch) { return (batch + BT - 1) / BT; }

int dicm_head_fwd_bwd(const float* head_in, int batch, int width, const float* labels, float inv_denominator,
                      const dicm_head_params_t* p, float* logits, float* d_head_in, float* partials,
                      float* loss_partials, dicm_stream_t stream) {
  using namespace dicm;
  if (width < 1 || width > MAXW) return fail(DICM_ERR_UNSUPPORTED, "head: input width %d not in [1, %d]", width, MAXW);
  if (batch <= 0) return DICM_OK;
  const size_t smem = sizeof(Smem);
  static bool attr = false;
  if (!attr) {
    int rc = check_cuda(cudaFuncSetAttribute(k_head<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                        "head smem attribute");
    if (rc) return rc;
    attr = true;
  }
  k_head<false><<<dicm_head_blocks(batch), THREADS, smem, (cudaStream_t)stream>>>(
      head_in, batch, width, labels, inv_denominator, *p, logits, d_head_in, partials, loss_partials);
  return last_launch("dicm_head_fwd_bwd");
}

int dicm_head_fwd(const float* head_in, int batch, int width, const dicm_head_params_t* p, float* logits,
                  dicm_stream_t stream) {
  using namespace dicm;
  if (width < 1 || width > MAXW) return fail(DICM_ERR_UNSUPPORTED, "head: input width %d not in [1, %d]", width, MAXW);
  if (batch <= 0) return DICM_OK;
  const size_t smem = sizeof(Smem);
  static int attr = check_cuda(cudaFuncSetAttribute(k_head<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                               "head smem attribute");
  if (attr) return attr;
  k_head<false><<<dicm_head_blocks(batch), THREADS, smem, (cudaStream_t)stream>>>(head_in, batch, width, nullptr, 0.f, *p,
                                                                         logits, nullptr, nullptr, nullptr);
  return last_launch("dicm_head_fwd");
}

size_t dicm_head_wide_workspace(int batch, int width) { return wide_carve(batch, width, nullptr, nullptr); }

int dicm_head_wide_fwd_bwd(const float* head_in, int batch, int width, const float* labels, float inv_denominator,
                           const dicm_head_params_t* p, float* logits, float* d_head_in, float* grads,
                           float* loss_partials, void* workspace, size_t workspace_bytes, dicm_stream_t stream) {
  using namespace dicm;
  if (width < 1 || width > DICM_HEAD_MAX_WIDE)
    return fail(DICM_ERR_UNSUPPORTED, "head: input width %d not in [1, %d]", width, DICM_HEAD_MAX_WIDE);
  if (!labels) return fail(DICM_ERR_VALUE, "dicm_head_wide_fwd_bwd: labels required");
  if (batch <= 0) return DICM_OK;
  if (workspace_bytes < wide_carve(batch, width, nullptr, nullptr))
    return fail(DICM_ERR_VALUE, "dicm_head_wide_fwd_bwd: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  WideWs w;
  wide_carve(batch, width, workspace, &w);
  const size_t smem = sizeof(Smem);
  static int attr = check_cuda(cudaFuncSetAttribute(k_head<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    (int)smem), "head smem attribute");
  if (attr) return attr;
  const int W = width;
  // a0 = X W0^T + b0
  sgemm(st, batch, H0, W, head_in, W, 1, p->w0, 1, W, p->b0, w.a0, H0);
  const int nblk = dicm_head_blocks(batch);
  k_head<true><<<nblk, THREADS, smem, st>>>(w.a0, batch, W, labels, inv_denominator, *p, logits, w.da0, w.part,
                                            loss_partials);
  // partial rows [a0 b0 | a1 b1 w1 b2 w2] -> the mlp/ gradient range around w0
  const int64_t rest = w.prow - 2 * H0;
  k_reduce_cols<<<1, 2 * H0, 0, st>>>(w.part, nblk, w.prow, 0, 2 * H0, grads);
  k_reduce_cols<<<(int)((rest + 255) / 256), 256, 0, st>>>(w.part, nblk, w.prow, 2 * H0, rest,
                                                           grads + 2 * H0 + (int64_t)H0 * W);
  // dW0 = da0^T X  -> grads[2 H0 ..), dX = da0 W0
  sgemm(st, H0, W, batch, w.da0, 1, H0, head_in, W, 1, nullptr, grads + 2 * H0, W);
  sgemm(st, batch, W, H0, w.da0, H0, 1, p->w0, W, 1, nullptr, d_head_in, W);
  return last_launch("dicm_head_wide_fwd_bwd");
}

int dicm_head_wide_fwd(const float* head_in, int batch, int width, const dicm_head_params_t* p, float* logits,
                       void* workspace, size_t workspace_bytes, dicm_stream_t stream) {
  using namespace dicm;
  if (width < 1 || width > DICM_HEAD_MAX_WIDE)
    return fail(DICM_ERR_UNSUPPORTED, "head: input width %d not in [1, %d]", width, DICM_HEAD_MAX_WIDE);
  if (batch <= 0) return DICM_OK;
  if (workspace_bytes < wide_carve(batch, width, nullptr, nullptr))
    return fail(DICM_ERR_VALUE, "dicm_head_wide_fwd: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  WideWs w;
  wide_carve(batch, width, workspace, &w);
  const size_t smem = sizeof(Smem);
  static int attr = check_cuda(cudaFuncSetAttribute(k_head<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    (int)smem), "head smem attribute");
  if (attr) return attr;
  sgemm(st, batch, H0, width, head_in, width, 1, p->w0, 1, width, p->b0, w.a0, H0);
  k_head<true><<<dicm_head_blocks(batch), THREADS, smem, st>>>(w.a0, batch, width, nullptr, 0.f, *p, logits, nullptr,
                                                              nullptr, nullptr);
  return last_launch("dicm_head_wide_fwd");
}

int dicm_loss_finalize(const float* loss_partials, int nblk, float scale, float* loss_out, int32_t* status,
                       dicm_stream_t stream) {
  k_loss_finalize<<<1, 256, 0, (cudaStream_t)stream>>>(loss_partials, nblk, scale, loss_out, status);
  return dicm::last_launch("dicm_loss_finalize");
}

int dicm_check_finite(const float* x, int64_t n, const int32_t* count_dev, int row_width, int bit,
                      int32_t* status, dicm_stream_t stream) {
  if (n <= 0) return DICM_OK;
  k_check_finite<<<dicm_grid(n, 256, 148 * 4), 256, 0, (cudaStream_t)stream>>>(x, n, count_dev, row_width, bit,
                                                                               status);
  return dicm::last_launch("dicm_check_finite");
}

}  // extern "C"
