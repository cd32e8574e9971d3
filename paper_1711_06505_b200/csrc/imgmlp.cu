// a4/a5: the image MLP d_raw -> 256 -> 64 -> 12 and its reverse path.
//
// Reference: image_net_apply (model.py:108-120) = linear+PReLU, linear+PReLU,
// linear (autograd.py:171-227); backward = the linear/prelu closures
// (autograd.py:201-204, 222-225).  Layer 0 is the only dense contraction of
// the whole step and carries ~98% of its FLOPs: it runs on tcgen05 tensor
// cores (imgmlp_sm100.cu) in the tf32/bf16 precision modes; the fp32 mode
// here (CUDA cores) is the strict-parity reference path.  Layers 1-2
// (256->64->12, 1.6% of the FLOPs) stay fp32 in every mode.
#include "common.cuh"
#include "gemm_simt.cuh"
#include "imgmlp_sm100.cuh"

namespace {
using namespace dicm;

constexpr int H1 = 256, H2 = 64;
constexpr int L2_BLOCKS = 296;  // fixed -> deterministic partial layout

// E = h2 W2^T + b2 with h2 = prelu(a1); one thread per row
__global__ void __launch_bounds__(128) k_layer2_fwd(const float* __restrict__ a1, const float* __restrict__ al1,
                                                    const float* __restrict__ w2, const float* __restrict__ b2,
                                                    const int32_t* __restrict__ count, int64_t n_max,
                                                    float* __restrict__ emb) {
  __shared__ float sw[DICM_D * H2], sb[DICM_D], sa[H2];
  for (int i = threadIdx.x; i < DICM_D * H2; i += blockDim.x) sw[i] = w2[i];
  for (int i = threadIdx.x; i < H2; i += blockDim.x) sa[i] = al1[i];
  if (threadIdx.x < DICM_D) sb[threadIdx.x] = b2[threadIdx.x];
  __syncthreads();
  const int64_t n = min((int64_t)*count, n_max);
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    float e[DICM_D];
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) e[c] = sb[c];
    const float4* row = reinterpret_cast<const float4*>(a1 + r * H2);
#pragma unroll 4
    for (int q = 0; q < H2 / 4; ++q) {
      const float4 v = __ldg(row + q);
      const float h[4] = {prelu(v.x, sa[4 * q]), prelu(v.y, sa[4 * q + 1]), prelu(v.z, sa[4 * q + 2]),
                          prelu(v.w, sa[4 * q + 3])};
#pragma unroll
      for (int c = 0; c < DICM_D; ++c)
#pragma unroll
        for (int i = 0; i < 4; ++i) e[c] = fmaf(sw[c * H2 + 4 * q + i], h[i], e[c]);
    }
    float4* out = reinterpret_cast<float4*>(emb + r * DICM_D);
    out[0] = make_float4(e[0], e[1], e[2], e[3]);
    out[1] = make_float4(e[4], e[5], e[6], e[7]);
    out[2] = make_float4(e[8], e[9], e[10], e[11]);
  }
}

// Reverse of layer 2 and the PReLU of layer 1, one column per thread:
// da1 = prelu'(a1) * (dE W2), and per-block partial sums of
// dW2 = dE^T h2, db2 = sum dE, dalpha1, db1.  Partial row layout:
// [w2 (12 x 64) | b2 (12) | a1 (64) | b1 (64)].
constexpr int L2_PART = DICM_D * H2 + DICM_D + H2 + H2;

__global__ void __launch_bounds__(256) k_layer2_bwd(const float* __restrict__ a1, const float* __restrict__ al1,
                                                    const float* __restrict__ w2, const float* __restrict__ demb,
                                                    const int32_t* __restrict__ count, int64_t n_max,
                                                    float* __restrict__ da1, float* __restrict__ part) {
  const int j = threadIdx.x & (H2 - 1), g = threadIdx.x >> 6;  // 4 row groups x 64 columns
  const int64_t n = min((int64_t)*count, n_max);
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * chunk, r1 = min(n, r0 + chunk);
  float wcol[DICM_D], accw[DICM_D];
#pragma unroll
  for (int c = 0; c < DICM_D; ++c) {
    wcol[c] = w2[c * H2 + j];
    accw[c] = 0.f;
  }
  const float alpha = al1[j];
  float acc_a = 0.f, acc_b = 0.f, acc_b2 = 0.f;
  for (int64_t r = r0 + g; r < r1; r += 4) {
    const Row12 d = load_row12(demb + r * DICM_D);
    const float a = a1[r * H2 + j];
    float dh = 0.f;
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) dh = fmaf(d.v[c], wcol[c], dh);
    const float dd = a > 0.f ? dh : alpha * dh;
    da1[r * H2 + j] = dd;
    if (!(a > 0.f)) acc_a = fmaf(a, dh, acc_a);
    acc_b += dd;
    const float h = prelu(a, alpha);
#pragma unroll
    for (int c = 0; c < DICM_D; ++c) accw[c] = fmaf(d.v[c], h, accw[c]);
    if (j < DICM_D) acc_b2 += d.v[j];
  }
  __shared__ float red[4][L2_PART];
#pragma unroll
  for (int c = 0; c < DICM_D; ++c) red[g][c * H2 + j] = accw[c];
  if (j < DICM_D) red[g][DICM_D * H2 + j] = acc_b2;
  red[g][DICM_D * H2 + DICM_D + j] = acc_a;
  red[g][DICM_D * H2 + DICM_D + H2 + j] = acc_b;
  __syncthreads();
  for (int i = threadIdx.x; i < L2_PART; i += blockDim.x)
    part[(int64_t)blockIdx.x * L2_PART + i] = ((red[0][i] + red[1][i]) + red[2][i]) + red[3][i];
}

// dh1 -> da0 = prelu'(a0) dh1 with per-block column partial sums of
// dalpha0 = sum_{a0<=0} a0*dh1 and db0 = sum da0 (rows of 64 per block-row)
struct EpPreluGrad {
  const float* a0;
  const float* alpha;
  float* da0;
  float* colpart;  // [gridDim.y][2][256]
  __device__ void operator()(float (&acc)[4][4], int m, int n, int Mr, int N, int split) const {
    __shared__ float red[2][16][simt::BN];
    float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
    for (int i = 0; i < 4; ++i) {
      if (m + i >= Mr) break;
      for (int jj = 0; jj < 4; ++jj) {
        const int64_t o = (int64_t)(m + i) * H1 + n + jj;
        const float x = a0[o], gg = acc[i][jj];
        const float d = x > 0.f ? gg : alpha[n + jj] * gg;
        da0[o] = d;
        sb[jj] += d;
        if (!(x > 0.f)) sa[jj] = fmaf(x, gg, sa[jj]);
      }
    }
    const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
    for (int jj = 0; jj < 4; ++jj) {
      red[0][ty][tx * 4 + jj] = sa[jj];
      red[1][ty][tx * 4 + jj] = sb[jj];
    }
    __syncthreads();
    if (threadIdx.x < 2 * simt::BN) {
      const int q = threadIdx.x / simt::BN, c = threadIdx.x % simt::BN;
      float s = 0.f;
      for (int t = 0; t < 16; ++t) s += red[q][t][c];
      colpart[((int64_t)blockIdx.y * 2 + q) * H1 + blockIdx.x * simt::BN + c] = s;
    }
  }
};

// out[j] (+)= sum_{b < nvalid} part[b*stride + off + j]; nvalid from the device
// row count when rows_per_blk > 0 (block rows past the count wrote nothing)
//
// Column sums over partial rows, deterministic (fixed association): block
// (32 columns x 8 row lanes) sums its chunk of rows with coalesced loads and
// reduces the 8 lanes in shared memory; with nchunk > 1 each chunk's sums go to
// tmp[chunk][n] and a second pass folds the chunks.
constexpr int RED_ROWS = 128;  // rows per chunk (16 per row lane)

__global__ void __launch_bounds__(256) k_colsum(const float* __restrict__ part, int nblk, int64_t stride, int64_t off,
                                                int64_t n, const int32_t* __restrict__ count, int rows_per_blk,
                                                int chunk_rows, float* __restrict__ out, int accumulate) {
  int nb = nblk;
  if (count && rows_per_blk > 0) nb = min(nblk, (int)((*count + rows_per_blk - 1) / rows_per_blk));
  const int64_t j = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int b0 = blockIdx.y * chunk_rows, b1 = min(nb, b0 + chunk_rows);
  float s = 0.f;
  if (j < n)
    for (int b = b0 + threadIdx.y; b < b1; b += 8) s += part[(int64_t)b * stride + off + j];
  __shared__ float red[8][33];
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && j < n) {
    float t = 0.f;
#pragma unroll
    for (int y = 0; y < 8; ++y) t += red[y][threadIdx.x];
    float* o = out + (int64_t)blockIdx.y * n + j;
    *o = accumulate ? *o + t : t;
  }
}

// several column ranges of one partial array, each into its own output, in
// one launch (blockIdx.y = range); same fixed association as k_colsum
struct ColSegs {
  int64_t off[8], n[8];
  float* out[8];
};
__global__ void __launch_bounds__(256) k_colsum_multi(const float* __restrict__ part, int nblk, int64_t stride,
                                                      const __grid_constant__ ColSegs segs) {
  const int sg = blockIdx.y;
  const int64_t j = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int64_t n = segs.n[sg];
  float s = 0.f;
  if (j < n)
    for (int b = threadIdx.y; b < nblk; b += 8) s += part[(int64_t)b * stride + segs.off[sg] + j];
  __shared__ float red[8][33];
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && j < n) {
    float t = 0.f;
#pragma unroll
    for (int y = 0; y < 8; ++y) t += red[y][threadIdx.x];
    segs.out[sg][j] = t;
  }
}

void reduce_multi(cudaStream_t st, const float* part, int nblk, int64_t stride, int nseg, const int64_t* off,
                  const int64_t* n, float* const* out) {
  ColSegs c{};
  int64_t mx = 1;
  for (int i = 0; i < nseg; ++i) {
    c.off[i] = off[i];
    c.n[i] = n[i];
    c.out[i] = out[i];
    mx = std::max(mx, n[i]);
  }
  k_colsum_multi<<<dim3((unsigned)((mx + 31) / 32), nseg), dim3(32, 8), 0, st>>>(part, nblk, stride, c);
}

// tmp: >= ceil(nblk / RED_ROWS) * n floats (or nullptr when nblk <= RED_ROWS)
void reduce_into(cudaStream_t st, const float* part, int nblk, int64_t stride, int64_t off, int64_t n, float* out,
                 float* tmp, int accumulate, const int32_t* count = nullptr, int rows_per_blk = 0) {
  if (n <= 0) return;
  const int nchunk = (nblk + RED_ROWS - 1) / RED_ROWS;
  const dim3 blk(32, 8);
  const unsigned gx = (unsigned)((n + 31) / 32);
  if (nchunk <= 1 || tmp == nullptr) {  // one chunk covering every row
    k_colsum<<<dim3(gx, 1), blk, 0, st>>>(part, nblk, stride, off, n, count, rows_per_blk, nblk > 0 ? nblk : 1, out,
                                          accumulate);
    return;
  }
  k_colsum<<<dim3(gx, nchunk), blk, 0, st>>>(part, nblk, stride, off, n, count, rows_per_blk, RED_ROWS, tmp, 0);
  k_colsum<<<dim3(gx, 1), blk, 0, st>>>(tmp, nchunk, n, 0, n, nullptr, 0, nchunk, out, accumulate);
}

size_t red_tmp_floats(int64_t rows_max) { return (size_t)(std::max<int64_t>(rows_max / 8192 + 2, 4)) * 16384; }

float* g_red_tmp = nullptr;  // set per call from the workspace

void reduce(cudaStream_t st, const float* part, int nblk, int64_t stride, int64_t off, int64_t n, float* out,
            const int32_t* count = nullptr, int rows_per_blk = 0) {
  reduce_into(st, part, nblk, stride, off, n, out, g_red_tmp, 0, count, rows_per_blk);
}

struct Ws {
  float *da1, *da0, *p2, *p0, *pw1, *pw0, *red, *pl12, *pdw1, *h1, *g3;
  int s1, s0;
};

int ksplit_dw1(int64_t rows_max) { return (int)std::max<int64_t>(1, std::min<int64_t>(148, rows_max / 256)); }
int ksplit_dw0(int64_t rows_max) { return (int)std::max<int64_t>(1, std::min<int64_t>(8, rows_max / 1024)); }

size_t carve(int64_t rows_max, int d_raw, Ws* w, char* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* p = base ? base + off : nullptr;
    off += (bytes + 255) / 256 * 256;
    return p;
  };
  Ws t;
  t.s1 = ksplit_dw1(rows_max);
  t.s0 = ksplit_dw0(rows_max);
  t.da1 = (float*)take((size_t)rows_max * H2 * 4);
  t.da0 = (float*)take((size_t)rows_max * H1 * 4);
  t.p2 = (float*)take((size_t)L2_BLOCKS * L2_PART * 4);
  t.p0 = (float*)take((size_t)((rows_max + 63) / 64) * 2 * H1 * 4);
  t.pw1 = (float*)take((size_t)t.s1 * H2 * H1 * 4);
  t.pw0 = (float*)take((size_t)t.s0 * H1 * d_raw * 4);
  t.red = (float*)take(red_tmp_floats(rows_max) * 4);
  t.pl12 = (float*)take((size_t)sm100::small_bwd_blocks(rows_max) * sm100::small_part_size() * 4);
  t.pdw1 = (float*)take((size_t)sm100::small_dw1_blocks(rows_max) * sm100::dw1_bf16_part_size() * 4);
  t.g3 = (float*)take((size_t)sm100::dw1_bf16_part_size() * 4);
  t.h1 = (float*)take((size_t)rows_max * H1 * 4);
  if (w) *w = t;
  return off + sm100::workspace_bytes(rows_max, d_raw);
}

int check_aligned(const void* a, const void* b, const void* c, const void* d) {
  if (((uintptr_t)a | (uintptr_t)b | (uintptr_t)c | (uintptr_t)d) & 15)
    return fail(DICM_ERR_VALUE, "image MLP: pool, act buffers and img/*/w must be 16-byte aligned");
  return DICM_OK;
}

int check_shapes(int d_raw, int64_t rows_max) {
  // the hidden widths are compiled (256 -> 64 -> 12); the row width is any
  // multiple of 64 (narrower image nets are zero-padded into these widths,
  // schema.KernelGeometry; the tensor-core paths need a multiple of 256)
  if (d_raw % 64 != 0 || d_raw < 64 || d_raw > (1 << 16))
    return fail(DICM_ERR_UNSUPPORTED,
                "image MLP: d_raw must be a multiple of 64 in [64, 65536] (256 -> 64 -> 12 hidden), got %d", d_raw);
  if (rows_max < 0 || rows_max > (int64_t)1 << 30) return fail(DICM_ERR_VALUE, "image MLP: rows_max out of range");
  return DICM_OK;
}

}  // namespace

extern "C" {

size_t dicm_imgmlp_workspace(int64_t rows_max, int d_raw, int precision) {
  return carve(rows_max < 1 ? 1 : rows_max, d_raw, nullptr, nullptr) + 1024;
}

int dicm_imgmlp_fwd(const void* pool, int pool_dtype, int d_raw, const int32_t* rows,
                    const int32_t* count_dev, int64_t rows_max, const dicm_imgmlp_params_t* p,
                    float* act0, float* act1, float* emb, int precision, void* workspace,
                    size_t workspace_bytes, dicm_stream_t stream) {
  using namespace dicm::simt;
  int rc = check_shapes(d_raw, rows_max);
  if (!rc) rc = check_aligned(pool, p->w0, p->w1, act0);
  if (rc) return rc;
  if (rows_max == 0) return DICM_OK;
  if (workspace_bytes < dicm_imgmlp_workspace(rows_max, d_raw, precision))
    return fail(DICM_ERR_VALUE, "image MLP fwd: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int M = (int)rows_max;
  // layer 0: act0 = X[rows] W0^T + b0
  if (precision == DICM_PREC_FP32) {
    if (pool_dtype == DICM_POOL_F32)
      gemm(st, LoadA_Rows<float>{(const float*)pool, d_raw, rows, nullptr}, LoadB_WT{p->w0, d_raw},
           EpBias{act0, H1, p->b0}, M, H1, d_raw, count_dev, nullptr, 1);
    else
      gemm(st, LoadA_Rows<__nv_bfloat16>{(const __nv_bfloat16*)pool, d_raw, rows, nullptr},
           LoadB_WT{p->w0, d_raw}, EpBias{act0, H1, p->b0}, M, H1, d_raw, count_dev, nullptr, 1);
  } else {
    Ws w;
    carve(rows_max, d_raw, &w, (char*)workspace);
    char* tc_ws = (char*)workspace + carve(rows_max, d_raw, nullptr, nullptr) - sm100::workspace_bytes(rows_max, d_raw);
    rc = sm100::fwd_layer0(pool, pool_dtype, d_raw, rows, count_dev, rows_max, p->w0, p->b0, act0, precision,
                           tc_ws, st);
    if (rc) return rc;
    if (precision == DICM_PREC_BF16) {
      // bf16 saved activations: act0 / act1 buffers hold bf16 rows
      rc = sm100::fwd_layers12_bf16(reinterpret_cast<const __nv_bfloat16*>(act0), count_dev, rows_max, p->a0, p->w1,
                                    p->b1, p->a1, p->w2, p->b2, reinterpret_cast<__nv_bfloat16*>(act1), emb, st);
      if (rc) return rc;
      return last_launch("dicm_imgmlp_fwd");
    }
    // layers 1-2 on tcgen05 (tf32) with the layer-2 epilogue fused
    rc = sm100::fwd_layers12(act0, count_dev, rows_max, p->a0, p->w1, p->b1, p->a1, p->w2, p->b2, act1, emb, w.h1,
                             st);
    if (rc) return rc;
    return last_launch("dicm_imgmlp_fwd");
  }
  // layer 1: act1 = prelu(act0) W1^T + b1   (fp32, CUDA cores)
  gemm(st, LoadA_Rows<float>{act0, H1, nullptr, p->a0}, LoadB_WT{p->w1, H1}, EpBias{act1, H2, p->b1}, M, H2,
       H1, count_dev, nullptr, 1);
  // layer 2: emb = prelu(act1) W2^T + b2
  k_layer2_fwd<<<dicm_grid(rows_max, 128, 148 * 8), 128, 0, st>>>(act1, p->a1, p->w2, p->b2, count_dev,
                                                                  rows_max, emb);
  return last_launch("dicm_imgmlp_fwd");
}

int dicm_imgmlp_bwd(const void* pool, int pool_dtype, int d_raw, const int32_t* rows,
                    const int32_t* count_dev, int64_t rows_max, const dicm_imgmlp_params_t* p,
                    const float* act0, const float* act1, const float* demb,
                    const dicm_imgmlp_grads_t* g, int precision, void* workspace,
                    size_t workspace_bytes, dicm_stream_t stream) {
  using namespace dicm::simt;
  int rc = check_shapes(d_raw, rows_max);
  if (!rc) rc = check_aligned(pool, p->w1, g->w0, act0);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (rows_max == 0) {
    // no rows: every image-net gradient is zero
    const float* none[1] = {nullptr};
    (void)none;
    cudaMemsetAsync(g->w0, 0, (size_t)H1 * d_raw * 4, st);
    cudaMemsetAsync(g->b0, 0, H1 * 4, st);
    cudaMemsetAsync(g->a0, 0, H1 * 4, st);
    cudaMemsetAsync(g->w1, 0, H2 * H1 * 4, st);
    cudaMemsetAsync(g->b1, 0, H2 * 4, st);
    cudaMemsetAsync(g->a1, 0, H2 * 4, st);
    cudaMemsetAsync(g->w2, 0, DICM_D * H2 * 4, st);
    cudaMemsetAsync(g->b2, 0, DICM_D * 4, st);
    return last_launch("dicm_imgmlp_bwd");
  }
  if (workspace_bytes < dicm_imgmlp_workspace(rows_max, d_raw, precision))
    return fail(DICM_ERR_VALUE, "image MLP bwd: workspace too small");
  Ws w;
  carve(rows_max, d_raw, &w, (char*)workspace);
  g_red_tmp = w.red;
  const int M = (int)rows_max;
  if (precision != DICM_PREC_FP32) {
    // tensor-core path: layers 2-1 fused on tcgen05, dW1 on tcgen05, then dW0
    char* tc_ws = (char*)workspace + carve(rows_max, d_raw, nullptr, nullptr) - sm100::workspace_bytes(rows_max, d_raw);
    const bool bf16 = precision == DICM_PREC_BF16;
    __nv_bfloat16* da0_bf16 = bf16 ? sm100::da0_bf16_ptr(tc_ws, rows_max, d_raw) : nullptr;
    if (bf16)
      rc = sm100::bwd_layers12_bf16(demb, reinterpret_cast<const __nv_bfloat16*>(act1),
                                    reinterpret_cast<const __nv_bfloat16*>(act0), count_dev, rows_max, p->a0, p->a1,
                                    p->w1, p->w2, reinterpret_cast<__nv_bfloat16*>(w.da1), da0_bf16, w.pl12, w.pdw1,
                                    st);
    else
      rc = sm100::bwd_layers12(demb, act1, act0, w.h1, count_dev, rows_max, p->a0, p->a1, p->w1, p->w2, w.da1, w.da0,
                             da0_bf16, w.pl12, w.pdw1, st);
    if (rc) return rc;
    // the layer-1/2 gradient reduces only feed the optimizer: they run on a
    // forked stream beside the layer-0 dW0 kernel (joined before returning)
    Fork* fk = side_fork(0);
    cudaStream_t rs = fork_begin(fk, st);
    const int nb = sm100::small_bwd_blocks(rows_max), ps = sm100::small_part_size();
    {
      // w2 | b2 | a1 | b1 (| a0 | b0 on the tf32 path) in one launch
      const int64_t off[6] = {0, DICM_D * H2, DICM_D * H2 + DICM_D, DICM_D * H2 + DICM_D + H2, L2_PART, L2_PART + H1};
      const int64_t n[6] = {DICM_D * H2, DICM_D, H2, H2, H1, H1};
      float* const out[6] = {g->w2, g->b2, g->a1, g->b1, g->a0, g->b0};
      reduce_multi(rs, w.pl12, nb, ps, bf16 ? 4 : 6, off, n, out);
    }
    if (bf16) {
      // dW1 / dalpha0 / db0 from the three row GEMMs of k_dw1b
      const int gp = sm100::dw1_bf16_part_size();
      reduce(rs, w.pdw1, sm100::small_dw1_blocks(rows_max), gp, 0, gp, w.g3);
      rc = sm100::l1_finish_bf16(w.g3, p->w1, p->a0, g->b1, g->w1, g->a0, g->b0, rs);
    } else {
      reduce(rs, w.pdw1, sm100::small_dw1_blocks(rows_max), (int64_t)H2 * H1, 0, (int64_t)H2 * H1, g->w1);
    }
    int rc0 = sm100::bwd_dw0(pool, pool_dtype, d_raw, rows, count_dev, rows_max, w.da0, g->w0, precision, tc_ws, st,
                             bf16);
    fork_end(fk, st);
    if (rc) return rc;
    if (rc0) return rc0;
    return last_launch("dicm_imgmlp_bwd");
  }
  // layer 2 + prelu 1
  k_layer2_bwd<<<L2_BLOCKS, 256, 0, st>>>(act1, p->a1, p->w2, demb, count_dev, rows_max, w.da1, w.p2);
  reduce(st, w.p2, L2_BLOCKS, L2_PART, 0, DICM_D * H2, g->w2);
  reduce(st, w.p2, L2_BLOCKS, L2_PART, DICM_D * H2, DICM_D, g->b2);
  reduce(st, w.p2, L2_BLOCKS, L2_PART, DICM_D * H2 + DICM_D, H2, g->a1);
  reduce(st, w.p2, L2_BLOCKS, L2_PART, DICM_D * H2 + DICM_D + H2, H2, g->b1);
  // dh1 = da1 W1 -> da0 (+ dalpha0, db0 partials)
  gemm(st, LoadA_Rows<float>{w.da1, H2, nullptr, nullptr}, LoadB_Rows<float>{p->w1, H1, nullptr, nullptr},
       EpPreluGrad{act0, p->a0, w.da0, w.p0}, M, H1, H2, count_dev, nullptr, 1);
  const int nrow_blk = (M + 63) / 64;
  reduce(st, w.p0, nrow_blk, 2 * H1, 0, H1, g->a0, count_dev, 64);
  reduce(st, w.p0, nrow_blk, 2 * H1, H1, H1, g->b0, count_dev, 64);
  // dW1 = da1^T prelu(a0)   (split-K over rows)
  gemm(st, LoadA_Cols{w.da1, H2}, LoadB_Rows<float>{act0, H1, nullptr, p->a0}, EpPartial{w.pw1, H2, H1}, H2, H1,
       M, nullptr, count_dev, w.s1);
  reduce(st, w.pw1, w.s1, (int64_t)H2 * H1, 0, (int64_t)H2 * H1, g->w1);
  // dW0 = da0^T X[rows]   (the big reduction over rows)
  if (precision == DICM_PREC_FP32) {
    if (pool_dtype == DICM_POOL_F32)
      gemm(st, LoadA_Cols{w.da0, H1}, LoadB_Rows<float>{(const float*)pool, d_raw, rows, nullptr},
           EpPartial{w.pw0, H1, d_raw}, H1, d_raw, M, nullptr, count_dev, w.s0);
    else
      gemm(st, LoadA_Cols{w.da0, H1},
           LoadB_Rows<__nv_bfloat16>{(const __nv_bfloat16*)pool, d_raw, rows, nullptr},
           EpPartial{w.pw0, H1, d_raw}, H1, d_raw, M, nullptr, count_dev, w.s0);
    reduce(st, w.pw0, w.s0, (int64_t)H1 * d_raw, 0, (int64_t)H1 * d_raw, g->w0);
  } else {
    char* tc_ws = (char*)workspace + carve(rows_max, d_raw, nullptr, nullptr) - sm100::workspace_bytes(rows_max, d_raw);
    rc = sm100::bwd_dw0(pool, pool_dtype, d_raw, rows, count_dev, rows_max, w.da0, g->w0, precision, tc_ws, st);
    if (rc) return rc;
  }
  return last_launch("dicm_imgmlp_bwd");
}

int dicm_reduce_partials(const float* partials, int nblk, int64_t n, float* out, int accumulate,
                         dicm_stream_t stream) {
  if (n <= 0) return DICM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  reduce_into(st, partials, nblk, n, 0, n, out, nullptr, accumulate);
  return dicm::last_launch("dicm_reduce_partials");
}

}  // extern "C"
