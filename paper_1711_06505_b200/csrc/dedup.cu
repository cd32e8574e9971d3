// a2: deduplication of keys with an inverse index, by dense-key-space bitmap.
//
// Reference semantics: unique = np.unique(keys) (model.py:187),
// inverse = np.searchsorted(unique, keys) (model.py:374, 378).  Keys are
// bounded ids (pool rows, vocabulary rows), so instead of sorting we mark a
// bitmap over the key space, prefix-scan the popcounts of its words, and read
// both results off the scan:
//   unique[r]  = the r-th set bit (ascending by construction),
//   inverse[i] = prefix(word(k)) + popc(word(k) & below(k)).
// Work is O(refs + key_space/32) with coalesced passes and no sort; results
// are bit-exact with numpy.
#include "common.cuh"

namespace {

constexpr int kScanThreads = 128;
constexpr int kWordsPerThread = 4;
constexpr int kTile = kScanThreads * kWordsPerThread;  // 512 words = 16384 keys: many blocks per pass

struct Segs {
  const int32_t* ids[DICM_MAX_SEGS];
  int64_t base[DICM_MAX_SEGS];
  int64_t vocab[DICM_MAX_SEGS];
  int64_t inv_off[DICM_MAX_SEGS];
  int64_t start[DICM_MAX_SEGS + 1];
  int nseg;
  const int32_t* n_dev;  // optional device-side length of a single segment
};

__device__ __forceinline__ int64_t seg_total(const Segs& s) {
  const int64_t t = s.start[s.nseg];
  return s.n_dev ? min(t, (int64_t)*s.n_dev) : t;
}

__device__ __forceinline__ int find_seg(const Segs& s, int64_t i) {
  int k = 0;
  while (k + 1 < s.nseg && i >= s.start[k + 1]) ++k;
  return k;
}

// Keys that share a bitmap word within a warp are combined first (one
// fire-and-forget RED.OR per distinct word and warp): small-vocabulary fields
// (scenario, ad_category: a handful of ids over the whole batch) and Zipf-hot
// keys would otherwise queue thousands of reductions on one word.
__global__ void k_mark(const __grid_constant__ Segs segs, uint32_t* __restrict__ bitmap, int tag,
                       int32_t* __restrict__ status) {
  const int64_t total = seg_total(segs);
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x - lane; i0 < total; i0 += stride) {
    const int64_t i = i0 + lane;
    uint32_t w = 0xffffffffu, bit = 0;
    if (i < total) {
      const int s = find_seg(segs, i);
      const int64_t id = segs.ids[s][i - segs.start[s]];
      if (id < 0 || id >= segs.vocab[s]) {
        if (atomicCAS(&status[DICM_ST_KEY_FLAG], 0, 1) == 0) {
          status[DICM_ST_KEY_VALUE] = (int32_t)id;
          status[DICM_ST_KEY_SEG] = tag * 16 + s;
        }
      } else {
        const uint32_t key = (uint32_t)(segs.base[s] + id);
        w = key >> 5;
        bit = 1u << (key & 31);
      }
    }
    const unsigned peers = __match_any_sync(0xffffffffu, w);
    uint32_t bits = 0;
#pragma unroll 8
    for (int src = 0; src < 32; ++src) {
      const uint32_t b = __shfl_sync(0xffffffffu, bit, src);
      if ((peers >> src) & 1u) bits |= b;
    }
    if (w != 0xffffffffu && lane == __ffs(peers) - 1) atomicOr(bitmap + w, bits);  // result unused: RED.OR
  }
}

__device__ __forceinline__ int block_excl_scan(int v, int* total) {
  __shared__ int warp_tot[kScanThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int t = lane < kScanThreads / 32 ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kScanThreads / 32) warp_tot[lane] = t;
  }
  __syncthreads();
  const int warp_off = wid ? warp_tot[wid - 1] : 0;
  *total = warp_tot[kScanThreads / 32 - 1];
  __syncthreads();
  return warp_off + x - v;
}

// per-tile popcount sums (coalesced: consecutive threads read consecutive uint4)
__global__ void k_tile_sums(const uint32_t* __restrict__ bitmap, int32_t* __restrict__ tile_sums) {
  const uint4* p = reinterpret_cast<const uint4*>(bitmap + (int64_t)blockIdx.x * kTile);
  int c = 0;
#pragma unroll
  for (int q = 0; q < kWordsPerThread / 4; ++q) {
    uint4 v = __ldcg(p + q * kScanThreads + threadIdx.x);
    c += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
  }
  int tot;
  block_excl_scan(c, &tot);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

// exclusive scan of the tile sums in one block; total -> count
__global__ void k_scan_tiles(int32_t* __restrict__ tile_sums, int ntiles, int32_t* count) {
  int carry = 0;
  for (int base = 0; base < ntiles; base += kScanThreads) {
    const int i = base + threadIdx.x;
    const int v = i < ntiles ? tile_sums[i] : 0;
    int tot;
    const int ex = block_excl_scan(v, &tot);
    if (i < ntiles) tile_sums[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *count = carry;
}

// word prefixes + emission of the unique keys.  Warp w of the block owns
// words [w*WPW, (w+1)*WPW) of the tile, 32 at a time with one word per lane:
// a warp scan of the popcounts places each lane's keys, which it then writes
// in ascending bit order (at most 32 short iterations per chunk).
__global__ void __launch_bounds__(kScanThreads) k_emit(const uint32_t* __restrict__ bitmap,
                                                       const int32_t* __restrict__ tile_off,
                                                       int32_t* __restrict__ word_prefix, int32_t* __restrict__ uniq) {
  constexpr int WPW = kTile / (kScanThreads / 32);  // words per warp
  __shared__ int32_t wtot[kScanThreads / 32];
  const int64_t tile_base = (int64_t)blockIdx.x * kTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t* mw = bitmap + tile_base + warp * WPW;
  uint32_t bits[WPW / 32];
  int c = 0;
#pragma unroll
  for (int q = 0; q < WPW / 32; ++q) {
    bits[q] = __ldcg(mw + q * 32 + lane);
    c += __popc(bits[q]);
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if (lane == 0) wtot[warp] = c;
  __syncthreads();
  int run = tile_off[blockIdx.x];
  for (int w = 0; w < warp; ++w) run += wtot[w];
#pragma unroll
  for (int q = 0; q < WPW / 32; ++q) {
    const int n = __popc(bits[q]);
    int incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int64_t wi = tile_base + warp * WPW + q * 32 + lane;
    int pos = run + incl - n;
    word_prefix[wi] = pos;
    uint32_t b = bits[q];
    const int32_t wkey = (int32_t)(wi << 5);
    while (b) {
      uniq[pos++] = wkey + (__ffs(b) - 1);
      b &= b - 1;
    }
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
}

__global__ void k_inverse(const __grid_constant__ Segs segs, const uint32_t* __restrict__ bitmap,
                          const int32_t* __restrict__ word_prefix, int32_t* __restrict__ inv) {
  const int64_t total = seg_total(segs);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int s = find_seg(segs, i);
    const int64_t j = i - segs.start[s];
    const int64_t id = segs.ids[s][j];
    int32_t r = 0;  // out-of-vocabulary: flagged by k_mark, index kept in bounds
    if (id >= 0 && id < segs.vocab[s]) {
      const uint32_t key = (uint32_t)(segs.base[s] + id);
      const uint32_t w = key >> 5;
      r = word_prefix[w] + __popc(__ldg(bitmap + w) & ((1u << (key & 31)) - 1u));
    }
    inv[segs.inv_off[s] + j] = r;
  }
}

int run_dedup(const Segs& s, int64_t key_space, void* workspace, int32_t* uniq_out, int32_t* inv_out,
              int32_t* count_dev, int32_t tag, int32_t* status, cudaStream_t st);

int64_t padded_words(int64_t key_space) {
  const int64_t w = (key_space + 31) / 32;
  return ((w + kTile - 1) / kTile) * kTile;
}

}  // namespace

extern "C" {

size_t dicm_dedup_workspace(int64_t key_space) {
  const int64_t W = padded_words(key_space < 1 ? 1 : key_space);
  return (size_t)(W * 4 * 2 + (W / kTile) * 4 + 256);
}

static int make_segs(const dicm_keyseg_t* segs, int nseg, int64_t key_space, size_t workspace_bytes, Segs& s) {
  using namespace dicm;
  if (nseg < 1 || nseg > DICM_MAX_SEGS) return fail(DICM_ERR_VALUE, "dedup: nseg %d not in [1, %d]", nseg, DICM_MAX_SEGS);
  if (key_space < 1 || key_space > (int64_t)1 << 31)
    return fail(DICM_ERR_VALUE, "dedup: key space %lld outside [1, 2^31]", (long long)key_space);
  if (workspace_bytes < dicm_dedup_workspace(key_space)) return fail(DICM_ERR_VALUE, "dedup: workspace too small");
  s = Segs{};
  s.nseg = nseg;
  s.start[0] = 0;
  for (int i = 0; i < nseg; ++i) {
    s.ids[i] = segs[i].ids;
    s.base[i] = segs[i].base;
    s.vocab[i] = segs[i].vocab;
    s.inv_off[i] = segs[i].inv_off;
    s.start[i + 1] = s.start[i] + segs[i].n;
    if (segs[i].n < 0 || segs[i].base < 0 || segs[i].base + segs[i].vocab > key_space)
      return fail(DICM_ERR_VALUE, "dedup: segment %d [%lld, +%lld) exceeds key space %lld", i,
                  (long long)segs[i].base, (long long)segs[i].vocab, (long long)key_space);
  }
  return DICM_OK;
}

int dicm_dedup(const dicm_keyseg_t* segs, int nseg, int64_t key_space, void* workspace,
               size_t workspace_bytes, int32_t* uniq_out, int32_t* inv_out, int32_t* count_dev,
               int32_t tag, int32_t* status, dicm_stream_t stream) {
  Segs s;
  if (int rc = make_segs(segs, nseg, key_space, workspace_bytes, s)) return rc;
  return run_dedup(s, key_space, workspace, uniq_out, inv_out, count_dev, tag, status, (cudaStream_t)stream);
}

int dicm_dedup_inverse(const dicm_keyseg_t* segs, int nseg, int64_t key_space, const void* workspace,
                       size_t workspace_bytes, int32_t* inv_out, dicm_stream_t stream) {
  using namespace dicm;
  Segs s;
  if (int rc = make_segs(segs, nseg, key_space, workspace_bytes, s)) return rc;
  const int64_t total = s.start[nseg];
  if (total <= 0) return DICM_OK;
  const int64_t W = padded_words(key_space);
  const uint32_t* bitmap = (const uint32_t*)workspace;
  const int32_t* word_prefix = (const int32_t*)(bitmap + W);
  k_inverse<<<dicm_grid(total, 256, 148 * 32), 256, 0, (cudaStream_t)stream>>>(s, bitmap, word_prefix, inv_out);
  return last_launch("dicm_dedup_inverse");
}

int dicm_dedup_devn(const int32_t* keys, const int32_t* n_dev, int64_t n_max, int64_t vocab, void* workspace,
                    size_t workspace_bytes, int32_t* uniq_out, int32_t* inv_out, int32_t* count_dev,
                    int32_t tag, int32_t* status, dicm_stream_t stream) {
  using namespace dicm;
  if (vocab < 1 || vocab > (int64_t)1 << 31) return fail(DICM_ERR_VALUE, "dedup: vocab %lld", (long long)vocab);
  if (n_max < 0) return fail(DICM_ERR_VALUE, "dedup: n_max < 0");
  if (workspace_bytes < dicm_dedup_workspace(vocab)) return fail(DICM_ERR_VALUE, "dedup: workspace too small");
  Segs s{};
  s.nseg = 1;
  s.ids[0] = keys;
  s.vocab[0] = vocab;
  s.start[1] = n_max;
  s.n_dev = n_dev;
  return run_dedup(s, vocab, workspace, uniq_out, inv_out, count_dev, tag, status, (cudaStream_t)stream);
}

}  // extern "C"

namespace {
int run_dedup(const Segs& s, int64_t key_space, void* workspace, int32_t* uniq_out, int32_t* inv_out,
              int32_t* count_dev, int32_t tag, int32_t* status, cudaStream_t st) {
  using namespace dicm;
  const int nseg = s.nseg;
  const int64_t W = padded_words(key_space);
  const int ntiles = (int)(W / kTile);
  uint32_t* bitmap = (uint32_t*)workspace;
  int32_t* word_prefix = (int32_t*)(bitmap + W);
  int32_t* tile_sums = word_prefix + W;
  int rc = check_cuda(cudaMemsetAsync(bitmap, 0, W * 4, st), "dedup memset");
  if (rc) return rc;
  const int64_t total = s.start[nseg];
  if (total > 0) k_mark<<<dicm_grid(total, 256, 148 * 32), 256, 0, st>>>(s, bitmap, tag, status);
  k_tile_sums<<<ntiles, kScanThreads, 0, st>>>(bitmap, tile_sums);
  k_scan_tiles<<<1, kScanThreads, 0, st>>>(tile_sums, ntiles, count_dev);
  k_emit<<<ntiles, kScanThreads, 0, st>>>(bitmap, tile_sums, word_prefix, uniq_out);
  if (total > 0 && inv_out)
    k_inverse<<<dicm_grid(total, 256, 148 * 32), 256, 0, st>>>(s, bitmap, word_prefix, inv_out);
  return last_launch("dicm_dedup");
}
}  // namespace
