// Counter-based initialisation of huge ID tables on the device.
//
// The reference draws every table as 0.05 * N(0, 1) from a per-name seeded
// generator (model.py:316-319) on the host; at 100M rows (cfg 5) that is
// 9.6 GB of f64 per table before it reaches a GPU.  Here row r, column c of
// table `key` is a pure function of (key, r * d + c): a splitmix64 hash of the
// counter gives two uniforms, Box-Muller one normal.  Every rank fills only
// the rows it owns (r = local * world + rank), and the values do not depend on
// the world size -- the same model at N = 1, 2, 4, 8 GPUs (not the
// reference's values: same distribution).
#include <math.h>

#include "common.cuh"

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void k_table_init(float* __restrict__ out, int64_t n_local, int d, int world, int rank, int64_t vocab,
                             uint64_t key, float scale) {
  const int64_t n = n_local * d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t local = i / d, c = i % d;
    const int64_t row = local * world + rank;
    if (row >= vocab) {  // padding rows of the last shard
      out[i] = 0.f;
      continue;
    }
    const uint64_t h = splitmix64(key ^ splitmix64((uint64_t)(row * d + c)));
    // two 26-bit uniforms in (0, 1], Box-Muller in double
    const double u1 = ((double)((h >> 38) & 0x3FFFFFF) + 1.0) / 67108864.0;
    const double u2 = (double)((h >> 6) & 0x3FFFFFF) / 67108864.0;
    const double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    out[i] = (float)(scale * z);
  }
}

}  // namespace

extern "C" int dicm_table_init(float* out, int64_t n_local, int d, int world, int rank, int64_t vocab, uint64_t key,
                               float scale, dicm_stream_t stream) {
  using namespace dicm;
  if (n_local <= 0) return DICM_OK;
  if (world < 1 || rank < 0 || rank >= world) return fail(DICM_ERR_VALUE, "table_init: rank %d of %d", rank, world);
  k_table_init<<<dicm_grid(n_local * d, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(out, n_local, d, world, rank,
                                                                                      vocab, key, scale);
  return last_launch("dicm_table_init");
}
