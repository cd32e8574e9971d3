// Epilogue helpers: a TMEM drain gives each lane one ROW of a 32x32 block
// (tcgen05.ld 32x32b); storing that directly writes 32 rows x 16 B per
// instruction (half-sector writes).  These helpers transpose the block through
// a per-warp shared-memory scratch so every store instruction writes whole
// 128-B row segments.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace dicm {
namespace epi {

constexpr int PITCH = 33;  // floats per scratch row (conflict-free transpose)
constexpr int SCRATCH_FLOATS = 32 * PITCH;

// v = columns [c0, c0+32) of row (row0 + lane); dst(row) = pointer to column
// c0 of that row; rows >= nrows are skipped.
template <typename RowPtr>
__device__ __forceinline__ void store_f32(const float (&v)[32], float* scratch, int lane, int row0, int nrows,
                                          RowPtr dst) {
#pragma unroll
  for (int j = 0; j < 32; ++j) scratch[lane * PITCH + j] = v[j];
  __syncwarp();
  const int sub = lane >> 3, ch = lane & 7;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = i * 4 + sub;
    if (row0 + r < nrows) {
      const float* s = scratch + r * PITCH + ch * 4;
      reinterpret_cast<float4*>(dst(row0 + r))[ch] = make_float4(s[0], s[1], s[2], s[3]);
    }
  }
  __syncwarp();
}

template <typename RowPtr>
__device__ __forceinline__ void store_bf16(const float (&v)[32], float* scratch, int lane, int row0, int nrows,
                                           RowPtr dst) {
#pragma unroll
  for (int j = 0; j < 32; ++j) scratch[lane * PITCH + j] = v[j];
  __syncwarp();
  const int sub = lane >> 2, ch = lane & 3;  // 8 rows x 4 chunks of 8 bf16 per pass
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = i * 8 + sub;
    if (row0 + r < nrows) {
      const float* s = scratch + r * PITCH + ch * 8;
      __nv_bfloat162 p0 = __floats2bfloat162_rn(s[0], s[1]), p1 = __floats2bfloat162_rn(s[2], s[3]);
      __nv_bfloat162 p2 = __floats2bfloat162_rn(s[4], s[5]), p3 = __floats2bfloat162_rn(s[6], s[7]);
      uint4 u;
      u.x = *reinterpret_cast<uint32_t*>(&p0);
      u.y = *reinterpret_cast<uint32_t*>(&p1);
      u.z = *reinterpret_cast<uint32_t*>(&p2);
      u.w = *reinterpret_cast<uint32_t*>(&p3);
      reinterpret_cast<uint4*>(dst(row0 + r))[ch] = u;
    }
  }
  __syncwarp();
}

}  // namespace epi
}  // namespace dicm
