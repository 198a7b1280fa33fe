// tensor_map.hpp -- TMA tensor maps for the swizzled stage loads of the inverse kernels.
//
// A batch of polynomials is viewed as a 2-D tensor of 128-byte rows (32 u32 words; a u16
// batch is moved byte-for-byte the same way).  One cp.async.bulk.tensor per stage copies a
// tile of rows with CU_TENSOR_MAP_SWIZZLE_128B: 16-byte chunk c of row r lands at chunk
// c ^ (r & 7) of its 128-byte shared-memory row, so the lanes' contiguous-ownership reads
// (lane j reads its own 32..128-byte segment) hit distinct banks -- the linear bulk copy
// left them 2-way (u16) / 4-way (u32) conflicted (profiles/r1b_ncu_full: 16 wavefronts per
// LDS.128 against an ideal 4).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace nttk_b200 {

constexpr uint32_t kRowBytes = 128;
// rows addressed by one tensor map (the TMA coordinates are signed 32-bit)
constexpr uint64_t kMaxMapRows = uint64_t(1) << 30;

// Encode a map over `rows` rows of 128 bytes starting at `base` (16-byte aligned), copied
// in boxes of `box_rows` (<= 256) rows.  cudaErrorNotSupported if the driver lacks the
// entry point, cudaErrorInvalidValue for unencodable arguments.
cudaError_t make_rows128_map(CUtensorMap* map, const void* base, uint64_t rows, uint32_t box_rows);

}  // namespace nttk_b200
