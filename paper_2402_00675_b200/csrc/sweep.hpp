// sweep.hpp -- reduction sweep launcher (sweep.cu).
#pragma once

#include <cuda_runtime.h>

#include "params.hpp"

namespace nttk_b200 {

// d_sum: device u64 accumulator (atomically added to; caller zeroes it); d_fires (optional,
// plantard_redc only): device u64 counter of the r == p corner (plantard_correction_fires)
cudaError_t sweep_launch(int variant, const Ctx& c, const int64_t* A, size_t na, const int64_t* B,
                         size_t nb, int64_t* r, unsigned long long* d_sum, cudaStream_t st,
                         unsigned long long* d_fires = nullptr);

}  // namespace nttk_b200
