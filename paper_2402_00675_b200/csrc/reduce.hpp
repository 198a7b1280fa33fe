// reduce.hpp -- launcher of the elementwise reduction kernels (reduce.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "../../include/nttk_gpu.h"

namespace nttk_b200 {

// out[i] = op(x[i] [, y[i]]); operand-range violations OR bits into d_flag[0]; d_flag points
// to 16 zeroed bytes whose second u64 (d_flag + 2) counts plantard_redc's r == p corner
cudaError_t reduce_launch(int op, const nttk_reduction_ctx& c, const int64_t* x, const int64_t* y,
                          int64_t* out, size_t n, unsigned* d_flag, cudaStream_t st);

// (xo[i], yo[i]) = butterfly(x[i], y[i], w[i] [, wq[i]]); violations OR bits into *d_flag
cudaError_t butterfly_launch(int op, const nttk_reduction_ctx& c, uint32_t aux0, uint32_t aux1,
                             const int64_t* x, const int64_t* y, const int64_t* w,
                             const int64_t* wq, int64_t* xo, int64_t* yo, size_t n,
                             unsigned* d_flag, cudaStream_t st);

}  // namespace nttk_b200
