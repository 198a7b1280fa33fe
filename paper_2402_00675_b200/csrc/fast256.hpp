// fast256.hpp -- launcher interface of the N = 256 sm_100a kernels (fast256.cu).
#pragma once

#include <cuda_runtime.h>

#include "params.hpp"

namespace nttk_b200 {

bool fast256_supports(int kind, int layers, int n_bits);
// dir 0 = forward (ntt_forward), 1 = inverse (intt_inverse).  variant 1 selects the
// paper-form n=16 Plantard tail ((h >> 16) + 1) p >> 16 (SASS census / A-B check).
cudaError_t fast256_launch(const HostParams& P, int kind, int dir, const void* in, void* out,
                           size_t batch, int elem_bytes, cudaStream_t st, int variant = 0);

}  // namespace nttk_b200

namespace nttk_b200 {

// v2: TMA bulk-copy fed kernels (fast256_tma.cu), u16/u32 storage, 16-byte aligned buffers
bool fast256_tma_supports(int elem_bytes, const void* in, const void* out);
cudaError_t fast256_tma_launch(const HostParams& P, int kind, int dir, const void* in, void* out,
                               size_t batch, int elem_bytes, cudaStream_t st);

}  // namespace nttk_b200

namespace nttk_b200 {

// fused polymul (polymul_tma.cu): c = inverse(product(forward(a), forward(b)))
cudaError_t polymul256_launch(const HostParams& P, int kind, const void* a, const void* b,
                              void* out, size_t batch, int elem_bytes, cudaStream_t st);

}  // namespace nttk_b200
