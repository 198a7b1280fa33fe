// product.hpp -- standalone slotwise product / degree-2 basemul kernels (product.cu).
#pragma once

#include <cuda_runtime.h>

#include "params.hpp"

namespace nttk_b200 {

// true when the 32-bit vectorised product kernel covers (P, kind, storage, alignment):
// improved / harvey / smont with fast-path encodings, u16 (p < 2^16) or u32 storage,
// 16-byte aligned buffers
bool product_supports(const HostParams& P, int kind, bool basemul, int elem, const void* l,
                      const void* r, const void* out);
// canonical l * r slotwise (pointwise_multiply, transform.hpp:349-370) or the degree-2
// basemul of a tree ending in degree-2 factors
cudaError_t product_launch(const HostParams& P, int kind, bool basemul, const void* l, const void* r,
                           void* out, size_t batch, int elem, cudaStream_t st);

}  // namespace nttk_b200
