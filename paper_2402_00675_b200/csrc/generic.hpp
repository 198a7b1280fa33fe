// generic.hpp -- launchers of the any-parameter kernels (generic.cu).
#pragma once

#include <cuda_runtime.h>

#include <functional>

#include "params.hpp"

namespace nttk_b200 {

cudaError_t generic_transform(const HostParams& P, const DeviceTables& T, int kind, int dir,
                              const void* in, void* out, size_t batch, int elem_bytes,
                              cudaStream_t st);
// canonical words between a storage width (2/4/8 bytes) and u64 (wide product path)
cudaError_t widen_to_u64(const void* src, int elem, uint64_t* dst, size_t n, cudaStream_t st);
cudaError_t narrow_from_u64(const uint64_t* src, void* dst, int elem, size_t n, cudaStream_t st);
// one polynomial, layer by layer, observe(layer) after each (state copied to h_state)
cudaError_t generic_transform_observed(const HostParams& P, const DeviceTables& T, int kind,
                                       int dir, uint64_t* d_io, uint64_t* h_state,
                                       const std::function<void(unsigned)>& observe,
                                       cudaStream_t st);
cudaError_t generic_pointwise(const HostParams& P, int kind, const void* l, const void* r,
                              void* out, size_t batch, int elem_bytes, cudaStream_t st);
// d_gamma: N/2 per-pair basemul moduli gamma_k (x^2 - gamma_k), device memory
cudaError_t generic_basemul(const HostParams& P, const uint64_t* d_gamma, int kind, const void* l,
                            const void* r, void* out, size_t batch, int elem_bytes,
                            cudaStream_t st);
cudaError_t check_canonical(const void* in, size_t n, int elem_bytes, uint64_t p,
                            unsigned* d_flag, cudaStream_t st);

}  // namespace nttk_b200
