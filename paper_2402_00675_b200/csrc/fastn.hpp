// fastn.hpp -- launchers of the N = 512 / 1024 TMA kernels (fastn_tma.cu).
#pragma once

#include <cuda_runtime.h>

#include "params.hpp"

namespace nttk_b200 {

// storage 2 or 4 bytes, full trees (layers == log2 N), 16-byte aligned buffers
bool fastn_supports(const HostParams& P, int elem_bytes, const void* in, const void* out);

// one transform direction (dir 0 forward, 1 inverse); tab = HostParams::fastn_table()
cudaError_t fastn_launch(const HostParams& P, int kind, int dir, const void* in, void* out,
                         size_t batch, int elem_bytes, const uint32_t* tab, cudaStream_t st);

}  // namespace nttk_b200
