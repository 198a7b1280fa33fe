// tensor_map.cpp -- host-side encoding of the 128-byte-row TMA tensor maps (tensor_map.hpp).
// cuTensorMapEncodeTiled is a driver-API function; it is resolved once through the
// runtime's driver entry point, so the static-cudart library needs no libcuda link.
#include "tensor_map.hpp"

#include <cudaTypedefs.h>

#include <atomic>

namespace nttk_b200 {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static std::atomic<PFN_cuTensorMapEncodeTiled_v12000> fn{nullptr};
  static std::atomic<bool> tried{false};
  PFN_cuTensorMapEncodeTiled_v12000 f = fn.load(std::memory_order_acquire);
  if (f || tried.load(std::memory_order_acquire)) return f;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess && p) {
    f = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    fn.store(f, std::memory_order_release);
  }
  tried.store(true, std::memory_order_release);
  return f;
}

}  // namespace

cudaError_t make_rows128_map(CUtensorMap* map, const void* base, uint64_t rows, uint32_t box_rows) {
  if (!map || !base || rows == 0 || rows > kMaxMapRows || box_rows == 0 || box_rows > 256 ||
      (reinterpret_cast<uintptr_t>(base) & 15))
    return cudaErrorInvalidValue;
  const auto f = encode_fn();
  if (!f) return cudaErrorNotSupported;
  const cuuint64_t dims[2] = {kRowBytes / 4, rows};
  const cuuint64_t strides[1] = {kRowBytes};  // bytes, dimension 1
  const cuuint32_t box[2] = {kRowBytes / 4, box_rows};
  const cuuint32_t estride[2] = {1, 1};
  const CUresult r = f(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(base), dims, strides,
                       box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace nttk_b200
