// launch_cache.hpp -- thread-safe, per-device launch-geometry caches for the persistent kernels.
//
// Each launcher instantiation owns one `OccCache` (a static local: kernels with the same
// signature share a function-pointer type, so the cache must not be keyed on the type).
// Entries are per device because the dynamic shared-memory attribute and the SM count are
// device properties; concurrent first calls from several host threads are benign (the
// attribute set is idempotent, the stored value identical).
#pragma once

#include <cuda_runtime.h>

#include <atomic>

namespace nttk_b200 {

constexpr int kMaxDevices = 64;
using OccCache = std::atomic<int>[kMaxDevices];

inline int current_device_index() {
  int d = 0;
  cudaGetDevice(&d);
  return d >= 0 && d < kMaxDevices ? d : 0;
}

inline int sm_count_current() {
  static std::atomic<int> cache[kMaxDevices];
  const int d = current_device_index();
  int v = cache[d].load(std::memory_order_acquire);
  if (!v) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    if (v <= 0) v = 148;
    cache[d].store(v, std::memory_order_release);
  }
  return v;
}

// resident CTAs per SM of `kern` at (threads, dynamic smem) on the current device
template <class Kern>
int occupancy_current(Kern kern, int threads, int smem, OccCache& cache) {
  const int d = current_device_index();
  int v = cache[d].load(std::memory_order_acquire);
  if (!v) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, threads, smem);
    if (v <= 0) v = 1;
    cache[d].store(v, std::memory_order_release);
  }
  return v;
}

}  // namespace nttk_b200
