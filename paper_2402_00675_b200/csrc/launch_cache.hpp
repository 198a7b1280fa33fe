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

// Launch with programmatic dependent launch (PDL) allowed: when the previous launch on the stream
// is one of the TMA kernels (which signal griddepcontrol.launch_dependents as they start), this
// grid's CTAs become resident as that grid's CTAs exit and run their prologue (barrier init,
// twiddle pins, table staging) under its tail; the producer warps block in griddepcontrol.wait
// until the previous grid has completed and its writes are visible before they touch global
// memory, and every consumer store depends on data the producer loaded after that wait.  After
// any other kernel, a copy or an event the launch is ordered as usual.  It removes the
// launch latency between back-to-back small launches (BASELINE configs 1 and 2).
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), int grid, int block, int smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(static_cast<unsigned>(block));
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace nttk_b200
