// copy_probe.cu -- HBM copy ceilings of the memory pipelines the N = 256 kernels can use
// (2 GiB in -> 2 GiB out, the Dilithium forward's traffic), CUDA events, best of 5.
//   A  grid-stride LDG.128 / STG.128 copy (4 vectors in flight per thread), CTAs/SM swept
//   B  TMA bulk copy HBM -> shared (1 producer lane, S stages of 16 KiB) -> LDS.128 -> STG.128
//      (the fast256_tma.cu pipeline with the butterflies removed), CTAs/SM and S swept
//   C  as B, but the consumers hand the landed stage straight back with a bulk shared -> HBM
//      store (no register pass)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/copy_probe tools/copy_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

__global__ void copy_ldg(const uint4* __restrict__ in, uint4* __restrict__ out, size_t n) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 a = __ldcs(in + i), b = __ldcs(in + i + stride), c = __ldcs(in + i + 2 * stride),
          d = __ldcs(in + i + 3 * stride);
    __stcs(out + i, a);
    __stcs(out + i + stride, b);
    __stcs(out + i + 2 * stride, c);
    __stcs(out + i + 3 * stride, d);
  }
  for (; i < n; i += stride) __stcs(out + i, __ldcs(in + i));
}

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

constexpr int kStageBytes = 16384;
constexpr int kConsumers = 8;

template <int S, bool BULK_STORE>
__global__ void __launch_bounds__((kConsumers + 1) * 32) copy_tma(const uint8_t* in, uint8_t* out, size_t tiles) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * kStageBytes);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[s])), "r"(kConsumers));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kConsumers) {
    if (lane == 0) {
      uint32_t s = 0, ph = 0, k = 0;
      for (size_t t = blockIdx.x; t < tiles; t += gridDim.x, ++k) {
        if (k >= S)
          asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(
                           sa(&empty[s])),
                       "r"(ph ^ 1)
                       : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(kStageBytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                sa(sm + s * kStageBytes)),
            "l"(in + t * kStageBytes), "r"(kStageBytes), "r"(sa(&full[s]))
            : "memory");
        if (++s == S) s = 0, ph ^= 1;
      }
    }
    return;
  }
  uint32_t s = 0, ph = 0;
  for (size_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(
                     sa(&full[s])),
                 "r"(ph)
                 : "memory");
    uint8_t* st = sm + s * kStageBytes + warp * 2048;
    if (BULK_STORE) {
      if (lane == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + t * kStageBytes + warp * 2048),
                     "r"(sa(st)), "r"(2048)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    } else {
      uint4 v[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = reinterpret_cast<const uint4*>(st)[lane + 32 * c];
      uint4* o = reinterpret_cast<uint4*>(out + t * kStageBytes + warp * 2048);
#pragma unroll
      for (int c = 0; c < 4; ++c) __stcs(o + lane + 32 * c, v[c]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
    if (++s == S) s = 0, ph ^= 1;
  }
  if (BULK_STORE && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <class F>
float best_ms(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r > 0 && ms < best) best = ms;
  }
  return best;
}

template <int S, bool BULK>
int run_tma(const uint8_t* in, uint8_t* out, size_t bytes, int sms) {
  auto k = copy_tma<S, BULK>;
  const int smem = S * kStageBytes + 2 * S * 8;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, (kConsumers + 1) * 32, smem));
  for (int c = 1; c <= occ; ++c) {
    const size_t tiles = bytes / kStageBytes;
    const float ms = best_ms([&] { k<<<sms * c, (kConsumers + 1) * 32, smem>>>(in, out, tiles); });
    CK(cudaGetLastError());
    printf("%s S=%d CTAs/SM=%d: %.4f ms  %.0f GB/s\n", BULK ? "C tma+bulkstore" : "B tma+stg", S, c, ms,
           2.0 * bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}

int main() {
  const size_t bytes = size_t(2) << 30;
  uint8_t *in, *out;
  CK(cudaMalloc(&in, bytes));
  CK(cudaMalloc(&out, bytes));
  CK(cudaMemset(in, 1, bytes));
  CK(cudaMemset(out, 0, bytes));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int c : {2, 4, 8}) {
    const float ms = best_ms([&] { copy_ldg<<<sms * c, 256>>>(reinterpret_cast<const uint4*>(in), reinterpret_cast<uint4*>(out), bytes / 16); });
    CK(cudaGetLastError());
    printf("A ldg/stg 256 thr CTAs/SM=%d: %.4f ms  %.0f GB/s\n", c, ms, 2.0 * bytes / (ms * 1e-3) / 1e9);
  }
  if (run_tma<2, false>(in, out, bytes, sms) || run_tma<3, false>(in, out, bytes, sms) ||
      run_tma<4, false>(in, out, bytes, sms) || run_tma<6, false>(in, out, bytes, sms) ||
      run_tma<3, true>(in, out, bytes, sms) || run_tma<4, true>(in, out, bytes, sms))
    return 1;
  return 0;
}
