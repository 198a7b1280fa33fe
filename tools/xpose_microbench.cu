// xpose_microbench.cu -- A/B of the phase switch of the N = 256 kernels: the XOR-swizzled
// shared-memory transpose they use (16 STS + 4 LDS.128 per lane, tma_common.cuh Xpose)
// against a register-only warp-shuffle transpose (4 SHFL.BFLY stages; in stage m a lane
// swaps the 8 registers whose bit m differs from its lane bit m with lane ^ m).  A half-warp
// holds one 16 x 16 tile (16 values per lane, the kernels' ownership); the loop repeats the
// transpose with a dependent add so nothing is hoisted.  Cycles per transpose per SMSP.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/xpose_mb.bin tools/xpose_microbench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__device__ __forceinline__ int swz(int i) {
  return (i & ~15) | ((((i >> 2) & 3) ^ ((i >> 5) & 3)) << 2) | (i & 3);
}

// shared-memory transpose: strided element i = j + 16 r at word swz(i); contiguous get4
__global__ void xpose_smem(uint32_t* out) {
  extern __shared__ uint32_t tiles[];  // one 256-word tile per half-warp
  const int j = threadIdx.x & 15;
  uint32_t* T = tiles + (threadIdx.x >> 4) * 256;
  uint32_t v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = threadIdx.x * 16 + r;
  for (int it = 0; it < ITERS; ++it) {
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 16; ++r) T[swz(j + 16 * r)] = v[r];
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 q = *reinterpret_cast<const uint4*>(&T[16 * j + 4 * (c ^ ((j >> 1) & 3))]);
      v[4 * c] += q.x;
      v[4 * c + 1] += q.y;
      v[4 * c + 2] += q.z;
      v[4 * c + 3] += q.w;
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) acc ^= v[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// register transpose with butterfly shuffles inside the half-warp
__global__ void xpose_shfl(uint32_t* out) {
  const int lane = threadIdx.x & 31, j = lane & 15;
  uint32_t v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = threadIdx.x * 16 + r;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int m = 8; m >= 1; m >>= 1) {
      const bool hi = (j & m) != 0;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r & m) continue;
        const uint32_t send = hi ? v[r] : v[r | m];
        const uint32_t got = __shfl_xor_sync(0xffffffffu, send, m);
        if (hi) v[r] = got;
        else v[r | m] = got;
      }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] += r;
  }
  uint32_t acc = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) acc ^= v[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* out;
  cudaMalloc(&out, size_t(sms) * 1024 * 4);
  auto run = [&](auto kern, const char* name) {
    for (int warps_per_smsp : {4, 6, 8}) {
      const int threads = 32 * 4 * warps_per_smsp;
      const int smem = threads / 16 * 256 * 4;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      kern<<<sms, threads, smem>>>(out);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      kern<<<sms, threads, smem>>>(out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      // per SMSP: warps_per_smsp warps x ITERS transposes (2 tiles per warp-transpose)
      const double per = ms * 1e-3 * clk * 1e3 / (double(warps_per_smsp) * ITERS);
      printf("%-44s warps/SMSP %d: %.1f cycles per warp-transpose (2 polys)\n", name, warps_per_smsp, per);
    }
  };
  run(xpose_smem, "smem XOR-swizzled (16 STS + 4 LDS.128)");
  run(xpose_shfl, "warp shuffle (4 SHFL.BFLY stages)");
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  return 0;
}
