// bf_microbench.cu -- how fast can one SM sub-partition run the n = 16 modified-Plantard CT
// butterfly (IMAD + IMAD.HI + 2 IADD3) with no memory traffic at all?  16 values per lane,
// 4 register-local layers per "phase" as in fast256_tma.cu, uniform twiddles from the
// constant bank.  Reports cycles per warp-butterfly per SMSP for several warp counts; the
// fmaheavy bound is 6 cycles (IMAD 2 + IMAD.HI 4).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o bf_mb tools/bf_microbench.cu && ./bf_mb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__constant__ uint32_t c_w[16];
__constant__ uint32_t c_p, c_zero;

template <int ITERS, int PAPER_MASK>
__global__ void bf_kernel(uint32_t* out) {
  uint32_t v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = threadIdx.x * 16 + r + blockIdx.x;
  const uint32_t p = c_p, z = c_zero;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int sl = 1; sl <= 4; ++sl) {
      const int h = 8 >> (sl - 1);
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r & h) continue;
        const uint32_t w = c_w[(1 << (sl - 1)) - 1 + (r >> (5 - sl))];
        const uint32_t hh = v[r + h] * w;
        const uint32_t rr = ((PAPER_MASK >> sl) & 1) ? (((hh >> 16) + 1u) * p) >> 16 : __umulhi(hh, p);
        const uint32_t x = v[r];
        v[r + h] = x + p - rr;
        v[r] = x + rr + z;
      }
    }
    // keep values bounded like the real transform (canonical-ish restart)
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] &= 0xffffu;
  }
  uint32_t acc = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) acc ^= v[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// pure fma-pipe mixes: 16 independent chains per thread, MODE 0: IMAD + IMAD.HI per step,
// 1: IMAD.HI only, 2: IMAD only
template <int ITERS, int MODE>
__global__ void chain_kernel(uint32_t* out) {
  uint32_t v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = threadIdx.x * 16 + r + blockIdx.x;
  const uint32_t p = c_p, w = c_w[0];
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (MODE == 0) v[r] = __umulhi(v[r] * w, p + r);
        else if (MODE == 1) v[r] = __umulhi(v[r], w + r);
        else v[r] = v[r] * w + r;
      }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) acc ^= v[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// butterfly-shaped mixes: MODE 0 standard (2 dependent IADD3 per bf), 1: same two ALU ops
// but independent of the product (accumulators), 2: one dependent IADD3 per bf
template <int ITERS, int MODE>
__global__ void mix_kernel(uint32_t* out) {
  uint32_t v[16], a0 = threadIdx.x, a1 = blockIdx.x;
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = threadIdx.x * 16 + r + blockIdx.x;
  const uint32_t p = c_p, z = c_zero;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int sl = 1; sl <= 4; ++sl) {
      const int h = 8 >> (sl - 1);
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r & h) continue;
        const uint32_t w = c_w[(1 << (sl - 1)) - 1 + (r >> (5 - sl))];
        const uint32_t rr = __umulhi(v[r + h] * w, p);
        const uint32_t x = v[r];
        if (MODE == 0) {
          v[r + h] = x + p - rr;
          v[r] = x + rr + z;
        } else if (MODE == 1) {
          v[r + h] = rr;
          v[r] = rr ^ x;  // LOP3 keeps the dependency chain but is one op
          a0 = a0 + x + z;
          a1 = a1 + p - a0;
        } else {
          v[r + h] = rr;
          v[r] = x + rr + z;
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] &= 0xffffu;
  }
  uint32_t acc = a0 ^ a1;
#pragma unroll
  for (int r = 0; r < 16; ++r) acc ^= v[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  uint32_t w[16];
  for (int i = 0; i < 16; ++i) w[i] = 0x9e3779b9u * (i + 1);
  const uint32_t p = 3329, z = 0;
  cudaMemcpyToSymbol(c_w, w, sizeof w);
  cudaMemcpyToSymbol(c_p, &p, 4);
  cudaMemcpyToSymbol(c_zero, &z, 4);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* out;
  cudaMalloc(&out, size_t(sms) * 1024 * 64 * 4);
  constexpr int ITERS = 4096;
  auto run = [&](auto kern, const char* name) {
    for (int warps_per_smsp : {4, 8}) {
      const int threads = 32 * 4 * warps_per_smsp;
      const int blocks = sms;
      kern<<<blocks, threads>>>(out);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      kern<<<blocks, threads>>>(out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double bf_per_smsp = double(warps_per_smsp) * ITERS * 32;
      const double cycles = ms * 1e-3 * clk * 1e3;
      printf("%-28s warps/SMSP %2d: %.2f cycles per warp-butterfly\n", name, warps_per_smsp,
             cycles / bf_per_smsp);
    }
  };
  auto run_chain = [&](auto kern, const char* name) {
    const int threads = 32 * 4 * 8, blocks = sms;
    kern<<<blocks, threads>>>(out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double steps = 8.0 * ITERS * 32;  // warp-steps per SMSP (8 warps x ITERS x 2 x 16)
    printf("%-28s %.2f cycles per warp-step per SMSP\n", name, ms * 1e-3 * clk * 1e3 / steps);
  };
  run_chain(chain_kernel<ITERS, 0>, "chain IMAD+IMAD.HI");
  run_chain(chain_kernel<ITERS, 1>, "chain IMAD.HI only");
  run_chain(chain_kernel<ITERS, 2>, "chain IMAD only");
  run(mix_kernel<ITERS, 0>, "mix: 2 dependent IADD3");
  run(mix_kernel<ITERS, 1>, "mix: LOP3 + 2 indep IADD3");
  run(mix_kernel<ITERS, 2>, "mix: 1 dependent IADD3");
  run(bf_kernel<ITERS, 0x0>, "umulhi all layers");
  run(bf_kernel<ITERS, 0x2>, "paper 1 of 4 layers");
  run(bf_kernel<ITERS, 0x6>, "paper 2 of 4 layers");
  run(bf_kernel<ITERS, 0xe>, "paper 3 of 4 layers");
  run(bf_kernel<ITERS, 0x1e>, "paper all layers");
  return 0;
}
