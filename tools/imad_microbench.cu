// imad_microbench.cu -- measured integer-multiply issue rates on the local GPU.
//
// The IMAD roofline of the north star ("IMAD ops per butterfly x butterflies") needs the
// per-SM throughput of IMAD / IMAD.HI / IMAD.WIDE on sm_100a, which MEASURED_PEAKS.json
// does not carry.  Each kernel runs 8 independent dependency chains per thread of one
// instruction type, all SMs, 8 warps per SMSP; result = warp-level instructions per
// cycle per SM and lane-ops per second for the chip.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/imad_microbench tools/imad_microbench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

template <int OP>
__global__ void bench(uint32_t* out, uint32_t a, uint32_t b, long long* cycles) {
  uint32_t v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = threadIdx.x + c * 977u;
  const long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (OP == 0) {  // IMAD
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[c]) : "r"(a), "r"(b));
      } else if (OP == 1) {  // IMAD.HI
        asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(v[c]) : "r"(a), "r"(b));
      } else if (OP == 2) {  // IMAD.WIDE (keep the low word in the chain)
        uint64_t w;
        asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w) : "r"(v[c]), "r"(a));
        v[c] = static_cast<uint32_t>(w) ^ static_cast<uint32_t>(w >> 32);
      } else if (OP == 3) {  // IADD3
        asm volatile("add.u32 %0, %0, %1;" : "+r"(v[c]) : "r"(a));
      } else if (OP == 4) {  // LOP3 / shift (alu)
        asm volatile("shr.u32 %0, %0, 1;" : "+r"(v[c]));
        asm volatile("xor.b32 %0, %0, %1;" : "+r"(v[c]) : "r"(b));
      } else if (OP == 6) {  // IDP.2A (dp2a)
        asm volatile("dp2a.lo.u32.u32 %0, %0, %1, %2;" : "+r"(v[c]) : "r"(b), "r"(a));
      } else if (OP >= 7 && OP <= 9) {  // even chains IDP.2A, odd chains IMAD / IMAD.HI / IADD3
        if (c & 1) {
          if (OP == 7) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[c]) : "r"(a), "r"(b));
          if (OP == 8) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(v[c]) : "r"(a), "r"(b));
          if (OP == 9) asm volatile("add.u32 %0, %0, %1;" : "+r"(v[c]) : "r"(a));
        } else {
          asm volatile("dp2a.lo.u32.u32 %0, %0, %1, %2;" : "+r"(v[c]) : "r"(b), "r"(a));
        }
      } else if (OP == 10 || OP == 11) {  // even chains IADD3 (10) / IMAD.HI (11), odd IMAD
        if (c & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[c]) : "r"(a), "r"(b));
        else if (OP == 10) asm volatile("add.u32 %0, %0, %1;" : "+r"(v[c]) : "r"(a));
        else asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(v[c]) : "r"(a), "r"(b));
      } else if (OP == 5) {  // Plantard n=16 tail: IMAD + IMAD.HI + 2 adds (a butterfly)
        uint32_t h = v[c] * a;
        uint32_t r = __umulhi(h, b);
        v[c] = v[c] + r + (v[c] ^ r);
      }
    }
  }
  const long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s ^= v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int instr_per_iter, int sms) {
  const int threads = 1024, blocks = sms;  // 32 warps per SM
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, size_t(threads) * blocks * 4);
  cudaMalloc(&cyc, blocks * 8);
  bench<OP><<<blocks, threads>>>(out, 3u, 5u, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<OP><<<blocks, threads>>>(out, 3u, 5u, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long hc[1024];
  cudaMemcpy(hc, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += hc[i];
  avg /= blocks;
  const double warp_instr_per_sm = double(threads / 32) * kIters * kChains * instr_per_iter;
  const double lane_ops = warp_instr_per_sm * 32 * blocks;
  printf("%-28s warp-instr/clk/SM = %6.3f   lane-ops/s (chip) = %.3e   (%.3f ms, %.0f cyc)\n",
         name, warp_instr_per_sm / avg, lane_ops / (ms * 1e-3), ms, avg);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("SMs=%d  max SM clock=%d MHz\n", sms, clk / 1000);
  run<0>("IMAD (mad.lo.u32)", 1, sms);
  run<1>("IMAD.HI (mad.hi.u32)", 1, sms);
  run<2>("IMAD.WIDE (mul.wide.u32)+LOP", 2, sms);
  run<3>("IADD3 (add.u32)", 1, sms);
  run<4>("SHF+LOP3", 2, sms);
  run<5>("plantard16 bfly (~5 instr)", 5, sms);
  run<6>("IDP.2A (dp2a)", 1, sms);
  run<7>("IDP.2A | IMAD (1:1)", 1, sms);
  run<8>("IDP.2A | IMAD.HI (1:1)", 1, sms);
  run<9>("IDP.2A | IADD3 (1:1)", 1, sms);
  run<10>("IADD3 | IMAD (1:1)", 1, sms);
  run<11>("IMAD.HI | IMAD (1:1)", 1, sms);
  return 0;
}
