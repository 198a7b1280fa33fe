// fp64_microbench.cu -- is the FP64 pipe a second modular-multiply unit on B200?
//
// The N = 256 butterflies are bound by the fmaheavy pipe (IMAD + IMAD.HI per modified-Plantard
// product).  B200 (sm_100a, unlike B300) keeps a full FP64 pipe; an exact double-precision
// modmul (floor via a round-down FMA against 2^52, two exact FMAs) would run beside the
// integer pipes.  Rates per SM per clock, 32 warps/SM, 8 independent chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_mb.bin tools/fp64_microbench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 2048;
constexpr int kChains = 8;

template <int OP>
__global__ void bench(double* outd, uint32_t* outi, double a, double b, uint32_t ia, uint32_t ib) {
  double d[kChains];
  uint32_t v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    d[c] = threadIdx.x + c * 977.0;
    v[c] = threadIdx.x + c * 977u;
  }
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (OP == 0) {  // DFMA
        asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[c]) : "d"(a), "d"(b));
      } else if (OP == 1) {  // DADD
        asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d[c]) : "d"(a));
      } else if (OP == 2) {  // FFMA (fp32)
        float f = __double2float_rn(0.0);
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f) : "f"(1.0f), "f"(2.0f));
        v[c] += __float_as_uint(f);
      } else if (OP == 3) {  // even chains DFMA, odd chains IMAD
        if (c & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[c]) : "r"(ia), "r"(ib));
        else asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[c]) : "d"(a), "d"(b));
      } else if (OP == 4) {  // even chains DFMA, odd chains IMAD.HI
        if (c & 1) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(v[c]) : "r"(ia), "r"(ib));
        else asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[c]) : "d"(a), "d"(b));
      } else if (OP == 5) {  // even chains DFMA, odd chains SHF+LOP (alu)
        if (c & 1) {
          asm volatile("shr.u32 %0, %0, 1;" : "+r"(v[c]));
          asm volatile("xor.b32 %0, %0, %1;" : "+r"(v[c]) : "r"(ib));
        } else {
          asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[c]) : "d"(a), "d"(b));
        }
      } else if (OP == 6) {  // integer improved-n16 butterfly (IMAD + IMAD.HI + 2 adds)
        uint32_t h = v[c] * ia;
        uint32_t r = __umulhi(h, ib);
        asm volatile("" : "+r"(r));
        v[c] = v[c] + r + (v[c] ^ r);
      } else if (OP == 7) {  // fp64 butterfly: 3 DFMA + 3 DADD (chain pairs)
        if (c & 1) continue;
        double x = d[c], y = d[c + 1];
        double qm = __fma_rd(y, a, 4503599627370496.0);
        double nqp = __fma_rn(qm, -3329.0, 4503599627370496.0 * 3329.0);
        double r = __fma_rn(y, b, nqp);
        asm volatile("" : "+d"(r));
        d[c] = x + r;
        d[c + 1] = (x + 3329.0) - r;
      } else if (OP == 8) {  // half the chains the integer butterfly, half the fp64 one
        if (c & 1) {
          uint32_t h = v[c] * ia;
          uint32_t r = __umulhi(h, ib);
          asm volatile("" : "+r"(r));
          v[c] = v[c] + r + (v[c] ^ r);
        } else {
          double x = d[c], y = d[c + 1];
          double qm = __fma_rd(y, a, 4503599627370496.0);
          double nqp = __fma_rn(qm, -3329.0, 4503599627370496.0 * 3329.0);
          double r = __fma_rn(y, b, nqp);
          asm volatile("" : "+d"(r));
          d[c] = x + r;
          d[c + 1] = (x + 3329.0) - r;
        }
      } else if (OP == 9) {  // 3 int butterflies : 1 fp64 butterfly per 4 chains
        if ((c & 3) != 0) {
          uint32_t h = v[c] * ia;
          uint32_t r = __umulhi(h, ib);
          asm volatile("" : "+r"(r));
          v[c] = v[c] + r + (v[c] ^ r);
        } else {
          double x = d[c], y = d[c + 1];
          double qm = __fma_rd(y, a, 4503599627370496.0);
          double nqp = __fma_rn(qm, -3329.0, 4503599627370496.0 * 3329.0);
          double r = __fma_rn(y, b, nqp);
          asm volatile("" : "+d"(r));
          d[c] = x + r;
          d[c + 1] = (x + 3329.0) - r;
        }
      } else if (OP == 10) {  // FP32 FFMA chains mixed with integer butterflies (fmalite use)
        if (c & 1) {
          uint32_t h = v[c] * ia;
          uint32_t r = __umulhi(h, ib);
          asm volatile("" : "+r"(r));
          v[c] = v[c] + r + (v[c] ^ r);
        } else {
          float f = __uint_as_float(v[c]);
          asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f) : "f"(1.0f), "f"(2.0f));
          asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f) : "f"(1.0f), "f"(2.0f));
          v[c] = __float_as_uint(f);
        }
      }
    }
  }
  double sd = 0;
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    sd += d[c];
    s ^= v[c];
  }
  outd[blockIdx.x * blockDim.x + threadIdx.x] = sd;
  outi[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
void run(const char* name, double units_per_iter, const char* unit, int sms) {
  const int threads = 1024, blocks = sms;
  double* od;
  uint32_t* oi;
  cudaMalloc(&od, size_t(threads) * blocks * 8);
  cudaMalloc(&oi, size_t(threads) * blocks * 4);
  bench<OP><<<blocks, threads>>>(od, oi, 1.0000001, 0.5, 3u, 5u);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<OP><<<blocks, threads>>>(od, oi, 1.0000001, 0.5, 3u, 5u);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cyc = ms * 1e-3 * clk * 1e3;
  const double warp_units = double(threads / 32) * kIters * units_per_iter;  // per SM
  printf("%-44s %s/clk/SM = %6.3f   cycles per unit per SMSP = %6.3f  (%.3f ms)\n", name, unit,
         warp_units / cyc, cyc / (warp_units / 4), ms);
  cudaFree(od);
  cudaFree(oi);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs=%d\n", sms);
  run<0>("DFMA", kChains, "warp-instr", sms);
  run<1>("DADD", kChains, "warp-instr", sms);
  run<2>("FFMA", kChains, "warp-instr", sms);
  run<3>("DFMA || IMAD (4+4 chains)", kChains, "warp-instr", sms);
  run<4>("DFMA || IMAD.HI (4+4 chains)", kChains, "warp-instr", sms);
  run<5>("DFMA || SHF+LOP (4 + 2x4)", kChains * 1.5, "warp-instr", sms);
  run<6>("int butterfly (IMAD+IMAD.HI+2 ALU)", kChains, "warp-bfly", sms);
  run<7>("fp64 butterfly (3 DFMA + 3 DADD)", kChains / 2, "warp-bfly", sms);
  run<8>("int || fp64 butterflies (1:1)", kChains, "warp-bfly", sms);
  run<9>("int || fp64 butterflies (3:1)", kChains, "warp-bfly", sms);
  run<10>("int butterfly || 2 FFMA (1:1)", kChains / 2, "warp-bfly(int)", sms);
  return 0;
}
