// bf_forms_microbench.cu -- instruction forms of the n = 16 modified-Plantard CT butterfly
// (x, y, w) -> (x + r, x + p - r), r = MP(w, y), measured in registers with no memory traffic
// (16 values per lane, 4 register-local layers per phase, uniform constant-bank twiddles, as
// in fast256_tma.cu).  Cycles per warp-butterfly per SMSP.
//
//   F0 umulhi        IMAD h; IMAD.HI r; IADD3 x + r; IADD3 x + p - r           (round-1 form)
//   F1 paper+LEA     IMAD h; SHF h >> 16; IMAD R = (h>>16) p + p; LEA.HI s = x + (R >> 16);
//                    IADD3 y' = 2x - s  (= x - r: the true x + p - r minus p; the kernel
//                    carries such offsets as compile-time multiples of p)
//   F2 wide-addend   IMAD h; IMAD.WIDE {lo, s} = h p + {lo_x, x} (s = x + r when the low
//                    words cannot carry); IADD3 y' = 2x - s  (u64 carriers per value)
//   mixes            per-layer choice between forms (mask bit s = layer s uses the 2nd form)
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bff_mb.bin tools/bf_forms_microbench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__constant__ uint32_t c_w[16];
__constant__ uint32_t c_p, c_zero;

__constant__ uint32_t c_two;
template <int FORM>
__device__ __forceinline__ void bf32(uint32_t& x, uint32_t& y, uint32_t w, uint32_t p, uint32_t z) {
  const uint32_t hh = y * w;
  if (FORM == 0) {
    const uint32_t rr = __umulhi(hh, p);
    y = x + p - rr;
    x = x + rr + z;
  } else if (FORM == 1) {
    const uint32_t R = (hh >> 16) * p + p;
    const uint32_t s = x + (R >> 16);
    y = x + x - s;
    x = s;
  } else {  // FORM 3: F1 with Y' = 2X - X' on the FMA pipe (IMAD by an opaque 2)
    const uint32_t R = (hh >> 16) * p + p;
    const uint32_t s = x + (R >> 16);
    uint32_t t;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(x), "r"(c_two), "r"(0u - s));
    y = t;
    x = s;
  }
}

// FORM_A for layers whose bit is clear in MASK, FORM_B otherwise (32-bit forms 0/1)
template <int ITERS, int FORM_A, int FORM_B, int MASK>
__global__ void bf32_kernel(uint32_t* out) {
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
        if ((MASK >> sl) & 1) bf32<FORM_B>(v[r], v[r + h], w, p, z);
        else bf32<FORM_A>(v[r], v[r + h], w, p, z);
      }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] &= 0xffffu;
  }
  uint32_t acc = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) acc ^= v[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// FORM 2 on {lo, value} register pairs (inline PTX mad.wide with a packed 64-bit addend);
// MASK bit s: layer s uses F0 instead.  RESET: zero the low words once per iteration.
__device__ __forceinline__ void madw(uint32_t& lo, uint32_t& hi, uint32_t a, uint32_t b, uint32_t clo,
                                     uint32_t chi) {
  asm("{\n.reg .b64 c, d;\nmov.b64 c, {%2, %3};\nmad.wide.u32 d, %4, %5, c;\nmov.b64 {%0, %1}, d;\n}"
      : "=r"(lo), "=r"(hi)
      : "r"(clo), "r"(chi), "r"(a), "r"(b));
}
template <int ITERS, int MASK, bool RESET>
__global__ void bf64_kernel(uint32_t* out) {
  uint32_t v[16], l[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    v[r] = threadIdx.x * 16 + r + blockIdx.x;
    l[r] = r;
  }
  const uint32_t p = c_p, z = c_zero;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int sl = 1; sl <= 4; ++sl) {
      const int h = 8 >> (sl - 1);
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r & h) continue;
        const uint32_t w = c_w[(1 << (sl - 1)) - 1 + (r >> (5 - sl))];
        const uint32_t x = v[r];
        const uint32_t hh = v[r + h] * w;
        if ((MASK >> sl) & 1) {
          const uint32_t rr = __umulhi(hh, p);
          v[r + h] = x + p - rr;
          v[r] = x + rr + z;
        } else {
          uint32_t s;
          madw(l[r], s, hh, p, l[r], x);
          v[r + h] = x + x - s;
          v[r] = s;
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      v[r] &= 0xffffu;
      if (RESET) l[r] = z;
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) acc ^= v[r] ^ l[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// GS (inverse) forms: (x, y, w) -> (x + y, MP(w, x + off - y)), off a constant-bank word
//   G0 umulhi   IADD3 t; IADD3 x + y; IMAD h; IMAD.HI r; XOR fence (the eager kernel form)
//   G1 paper    IADD3 t; IADD3 x + y; IMAD h; SHF; IMAD (h>>16) p + p; SHF
__constant__ uint32_t c_off;
//   G2 balanced IADD3 t; IMAD x + y (opaque 1); IMAD h; SHF; IMAD; SHF  (3 IMAD + 3 ALU)
__constant__ uint32_t c_one;
template <int FORM>
__device__ __forceinline__ void gs32(uint32_t& x, uint32_t& y, uint32_t w, uint32_t p, uint32_t z) {
  const uint32_t t = x + c_off - y;
  if (FORM == 2) {
    uint32_t s;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(s) : "r"(x), "r"(c_one), "r"(y));
    x = s;
  } else {
    x = x + y + z;
  }
  const uint32_t h = t * w;
  if (FORM == 0) y = __umulhi(h, p) ^ z;
  else y = (((h >> 16) + 1u) * p) >> 16;
}
template <int ITERS, int FORM>
__global__ void gs_kernel(uint32_t* out) {
  uint32_t v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = threadIdx.x * 16 + r;
  const uint32_t p = c_p, z = c_zero;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int sl = 1; sl <= 4; ++sl) {
      const int h = 1 << (sl - 1);
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r & h) continue;
        gs32<FORM>(v[r], v[r + h], c_w[(1 << (sl - 1)) - 1 + (r >> sl)], p, z);
      }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] &= 0xffffu;
  }
  uint32_t acc = 0;
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
  const uint32_t two = 2;
  cudaMemcpyToSymbol(c_two, &two, 4);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* out;
  cudaMalloc(&out, size_t(sms) * 1024 * 64 * 4);
  constexpr int ITERS = 2048;
  auto run = [&](auto kern, const char* name) {
    for (int warps_per_smsp : {4, 6, 8}) {
      const int threads = 32 * 4 * warps_per_smsp;
      kern<<<sms, threads>>>(out);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      kern<<<sms, threads>>>(out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double bf_per_smsp = double(warps_per_smsp) * ITERS * 32;
      printf("%-40s warps/SMSP %d: %.2f cycles per warp-butterfly\n", name, warps_per_smsp,
             ms * 1e-3 * clk * 1e3 / bf_per_smsp);
    }
  };
  run(bf32_kernel<ITERS, 0, 0, 0>, "F0 umulhi (all layers)");
  run(bf32_kernel<ITERS, 1, 1, 0>, "F1 paper+LEA.HI (all layers)");
  run(bf64_kernel<ITERS, 0, false>, "F2 wide-addend (all layers)");
  run(bf64_kernel<ITERS, 0, true>, "F2 wide-addend + low reset");
  run(bf32_kernel<ITERS, 0, 1, 0x2>, "F0, F1 on layer 1");
  run(bf32_kernel<ITERS, 0, 1, 0x6>, "F0, F1 on layers 1-2");
  run(bf32_kernel<ITERS, 0, 1, 0xa>, "F0, F1 on layers 1,3");
  run(bf32_kernel<ITERS, 0, 1, 0xe>, "F0, F1 on layers 1-3");
  run(bf64_kernel<ITERS, 0x2, true>, "F2, F0 on layer 1");
  run(bf64_kernel<ITERS, 0x6, true>, "F2, F0 on layers 1-2");
  const uint32_t off = 2 * p;
  cudaMemcpyToSymbol(c_off, &off, 4);
  run(bf32_kernel<ITERS, 3, 3, 0>, "F3 F1 with IMAD 2X - X' (all layers)");
  run(gs_kernel<ITERS, 0>, "G0 GS umulhi + fence");
  run(gs_kernel<ITERS, 1>, "G1 GS paper form");
  const uint32_t one = 1;
  cudaMemcpyToSymbol(c_one, &one, 4);
  run(gs_kernel<ITERS, 2>, "G2 GS paper form, X + Y as IMAD");
  return 0;
}
