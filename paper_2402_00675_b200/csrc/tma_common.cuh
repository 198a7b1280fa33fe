// tma_common.cuh -- shared pieces of the TMA-fed N = 256 kernels (fast256_tma.cu,
// polymul_tma.cu): stage geometry, mbarrier / bulk-copy wrappers, the proxy-fenced stage
// release, the swizzled transpose tile, and the producer loop.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "arith.cuh"

namespace nttk_b200 {
namespace tma {

constexpr int kConsumers = 8;                 // default consumer warps per CTA
constexpr int kThreads = (kConsumers + 1) * 32;
constexpr int kTile = 2 * kConsumers;          // polynomials per stage
constexpr int kScratchWords = 2 * 272;         // per-warp transpose scratch (u32)

// A stage holds one tile of kTile polynomials as two contiguous halves (one bulk copy
// each: polynomials 0..7 and 8..15 of the tile).  Consumer warp w owns polynomial w of
// the first half and polynomial w of the second; the second half starts kPad bytes
// later so the two polynomials of a warp sit on disjoint bank halves.
// Stage counts per use (DIR 0 forward, 1 inverse, 2 fused polymul).  Fewer bytes in flight
// per SM can be faster: a TMA -> STG copy peaks at 48-64 KiB per SM (tools/copy_probe.cu:
// 6.59 TB/s at 1 CTA x 3 stages vs 6.16 at 3 CTAs x 3 stages).  Measured (B200, 3 CTAs/SM):
// u32 forward 2 stages 0.806 -> 0.776 ms, u16 inverse 2 stages 1.152 -> 1.123 ms; the u16
// forward keeps 4 (2: +1.5 %), the u32 inverse 3 (profiles/r1b_stage_sweep.txt).
template <int DIR, int BYTES>
constexpr int stages_of() {
  return DIR == 0 ? (BYTES == 2 ? 4 : 2) : DIR == 1 ? (BYTES == 2 ? 2 : 3) : (BYTES == 2 ? 4 : 3);
}
// C = consumer warps per CTA (fast256_tma.cu picks it per kernel, see cons_of there)
template <class IO, int DIR = 2, int C = kConsumers>
struct Geo {
  static constexpr int kC = C;
  static constexpr int kTileP = 2 * kC;              // polynomials per stage
  static constexpr int kThreadsP = (kC + 1) * 32;    // + the producer warp
  static constexpr int kPolyBytes = 256 * int(sizeof(IO));
  static constexpr int kPad = sizeof(IO) == 2 ? 32 : 64;
  static constexpr int kHalfBytes = kC * kPolyBytes;
  static constexpr int kStages = stages_of<DIR, int(sizeof(IO))>();
  static constexpr int kStageBytes = 2 * kHalfBytes + kPad + 64;  // keep stages 128B-aligned
  static constexpr int kSmem = kStages * kStageBytes + kC * kScratchWords * 4 + 2 * kStages * 8;
  // byte offset of the polynomial of warp w, half h inside a stage
  __device__ static constexpr int poly_offset(int w, int h) {
    return h * (kHalfBytes + kPad) + w * kPolyBytes;
  }
};

// Inverse kernels on u32 words: the stage is one TMA tensor box of kTile polynomials
// (128-byte rows, SWIZZLE_128B, tensor_map.hpp) instead of two padded linear bulk copies
// (measured: u32 -3.3 %; u16 +0.4 %, so u16 keeps the linear copies).
template <class IO>
constexpr bool inv_swz() {
  return sizeof(IO) == 4;
}

template <class IO, int DIR = 2, int C = kConsumers>
struct GeoSwz {
  using G = Geo<IO, DIR, C>;
  static constexpr int kPolyBytes = 256 * int(sizeof(IO));
  static constexpr int kRowsPerPoly = kPolyBytes / 128;
  static constexpr int kBoxRows = G::kTileP * kRowsPerPoly;  // <= 256
  static constexpr int kStageBytes = kBoxRows * 128;     // multiple of 1024
  static constexpr int kUsed = G::kStages * kStageBytes + G::kC * kScratchWords * 4 + 2 * G::kStages * 8;
  static constexpr int kSmem = kUsed + 1024;  // + alignment slack for the 1024-byte base
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}
// Programmatic dependent launch (launch_cache.hpp launch_pdl): the producer calls pdl_wait()
// before its first global read; init_barriers() signals launch_dependents.  Both are no-ops for
// a launch without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(b))
      : "memory");
}

// 2-D tiled tensor copy global -> shared through a TMA tensor map (tensor_map.hpp): box
// origin (x, y) in elements; the full box is written (rows past the tensor end are
// zero-filled) and counted on the mbarrier.
__device__ __forceinline__ void bulk_tensor_g2s(void* dst, const CUtensorMap* map, int x, int y,
                                                uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_addr(b))
      : "memory");
}

// Byte offset of linear offset L inside a CU_TENSOR_MAP_SWIZZLE_128B destination (1024-byte
// aligned): 16-byte chunk c of 128-byte row r sits at chunk c ^ (r & 7).
__host__ __device__ constexpr uint32_t swz128(uint32_t L) {
  return (L & ~127u) | ((((L >> 4) & 7u) ^ ((L >> 7) & 7u)) << 4);
}

// producer over 128-byte-row tensor boxes: tile t = rows [t NBOX BOX_ROWS, (t+1) NBOX BOX_ROWS),
// NBOX boxes per stage (a box is at most 256 rows)
template <int BOX_ROWS, int STAGES, int NBOX = 1>
__device__ __forceinline__ void produce_rows(const CUtensorMap* map, uint32_t ntiles, uint8_t* stages,
                                             uint64_t* full, uint64_t* empty) {
  constexpr uint32_t kBytes = BOX_ROWS * 128;
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
  pdl_wait();
  uint32_t s = 0, phase = 0, k = 0;
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    if (k >= uint32_t(STAGES)) mbar_wait(&empty[s], phase ^ 1);
    mbar_expect_tx(&full[s], NBOX * kBytes);
#pragma unroll
    for (int b = 0; b < NBOX; ++b)
      bulk_tensor_g2s(stages + (s * NBOX + b) * kBytes, map, 0, int((t * NBOX + b) * BOX_ROWS), &full[s]);
    if (++s == uint32_t(STAGES)) {
      s = 0;
      phase ^= 1;
    }
  }
}

// Hand a consumed stage back to the producer.  The stage was read through the generic
// proxy (LDS) and will be overwritten by the async proxy (the next bulk copy): the
// proxy fence orders this warp's reads before the refill (WAR across proxies), the
// warp barrier collects all lanes, one lane arrives.
__device__ __forceinline__ void release_stage(uint64_t* empty, int lane) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // tools/stress_fwd.py
  __syncwarp();
  if (lane == 0) mbar_arrive(empty);
}

__device__ __forceinline__ int swz(int i) {
  return (i & ~15) | ((((i >> 2) & 3) ^ ((i >> 5) & 3)) << 2) | (i & 3);
}

// Per-lane shared-window addresses into a half-warp's 272-word transpose tile, hoisted
// out of the loop (32-bit registers + immediate offsets: no address IMADs per access).
// Element i = j + 16 r (strided ownership, lane j) lives at word swz(i) = 16 r + (j ^ 4m),
// m = (r >> 1) & 3; chunk c of row j (contiguous ownership) at 16 j + 4 (c ^ ((j>>1)&3)).
struct Xpose {
  uint32_t sp[4], cp[4];
  __device__ __forceinline__ void init(const uint32_t* tile, int j) {
    const uint32_t b = smem_addr(tile);
#pragma unroll
    for (int m = 0; m < 4; ++m) sp[m] = b + 4u * uint32_t(j ^ (4 * m));
    const int g = (j >> 1) & 3;
#pragma unroll
    for (int c = 0; c < 4; ++c) cp[c] = b + 64u * j + 16u * uint32_t(c ^ g);
  }
  __device__ __forceinline__ void put(int r, uint32_t v) const {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(sp[(r >> 1) & 3] + 64u * r), "r"(v) : "memory");
  }
  __device__ __forceinline__ uint32_t get(int r) const {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(sp[(r >> 1) & 3] + 64u * r) : "memory");
    return v;
  }
  __device__ __forceinline__ void put4(int c, uint32_t a, uint32_t b, uint32_t d, uint32_t e) const {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(cp[c]), "r"(a), "r"(b), "r"(d),
                 "r"(e)
                 : "memory");
  }
  __device__ __forceinline__ void get4(int c, uint32_t& a, uint32_t& b, uint32_t& d,
                                       uint32_t& e) const {
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(d), "=r"(e)
                 : "r"(cp[c])
                 : "memory");
  }
};

template <class T>
__device__ __forceinline__ T pin(T x) {  // opaque copy: value lives in registers
  if constexpr (sizeof(T) == 4) {
    asm volatile("mov.b32 %0, %0;" : "+r"(x));
  } else {
    asm volatile("mov.b32 %0, %0;" : "+r"(x.x));
    asm volatile("mov.b32 %0, %0;" : "+r"(x.y));
  }
  return x;
}

template <class IO, bool SGN>
__device__ __forceinline__ uint32_t widen(IO x) {
  if constexpr (sizeof(IO) == 2)
    return SGN ? static_cast<uint32_t>(static_cast<int32_t>(static_cast<int16_t>(x))) : uint32_t(x);
  else
    return x;
}

// canonical residue of a loaded coefficient (transform.hpp:38-40,243)
// FAST (host-validated, A.flags bits 0/1): Barrett for u16, shift reduction for u32
template <class IO, bool SGN, bool FAST>
__device__ __forceinline__ uint32_t canon(uint32_t x, const FastArgs& A) {
  if (SGN) return mod_s32(x, A);
  if constexpr (sizeof(IO) == 2) return FAST ? mod_cb(x, A) : mod_u16(x, A);
  return FAST ? mod_cs(x, A) : mod_u32(x, A);
}

// Minimum CTAs per SM for the forward's register allocator (shared memory admits 4 for u16
// and 3 for u32 stages).  Measured on B200: capping the u32 forward to 3 CTAs (72 regs, was
// 2 CTAs at 92) is 3.5% faster; the same cap on the u32 inverse is 1.7% slower and capping
// the u16 kernels to 4 CTAs (56 regs) is 2-6% slower.  Lane twiddles stay in registers:
// staging them in shared memory (fewer registers, more CTAs) measured slower everywhere
// (u32 inverse 1.032 -> 1.050 ms at 3 CTAs/SM): these kernels are bound by FMA/ALU pipe
// scheduling, not by occupancy.
template <class IO>
constexpr int fwd_minb() {
  return sizeof(IO) == 4 ? 3 : 1;
}

// Lane-dependent twiddles read from shared memory (the fused polymul keeps both directions'
// tables there): entry i of lane j at S[16 i + j] -- consecutive lanes, consecutive words,
// the two half-warps broadcast.
template <class Tw>
struct TwSmem {
  const Tw* base;  // S + j
  __device__ __forceinline__ Tw operator[](int i) const { return base[16 * i]; }
};

// producer: stream tiles of kTile polynomials into the stage ring
template <class IO, int DIR = 2, int C = kConsumers>
__device__ __forceinline__ void produce(const IO* in, size_t batch, uint8_t* stages, uint64_t* full,
                                        uint64_t* empty) {
  using G = Geo<IO, DIR, C>;
  constexpr int kTile = G::kTileP, kConsumers = G::kC;
  const size_t ntiles = (batch + kTile - 1) / kTile;
  int k = 0;
  pdl_wait();
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int s = k % G::kStages;
    if (k >= G::kStages) mbar_wait(&empty[s], ((k / G::kStages) & 1) ^ 1);
    const size_t first = t * kTile;
    const int n = batch - first < size_t(kTile) ? int(batch - first) : kTile;
    const int n0 = n < kConsumers ? n : kConsumers, n1 = n - n0;
    mbar_expect_tx(&full[s], uint32_t(n) * G::kPolyBytes);
    uint8_t* base = stages + s * G::kStageBytes;
    bulk_g2s(base, in + first * 256, uint32_t(n0) * G::kPolyBytes, &full[s]);
    if (n1 > 0)
      bulk_g2s(base + G::poly_offset(0, 1), in + (first + kConsumers) * 256,
               uint32_t(n1) * G::kPolyBytes, &full[s]);
  }
}



// ---------------------------------------------------------------------------
// Transform bodies shared by the standalone and the fused kernels.  A half-warp owns one
// polynomial, lane j holds 16 coefficients in v[]:
//   strided ownership     v[r] = a[j + 16 r]   (index bits 7..4 in the register index)
//   contiguous ownership  v[r] = a[16 j + r]   (index bits 3..0 in the register index)

// lane-dependent twiddles of the forward transform (pinned in registers)
template <class K, int L, bool PER_INDEX>
__device__ __forceinline__ void fwd_twiddles(typename K::Tw (&twl)[15], const FastArgs& A, int j) {
  if (PER_INDEX) {  // DIF per-index schedule, phase 1: j_index = j + 16 (r mod len/16)
#pragma unroll
    for (int r = 0; r < 8; ++r) twl[r] = pin(K::tw(A, 0 + j + 16 * r));
#pragma unroll
    for (int r = 0; r < 4; ++r) twl[8 + r] = pin(K::tw(A, 128 + j + 16 * r));
#pragma unroll
    for (int r = 0; r < 2; ++r) twl[12 + r] = pin(K::tw(A, 192 + j + 16 * r));
    twl[14] = pin(K::tw(A, 224 + j));
  } else {  // CT per-block schedule, phase 2: block = j 2^{s-5} + (r >> (9 - s))
    twl[0] = pin(K::tw(A, 15 + j));
#pragma unroll
    for (int q = 0; q < 2; ++q) twl[1 + q] = pin(K::tw(A, 31 + 2 * j + q));
#pragma unroll
    for (int q = 0; q < 4; ++q) twl[3 + q] = pin(K::tw(A, 63 + 4 * j + q));
    if (L >= 8) {
#pragma unroll
      for (int q = 0; q < 8; ++q) twl[7 + q] = pin(K::tw(A, 127 + 8 * j + q));
    }
  }
}

// lane-dependent twiddles of the inverse transform (merge-order table, phase 1)
template <class K, int L>
__device__ __forceinline__ void inv_twiddles(typename K::Tw (&twl)[15], const FastArgs& A, int j) {
  constexpr int TL = 1 << L;
  twl[0] = pin(K::tw(A, TL - 32 + j));
#pragma unroll
  for (int q = 0; q < 2; ++q) twl[1 + q] = pin(K::tw(A, TL - 64 + 2 * j + q));
#pragma unroll
  for (int q = 0; q < 4; ++q) twl[3 + q] = pin(K::tw(A, TL - 128 + 4 * j + q));
  if (L >= 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) twl[7 + q] = pin(K::tw(A, TL - 256 + 8 * j + q));
  }
}

// Forward layers whose block-0 product is multiply-free (1..4).  Measured: 2 is best for
// Kyber (0.996 ms vs 1.014 at 3 or 4 -- the extra min ops and the changed schedule cost
// more than the 3 saved multiplies); Dilithium is flat within noise.
constexpr int kW1Layers = 2;

// run_split_layers (transform.hpp:77-96): strided in -> contiguous out.
// W1 (A.flags bit 4, improved kinds on the cyclic tree): block 0 of layers 1..4 has
// twiddle omega^0 = 1 and inputs below s p, so its Plantard product is a canonical
// reduction without a multiply (fwd_w1); input coefficients must be canonical (the
// ntt_forward contract).
template <class K, int L, bool PER_INDEX, bool W1 = false, class TWL>
__device__ __forceinline__ void fwd_body(uint32_t (&v)[16], const TWL& twl, const FastArgs& A,
                                         const Xpose& X) {
  using Tw = typename K::Tw;
#pragma unroll
  for (int sl = 1; sl <= 4; ++sl) {  // phase 1: layers 1..4
    const int h = 8 >> (sl - 1);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & h) continue;
      if constexpr (W1 && !PER_INDEX) {
        if (sl <= kW1Layers && (r >> (5 - sl)) == 0) {
          K::fwd_w1(v[r], v[r + h], sl, A);
          continue;
        }
      }
      Tw w;
      if (PER_INDEX) {
        const int base = sl == 1 ? 0 : sl == 2 ? 8 : sl == 3 ? 12 : 14;
        w = twl[base + (r & (h - 1))];
      } else {
        w = K::tw(A, (1 << (sl - 1)) - 1 + (r >> (5 - sl)));
      }
      K::fwd(v[r], v[r + h], w, A);
    }
  }
  __syncwarp();  // the tile is free (previous readers done)
#pragma unroll
  for (int r = 0; r < 16; ++r) X.put(r, v[r]);
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 4; ++c) X.get4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
#pragma unroll
  for (int sl = 5; sl <= 8; ++sl) {  // phase 2: layers 5..L
    if (sl > L) break;
    const int h = 1 << (8 - sl);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & h) continue;
      Tw w;
      if (PER_INDEX) {
        w = K::tw(A, 256 - (1 << (9 - sl)) + (r & (h - 1)));
      } else {
        const int base = sl == 5 ? 0 : sl == 6 ? 1 : sl == 7 ? 3 : 7;
        w = twl[base + (r >> (9 - sl))];
      }
      K::fwd(v[r], v[r + h], w, A);
    }
  }
}

// F1 forward (ImprovedN16, cyclic L = 8 with the W1 blocks, A.flags bit 10).  Layers 2..7
// use the paper-form product with the final shift fused into the add:
//   g = (y w_hat mu) >> 16;  R = g p + p;  X' = X + (R >> 16)  (LEA.HI);  Y' = 2X - X'
// i.e. IMAD + SHF + IMAD + LEA.HI + IADD3 (2 fmaheavy + 3 ALU issue slots instead of IMAD +
// IMAD.HI + 2 IADD3: 7.1 vs 7.7 cycles per warp-butterfly in registers,
// profiles/r2_bf_forms_microbench.txt).  Y' = X - r is the reference's X + p - r minus p, so
// every word carries a surplus sigma p (exact mod p, so the products are unchanged): layer 1
// (twiddle 1 everywhere) injects S = kF1Surplus into both outputs for free, each F1 Y-step
// spends one, and an X input always keeps sigma >= 1 (S = 6 covers the 5 F1 layers before
// the last).  Layer 8 runs the umulhi form and subtracts the surplus in its IADD3s: for the
// X position i = 16 j + r of the contiguous phase sigma = S - [i7 & i6] - popcount(i5..i1)
// (block 0 of layer 2 is a W1 block, which spends none) -- a lane part cj and a register
// part; E[m] = (m - cj) p are per-lane registers.  Largest word (9 + S) p, host-validated
// against Prop. 4.  A CPU model of this schedule is checked against the reference loop in
// tests/test_oracle.py.
// IMAD_Y: Y' = 2 X - X' as one IMAD by the opaque constant A.two, so 3 IMAD (fmaheavy) +
// SHF + LEA.HI (ALU) balance the two pipes -- 6.1 cycles per warp-butterfly in registers
// against 7.1 with Y' = X + X - X' as an IADD3 and 7.7 for the umulhi form
// (profiles/r2_bf_forms_microbench.txt).  In the kernels it pays where the ALU pipe is the
// busier one: the N = 256 Kyber forward 0.911 -> 0.879 ms; the N = 512/1024 forwards and the
// fused polymul measured 1.5-3 % slower with it and keep the IADD3 (profiles/r2_f3_ab.txt).
template <bool IMAD_Y = false>
__device__ __forceinline__ void f1_bf(uint32_t& x, uint32_t& y, uint32_t w, const FastArgs& A) {
  const uint32_t R = ((y * w) >> 16) * A.p + A.p;
  const uint32_t s = x + (R >> 16);
  if constexpr (IMAD_Y) {
    uint32_t t;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(x), "r"(A.two), "r"(0u - s));
    y = t;
  } else {
    y = x + x - s;
  }
  x = s;
}

template <class K, class TWL>
__device__ __forceinline__ void fwd_body_f1(uint32_t (&v)[16], const TWL& twl, const FastArgs& A,
                                            const Xpose& X, const uint32_t (&E)[5]) {
  static_assert(kW1Layers == 2, "the surplus schedule assumes W1 blocks on layers 1-2");
#pragma unroll
  for (int r = 0; r < 8; ++r) {  // layer 1: one block, twiddle 1, r = Y (canonical input)
    const uint32_t x = v[r], y = v[r + 8];
    v[r] = x + y + A.f1_sp;
    v[r + 8] = x + A.f1_sp1 - y;
  }
#pragma unroll
  for (int sl = 2; sl <= 4; ++sl) {  // layers 2..4 (strided phase)
    const int h = 8 >> (sl - 1);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & h) continue;
      const int blk = r >> (5 - sl);
      if (sl == 2 && blk == 0) {  // W1 block: canonical residue of Y = y_ref + S p (< (2 + S) p)
        uint32_t c = v[r + h] - A.f1_sp;
        c = umin32(c, c - A.p);
        const uint32_t x = v[r];
        v[r + h] = x + A.p - c;
        v[r] = x + c + A.zero;
        continue;
      }
      f1_bf<true>(v[r], v[r + h], K::tw(A, (1 << (sl - 1)) - 1 + blk), A);
    }
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 16; ++r) X.put(r, v[r]);
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 4; ++c) X.get4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
#pragma unroll
  for (int sl = 5; sl <= 7; ++sl) {  // layers 5..7 (contiguous phase)
    const int h = 1 << (8 - sl);
    const int base = sl == 5 ? 0 : sl == 6 ? 1 : 3;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & h) continue;
      f1_bf<true>(v[r], v[r + h], twl[base + (r >> (9 - sl))], A);
    }
  }
#pragma unroll
  for (int r = 0; r < 16; r += 2) {  // layer 8: umulhi form, surplus removed
    const int k = ((r >> 1) & 1) + ((r >> 2) & 1) + ((r >> 3) & 1);
    const uint32_t rr = mp_n16<false>(v[r + 1], twl[7 + (r >> 1)], A.p);
    const uint32_t x = v[r];
    v[r + 1] = x - rr + E[k + 1];
    v[r] = x + rr + E[k];
  }
}

// F1 forward of the 7-layer negacyclic tree (the Kyber NTT, row a22; A.flags bit 10 at L = 7).
// No layer has twiddle 1, so layer 1 runs the umulhi product and injects the surplus S = L - 2 = 5
// inside its two IADD3s, layers 2..6 run the F3 form (each Y-step spends one), and layer 7
// (register distance 2: the tree ends in degree-2 factors) runs the umulhi form and removes
// sigma = S - popcount(i6..i2) of its X position i = 16 j + r: lane part cj = S - popcount(j & 7),
// register part k = r3 + r2, E[m] = (m - cj) p.  Largest word (2 L - 1) p, host-validated.
template <class K, class TWL>
__device__ __forceinline__ void fwd_body_f1_nega7(uint32_t (&v)[16], const TWL& twl, const FastArgs& A,
                                                  const Xpose& X, const uint32_t (&E)[5]) {
#pragma unroll
  for (int r = 0; r < 8; ++r) {  // layer 1: one block, umulhi product, surplus injected
    const uint32_t x = v[r], c = mp_n16<false>(v[r + 8], K::tw(A, 0), A.p);
    v[r] = x + c + A.f1_sp;
    v[r + 8] = x + A.f1_sp1 - c;
  }
#pragma unroll
  for (int sl = 2; sl <= 4; ++sl) {  // layers 2..4 (strided phase)
    const int h = 8 >> (sl - 1);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & h) continue;
      f1_bf<true>(v[r], v[r + h], K::tw(A, (1 << (sl - 1)) - 1 + (r >> (5 - sl))), A);
    }
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 16; ++r) X.put(r, v[r]);
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 4; ++c) X.get4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
#pragma unroll
  for (int sl = 5; sl <= 6; ++sl) {  // layers 5, 6 (contiguous phase)
    const int h = 1 << (8 - sl);
    const int base = sl == 5 ? 0 : 1;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & h) continue;
      f1_bf<true>(v[r], v[r + h], twl[base + (r >> (9 - sl))], A);
    }
  }
#pragma unroll
  for (int r = 0; r < 16; ++r) {  // layer 7: umulhi form, surplus removed
    if (r & 2) continue;
    const int k = ((r >> 2) & 1) + ((r >> 3) & 1);
    const uint32_t rr = mp_n16<false>(v[r + 2], twl[3 + (r >> 2)], A.p);
    const uint32_t x = v[r];
    v[r + 2] = x - rr + E[k + 1];
    v[r] = x + rr + E[k];
  }
}

// F1 forward whose words are free (the fused polymul: only its canonical product is pinned):
// the same paper-form layers as fwd_body_f1 on every layer after the first, no final
// correction -- outputs are exact mod p, below (L + 1 + S) p with S = L - 1 (host-validated,
// ProdArgs::lazy).  Layer 1 injects the surplus (W1 block on the cyclic tree, umulhi product
// on the negacyclic one); block 0 of layer 2 keeps its W1 form on the cyclic tree.
template <class K, int L, bool W1, class TWL>
__device__ __forceinline__ void fwd_body_f1_free(uint32_t (&v)[16], const TWL& twl, const FastArgs& A,
                                                 const Xpose& X, uint32_t sp, uint32_t sp1) {
#pragma unroll
  for (int r = 0; r < 8; ++r) {  // layer 1: one block
    const uint32_t x = v[r], y = v[r + 8];
    const uint32_t c = W1 ? y : mp_n16<false>(y, K::tw(A, 0), A.p);
    v[r] = x + c + sp;
    v[r + 8] = x + sp1 - c;
  }
#pragma unroll
  for (int sl = 2; sl <= 4; ++sl) {
    const int h = 8 >> (sl - 1);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & h) continue;
      const int blk = r >> (5 - sl);
      if (W1 && sl == 2 && blk == 0) {
        uint32_t c = v[r + h] - sp;
        c = umin32(c, c - A.p);
        const uint32_t x = v[r];
        v[r + h] = x + A.p - c;
        v[r] = x + c + A.zero;
        continue;
      }
      f1_bf(v[r], v[r + h], K::tw(A, (1 << (sl - 1)) - 1 + blk), A);
    }
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 16; ++r) X.put(r, v[r]);
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 4; ++c) X.get4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
#pragma unroll
  for (int sl = 5; sl <= L; ++sl) {
    const int h = 1 << (8 - sl);
    const int base = sl == 5 ? 0 : sl == 6 ? 1 : sl == 7 ? 3 : 7;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & h) continue;
      f1_bf(v[r], v[r + h], twl[base + (r >> (9 - sl))], A);
    }
  }
}

template <class K, class = void>
struct lazy_of {
  static constexpr bool value = false;
};
template <class K>
struct lazy_of<K, std::void_t<decltype(K::kLazy)>> {
  static constexpr bool value = K::kLazy;
};

template <class K, class = void>
struct w1_of {
  static constexpr bool value = false;
};
template <class K>
struct w1_of<K, std::void_t<decltype(&K::fwd_w1)>> {
  static constexpr bool value = true;
};

// inv_body with lazy merge outputs (policy kLazy, see ImprovedN16::inv_hh): after a merge
// layer of half-span h the words at (r & h) hold pre-quotient h-values; the next layer
// (span 2h) pairs them with each other, so "both inputs lazy" is the compile-time test
// r & (h_prev).  Lazy words are materialised before the transpose.
//
// The inverse output is canonical (hence unique), so its intermediate words are free as
// long as every value stays exact mod p inside the multiplies' valid ranges.  Two
// host-validated options use that freedom:
//   TW1   (A.flags bit 5, cyclic tree, L = 8): block 0 of merge layers len = 16, 32, 64
//         has twiddle omega^0 = 1, so Y' = X + off - Y is kept unreduced instead of
//         MP(1^, T) -- 7 of the 72 products per lane disappear.  Every value of merge
//         depth d stays < 2^d p (T < X + off with off = 2^{d-1} p), the standard bound.
//   DEFER (A.flags bit 6, u16 input, improved n = 16, L = 8): no input canonicalisation.
//         Raw words (< 2^16) flow through phase 1; only the "sum chain" (the positions
//         whose X input is a sum of 2^m raw words: r & (h - 1) == 0) needs the larger
//         offset h K p (A.skp), and its single survivor v[0] (< 16 (2^16 - 1)) is reduced
//         with one Plantard product by 1^ before the transpose.  Replaces 8 Barrett
//         reductions per lane by one product.
// Phase 2 tracks which words are lazy at compile time (lz[], constant-folded by the full
// unroll): TW1 outputs are materialised, and a pair with one lazy word materialises it.
// PACKED (DEFER only): the caller leaves the 8 raw packed u16 words of the lane in v[8..15];
// the first merge layer pairs the two halves of one word, so X + Y and X + Kp - Y come from
// two dp2a dot products (IDP.2A) with byte vectors (1, 1) and (1, -1) instead of two
// unpack ops and two adds.
// OSH = 1: inputs only partially reduced to [0, 2p) (u32 inverse, A.flags bit 7), every
// bound doubles, so merge depth d takes the offset of depth d + 1.
template <class K, int L, bool FUSE, bool TW1 = false, bool DEFER = false, bool PACKED = false,
          int OSH = 0, class TWL>
__device__ __forceinline__ void inv_body_lazy(uint32_t (&v)[16], const TWL& twl, const FastArgs& A,
                                              const Xpose& X) {
  using Tw = typename K::Tw;
  constexpr int TL = 1 << L;
  static_assert(!DEFER || (FUSE && L == 8), "DEFER needs the fused u16 first layer at L = 8");
  static_assert(!TW1 || L == 8, "TW1 needs the full 8-layer tree");
#pragma unroll
  for (int sl = 8; sl >= 5; --sl) {  // phase 1: merge layers s = L..5
    if (sl > L) continue;
    const int h = 1 << (8 - sl);
    const uint32_t off = A.off[L - sl + 1 + OSH];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & h) continue;
      const int base = sl == 5 ? 0 : sl == 6 ? 1 : sl == 7 ? 3 : 7;
      const Tw w = twl[base + (r >> (9 - sl))];
      if (sl == L) {  // first merge layer: materialised (raw u16 if FUSE) inputs
        if constexpr (PACKED) {
          static_assert(DEFER, "PACKED input needs DEFER");
          const uint32_t pw = v[8 + r / 2];
          uint32_t sum, dif;
          asm("dp2a.lo.u32.u32 %0, %1, %2, %3;" : "=r"(sum) : "r"(pw), "r"(0x0101u), "r"(0u));
          asm("dp2a.lo.u32.s32 %0, %1, %2, %3;" : "=r"(dif) : "r"(pw), "r"(0xff01u), "r"(A.kp));
          v[r] = sum;
          v[r + h] = dif * w;
          continue;
        }
        const uint32_t x = v[r], y = v[r + h];
        if constexpr (DEFER) {
          v[r] = x + y + A.zero;
          v[r + h] = (x + A.kp - y) * w;
        } else if constexpr (FUSE) {
          v[r] = mod_cb(x + y + A.zero, A);
          v[r + h] = (x + A.kp - y) * w;
        } else {
          K::inv_h(v[r], v[r + h], w, off, A);
        }
      } else if (r & (h >> 1)) {
        K::inv_hh(v[r], v[r + h], w, off, A);
      } else if (DEFER && (r & (h - 1)) == 0) {  // sum chain: inputs < h (2^16 - 1)
        K::inv_h(v[r], v[r + h], w, A.skp[sl == 7 ? 1 : sl == 6 ? 2 : 3], A);
      } else {
        K::inv_h(v[r], v[r + h], w, off, A);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 16; ++r)
    if (r & 8) v[r] = K::materialize(v[r], A);
  if constexpr (DEFER) v[0] = __umulhi(v[0] * A.one_lo, A.p);  // MP(1^, v0): canonical
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 4; ++c) X.put4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = X.get(r);
  bool lz[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) lz[r] = false;
#pragma unroll
  for (int sl = 4; sl >= 1; --sl) {  // phase 2: merge layers s = 4..1, materialised start
    const int h = 1 << (4 - sl);
    const uint32_t off = A.off[L - sl + 1 + OSH];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & h) continue;
      bool lx = lz[r], ly = lz[r + h];
      if (lx != ly) {  // mixed pair (after a TW1 block): materialise the lazy word
        if (lx) v[r] = K::materialize(v[r], A);
        else v[r + h] = K::materialize(v[r + h], A);
        lx = ly = false;
      }
      if (sl == 1) {  // N^{-1} folded into the last merge layer
        if (lx) K::inv_last_hh(v[r], v[r + h], off, A);
        else K::inv_last(v[r], v[r + h], off, A);
        lz[r] = lz[r + h] = false;
      } else if (TW1 && (r >> (5 - sl)) == 0) {  // twiddle 1: Y' = T unreduced
        uint32_t x = v[r], y = v[r + h];
        if (lx) {
          uint32_t Xm;
          const uint32_t S = K::sum_hh(x, y, Xm, A);
          v[r] = S;
          v[r + h] = Xm + Xm + off - S + A.zero;
        } else {
          v[r] = x + y + A.zero;
          v[r + h] = x + off - y;
        }
        lz[r] = lz[r + h] = false;
      } else {
        const Tw w = K::tw(A, TL - (2 << (sl - 1)) + (r >> (5 - sl)));
        if (lx) K::inv_hh(v[r], v[r + h], w, off, A);
        else K::inv_h(v[r], v[r + h], w, off, A);
        lz[r] = false;
        lz[r + h] = true;
      }
    }
  }
}

// run_merge_layers + final N^{-1} (transform.hpp:99-116, 323-335): contiguous in
// (canonical unless FUSE) -> strided out (canonical).  FUSE: u16 raw input, fused first
// merge layer (A.flags bit 2, improved n = 16 only).
// TW1 (policies with inv_w1: harvey, ntl; A.flags bit 5): phase-2 block-0 merges without
// a product, as in inv_body_lazy.
template <class K, class = void>
struct inv_w1_of {
  static constexpr bool value = false;
};
template <class K>
struct inv_w1_of<K, std::void_t<decltype(&K::inv_w1)>> {
  static constexpr bool value = true;
};

template <class K, int L, bool FUSE, bool TW1 = false, class TWL>
__device__ __forceinline__ void inv_body_eager(uint32_t (&v)[16], const TWL& twl, const FastArgs& A,
                                               const Xpose& X) {
  using Tw = typename K::Tw;
  constexpr int TL = 1 << L;
#pragma unroll
  for (int sl = 8; sl >= 5; --sl) {  // phase 1: merge layers s = L..5
    if (sl > L) continue;
    const int h = 1 << (8 - sl);
    const uint32_t off = A.off[L - sl + 1];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & h) continue;
      const int base = sl == 5 ? 0 : sl == 6 ? 1 : sl == 7 ? 3 : 7;
      const Tw w = twl[base + (r >> (9 - sl))];
      if constexpr (FUSE) {
        if (sl == L) {
          const uint32_t x = v[r], y = v[r + h];
          v[r] = mod_cb(x + y + A.zero, A);
          v[r + h] = fence_val(mp_n16<false>(x + A.kp - y, w, A.p), A);
          continue;
        }
      }
      K::inv(v[r], v[r + h], w, off, A);
    }
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 4; ++c) X.put4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = X.get(r);
#pragma unroll
  for (int sl = 4; sl >= 1; --sl) {  // phase 2: merge layers s = 4..1
    const int h = 1 << (4 - sl);
    const uint32_t off = A.off[L - sl + 1];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & h) continue;
      if (K::kFold && sl == 1) {  // N^{-1} folded into the last merge layer
        K::inv_last(v[r], v[r + h], off, A);
      } else if constexpr (TW1) {
        static_assert(inv_w1_of<K>::value && L == 8, "TW1 needs inv_w1 and the 8-layer tree");
        if ((r >> (5 - sl)) == 0) K::inv_w1(v[r], v[r + h], A);
        else K::inv(v[r], v[r + h], K::tw(A, TL - (2 << (sl - 1)) + (r >> (5 - sl))), off, A);
      } else
        K::inv(v[r], v[r + h], K::tw(A, TL - (2 << (sl - 1)) + (r >> (5 - sl))), off, A);
    }
  }
  if (!K::kFold) {
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = K::scale(v[r], A);
  }
}

// Narrow inverse (HostParams::narrow[1]: ImprovedN16 on an n = 32 improved parameter set,
// e.g. the paper's Table 2 presets).  The inverse output is canonical, so its words are free,
// but every GS operand must stay inside n = 16's Prop. 4 range W T < 2^16 (2^16 - p), i.e.
// T < 2^EMAX p (host-validated, FastArgs::flags bit 9 with EMAX = kNarrowEmax).  e[]
// (compile-time after the unroll) is the bound exponent of each register's word (word <
// 2^e p): X' = X + Y < 2^{max e + 1} p, Y' = MP(w, T) is canonical; the GS offset is
// 2^{max e} p >= Y.  A butterfly that would exceed 2^EMAX p first reduces its inputs with one
// Plantard product by 1^ (canonical).  Words are reduced before the transpose, so phase 2
// starts canonical and its e[] stays compile-time.

// Butterflies of the narrow inverse: paper-form products (IMAD + SHF + IMAD + SHF) and X + Y as
// an IMAD by the opaque A.one, so the fmaheavy and ALU pipes carry 3 + 3 slots (G2 in
// profiles/r2_bf_forms_microbench.txt: 6.7 cycles per warp-butterfly in registers against 8.9
// for the eager umulhi form with its fence).  Measured (profiles/r2_narrow_form_ab.txt):
// newhope512 inverse 0.879 -> 0.786, newhope1024 1.755 -> 1.662, kyber256 0.415 -> 0.405
// ns/poly.  The words are free (canonical output), every product operand stays in Prop. 4's
// range by the bound exponents below.
template <class K>
__device__ __forceinline__ void narrow_bf(uint32_t& x, uint32_t& y, int& ex, int& ey,
                                          typename K::Tw w, bool last, const FastArgs& A) {
  int em = ex > ey ? ex : ey;
  if (em + 1 > kNarrowEmax) {
    if (ex) x = K::canon1(x, A);
    if (ey) y = K::canon1(y, A);
    em = 0;
  }
  const uint32_t t = x + A.off[em + 1] - y;
  uint32_t s;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(s) : "r"(x), "r"(A.one), "r"(y));
  if (last) {  // N^{-1} folded: (MP(n^, X + Y), MP((w N^{-1})^, T)), both canonical
    x = mp_n16<true>(s, A.scale_lo, A.p);
    y = mp_n16<true>(t, A.fold_lo, A.p);
  } else {
    x = s;
    y = mp_n16<true>(t, w, A.p);
  }
  ex = em + 1;
  ey = 0;
}

template <class K, int L, class TWL>
__device__ __forceinline__ void inv_body_narrow(uint32_t (&v)[16], const TWL& twl, const FastArgs& A,
                                                const Xpose& X) {
  using Tw = typename K::Tw;
  constexpr int TL = 1 << L;
  int e[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) e[r] = 0;
#pragma unroll
  for (int sl = 8; sl >= 5; --sl) {  // phase 1: merge layers s = L..5
    if (sl > L) continue;
    const int h = 1 << (8 - sl);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & h) continue;
      const int base = sl == 5 ? 0 : sl == 6 ? 1 : sl == 7 ? 3 : 7;
      narrow_bf<K>(v[r], v[r + h], e[r], e[r + h], twl[base + (r >> (9 - sl))], false, A);
    }
  }
#pragma unroll
  for (int r = 0; r < 16; ++r)
    if (e[r]) v[r] = K::canon1(v[r], A);
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 4; ++c) X.put4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    v[r] = X.get(r);
    e[r] = 0;
  }
#pragma unroll
  for (int sl = 4; sl >= 1; --sl) {  // phase 2: merge layers s = 4..1, N^{-1} folded into s = 1
    const int h = 1 << (4 - sl);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & h) continue;
      const Tw w = sl == 1 ? Tw{} : K::tw(A, TL - (2 << (sl - 1)) + (r >> (5 - sl)));
      narrow_bf<K>(v[r], v[r + h], e[r], e[r + h], w, sl == 1, A);
    }
  }
}

// CT-form inverse (HostParams::fast_ctinv, A.flags bit 11; params.cpp fill_ct_inverse has the
// derivation and the bound checks).  Radix-2 DIT on the bit-reversed spectrum with omega^{-1}:
// contiguous phase len = 1, 2, 4, 8 (uniform twiddles A.lo[(128 / len) jb], the jb = 0
// butterfly of every block multiply-free with the host's offsets A.ct_c), transpose, strided
// phase len = 16, 32, 64 (lane twiddles), then len = 128 with N^{-1} folded into two Plantard
// products per butterfly and a min to the canonical residue.  Raw packed u16 words in v[8..15]
// (the first layer pairs the halves of one word: dp2a).  Products: F1 with the IADD3 Y in the
// contiguous phase, F3 (IMAD Y) in the strided one -- the best of the per-layer masks measured
// (0.939 vs 0.942 ms all-F3, 0.958 all-F1; profiles/r2_ct_inverse_ab.txt).
template <class K>
__device__ __forceinline__ void ct_twiddles(uint32_t (&twl)[15], const FastArgs& A, int j) {
  twl[0] = pin(A.lo[8 * j]);  // len 16: omega^{-8 j}
#pragma unroll
  for (int b = 0; b < 2; ++b) twl[1 + b] = pin(A.lo[4 * (j + 16 * b)]);  // len 32
#pragma unroll
  for (int b = 0; b < 4; ++b) twl[3 + b] = pin(A.lo[2 * (j + 16 * b)]);  // len 64
#pragma unroll
  for (int b = 0; b < 8; ++b) twl[7 + b] = pin(A.lo[128 + j + 16 * b]);  // len 128, N^{-1} folded
}

// PACKED: raw u16 words, two per register in v[8..15]; else canonicalised words in v[0..15] (u32
// storage of an n = 16 set, or the narrow image of an n = 32 set: HostParams::fast_ctinv_c).
template <bool PACKED = true, class TWL>
__device__ __forceinline__ void inv_body_ct(uint32_t (&v)[16], const TWL& twl, const FastArgs& A,
                                            const Xpose& X) {
  if constexpr (PACKED) {
    uint32_t t[16];
#pragma unroll
    for (int m = 0; m < 8; ++m) {  // len 1: positions 2m, 2m + 1 = the halves of word m
      const uint32_t pw = v[8 + m];
      asm("dp2a.lo.u32.u32 %0, %1, %2, %3;" : "=r"(t[2 * m]) : "r"(pw), "r"(0x0101u), "r"(A.ct_c[0]));
      asm("dp2a.lo.u32.s32 %0, %1, %2, %3;" : "=r"(t[2 * m + 1]) : "r"(pw), "r"(0xff01u), "r"(A.ct_c[1]));
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = t[r];
  } else {
#pragma unroll
    for (int m = 0; m < 8; ++m) {  // len 1
      const uint32_t u = v[2 * m], w = v[2 * m + 1];
      v[2 * m] = u + w + A.ct_c[0];
      v[2 * m + 1] = u - w + A.ct_c[1];
    }
  }
#pragma unroll
  for (int li = 1; li <= 3; ++li) {  // len 2, 4, 8
    const int len = 1 << li;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & len) continue;
      const int jb = r & (len - 1);
      if (jb == 0) {
        const uint32_t u = v[r], w = v[r + len];
        v[r] = u + w + A.ct_c[2 * li];
        v[r + len] = u - w + A.ct_c[2 * li + 1];
      } else {
        f1_bf<false>(v[r], v[r + len], A.lo[(128 >> li) * jb], A);  // IADD3 Y (ALU)
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 4; ++c) X.put4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = X.get(r);
#pragma unroll
  for (int h = 1; h <= 4; h *= 2) {  // len 16, 32, 64
    const int base = h == 1 ? 0 : h == 2 ? 1 : 3;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & h) continue;
      f1_bf<true>(v[r], v[r + h], twl[base + (r & (h - 1))], A);  // IMAD Y (fmaheavy)
    }
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {  // len 128: (u + w v) N^{-1}, (u - w v) N^{-1}, canonical
    const uint32_t a = mp_n16<true>(v[r], A.scale_lo, A.p);
    const uint32_t b = mp_n16<true>(v[r + 8], twl[7 + r], A.p);
    const uint32_t s = a + b, d = a + A.p - b;
    v[r] = umin32(s, s - A.p);
    v[r + 8] = umin32(d, d - A.p);
  }
}

// n = 32 twin (Dilithium, u32; params.cpp fill_ct_inverse32): inputs partially reduced to
// [0, 2p), ImprovedN32's umulhi-form products in the CT butterfly (X + r, X + p - r), the
// multiply-free jb = 0 butterflies add A.ct_c[2 li + 1] >= their Y input, N^{-1} folded.
__device__ __forceinline__ void ct_twiddles32(uint2 (&twl)[15], const FastArgs& A, int j) {
  auto tw = [&](int e) { return make_uint2(A.lo[e], A.hi[e]); };
  twl[0] = pin(tw(8 * j));
#pragma unroll
  for (int b = 0; b < 2; ++b) twl[1 + b] = pin(tw(4 * (j + 16 * b)));
#pragma unroll
  for (int b = 0; b < 4; ++b) twl[3 + b] = pin(tw(2 * (j + 16 * b)));
#pragma unroll
  for (int b = 0; b < 8; ++b) twl[7 + b] = pin(tw(128 + j + 16 * b));
}

template <class TWL>
__device__ __forceinline__ void inv_body_ct32(uint32_t (&v)[16], const TWL& twl, const FastArgs& A,
                                              const Xpose& X) {
#pragma unroll
  for (int li = 0; li <= 3; ++li) {  // len 1, 2, 4, 8 (contiguous)
    const int len = 1 << li;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & len) continue;
      const int jb = r & (len - 1);
      if (jb == 0) {
        const uint32_t u = v[r], w = v[r + len];
        v[r] = u + w + A.zero;
        v[r + len] = u + A.ct_c[2 * li + 1] - w;
      } else {
        const int e = (128 >> li) * jb;
        ImprovedN32::fwd(v[r], v[r + len], make_uint2(A.lo[e], A.hi[e]), A);
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 4; ++c) X.put4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = X.get(r);
#pragma unroll
  for (int h = 1; h <= 4; h *= 2) {  // len 16, 32, 64 (strided)
    const int base = h == 1 ? 0 : h == 2 ? 1 : 3;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & h) continue;
      ImprovedN32::fwd(v[r], v[r + h], twl[base + (r & (h - 1))], A);
    }
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {  // len 128, N^{-1} folded
    const uint32_t a = mp_n32(v[r], A.scale_lo, A.scale_hi, A.p);
    const uint32_t b = mp_n32(v[r + 8], twl[7 + r].x, twl[7 + r].y, A.p);
    const uint32_t s = a + b, d = a + A.p - b;
    v[r] = umin32(s, s - A.p);
    v[r + 8] = umin32(d, d - A.p);
  }
}

// LAZY: inv_body_lazy (policy kLazy, host-validated A.flags bit 3); TW1 / DEFER: see there.
template <class K, int L, bool FUSE, bool LAZY = false, bool TW1 = false, bool DEFER = false,
          bool PACKED = false, int OSH = 0, class TWL>
__device__ __forceinline__ void inv_body(uint32_t (&v)[16], const TWL& twl, const FastArgs& A,
                                         const Xpose& X) {
  if constexpr (LAZY) {
    static_assert(lazy_of<K>::value, "policy has no lazy merge");
    inv_body_lazy<K, L, FUSE, TW1, DEFER, PACKED, OSH>(v, twl, A, X);
  } else {
    static_assert(OSH == 0, "partial canonicalisation needs the lazy body");
    inv_body_eager<K, L, FUSE, TW1>(v, twl, A, X);
  }
}

// stores
// AL32 (u16): the output is 32-byte aligned, so a lane's 16 coefficients leave in one 256-bit
// store (STG.256, one full sector per lane) instead of two 128-bit stores of half a sector each
template <class IO>
__device__ __forceinline__ void store_contiguous(IO* out_poly, int j, const uint32_t (&v)[16],
                                                 bool al32 = false) {
  if constexpr (sizeof(IO) == 2) {
    if (al32) {
      asm volatile("st.global.cs.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(out_poly + 16 * j),
                   "r"(__byte_perm(v[0], v[1], 0x5410)), "r"(__byte_perm(v[2], v[3], 0x5410)),
                   "r"(__byte_perm(v[4], v[5], 0x5410)), "r"(__byte_perm(v[6], v[7], 0x5410)),
                   "r"(__byte_perm(v[8], v[9], 0x5410)), "r"(__byte_perm(v[10], v[11], 0x5410)),
                   "r"(__byte_perm(v[12], v[13], 0x5410)), "r"(__byte_perm(v[14], v[15], 0x5410))
                   : "memory");
      return;
    }
    uint4* dst = reinterpret_cast<uint4*>(out_poly) + 2 * j;
    uint4 a, b;  // PRMT packs two low halves in one ALU op
    a.x = __byte_perm(v[0], v[1], 0x5410);
    a.y = __byte_perm(v[2], v[3], 0x5410);
    a.z = __byte_perm(v[4], v[5], 0x5410);
    a.w = __byte_perm(v[6], v[7], 0x5410);
    b.x = __byte_perm(v[8], v[9], 0x5410);
    b.y = __byte_perm(v[10], v[11], 0x5410);
    b.z = __byte_perm(v[12], v[13], 0x5410);
    b.w = __byte_perm(v[14], v[15], 0x5410);
    __stcs(dst, a);
    __stcs(dst + 1, b);
  } else {
    uint4* dst = reinterpret_cast<uint4*>(out_poly) + 4 * j;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      __stcs(dst + c, make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]));
  }
}

// u32 contiguous ownership -> coalesced stores through the half-warp's transpose tile: 4
// swizzled 16-byte chunk writes per lane (Xpose::put4), then lane j stores chunks j + 16 k,
// so each store instruction writes 256 contiguous bytes instead of 16 chunks 64 B apart
__device__ __forceinline__ void store_contiguous_coalesced(uint32_t* out_poly, int j, const uint32_t (&v)[16],
                                                           const Xpose& X, const uint32_t* tile,
                                                           bool valid) {
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 4; ++c) X.put4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  __syncwarp();
  if (!valid) return;
  const uint32_t b = smem_addr(tile);
  uint4* dst = reinterpret_cast<uint4*>(out_poly);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int row = (j >> 2) + 4 * k, ch = (j & 3) ^ ((row >> 1) & 3);
    uint4 w;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                 : "r"(b + 64u * row + 16u * ch)
                 : "memory");
    __stcs(dst + j + 16 * k, w);
  }
}

// strided ownership -> coalesced 128-bit stores through the transpose tile
template <class IO>
__device__ __forceinline__ void store_strided(IO* out_poly, int j, const uint32_t (&v)[16],
                                              const uint32_t* S, const Xpose& X, bool valid) {
  if constexpr (sizeof(IO) == 2) {
    // u16 tile in natural order: 16 scalar 16-bit stores (two lanes share a word, one
    // wavefront), then each lane reads two packed 16-byte vectors -- no pack ops, and
    // consecutive lanes read consecutive chunks (conflict-free without a swizzle)
    const uint32_t b = smem_addr(S);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 16; ++r)
      asm volatile("st.shared.u16 [%0], %1;" ::"r"(b + 2u * j + 32u * r), "h"(static_cast<unsigned short>(v[r]))
                   : "memory");
    __syncwarp();
    if (!valid) return;
    uint4* dst = reinterpret_cast<uint4*>(out_poly);
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      uint4 w;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                   : "r"(b + 16u * (j + 16 * kk))
                   : "memory");
      __stcs(dst + j + 16 * kk, w);
    }
    return;
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 16; ++r) X.put(r, v[r]);
  __syncwarp();
  if (!valid) return;
  constexpr int PV = 16 / int(sizeof(IO));  // coefficients per 16-byte vector
  constexpr int V = 16 / PV;                // vectors per lane
  uint4* dst = reinterpret_cast<uint4*>(out_poly);
#pragma unroll
  for (int kk = 0; kk < V; ++kk) {
    const int i0 = (j + 16 * kk) * PV;
    uint4 w;
    if constexpr (PV == 8) {
      const uint4 q0 = *reinterpret_cast<const uint4*>(S + swz(i0));
      const uint4 q1 = *reinterpret_cast<const uint4*>(S + swz(i0 + 4));
      w.x = (q0.x & 0xffffu) | (q0.y << 16);
      w.y = (q0.z & 0xffffu) | (q0.w << 16);
      w.z = (q1.x & 0xffffu) | (q1.y << 16);
      w.w = (q1.z & 0xffffu) | (q1.w << 16);
    } else {
      w = *reinterpret_cast<const uint4*>(S + swz(i0));
    }
    __stcs(dst + j + 16 * kk, w);
  }
}

// strided read of one polynomial from a landed stage slot: one 32-bit shared-window base
// register, immediate offsets (ptxas otherwise rebuilds each address with an IMAD)
template <class IO, bool SGN>
__device__ __forceinline__ void load_strided(uint32_t (&v)[16], const IO* src, int j) {
  const uint32_t base = smem_addr(src) + uint32_t(sizeof(IO)) * j;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    uint32_t x;
    if constexpr (sizeof(IO) == 2) {
      if (SGN)
        asm volatile("ld.shared.s16 %0, [%1];" : "=r"(x) : "r"(base + 32u * r) : "memory");
      else
        asm volatile("ld.shared.u16 %0, [%1];" : "=r"(x) : "r"(base + 32u * r) : "memory");
    } else {
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(base + 64u * r) : "memory");
    }
    v[r] = x;
  }
}

// contiguous read (16 consecutive coefficients of lane j)
template <class IO, bool SGN>
__device__ __forceinline__ void load_contiguous(uint32_t (&v)[16], const IO* poly, int j) {
  const uint4* src = reinterpret_cast<const uint4*>(poly) + j * (16 * int(sizeof(IO)) / 16);
  if constexpr (sizeof(IO) == 2) {
    const uint4 a = src[0], b = src[1];
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      v[2 * e] = widen<uint16_t, SGN>(static_cast<uint16_t>(w[e] & 0xffffu));
      v[2 * e + 1] = widen<uint16_t, SGN>(static_cast<uint16_t>(w[e] >> 16));
    }
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 a = src[c];
      v[4 * c] = a.x;
      v[4 * c + 1] = a.y;
      v[4 * c + 2] = a.z;
      v[4 * c + 3] = a.w;
    }
  }
}

// barrier setup shared by every TMA kernel
// contiguous read v[r] = a[16 j + r] from a 128B-swizzled stage: chunk c of the lane's
// segment at stage + off[c] (off = swz128 of its linear offset, hoisted per lane)
template <class IO, bool SGN>
__device__ __forceinline__ void load_contiguous_swz(uint32_t (&v)[16], uint32_t stage,
                                                    const uint32_t (&off)[4]) {
  if constexpr (sizeof(IO) == 2) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t w[4];
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                   : "r"(stage + off[c])
                   : "memory");
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        v[8 * c + 2 * e] = widen<uint16_t, SGN>(static_cast<uint16_t>(w[e] & 0xffffu));
        v[8 * c + 2 * e + 1] = widen<uint16_t, SGN>(static_cast<uint16_t>(w[e] >> 16));
      }
    }
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v[4 * c]), "=r"(v[4 * c + 1]), "=r"(v[4 * c + 2]), "=r"(v[4 * c + 3])
                   : "r"(stage + off[c])
                   : "memory");
  }
}

__device__ __forceinline__ void init_barriers(uint64_t* full, uint64_t* empty, int stages,
                                              int consumers = kConsumers) {
  if (threadIdx.x == 0) {
    pdl_launch_dependents();
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], consumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

}  // namespace tma
}  // namespace nttk_b200
