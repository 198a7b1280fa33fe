// fast256_tma.cu -- TMA-fed batched N = 256 NTT kernels for sm_100a (hot path, v2).
//
// Same arithmetic, layer schedule and twiddle indexing as fast256.cu (bit-exact with
// the reference drivers transform.hpp:77-116 via the arith.cuh policies), with the
// memory side rebuilt around Blackwell's bulk-copy engine:
//   * one producer warp per CTA streams tiles of 16 polynomials HBM -> shared memory
//     with cp.async.bulk (one 512 B / 1 KiB copy per polynomial into a padded slot,
//     SASS UBLKCP), completion signalled through mbarrier transaction counts; an
//     S-stage ring keeps ~100+ KiB per SM in flight (the HBM bandwidth-delay product)
//     without spending registers or LSU issue slots on prefetching;
//   * 8 consumer warps (a half-warp per polynomial, 16 coefficients per lane) read
//     their coefficients straight from the landed slot, release it with one
//     mbarrier arrive per warp, and run all butterfly layers in registers with one
//     shared-memory transpose between the two 4-layer phases;
//   * the 15 lane-dependent twiddles are pinned in registers (an opaque move keeps
//     ptxas from re-loading them from the constant bank inside the loop); the uniform
//     ones are constant-bank IMAD operands.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "arith.cuh"
#include "fast256.hpp"

namespace nttk_b200 {
namespace {

constexpr int kConsumers = 8;                  // consumer warps per CTA
constexpr int kThreads = (kConsumers + 1) * 32;
constexpr int kTile = 2 * kConsumers;          // polynomials per stage
constexpr int kScratchWords = 2 * 272;         // per-warp transpose scratch (u32)

// A stage holds one tile of kTile polynomials as two contiguous halves (one bulk copy
// each: polynomials 0..7 and 8..15 of the tile).  Consumer warp w owns polynomial w of
// the first half and polynomial w of the second; the second half starts kPad bytes
// later so the two polynomials of a warp sit on disjoint bank halves.
template <class IO>
struct Geo {
  static constexpr int kPolyBytes = 256 * int(sizeof(IO));
  static constexpr int kPad = sizeof(IO) == 2 ? 32 : 64;
  static constexpr int kHalfBytes = kConsumers * kPolyBytes;
  static constexpr int kStages = sizeof(IO) == 2 ? 4 : 3;
  static constexpr int kStageBytes = 2 * kHalfBytes + kPad + 64;  // keep stages 128B-aligned
  static constexpr int kSmem = kStages * kStageBytes + kConsumers * kScratchWords * 4 +
                               2 * kStages * 8;
  // byte offset of the polynomial of warp w, half h inside a stage
  __device__ static constexpr int poly_offset(int w, int h) {
    return h * (kHalfBytes + kPad) + w * kPolyBytes;
  }
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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(b))
      : "memory");
}

// Hand a consumed stage back to the producer.  The stage was read through the generic
// proxy (LDS) and will be overwritten by the async proxy (the next bulk copy): the
// proxy fence orders this warp's reads before the refill (WAR across proxies), the
// warp barrier collects all lanes, one lane arrives.
__device__ __forceinline__ void release_stage(uint64_t* empty, int lane) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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

#ifndef NTTK_ALT_MASK
#define NTTK_ALT_MASK 0x22  // forward layers (bit s) using the alternative Plantard form
#endif
#ifndef NTTK_INV_ALT_MASK
#define NTTK_INV_ALT_MASK 0x0  // inverse merge layers (bit s) using the alternative form
#endif

// Minimum CTAs per SM for the register allocator (shared memory admits 4 for u16 and 3
// for u32 stages).  Measured: capping the n=32 kernels to 3 CTAs (72 regs) is ~2% slower.
#ifndef NTTK_MINB
#define NTTK_MINB(IO) 1
#endif

template <class K, class Tw>
__device__ __forceinline__ void inv_bf(int sl, uint32_t& x, uint32_t& y, Tw w, uint32_t off,
                                       const FastArgs& A) {
  if ((NTTK_INV_ALT_MASK >> sl) & 1) K::inv_alt(x, y, w, off, A);
  else K::inv(x, y, w, off, A);
}

// producer: stream tiles of kTile polynomials into the stage ring
template <class IO>
__device__ __forceinline__ void produce(const IO* in, size_t batch, uint8_t* stages, uint64_t* full,
                                        uint64_t* empty) {
  using G = Geo<IO>;
  const size_t ntiles = (batch + kTile - 1) / kTile;
  int k = 0;
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
template <class K, class IO, int L, bool PER_INDEX>
__global__ void __launch_bounds__(kThreads, NTTK_MINB(IO))
    fwd256_tma_kernel(const IO* __restrict__ in, IO* __restrict__ out, size_t batch,
                      const __grid_constant__ FastArgs A) {
  using G = Geo<IO>;
  using Tw = typename K::Tw;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stages = smem;
  uint32_t* scratch = reinterpret_cast<uint32_t*>(smem + G::kStages * G::kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(scratch + kConsumers * kScratchWords);
  uint64_t* empty = full + G::kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < G::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kConsumers) {
    if (lane == 0) produce<IO>(in, batch, stages, full, empty);
    return;
  }
  const int j = lane & 15, half = lane >> 4;
  Xpose X;
  X.init(scratch + warp * kScratchWords + half * 272, j);

  Tw twl[15];
  if (PER_INDEX) {
#pragma unroll
    for (int r = 0; r < 8; ++r) twl[r] = pin(K::tw(A, 0 + j + 16 * r));
#pragma unroll
    for (int r = 0; r < 4; ++r) twl[8 + r] = pin(K::tw(A, 128 + j + 16 * r));
#pragma unroll
    for (int r = 0; r < 2; ++r) twl[12 + r] = pin(K::tw(A, 192 + j + 16 * r));
    twl[14] = pin(K::tw(A, 224 + j));
  } else {
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

  const size_t ntiles = (batch + kTile - 1) / kTile;
  int k = 0;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int s = k % G::kStages;
    const size_t poly = t * kTile + half * kConsumers + warp;
    mbar_wait(&full[s], (k / G::kStages) & 1);
    const IO* src = reinterpret_cast<const IO*>(stages + s * G::kStageBytes + G::poly_offset(warp, half));
    uint32_t v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = widen<IO, K::kSigned>(src[j + 16 * r]);
    __syncwarp();
    release_stage(&empty[s], lane);

    // phase 1: layers 1..4 (index bits 7..4 in registers)
#pragma unroll
    for (int sl = 1; sl <= 4; ++sl) {
      const int h = 8 >> (sl - 1);
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r & h) continue;
        Tw w;
        if (PER_INDEX) {
          const int base = sl == 1 ? 0 : sl == 2 ? 8 : sl == 3 ? 12 : 14;
          w = twl[base + (r & (h - 1))];
        } else {
          w = K::tw(A, (1 << (sl - 1)) - 1 + (r >> (5 - sl)));
        }
        if ((NTTK_ALT_MASK >> sl) & 1) K::fwd_alt(v[r], v[r + h], w, A);
        else K::fwd(v[r], v[r + h], w, A);
      }
    }
    // transpose: strided -> contiguous ownership
#pragma unroll
    for (int r = 0; r < 16; ++r) X.put(r, v[r]);
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 4; ++c) X.get4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
    // phase 2: layers 5..L (index bits 3..0 in registers)
#pragma unroll
    for (int sl = 5; sl <= 8; ++sl) {
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
        if ((NTTK_ALT_MASK >> sl) & 1) K::fwd_alt(v[r], v[r + h], w, A);
        else K::fwd(v[r], v[r + h], w, A);
      }
    }
    if (poly < batch) {
      if constexpr (sizeof(IO) == 2) {
        uint4* dst = reinterpret_cast<uint4*>(out + poly * 256) + 2 * j;
        uint4 a, b;
        a.x = (v[0] & 0xffffu) | (v[1] << 16);
        a.y = (v[2] & 0xffffu) | (v[3] << 16);
        a.z = (v[4] & 0xffffu) | (v[5] << 16);
        a.w = (v[6] & 0xffffu) | (v[7] << 16);
        b.x = (v[8] & 0xffffu) | (v[9] << 16);
        b.y = (v[10] & 0xffffu) | (v[11] << 16);
        b.z = (v[12] & 0xffffu) | (v[13] << 16);
        b.w = (v[14] & 0xffffu) | (v[15] << 16);
        __stcs(dst, a);
        __stcs(dst + 1, b);
      } else {
        uint4* dst = reinterpret_cast<uint4*>(out + poly * 256) + 4 * j;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          __stcs(dst + c, make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]));
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// MODE 0: generic canonicalisation; 1: host-validated fast canonicalisation (A.flags
// bits 0/1); 2: u16 input with the fused first merge layer (A.flags bit 2, improved n=16):
// X' = (X + Y) mod p, Y' = MP(w, X + K p - Y) replaces canonicalise-then-merge
template <class K, class IO, int L, int MODE>
__global__ void __launch_bounds__(kThreads, NTTK_MINB(IO))
    inv256_tma_kernel(const IO* __restrict__ in, IO* __restrict__ out, size_t batch,
                      const __grid_constant__ FastArgs A) {
  using G = Geo<IO>;
  using Tw = typename K::Tw;
  constexpr int TL = 1 << L;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stages = smem;
  uint32_t* scratch = reinterpret_cast<uint32_t*>(smem + G::kStages * G::kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(scratch + kConsumers * kScratchWords);
  uint64_t* empty = full + G::kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < G::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kConsumers) {
    if (lane == 0) produce<IO>(in, batch, stages, full, empty);
    return;
  }
  const int j = lane & 15, half = lane >> 4;
  uint32_t* S = scratch + warp * kScratchWords + half * 272;
  Xpose X;
  X.init(S, j);

  Tw twl[15];
  twl[0] = pin(K::tw(A, TL - 32 + j));
#pragma unroll
  for (int q = 0; q < 2; ++q) twl[1 + q] = pin(K::tw(A, TL - 64 + 2 * j + q));
#pragma unroll
  for (int q = 0; q < 4; ++q) twl[3 + q] = pin(K::tw(A, TL - 128 + 4 * j + q));
  if (L >= 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) twl[7 + q] = pin(K::tw(A, TL - 256 + 8 * j + q));
  }

  const size_t ntiles = (batch + kTile - 1) / kTile;
  int k = 0;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int s = k % G::kStages;
    const size_t poly = t * kTile + half * kConsumers + warp;
    mbar_wait(&full[s], (k / G::kStages) & 1);
    const uint4* src =
        reinterpret_cast<const uint4*>(stages + s * G::kStageBytes + G::poly_offset(warp, half)) +
        j * (16 * sizeof(IO) / 16);
    uint32_t v[16];
    if constexpr (sizeof(IO) == 2) {
      const uint4 a = src[0], b = src[1];
      const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        v[2 * e] = widen<uint16_t, K::kSigned>(static_cast<uint16_t>(w[e] & 0xffffu));
        v[2 * e + 1] = widen<uint16_t, K::kSigned>(static_cast<uint16_t>(w[e] >> 16));
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
    __syncwarp();
    release_stage(&empty[s], lane);
    if (MODE != 2) {
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = canon<IO, K::kSigned, MODE == 1>(v[r], A);
    }

    // phase 1: merge layers s = L..5 (contiguous ownership)
#pragma unroll
    for (int sl = 8; sl >= 5; --sl) {
      if (sl > L) continue;
      const int h = 1 << (8 - sl);
      const uint32_t off = A.off[L - sl + 1];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r & h) continue;
        const int base = sl == 5 ? 0 : sl == 6 ? 1 : sl == 7 ? 3 : 7;
        const Tw w = twl[base + (r >> (9 - sl))];
        if constexpr (MODE == 2) {
          if (sl == L) {
            const uint32_t x = v[r], y = v[r + h];
            v[r] = mod_cb(x + y + A.zero, A);
            v[r + h] = fence_val(mp_n16<false>(x + A.kp - y, w, A.p), A);
          } else {
            inv_bf<K>(sl, v[r], v[r + h], w, off, A);
          }
        } else {
          inv_bf<K>(sl, v[r], v[r + h], w, off, A);
        }
      }
    }
    // transpose: contiguous -> strided ownership
#pragma unroll
    for (int c = 0; c < 4; ++c) X.put4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = X.get(r);
    // phase 2: merge layers s = 4..1, uniform twiddles
#pragma unroll
    for (int sl = 4; sl >= 1; --sl) {
      const int h = 1 << (4 - sl);
      const uint32_t off = A.off[L - sl + 1];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r & h) continue;
        if (K::kFold && sl == 1)  // N^{-1} folded into the last merge layer
          K::inv_last(v[r], v[r + h], off, A);
        else
          inv_bf<K>(sl, v[r], v[r + h], K::tw(A, TL - (2 << (sl - 1)) + (r >> (5 - sl))), off, A);
      }
    }
    if (!K::kFold) {
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = K::scale(v[r], A);
    }
    // strided -> contiguous through the scratch for coalesced 128-bit stores
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 16; ++r) X.put(r, v[r]);
    __syncwarp();
    if (poly < batch) {
      constexpr int PV = 16 / int(sizeof(IO));  // coefficients per 16-byte vector
      constexpr int V = 16 / PV;                // vectors per lane
      uint4* dst = reinterpret_cast<uint4*>(out + poly * 256);
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
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
int g_sms = 0;

template <class Kern>
int grid_for(Kern kern, int smem, int& occ, size_t batch) {
  if (!occ) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kThreads, smem);
    occ = o > 0 ? o : 1;
    if (!g_sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
      if (g_sms <= 0) g_sms = 148;
    }
  }
  const size_t tiles = (batch + kTile - 1) / kTile;
  const size_t full = size_t(g_sms) * occ;
  return static_cast<int>(tiles < full ? tiles : full);
}

template <class K, class IO, int L, bool PER_INDEX>
cudaError_t fwd_launch(const void* in, void* out, size_t batch, const FastArgs& A, cudaStream_t st) {
  static int occ = 0;
  auto kern = fwd256_tma_kernel<K, IO, L, PER_INDEX>;
  const int blocks = grid_for(kern, Geo<IO>::kSmem, occ, batch);
  kern<<<blocks, kThreads, Geo<IO>::kSmem, st>>>(static_cast<const IO*>(in), static_cast<IO*>(out),
                                                 batch, A);
  return cudaGetLastError();
}

template <class K, class IO, int L>
cudaError_t inv_launch(const void* in, void* out, size_t batch, const FastArgs& A, cudaStream_t st) {
  constexpr bool kCanFuse = sizeof(IO) == 2 && std::is_same<K, ImprovedN16<false>>::value;
  const unsigned fast_bit = sizeof(IO) == 2 ? 1u : 2u;
  if (kCanFuse && (A.flags & 4)) {
    static int occ = 0;
    auto kern = inv256_tma_kernel<K, IO, L, kCanFuse ? 2 : 1>;
    const int blocks = grid_for(kern, Geo<IO>::kSmem, occ, batch);
    kern<<<blocks, kThreads, Geo<IO>::kSmem, st>>>(static_cast<const IO*>(in),
                                                   static_cast<IO*>(out), batch, A);
  } else if (!K::kSigned && (A.flags & fast_bit)) {
    static int occ = 0;
    auto kern = inv256_tma_kernel<K, IO, L, 1>;
    const int blocks = grid_for(kern, Geo<IO>::kSmem, occ, batch);
    kern<<<blocks, kThreads, Geo<IO>::kSmem, st>>>(static_cast<const IO*>(in),
                                                   static_cast<IO*>(out), batch, A);
  } else {
    static int occ = 0;
    auto kern = inv256_tma_kernel<K, IO, L, 0>;
    const int blocks = grid_for(kern, Geo<IO>::kSmem, occ, batch);
    kern<<<blocks, kThreads, Geo<IO>::kSmem, st>>>(static_cast<const IO*>(in),
                                                   static_cast<IO*>(out), batch, A);
  }
  return cudaGetLastError();
}

template <class K, class IO, bool PER_INDEX>
cudaError_t by_layers(int dir, int L, const void* in, void* out, size_t batch, const FastArgs& A,
                      cudaStream_t st) {
  if (L == 8)
    return dir == 0 ? fwd_launch<K, IO, 8, PER_INDEX>(in, out, batch, A, st)
                    : inv_launch<K, IO, 8>(in, out, batch, A, st);
  if (L == 7)
    return dir == 0 ? fwd_launch<K, IO, 7, PER_INDEX>(in, out, batch, A, st)
                    : inv_launch<K, IO, 7>(in, out, batch, A, st);
  return cudaErrorInvalidValue;
}

template <class K, bool PER_INDEX>
cudaError_t by_io(int dir, int L, int elem, const void* in, void* out, size_t batch,
                  const FastArgs& A, cudaStream_t st) {
  if (elem == 2) return by_layers<K, uint16_t, PER_INDEX>(dir, L, in, out, batch, A, st);
  if (elem == 4) return by_layers<K, uint32_t, PER_INDEX>(dir, L, in, out, batch, A, st);
  return cudaErrorInvalidValue;
}

}  // namespace

bool fast256_tma_supports(int elem_bytes, const void* in, const void* out) {
  // bulk copies need 16-byte aligned global addresses
  return (elem_bytes == 2 || elem_bytes == 4) &&
         !(reinterpret_cast<uintptr_t>(in) & 15) && !(reinterpret_cast<uintptr_t>(out) & 15);
}

cudaError_t fast256_tma_launch(const HostParams& P, int kind, int dir, const void* in, void* out,
                               size_t batch, int elem_bytes, cudaStream_t st) {
  const FastArgs& A = P.fast[kind][dir];
  const int L = static_cast<int>(P.layers);
  const bool n16 = P.n_bits == 16;
  const bool cyclic = P.tree == NTTK_CYCLIC;
  if (batch == 0) return cudaSuccess;
  switch (kind) {
    case NTTK_IMPROVED:
      return n16 ? by_io<ImprovedN16<false>, false>(dir, L, elem_bytes, in, out, batch, A, st)
                 : by_io<ImprovedN32, false>(dir, L, elem_bytes, in, out, batch, A, st);
    case NTTK_HARVEY:
      if (cyclic)
        return n16 ? by_io<Harvey<16, false>, true>(dir, L, elem_bytes, in, out, batch, A, st)
                   : by_io<Harvey<32, false>, true>(dir, L, elem_bytes, in, out, batch, A, st);
      return n16 ? by_io<Harvey<16, true>, false>(dir, L, elem_bytes, in, out, batch, A, st)
                 : by_io<Harvey<32, true>, false>(dir, L, elem_bytes, in, out, batch, A, st);
    case NTTK_SMONT:
      return n16 ? by_io<Smont<16>, false>(dir, L, elem_bytes, in, out, batch, A, st)
                 : by_io<Smont<32>, false>(dir, L, elem_bytes, in, out, batch, A, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace nttk_b200
