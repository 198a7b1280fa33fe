// fastn_tma.cu -- TMA-fed batched NTT for N = 512 and N = 1024 (the paper's Table 2
// parameter sets: newhope/falcon/remblem 512, newhope/falcon/hila5 1024, params.hpp:273-306).
//
// Same pipeline as fast256_tma.cu (one producer warp streaming tiles with cp.async.bulk on
// an mbarrier ring, 8 consumer warps) and the same butterfly policies (arith.cuh), scaled
// to 32 coefficients per lane: G = N / 32 lanes own a polynomial (a half-warp at N = 512,
// a warp at N = 1024), so 5 layers are register-local per phase:
//   strided ownership     v[k] = a[j + G k]    (index bits LOGN-1..LOGN-5 in k)
//   contiguous ownership  v[k] = a[32 j + k]   (index bits 4..0 in k)
// Forward: layers 1..5 strided, one XOR-swizzled transpose, layers 6..LOGN contiguous.
// Inverse: merge layers LOGN..6 contiguous, transpose, 5..1 strided (N^{-1} folded into
// the last layer), natural-order coalesced stores through the same tile.
// Twiddles: the warp-uniform ones are constant-bank operands (FastArgs, compact order
// written by params.cpp fill_fast); the lane-dependent ones come from a shared-memory copy
// of the whole direction table (HostParams::fastn_table).
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "arith.cuh"
#include "fastn.hpp"
#include "launch_cache.hpp"
#include "tensor_map.hpp"
#include "tma_common.cuh"

namespace nttk_b200 {
namespace {

using namespace tma;

// C = consumer warps per CTA (the forward may use more than the inverse, whose swizzled
// tensor box of kTileN polynomials is limited to 256 rows)
template <int LOGN, class IO, int C = kConsumers>
struct GeoN {
  static constexpr int kConsumers = C;
  static constexpr int kThreadsN = (C + 1) * 32;
  static constexpr int N = 1 << LOGN;
  static constexpr int G = N / 32;                  // lanes per polynomial
  static constexpr int PPW = 32 / G;                // polynomials per warp (2 or 1)
  static constexpr int kTileN = kConsumers * PPW;   // polynomials per stage
  static constexpr int kPolyBytes = N * int(sizeof(IO));
  static constexpr int kHalfBytes = kConsumers * kPolyBytes;
  static constexpr int kPad = PPW == 2 ? 64 : 0;    // second half-warp: disjoint bank half
  static constexpr int kStages = sizeof(IO) == 2 ? 3 : 2;
  static constexpr int kStageBytes = (PPW * kHalfBytes + kPad + 127) / 128 * 128;
  static constexpr int kRegionWords = N + (PPW == 2 ? 16 : 0);  // transpose tile per poly
  static constexpr int kScratchWords = PPW * kRegionWords;       // per warp
  static constexpr int kSmem = kStages * kStageBytes + kConsumers * kScratchWords * 4 +
                               N * 8 /* twiddle table */ + 2 * kStages * 8;
  __device__ static constexpr int poly_offset(int w, int h) {
    return h * (kHalfBytes + kPad) + w * kPolyBytes;
  }
  // inverse with 128B-swizzled tensor-map stages (tma_common.cuh inv_swz): one box of
  // kTileN polynomials, 1024-byte aligned, no pad
  static constexpr int kRowsPerPoly = kPolyBytes / 128;
  static constexpr int kTileRows = kTileN * kRowsPerPoly;
  static constexpr int kBoxRows = kTileRows < 256 ? kTileRows : 256;  // TMA box limit
  static constexpr int kBoxes = kTileRows / kBoxRows;                  // boxes per stage
  static constexpr int kSwzStageBytes = kTileRows * 128;
  static constexpr int kSwzSmem = 1024 + kStages * kSwzStageBytes + kConsumers * kScratchWords * 4 +
                                  N * 8 + 2 * kStages * 8;
};

// Transpose tile of one polynomial: 32-word rows, 16-byte chunk c of row r stored at chunk
// c ^ (r & 7).  Strided puts/gets (lane j, register k, element j + G k) and contiguous
// 128-bit gets/puts (lane j, row j) are both bank-conflict-free; the two polynomials of
// a half-warp pair sit 16 words apart.  Addresses are hoisted 32-bit shared-window words.
template <int G>
struct XposeN {
  uint32_t sp[8], cp[8], base;
  __device__ __forceinline__ void init(const uint32_t* tile, int j) {
    base = smem_addr(tile);
    // strided element i = j + G k: row = (G k + j) >> 5, column = (G k + j) & 31
    // G = 32: row k, col j -> chunk (j >> 2) ^ (k & 7)
    // G = 16: row k >> 1, col j + 16 (k & 1) -> chunk (j >> 2) ^ ((k >> 1) & 7) ^ 4 (k & 1)
#pragma unroll
    for (int m = 0; m < 8; ++m) sp[m] = base + 4u * ((uint32_t((j >> 2) ^ m) << 2) | uint32_t(j & 3));
#pragma unroll
    for (int c = 0; c < 8; ++c) cp[c] = base + 4u * (32u * j + (uint32_t(c ^ (j & 7)) << 2));
  }
  __device__ __forceinline__ uint32_t saddr(int k) const {
    if constexpr (G == 32) return sp[k & 7] + 128u * k;
    else return sp[((k >> 1) & 7) ^ (4 * (k & 1))] + 128u * (k >> 1);
  }
  __device__ __forceinline__ void put(int k, uint32_t v) const {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(saddr(k)), "r"(v) : "memory");
  }
  __device__ __forceinline__ uint32_t get(int k) const {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr(k)) : "memory");
    return v;
  }
  __device__ __forceinline__ void put4(int c, uint32_t a, uint32_t b, uint32_t d, uint32_t e) const {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(cp[c]), "r"(a), "r"(b), "r"(d),
                 "r"(e)
                 : "memory");
  }
  __device__ __forceinline__ void get4(int c, uint32_t& a, uint32_t& b, uint32_t& d, uint32_t& e) const {
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(d), "=r"(e)
                 : "r"(cp[c])
                 : "memory");
  }
  // chunk q (natural order: elements 4q..4q+3) of the tile
  __device__ __forceinline__ uint4 chunk(int q) const {
    const int row = q >> 3, c = q & 7;
    uint4 w;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                 : "r"(base + 128u * row + 16u * uint32_t(c ^ (row & 7)))
                 : "memory");
    return w;
  }
};

template <class Tw>
__device__ __forceinline__ Tw mk_tw(uint2 e) {
  if constexpr (std::is_same<Tw, uint32_t>::value) return e.x;
  else return e;
}

template <class Tw>
__device__ __forceinline__ Tw tw_smem(const uint2* tws, int idx) {
  return mk_tw<Tw>(tws[idx]);
}

template <int LOGN, class IO, int C = kConsumers>
__device__ __forceinline__ void produce_n(const IO* in, size_t batch, uint8_t* stages, uint64_t* full,
                                          uint64_t* empty) {
  using GN = GeoN<LOGN, IO, C>;
  constexpr int kConsumers = C;
  const size_t ntiles = (batch + GN::kTileN - 1) / GN::kTileN;
  int k = 0;
  pdl_wait();
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int s = k % GN::kStages;
    if (k >= GN::kStages) mbar_wait(&empty[s], ((k / GN::kStages) & 1) ^ 1);
    const size_t first = t * GN::kTileN;
    const int n = batch - first < size_t(GN::kTileN) ? int(batch - first) : GN::kTileN;
    const int n0 = n < kConsumers ? n : kConsumers, n1 = n - n0;
    mbar_expect_tx(&full[s], uint32_t(n) * GN::kPolyBytes);
    uint8_t* base = stages + s * GN::kStageBytes;
    bulk_g2s(base, in + first * GN::N, uint32_t(n0) * GN::kPolyBytes, &full[s]);
    if (n1 > 0)
      bulk_g2s(base + GN::poly_offset(0, 1), in + (first + kConsumers) * GN::N,
               uint32_t(n1) * GN::kPolyBytes, &full[s]);
  }
}

// strided read v[k] = a[j + G k] from a landed stage slot (consecutive lanes, consecutive
// words: conflict-free)
template <class IO, int G, bool SGN>
__device__ __forceinline__ void load_strided_n(uint32_t (&v)[32], const IO* src, int j) {
  const uint32_t b = smem_addr(src) + uint32_t(sizeof(IO)) * j;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    uint32_t x;
    if constexpr (sizeof(IO) == 2) {
      if (SGN)
        asm volatile("ld.shared.s16 %0, [%1];" : "=r"(x) : "r"(b + 2u * G * k) : "memory");
      else
        asm volatile("ld.shared.u16 %0, [%1];" : "=r"(x) : "r"(b + 2u * G * k) : "memory");
    } else {
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(b + 4u * G * k) : "memory");
    }
    v[k] = x;
  }
}

// contiguous read v[k] = a[32 j + k]
template <class IO, bool SGN>
__device__ __forceinline__ void load_contiguous_n(uint32_t (&v)[32], const IO* poly, int j) {
  const uint4* src = reinterpret_cast<const uint4*>(poly + 32 * j);
  if constexpr (sizeof(IO) == 2) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 a = src[c];
      const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        v[8 * c + 2 * e] = widen<uint16_t, SGN>(static_cast<uint16_t>(w[e] & 0xffffu));
        v[8 * c + 2 * e + 1] = widen<uint16_t, SGN>(static_cast<uint16_t>(w[e] >> 16));
      }
    }
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint4 a = src[c];
      v[4 * c] = a.x;
      v[4 * c + 1] = a.y;
      v[4 * c + 2] = a.z;
      v[4 * c + 3] = a.w;
    }
  }
}

// contiguous read from a 128B-swizzled stage: chunk c of the lane's segment at stage + off[c]
template <class IO, bool SGN>
__device__ __forceinline__ void load_contiguous_n_swz(uint32_t (&v)[32], uint32_t stage,
                                                      const uint32_t (&off)[8]) {
  if constexpr (sizeof(IO) == 2) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
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
    for (int c = 0; c < 8; ++c)
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v[4 * c]), "=r"(v[4 * c + 1]), "=r"(v[4 * c + 2]), "=r"(v[4 * c + 3])
                   : "r"(stage + off[c])
                   : "memory");
  }
}

// The u32 forward writes its output through the transpose tile (coalesced stores, +10-11 %,
// profiles/r1b_fastn_store.txt); u16 stores straight from registers.

// contiguous ownership -> global (lane j writes its 32 consecutive coefficients)
template <class IO>
__device__ __forceinline__ void store_contiguous_n(IO* out_poly, int j, const uint32_t (&v)[32]) {
  uint4* dst = reinterpret_cast<uint4*>(out_poly + 32 * j);
  if constexpr (sizeof(IO) == 2) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      __stcs(dst + c, make_uint4(__byte_perm(v[8 * c], v[8 * c + 1], 0x5410),
                                 __byte_perm(v[8 * c + 2], v[8 * c + 3], 0x5410),
                                 __byte_perm(v[8 * c + 4], v[8 * c + 5], 0x5410),
                                 __byte_perm(v[8 * c + 6], v[8 * c + 7], 0x5410)));
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      __stcs(dst + c, make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]));
  }
}

// natural-order coalesced 128-bit stores of the transpose tile (lane j: chunks j + G t)
template <class IO, int G>
__device__ __forceinline__ void store_tile_n(IO* out_poly, int j, const XposeN<G>& X) {
  constexpr int N = 32 * G;
  uint4* dst = reinterpret_cast<uint4*>(out_poly);
  if constexpr (sizeof(IO) == 2) {  // 8 coefficients per 16-byte vector
#pragma unroll
    for (int t = 0; t < N / 8 / G; ++t) {
      const int q = j + G * t;
      const uint4 a = X.chunk(2 * q), b = X.chunk(2 * q + 1);
      __stcs(dst + q, make_uint4(__byte_perm(a.x, a.y, 0x5410), __byte_perm(a.z, a.w, 0x5410),
                                 __byte_perm(b.x, b.y, 0x5410), __byte_perm(b.z, b.w, 0x5410)));
    }
  } else {
#pragma unroll
    for (int t = 0; t < N / 4 / G; ++t) {
      const int q = j + G * t;
      __stcs(dst + q, X.chunk(q));
    }
  }
}

// strided ownership -> natural-order coalesced 128-bit stores through the transpose tile
template <class IO, int G>
__device__ __forceinline__ void store_strided_n(IO* out_poly, int j, const uint32_t (&v)[32],
                                                const XposeN<G>& X, bool valid) {
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 32; ++k) X.put(k, v[k]);
  __syncwarp();
  if (valid) store_tile_n<IO, G>(out_poly, j, X);
}

// contiguous ownership (forward output) -> the same coalesced stores: 8 conflict-free
// 16-byte row writes per lane instead of 8 stores whose lanes sit 64 / 128 B apart
template <class IO, int G>
__device__ __forceinline__ void store_contiguous_n_coalesced(IO* out_poly, int j, const uint32_t (&v)[32],
                                                             const XposeN<G>& X, bool valid) {
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 8; ++c) X.put4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  __syncwarp();
  if (valid) store_tile_n<IO, G>(out_poly, j, X);
}

// Stage the direction table into shared memory.  The lane-dependent segments (per-block
// layers s >= 6: lane j reads blocks j c + q, q < c = 2^{s-1} / G) are stored transposed,
// entry j c + q at q G + j, so a warp's reads hit consecutive words; without this layer
// LOGN has lanes 128 B apart (a 32-way bank conflict).  SEG(s) = first entry of layer s.
template <int LOGN, bool MERGE>
__device__ __forceinline__ constexpr int seg_base(int s) {
  return MERGE ? (1 << LOGN) - (2 << (s - 1)) : (1 << (s - 1)) - 1;
}

// ---------------------------------------------------------------------------
// forward: run_split_layers (transform.hpp:77-96) for N = 2^LOGN, strided in ->
// contiguous out.  PER_INDEX: DIF per-index schedule (ntl / harvey / scott, cyclic).
template <class K, int LOGN, bool PER_INDEX>
__device__ __forceinline__ void fwd_body_n(uint32_t (&v)[32], const uint2* tws, const FastArgs& A,
                                           const XposeN<(1 << LOGN) / 32>& X, int j) {
  using Tw = typename K::Tw;
  constexpr int N = 1 << LOGN, G = N / 32;
#pragma unroll
  for (int s = 1; s <= 5; ++s) {  // phase 1: register distance h = 2^{5-s}
    const int h = 16 >> (s - 1);
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k & h) continue;
      Tw w;
      if (PER_INDEX)  // index within the half block: j + G (k mod h); cursor N - 2^{LOGN-s+1}
        w = tw_smem<Tw>(tws, N - (N >> (s - 1)) + j + G * (k & (h - 1)));
      else  // block k >> (6 - s), CT per-block cursor 2^{s-1} - 1 (constant bank)
        w = K::tw(A, (1 << (s - 1)) - 1 + (k >> (6 - s)));
      K::fwd(v[k], v[k + h], w, A);
    }
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 32; ++k) X.put(k, v[k]);
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 8; ++c) X.get4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
#pragma unroll
  for (int s = 6; s <= LOGN; ++s) {  // phase 2: register distance h = 2^{LOGN-s}
    const int h = 1 << (LOGN - s);
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k & h) continue;
      Tw w;
      if (PER_INDEX)  // uniform index k mod h, compact constant-bank order
        w = K::tw(A, 32 - 2 * h + (k & (h - 1)));
      else  // block (32 j + k) >> (LOGN - s + 1) = j c + (k >> (LOGN - s + 1)), transposed
        w = tw_smem<Tw>(tws, seg_base<LOGN, false>(s) + (k >> (LOGN - s + 1)) * G + j);
      K::fwd(v[k], v[k + h], w, A);
    }
  }
}

// F1 forward for N = 512 / 1024 (ImprovedN16 -- the narrow image of the Table 2 presets --
// A.flags bit 10; tma_common.cuh fwd_body_f1 has the derivation): layer 1 (twiddle 1) injects
// the surplus S = L - 2 (A.f1_sp), layers 2..L-1 run the F1 form (Y' = X - r spends one), the
// last layer runs the umulhi form and removes sigma = S - popcount(i bits L-2..1) of the X
// position i = 32 j + k with the per-lane registers E[m] = (m - cj) p.
template <class K, int LOGN>
__device__ __forceinline__ void fwd_body_n_f1(uint32_t (&v)[32], const uint2* tws, const FastArgs& A,
                                              const XposeN<(1 << LOGN) / 32>& X, int j,
                                              const uint32_t (&E)[6]) {
  using Tw = typename K::Tw;
  constexpr int N = 1 << LOGN, G = N / 32;
#pragma unroll
  for (int k = 0; k < 16; ++k) {  // layer 1: one block, twiddle 1, r = Y (canonical input)
    const uint32_t x = v[k], y = v[k + 16];
    v[k] = x + y + A.f1_sp;
    v[k + 16] = x + A.f1_sp1 - y;
  }
#pragma unroll
  for (int s = 2; s <= 5; ++s) {  // phase 1 (strided), uniform twiddles
    const int h = 16 >> (s - 1);
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k & h) continue;
      f1_bf(v[k], v[k + h], K::tw(A, (1 << (s - 1)) - 1 + (k >> (6 - s))), A);
    }
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 32; ++k) X.put(k, v[k]);
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 8; ++c) X.get4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
#pragma unroll
  for (int s = 6; s < LOGN; ++s) {  // phase 2 (contiguous), lane twiddles from shared memory
    const int h = 1 << (LOGN - s);
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k & h) continue;
      f1_bf(v[k], v[k + h], tw_smem<Tw>(tws, seg_base<LOGN, false>(s) + (k >> (LOGN - s + 1)) * G + j), A);
    }
  }
#pragma unroll
  for (int k = 0; k < 32; k += 2) {  // layer L: umulhi form, surplus removed
    const int kk = ((k >> 1) & 1) + ((k >> 2) & 1) + ((k >> 3) & 1) + ((k >> 4) & 1);
    const uint32_t r = mp_n16<false>(v[k + 1], tw_smem<Tw>(tws, seg_base<LOGN, false>(LOGN) + (k >> 1) * G + j), A.p);
    const uint32_t x = v[k];
    v[k + 1] = x - r + E[kk + 1];
    v[k] = x + r + E[kk];
  }
}

// inverse: run_merge_layers + N^{-1} (transform.hpp:99-116, 323-335), contiguous
// canonical in -> strided canonical out
template <class K, int LOGN>
__device__ __forceinline__ void inv_body_n(uint32_t (&v)[32], const uint2* tws, const FastArgs& A,
                                           const XposeN<(1 << LOGN) / 32>& X, int j) {
  using Tw = typename K::Tw;
  constexpr int G = (1 << LOGN) / 32;
#pragma unroll
  for (int s = LOGN; s >= 6; --s) {  // phase 1: merge depth m = LOGN - s + 1
    const int h = 1 << (LOGN - s);
    const uint32_t off = A.off[LOGN - s + 1];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k & h) continue;
      const Tw w = tw_smem<Tw>(tws, seg_base<LOGN, true>(s) + (k >> (LOGN - s + 1)) * G + j);
      K::inv(v[k], v[k + h], w, off, A);
    }
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 8; ++c) X.put4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = X.get(k);
#pragma unroll
  for (int s = 5; s >= 1; --s) {  // phase 2: register distance h = 2^{5-s}
    const int h = 1 << (5 - s);
    const uint32_t off = A.off[LOGN - s + 1];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k & h) continue;
      if (K::kFold && s == 1)
        K::inv_last(v[k], v[k + h], off, A);
      else  // block k >> (6 - s), compact merge order 32 - 2^s + b (constant bank)
        K::inv(v[k], v[k + h], K::tw(A, 32 - (2 << (s - 1)) + (k >> (6 - s))), off, A);
    }
  }
  if (!K::kFold) {
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = K::scale(v[k], A);
  }
}

// inv_body_n with lazy merge outputs (policy kLazy, A.flags bit 3; see tma_common.cuh
// inv_body_lazy): after a layer of register half-span h the words at (k & h) hold
// pre-quotient values, paired with each other by the next layer; materialised before the
// transpose, and phase 2 starts materialised.
// TW1 (A.flags bit 5, cyclic full tree): block 0 of the phase-2 merge layers (len >= N/32)
// has twiddle 1 and is uniform across lanes; Y' = X + off - Y stays unreduced (every value
// of merge depth d < 2^d p, as in tma_common.cuh inv_body_lazy).
template <class K, int LOGN, bool TW1 = false>
__device__ __forceinline__ void inv_body_n_lazy(uint32_t (&v)[32], const uint2* tws,
                                                const FastArgs& A,
                                                const XposeN<(1 << LOGN) / 32>& X, int j) {
  using Tw = typename K::Tw;
  constexpr int G = (1 << LOGN) / 32;
#pragma unroll
  for (int s = LOGN; s >= 6; --s) {  // phase 1: contiguous, register half-span h = 2^{LOGN-s}
    const int h = 1 << (LOGN - s);
    const uint32_t off = A.off[LOGN - s + 1];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k & h) continue;
      const Tw w = tw_smem<Tw>(tws, seg_base<LOGN, true>(s) + (k >> (LOGN - s + 1)) * G + j);
      if (s < LOGN && (k & (h >> 1))) K::inv_hh(v[k], v[k + h], w, off, A);
      else K::inv_h(v[k], v[k + h], w, off, A);
    }
  }
  constexpr int hl = 1 << (LOGN - 6);  // half-span of the last phase-1 layer: lazy words
#pragma unroll
  for (int k = 0; k < 32; ++k)
    if (k & hl) v[k] = K::materialize(v[k], A);
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 8; ++c) X.put4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = X.get(k);
  bool lz[32];  // lazy words of phase 2 (compile-time after the unroll; see inv_body_lazy)
#pragma unroll
  for (int k = 0; k < 32; ++k) lz[k] = false;
#pragma unroll
  for (int s = 5; s >= 1; --s) {  // phase 2: strided, h = 2^{5-s}, materialised start
    const int h = 1 << (5 - s);
    const uint32_t off = A.off[LOGN - s + 1];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k & h) continue;
      bool lx = lz[k], ly = lz[k + h];
      if (lx != ly) {  // mixed pair after a TW1 block: materialise the lazy word
        if (lx) v[k] = K::materialize(v[k], A);
        else v[k + h] = K::materialize(v[k + h], A);
        lx = ly = false;
      }
      if (s == 1) {
        if (lx) K::inv_last_hh(v[k], v[k + h], off, A);
        else K::inv_last(v[k], v[k + h], off, A);
        lz[k] = lz[k + h] = false;
      } else if (TW1 && (k >> (6 - s)) == 0) {  // block 0: twiddle 1, Y' = T unreduced
        const uint32_t x = v[k], y = v[k + h];
        if (lx) {
          uint32_t Xm;
          const uint32_t S = K::sum_hh(x, y, Xm, A);
          v[k] = S;
          v[k + h] = Xm + Xm + off - S + A.zero;
        } else {
          v[k] = x + y + A.zero;
          v[k + h] = x + off - y;
        }
        lz[k] = lz[k + h] = false;
      } else {
        const Tw w = K::tw(A, 32 - (2 << (s - 1)) + (k >> (6 - s)));
        if (lx) K::inv_hh(v[k], v[k + h], w, off, A);
        else K::inv_h(v[k], v[k + h], w, off, A);
        lz[k] = false;
        lz[k + h] = true;
      }
    }
  }
}

// narrow inverse (ImprovedN16 on an n = 32 improved parameter set; tma_common.cuh
// inv_body_narrow): compile-time bound exponents e[], reduction by MP(1^, .) before a merge
// that would leave n = 16's Prop. 4 range and before the transpose
template <class K, int LOGN>
__device__ __forceinline__ void inv_body_n_narrow(uint32_t (&v)[32], const uint2* tws, const FastArgs& A,
                                                  const XposeN<(1 << LOGN) / 32>& X, int j) {
  using Tw = typename K::Tw;
  constexpr int G = (1 << LOGN) / 32;
  int e[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) e[k] = 0;
#pragma unroll
  for (int s = LOGN; s >= 6; --s) {  // phase 1: contiguous, register half-span h = 2^{LOGN-s}
    const int h = 1 << (LOGN - s);
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k & h) continue;
      const Tw w = tw_smem<Tw>(tws, seg_base<LOGN, true>(s) + (k >> (LOGN - s + 1)) * G + j);
      narrow_bf<K>(v[k], v[k + h], e[k], e[k + h], w, false, A);
    }
  }
#pragma unroll
  for (int k = 0; k < 32; ++k)
    if (e[k]) v[k] = K::canon1(v[k], A);
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 8; ++c) X.put4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    v[k] = X.get(k);
    e[k] = 0;
  }
#pragma unroll
  for (int s = 5; s >= 1; --s) {  // phase 2: strided, h = 2^{5-s}, N^{-1} folded into s = 1
    const int h = 1 << (5 - s);
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k & h) continue;
      const Tw w = s == 1 ? Tw{} : K::tw(A, 32 - (2 << (s - 1)) + (k >> (6 - s)));
      narrow_bf<K>(v[k], v[k + h], e[k], e[k + h], w, s == 1, A);
    }
  }
}

// CT-form inverse of the narrow image at N = 512 / 1024 (A.flags bit 11; params.cpp
// fill_ct_inverse_n, tma_common.cuh inv_body_ct has the N = 256 derivation).  Radix-2 DIT on the
// bit-reversed spectrum with omega^{-1}.  Contiguous phase (position 32 j + k, len = 1..16): the
// jb = 0 butterfly of every block is multiply-free, the others run the F1 form with the uniform
// twiddles A.lo[(16 / len) jb].  Strided phase (position j + G k, len = G h): F-form butterflies
// with the lane twiddles of the shared-memory table (segment (h - 1) G, entry kk G + j), then
// h = 16 with N^{-1} folded into two Plantard products per butterfly and a min to the canonical
// residue.  The value interval [lo p, hi p) of every register is tracked at compile time (the
// arrays below fold away in the full unroll): an F butterfly's X input needs lo >= 1 + the floor
// its Y output must keep for the F layers still ahead (rq[]), the multiply-free butterflies set
// their outputs' floors with the offsets A.pm[m] = m p, and an input wider than kT[li] p is first
// reduced by one product by 1^ (four per lane in all).  Every product operand stays below
// kCtLimN p, host-checked against Prop. 4's n = 16 range.
template <class K, int LOGN, bool F3C, bool F3S>
__device__ __forceinline__ void inv_body_n_ct(uint32_t (&v)[32], const uint32_t* tws, const FastArgs& A,
                                              const XposeN<(1 << LOGN) / 32>& X, int j) {
  constexpr int G = (1 << LOGN) / 32;
  constexpr int H0 = LOGN == 10 ? 1 : 2;   // first strided register distance
  constexpr int FS = LOGN == 10 ? 4 : 3;   // strided F layers (h = H0 .. 8)
  constexpr int kT[5] = {1, 2, 4, 1, 2};   // widest multiply-free input per layer
  int rq[6][32];  // rq[li][k]: floor register k needs before contiguous layer li
#pragma unroll
  for (int k = 0; k < 32; ++k) rq[5][k] = FS;
#pragma unroll
  for (int li = 4; li >= 0; --li) {
    const int len = 1 << li;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k & len) continue;
      if ((k & (len - 1)) == 0) {
        rq[li][k] = rq[li][k + len] = 0;
      } else {
        const int a = rq[li + 1][k], b = rq[li + 1][k + len] + 1;
        rq[li][k] = a > b ? a : b;
        rq[li][k + len] = 0;
      }
    }
  }
  int lo[32], hi[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) lo[k] = 0, hi[k] = 1;  // canonical input
#pragma unroll
  for (int li = 0; li < 5; ++li) {  // contiguous phase: len = 1, 2, 4, 8, 16
    const int len = 1 << li;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k & len) continue;
      const int jb = k & (len - 1), m = k + len;
      if (jb == 0) {
        if (hi[k] - lo[k] > kT[li]) v[k] = K::canon1(v[k], A), lo[k] = 0, hi[k] = 1;
        if (hi[m] - lo[m] > kT[li]) v[m] = K::canon1(v[m], A), lo[m] = 0, hi[m] = 1;
        const int c1 = rq[li + 1][k] - (lo[k] + lo[m]), c2 = rq[li + 1][m] - (lo[k] - hi[m]);
        const uint32_t u = v[k], w = v[m];
        v[k] = u + w + A.pm[c1 < 0 ? 0 : c1];
        v[m] = u - w + A.pm[c2 < 0 ? 0 : c2];
        const int xl = lo[k] + lo[m] + (c1 < 0 ? 0 : c1), xh = hi[k] + hi[m] + (c1 < 0 ? 0 : c1);
        const int yl = lo[k] - hi[m] + (c2 < 0 ? 0 : c2), yh = hi[k] - lo[m] + (c2 < 0 ? 0 : c2);
        lo[k] = xl, hi[k] = xh, lo[m] = yl, hi[m] = yh;
      } else {
        f1_bf<F3C>(v[k], v[m], A.lo[(16 >> li) * jb], A);
        lo[m] = lo[k] - 1, hi[m] = hi[k];
        hi[k] = hi[k] + 1;
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 8; ++c) X.put4(c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = X.get(k);
#pragma unroll
  for (int h = H0; h <= 8; h *= 2) {  // strided phase: len = G h
    const uint32_t* seg = tws + (h - 1) * G + j;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k & h) continue;
      f1_bf<F3S>(v[k], v[k + h], seg[(k & (h - 1)) * G], A);
    }
  }
  const uint32_t* seg = tws + 15 * G + j;
#pragma unroll
  for (int k = 0; k < 16; ++k) {  // len = N / 2: (u + w v) N^{-1}, (u - w v) N^{-1}, canonical
    const uint32_t a = mp_n16<true>(v[k], A.scale_lo, A.p);
    const uint32_t b = mp_n16<true>(v[k + 16], seg[k * G], A.p);
    const uint32_t s = a + b, d = a + A.p - b;
    v[k] = umin32(s, s - A.p);
    v[k + 16] = umin32(d, d - A.p);
  }
}

template <int LOGN, bool TRANSPOSE, bool MERGE>
__device__ __forceinline__ void stage_table(uint2* tws, const uint32_t* tab) {
  constexpr int N = 1 << LOGN, G = N / 32;
  const uint2* src = reinterpret_cast<const uint2*>(tab);
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    int dst = i;
    if (TRANSPOSE) {
#pragma unroll
      for (int s = 6; s <= LOGN; ++s) {
        const int b0 = seg_base<LOGN, MERGE>(s), size = 1 << (s - 1), c = size / G;
        if (i >= b0 && i < b0 + size) {
          const int b = i - b0;
          dst = b0 + (b % c) * G + b / c;
        }
      }
    }
    tws[dst] = src[i];
  }
}

// consumer warps of the N = 512 / 1024 forward: 16 (falcon512 improved -3 %, falcon1024
// harvey -12 %, improved +0.7 % vs 8, profiles/r1b_fastn_store.txt)
constexpr int kFwdConsN = 16;

template <class K, class IO, int LOGN, bool PER_INDEX, bool F1 = false>
__global__ void __launch_bounds__(GeoN<LOGN, IO, kFwdConsN>::kThreadsN)
    fwdn_tma_kernel(const IO* __restrict__ in, IO* __restrict__ out, size_t batch,
                    const uint32_t* __restrict__ tab, const __grid_constant__ FastArgs A) {
  using GN = GeoN<LOGN, IO, kFwdConsN>;
  constexpr int kConsumers = GN::kConsumers;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stages = smem;
  uint32_t* scratch = reinterpret_cast<uint32_t*>(smem + GN::kStages * GN::kStageBytes);
  uint2* tws = reinterpret_cast<uint2*>(scratch + kConsumers * GN::kScratchWords);
  uint64_t* full = reinterpret_cast<uint64_t*>(tws + GN::N);
  uint64_t* empty = full + GN::kStages;
  stage_table<LOGN, !PER_INDEX, false>(tws, tab);
  init_barriers(full, empty, GN::kStages, kConsumers);  // __syncthreads: table visible
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == kConsumers) {
    if (lane == 0) produce_n<LOGN, IO, kConsumers>(in, batch, stages, full, empty);
    return;
  }
  constexpr int G = GN::G;
  const int j = lane & (G - 1), half = GN::PPW == 2 ? lane >> 4 : 0;
  XposeN<G> X;
  X.init(scratch + warp * GN::kScratchWords + half * GN::kRegionWords, j);
  uint32_t E[6];  // F1: last-layer surplus corrections (fwd_body_n_f1)
  if constexpr (F1) {
    const int cj = LOGN - 2 - __popc(uint32_t(j) & ((1u << (LOGN - 6)) - 1u));
#pragma unroll
    for (int m = 0; m < 6; ++m) E[m] = pin(uint32_t(m - cj) * A.p);
  }
  const size_t ntiles = (batch + GN::kTileN - 1) / GN::kTileN;
  int it = 0;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int s = it % GN::kStages;
    const size_t poly = t * GN::kTileN + half * kConsumers + warp;
    mbar_wait(&full[s], (it / GN::kStages) & 1);
    uint32_t v[32];
    load_strided_n<IO, G, K::kSigned>(
        v, reinterpret_cast<const IO*>(stages + s * GN::kStageBytes + GN::poly_offset(warp, half)), j);
    release_stage(&empty[s], lane);
    if constexpr (F1)
      fwd_body_n_f1<K, LOGN>(v, tws, A, X, j, E);
    else
      fwd_body_n<K, LOGN, PER_INDEX>(v, tws, A, X, j);
    if constexpr (sizeof(IO) == 4)
      store_contiguous_n_coalesced<IO, G>(out + poly * GN::N, j, v, X, poly < batch);
    else if (poly < batch)
      store_contiguous_n<IO>(out + poly * GN::N, j, v);
  }
}

// MODE bits 0-1 -- 0: generic canonicalisation of the input words; 1: host-validated fast
// form.  MODE bit 2: lazy merge (policy kLazy, A.flags bit 3); bit 3: TW1 (A.flags bit 5);
// bit 5: narrow image (A.flags bit 9, inv_body_n_narrow); bit 6: CT-form narrow inverse (A.flags
// bit 11, inv_body_n_ct; the table is staged verbatim).
// Product forms of the CT-form inverse (f1_bf: Y' = 2 X - X' as an IADD3 or as an IMAD) in the
// contiguous / strided phase.  Measured (profiles/r2_ctn_inverse_ab.txt, ns/poly at 2^17):
// N = 512 IADD3 / IMAD 0.705 (IMAD / IADD3 0.722, all-IMAD 0.721, all-IADD3 0.722);
// N = 1024 IMAD / IADD3 1.405 (IADD3 / IMAD 1.426, all-IMAD 1.411, all-IADD3 1.439).
template <int LOGN>
constexpr bool ct_f3_contiguous() {
  return LOGN == 10;
}

template <class K, class IO, int LOGN, int MODE, int C = kConsumers>
__global__ void __launch_bounds__((C + 1) * 32)
    invn_tma_kernel(const IO* __restrict__ in, IO* __restrict__ out, size_t batch,
                    const uint32_t* __restrict__ tab, const __grid_constant__ FastArgs A,
                    const __grid_constant__ CUtensorMap tmap) {
  using GN = GeoN<LOGN, IO, C>;
  constexpr int kConsumers = C;
  constexpr bool SWZ = inv_swz<IO>();
  constexpr int kStageBytes = SWZ ? GN::kSwzStageBytes : GN::kStageBytes;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = SWZ ? smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u) : smem_raw;
  uint8_t* stages = smem;
  uint32_t* scratch = reinterpret_cast<uint32_t*>(smem + GN::kStages * kStageBytes);
  uint2* tws = reinterpret_cast<uint2*>(scratch + kConsumers * GN::kScratchWords);
  uint64_t* full = reinterpret_cast<uint64_t*>(tws + GN::N);
  uint64_t* empty = full + GN::kStages;
  stage_table<LOGN, (MODE & 64) == 0, true>(tws, tab);
  init_barriers(full, empty, GN::kStages, kConsumers);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == kConsumers) {
    if (lane == 0) {
      if constexpr (SWZ)
        produce_rows<GN::kBoxRows, GN::kStages, GN::kBoxes>(
            &tmap, static_cast<uint32_t>((batch + GN::kTileN - 1) / GN::kTileN), stages, full, empty);
      else
        produce_n<LOGN, IO, kConsumers>(in, batch, stages, full, empty);
    }
    return;
  }
  constexpr int G = GN::G;
  const int j = lane & (G - 1), half = GN::PPW == 2 ? lane >> 4 : 0;
  XposeN<G> X;
  X.init(scratch + warp * GN::kScratchWords + half * GN::kRegionWords, j);
  uint32_t soff[8];  // swizzled stage: polynomial half * 8 + warp, lane segment j
#pragma unroll
  for (int c = 0; c < 8; ++c)
    soff[c] = swz128(uint32_t((half * kConsumers + warp) * GN::kPolyBytes + j * 32 * int(sizeof(IO)) + 16 * c));
  const uint32_t sbase = smem_addr(stages);
  const size_t ntiles = (batch + GN::kTileN - 1) / GN::kTileN;
  int it = 0;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int s = it % GN::kStages;
    const size_t poly = t * GN::kTileN + half * kConsumers + warp;
    mbar_wait(&full[s], (it / GN::kStages) & 1);
    uint32_t v[32];
    if constexpr (SWZ)
      load_contiguous_n_swz<IO, K::kSigned>(v, sbase + s * kStageBytes, soff);
    else
      load_contiguous_n<IO, K::kSigned>(
          v, reinterpret_cast<const IO*>(stages + s * GN::kStageBytes + GN::poly_offset(warp, half)), j);
    release_stage(&empty[s], lane);
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = canon<IO, K::kSigned, (MODE & 3) == 1>(v[k], A);
    if constexpr ((MODE & 64) != 0)
      inv_body_n_ct<K, LOGN, ct_f3_contiguous<LOGN>(), !ct_f3_contiguous<LOGN>()>(v, reinterpret_cast<const uint32_t*>(tws), A, X, j);
    else if constexpr ((MODE & 32) != 0) inv_body_n_narrow<K, LOGN>(v, tws, A, X, j);
    else if constexpr ((MODE & 4) != 0) inv_body_n_lazy<K, LOGN, (MODE & 8) != 0>(v, tws, A, X, j);
    else inv_body_n<K, LOGN>(v, tws, A, X, j);
    store_strided_n<IO, G>(out + poly * GN::N, j, v, X, poly < batch);
  }
}

template <class Kern>
int grid_n(Kern kern, int smem, OccCache& occ, size_t tiles, int threads = kThreads) {
  const size_t full = size_t(sm_count_current()) * occupancy_current(kern, threads, smem, occ);
  return static_cast<int>(tiles < full ? tiles : full);
}

template <class K, class IO, int LOGN, bool PER_INDEX, bool F1>
cudaError_t fwd_n_f(const void* in, void* out, size_t batch, const uint32_t* tab, const FastArgs& A,
                    cudaStream_t st) {
  using GN = GeoN<LOGN, IO, kFwdConsN>;
  static OccCache occ;
  auto kern = fwdn_tma_kernel<K, IO, LOGN, PER_INDEX, F1>;
  const int blocks = grid_n(kern, GN::kSmem, occ, (batch + GN::kTileN - 1) / GN::kTileN, GN::kThreadsN);
  return launch_pdl(kern, blocks, GN::kThreadsN, GN::kSmem, st, static_cast<const IO*>(in), static_cast<IO*>(out),
                    batch, tab, A);
}

// consumer warps of the N = 512 / 1024 inverse (two 256-row tensor boxes per stage at 16)
constexpr int inv_cons_n() {
  return 16;
}

template <class K, class IO, int LOGN, bool PER_INDEX>
cudaError_t fwd_n(const void* in, void* out, size_t batch, const uint32_t* tab, const FastArgs& A,
                  cudaStream_t st) {
  if constexpr (std::is_same<K, ImprovedN16<false>>::value && !PER_INDEX) {
    if (A.flags & 1024) return fwd_n_f<K, IO, LOGN, PER_INDEX, true>(in, out, batch, tab, A, st);
  }
  return fwd_n_f<K, IO, LOGN, PER_INDEX, false>(in, out, batch, tab, A, st);
}

template <class K, class IO, int LOGN, int MODE>
cudaError_t inv_n_mode(const void* in, void* out, size_t batch, const uint32_t* tab,
                       const FastArgs& A, cudaStream_t st) {
  constexpr int C = inv_cons_n();
  using GN = GeoN<LOGN, IO, C>;
  static OccCache occ;
  auto kern = invn_tma_kernel<K, IO, LOGN, MODE, C>;
  constexpr bool SWZ = inv_swz<IO>();
  constexpr int smem = SWZ ? GN::kSwzSmem : GN::kSmem;
  // the swizzled input is addressed through a tensor map of <= kMaxMapRows rows
  constexpr size_t kMaxBatch = SWZ ? size_t(kMaxMapRows / GN::kRowsPerPoly) : ~size_t(0);
  for (size_t done = 0; done < batch;) {
    const size_t n = batch - done < kMaxBatch ? batch - done : kMaxBatch;
    const IO* src = static_cast<const IO*>(in) + done * GN::N;
    CUtensorMap map{};
    if constexpr (SWZ) {
      const cudaError_t e = make_rows128_map(&map, src, uint64_t(n) * GN::kRowsPerPoly, GN::kBoxRows);
      if (e != cudaSuccess) return e;
    }
    const int blocks = grid_n(kern, smem, occ, (n + GN::kTileN - 1) / GN::kTileN, GN::kThreadsN);
    const cudaError_t e = launch_pdl(kern, blocks, GN::kThreadsN, smem, st, src,
                                     static_cast<IO*>(out) + done * GN::N, n, tab, A, map);
    if (e != cudaSuccess) return e;
    done += n;
  }
  return cudaSuccess;
}

template <class K, class IO, int LOGN, int LZ>
cudaError_t inv_n_canon(const void* in, void* out, size_t batch, const uint32_t* tab,
                        const FastArgs& A, cudaStream_t st) {
  const unsigned fast_bit = sizeof(IO) == 2 ? 1u : 2u;
  if (!K::kSigned && (A.flags & fast_bit))
    return inv_n_mode<K, IO, LOGN, 1 | LZ>(in, out, batch, tab, A, st);
  return inv_n_mode<K, IO, LOGN, 0 | LZ>(in, out, batch, tab, A, st);
}

template <class K, class IO, int LOGN>
cudaError_t inv_n(const void* in, void* out, size_t batch, const uint32_t* tab, const FastArgs& A,
                  cudaStream_t st) {
  if constexpr (std::is_same<K, ImprovedN16<false>>::value) {
    if (A.flags & 2048) return inv_n_canon<K, IO, LOGN, 64>(in, out, batch, tab, A, st);  // CT form
    if (A.flags & 512) return inv_n_canon<K, IO, LOGN, 32>(in, out, batch, tab, A, st);  // narrow
  }
  if constexpr (lazy_of<K>::value) {
    if (A.flags & 8) {
      if (A.flags & 32) return inv_n_canon<K, IO, LOGN, 4 | 8>(in, out, batch, tab, A, st);
      return inv_n_canon<K, IO, LOGN, 4>(in, out, batch, tab, A, st);
    }
  }
  return inv_n_canon<K, IO, LOGN, 0>(in, out, batch, tab, A, st);
}

template <class K, bool PER_INDEX, class IO>
cudaError_t by_logn(int dir, int logn, const void* in, void* out, size_t batch, const uint32_t* tab,
                    const FastArgs& A, cudaStream_t st) {
  if (logn == 9)
    return dir == 0 ? fwd_n<K, IO, 9, PER_INDEX>(in, out, batch, tab, A, st)
                    : inv_n<K, IO, 9>(in, out, batch, tab, A, st);
  if (logn == 10)
    return dir == 0 ? fwd_n<K, IO, 10, PER_INDEX>(in, out, batch, tab, A, st)
                    : inv_n<K, IO, 10>(in, out, batch, tab, A, st);
  return cudaErrorInvalidValue;
}

template <class K, bool PER_INDEX>
cudaError_t by_elem(int dir, int logn, int elem, const void* in, void* out, size_t batch,
                    const uint32_t* tab, const FastArgs& A, cudaStream_t st) {
  if (elem == 2) return by_logn<K, PER_INDEX, uint16_t>(dir, logn, in, out, batch, tab, A, st);
  if (elem == 4) return by_logn<K, PER_INDEX, uint32_t>(dir, logn, in, out, batch, tab, A, st);
  return cudaErrorInvalidValue;
}

}  // namespace

bool fastn_supports(const HostParams& P, int elem_bytes, const void* in, const void* out) {
  return (P.N == 512 || P.N == 1024) && P.layers == P.log2N && (elem_bytes == 2 || elem_bytes == 4) &&
         !(reinterpret_cast<uintptr_t>(in) & 15) && !(reinterpret_cast<uintptr_t>(out) & 15);
}

cudaError_t fastn_launch(const HostParams& P, int kind, int dir, const void* in, void* out,
                         size_t batch, int elem_bytes, const uint32_t* tab, cudaStream_t st) {
  const FastArgs& A = P.fast[kind][dir];
  const int logn = static_cast<int>(P.log2N);
  const bool n16 = P.n_bits == 16, cyclic = P.tree == NTTK_CYCLIC;
  if (batch == 0) return cudaSuccess;
  switch (kind) {
    case NTTK_IMPROVED:
      if (P.image(kind, dir) == kNarrow || P.image(kind, dir) == kCtN)  // n = 32 parameters on the
        return by_elem<ImprovedN16<false>, false>(dir, logn, elem_bytes, in, out, batch, tab,  // n = 16 product
                                                  P.fast[P.image(kind, dir)][dir], st);
      return n16 ? by_elem<ImprovedN16<false>, false>(dir, logn, elem_bytes, in, out, batch, tab, A, st)
                 : by_elem<ImprovedN32, false>(dir, logn, elem_bytes, in, out, batch, tab, A, st);
    case NTTK_HARVEY:
      if (cyclic)
        return n16 ? by_elem<Harvey<16, false>, true>(dir, logn, elem_bytes, in, out, batch, tab, A, st)
                   : by_elem<Harvey<32, false>, true>(dir, logn, elem_bytes, in, out, batch, tab, A, st);
      return n16 ? by_elem<Harvey<16, true>, false>(dir, logn, elem_bytes, in, out, batch, tab, A, st)
                 : by_elem<Harvey<32, true>, false>(dir, logn, elem_bytes, in, out, batch, tab, A, st);
    case NTTK_SMONT:
      return n16 ? by_elem<Smont<16>, false>(dir, logn, elem_bytes, in, out, batch, tab, A, st)
                 : by_elem<Smont<32>, false>(dir, logn, elem_bytes, in, out, batch, tab, A, st);
    case NTTK_NTL:
      return n16 ? by_elem<Ntl<16>, true>(dir, logn, elem_bytes, in, out, batch, tab, A, st)
                 : by_elem<Ntl<32>, true>(dir, logn, elem_bytes, in, out, batch, tab, A, st);
    case NTTK_SCOTT:
      if (n16 || !cyclic) return cudaErrorInvalidValue;
      return by_elem<Scott32, true>(dir, logn, elem_bytes, in, out, batch, tab, A, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace nttk_b200
