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
#include <cstdlib>
#include <type_traits>

#include "arith.cuh"
#include "fast256.hpp"
#include "launch_cache.hpp"
#include "tensor_map.hpp"
#include "tma_common.cuh"

namespace nttk_b200 {
namespace {

using namespace tma;

// Consumer warps per CTA (cons_of below).  Measured (B200, round 1,
// profiles/r1b_consumer_sweep.txt, r1b_consumer_batch.txt): 12 consumers (2 CTAs/SM: 24
// consumer warps, 2 producer warps instead of 3) beat 8 for the improved u16 cyclic forward
// (0.994 -> 0.983 ms); one CTA of 16 consumers per SM beats both for the improved inverses
// (u16 1.123 -> 1.088 -> 1.026 ms, u32 0.872 -> 0.862 -> 0.824 ms; the u32 tile is then one
// 256-row tensor box).  The u32 forward keeps 8 at 3 CTAs/SM (12: 0.776 -> 0.826), the
// 7-layer negacyclic forward keeps 8 at every batch size (4096 polys 5.5 -> 4.2 us), and the
// other kinds keep 8: most use 79-128 registers, where more consumers leave fewer warps.
// The u32 forward writes its output through the transpose tile with coalesced stores
// (Dilithium forward 0.777 -> 0.748 ms, profiles/r1b_store_variants.txt); the compute-bound
// u16 forward stores straight from registers (its coalesced twin measured 0.982 -> 0.999 ms).
// Consumer counts: 12 for the improved u16 cyclic W1 forward, 16 (one 94-register CTA per
// SM: 0.748 -> 0.695 ms; 12 or 20: 0.743) for the improved u32 cyclic W1 forward, 16 for
// every inverse (improved u16 1.039 -> 1.026 ms vs 12, 20 equal, 24 / 26 slower; u32 0.836
// -> 0.824 ms vs 12, 14: 0.918; the comparison kinds gain 2-11 %), 8 otherwise.
template <class K, class IO, int DIR, int L = 8, bool W1 = true>
struct cons_of {
  static constexpr bool kN16 = std::is_same<K, ImprovedN16<false>>::value && sizeof(IO) == 2;
  static constexpr int value =
      kN16 && W1 && DIR == 0 && L == 8                                                   ? 12
      : sizeof(IO) == 4 && DIR == 0 && std::is_same<K, ImprovedN32>::value && L == 8 && W1 ? 16
      : DIR == 1                                                                         ? 16
                                                                                         : kConsumers;
};
template <class K, class IO, int DIR, int L = 8, bool W1 = true>
using GeoK = Geo<IO, DIR, cons_of<K, IO, DIR, L, W1>::value>;
template <class K, class IO, int DIR>
using GeoSwzK = GeoSwz<IO, DIR, cons_of<K, IO, DIR>::value>;

// ---------------------------------------------------------------------------
template <class K, class IO, int L, bool PER_INDEX, bool W1, bool F1 = false>
__global__ void __launch_bounds__(GeoK<K, IO, 0, L, W1>::kThreadsP,
                                  GeoK<K, IO, 0, L, W1>::kC >= 16 ? 1 : fwd_minb<IO>())
    fwd256_tma_kernel(const IO* __restrict__ in, IO* __restrict__ out, size_t batch,
                      const __grid_constant__ FastArgs A) {
  using G = GeoK<K, IO, 0, L, W1>;
  constexpr int kConsumers = G::kC, kTile = G::kTileP;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stages = smem;
  uint32_t* scratch = reinterpret_cast<uint32_t*>(smem + G::kStages * G::kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(scratch + kConsumers * kScratchWords);
  uint64_t* empty = full + G::kStages;
  using Tw = typename K::Tw;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  init_barriers(full, empty, G::kStages, kConsumers);
  if (warp == kConsumers) {
    if (lane == 0) produce<IO, 0, kConsumers>(in, batch, stages, full, empty);
    return;
  }
  const int j = lane & 15, half = lane >> 4;
  Xpose X;
  X.init(scratch + warp * kScratchWords + half * 272, j);
  // u16 output 32-byte aligned: one 256-bit store per lane (store_contiguous; Kyber forward
  // 0.888 -> 0.878 ms, profiles/r2_stg256_ab.txt); a 16-byte aligned buffer keeps the two 128-bit stores
  const bool al32 = (reinterpret_cast<uintptr_t>(out) & 31) == 0;
  // F1: per-lane surplus corrections E[m] = (m - cj) p of the last layer (fwd_body_f1)
  uint32_t E[5];
  if constexpr (F1) {
    const int cj = L == 8 ? int(kF1Surplus) - ((j >> 3) & (j >> 2) & 1) - ((j >> 1) & 1) - (j & 1)
                          : int(kF1SurplusNega7) - __popc(uint32_t(j) & 7u);  // fwd_body_f1_nega7
#pragma unroll
    for (int m = 0; m < 5; ++m) E[m] = pin(uint32_t(m - cj) * A.p);
  }
  auto run = [&](const auto& twl) {
    // 32-bit tile/poly counters (the launcher splits batches >= 2^31), a stride pointer for
    // the output and incremental stage/phase: loop bookkeeping off the 64-bit datapath
    const uint32_t ntiles = static_cast<uint32_t>((batch + kTile - 1) / kTile);
    const uint32_t nb = static_cast<uint32_t>(batch), pstep = gridDim.x * kTile;
    uint32_t poly = blockIdx.x * kTile + half * kConsumers + warp, s = 0, phase = 0;
    IO* optr = out + size_t(poly) * 256;
    const size_t ostep = size_t(pstep) * 256;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      mbar_wait(&full[s], phase);
      uint32_t v[16];
      load_strided<IO, K::kSigned>(
          v, reinterpret_cast<const IO*>(stages + s * G::kStageBytes + G::poly_offset(warp, half)), j);
      release_stage(&empty[s], lane);
      if constexpr (F1 && L == 8)
        fwd_body_f1<K>(v, twl, A, X, E);
      else if constexpr (F1)
        fwd_body_f1_nega7<K>(v, twl, A, X, E);
      else
        fwd_body<K, L, PER_INDEX, W1>(v, twl, A, X);
      if constexpr (sizeof(IO) == 4)
        store_contiguous_coalesced(reinterpret_cast<uint32_t*>(optr), j, v, X,
                                   scratch + warp * kScratchWords + half * 272, poly < nb);
      else if (poly < nb)
        store_contiguous<IO>(optr, j, v, al32);
      poly += pstep;
      optr += ostep;
      if (++s == G::kStages) {
        s = 0;
        phase ^= 1;
      }
    }
  };
  Tw twl[15];
  fwd_twiddles<K, L, PER_INDEX>(twl, A, j);
  run(twl);
}

// u16 DEFER inverse: first merge layer from packed words with dp2a (Kyber inverse 1.088 ->
// 1.040 ms, profiles/r1b_idp.txt)

// ---------------------------------------------------------------------------
// MODE bits 0-1 -- 0: generic canonicalisation; 1: host-validated fast canonicalisation
// (A.flags bits 0/1); 2: u16 input with the fused first merge layer (A.flags bit 2,
// improved n=16); 3: u32 partial canonicalisation to [0, 2p) with doubled merge offsets
// (A.flags bit 7, lazy improved n=32).  MODE bit 2: lazy merge outputs (A.flags bit 3, improved).  Bit 3: TW1
// multiply-free block-0 merges (A.flags bit 5); bit 4: DEFER, no input canonicalisation
// (A.flags bit 6, u16 improved n=16) -- see inv_body_lazy.  Bit 5: narrow image
// (A.flags bit 9, ImprovedN16 on n = 32 parameters) -- see inv_body_narrow.
template <class K, class IO, int L, int MODE>
__global__ void __launch_bounds__(GeoK<K, IO, 1>::kThreadsP, 1)
    inv256_tma_kernel(const IO* __restrict__ in, IO* __restrict__ out, size_t batch,
                      const __grid_constant__ FastArgs A, const __grid_constant__ CUtensorMap tmap) {
  using G = GeoK<K, IO, 1>;
  using GS = GeoSwzK<K, IO, 1>;
  constexpr int kConsumers = G::kC, kTile = G::kTileP;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // SWIZZLE_128B destinations must be 1024-byte aligned (GS::kSmem carries the slack)
  uint8_t* smem = inv_swz<IO>() ? smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u) : smem_raw;
  constexpr int kStageBytes = inv_swz<IO>() ? GS::kStageBytes : G::kStageBytes;
  uint8_t* stages = smem;
  uint32_t* scratch = reinterpret_cast<uint32_t*>(smem + G::kStages * kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(scratch + kConsumers * kScratchWords);
  uint64_t* empty = full + G::kStages;
  using Tw = typename K::Tw;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  init_barriers(full, empty, G::kStages, kConsumers);
  if (warp == kConsumers) {
    if (lane == 0) {
      if constexpr (inv_swz<IO>())
        produce_rows<GS::kBoxRows, G::kStages>(&tmap, static_cast<uint32_t>((batch + kTile - 1) / kTile),
                                               stages, full, empty);
      else
        produce<IO, 1, kConsumers>(in, batch, stages, full, empty);
    }
    return;
  }
  const int j = lane & 15, half = lane >> 4;
  uint32_t* S = scratch + warp * kScratchWords + half * 272;
  Xpose X;
  X.init(S, j);
  // swizzled stage: polynomial half * 8 + warp of the tile, lane segment j (16 coefficients)
  uint32_t soff[4];
#pragma unroll
  for (int c = 0; c < 4; ++c)
    soff[c] = swz128(uint32_t((half * kConsumers + warp) * G::kPolyBytes + j * 16 * int(sizeof(IO)) + 16 * c));
  const uint32_t sbase = smem_addr(stages);
  auto run = [&](const auto& twl) {
    const uint32_t ntiles = static_cast<uint32_t>((batch + kTile - 1) / kTile);
    const uint32_t nb = static_cast<uint32_t>(batch), pstep = gridDim.x * kTile;
    uint32_t poly = blockIdx.x * kTile + half * kConsumers + warp, s = 0, phase = 0;
    IO* optr = out + size_t(poly) * 256;
    const size_t ostep = size_t(pstep) * 256;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      mbar_wait(&full[s], phase);
      uint32_t v[16];
      constexpr bool kPacked = (MODE & 16) && sizeof(IO) == 2 && !inv_swz<IO>();
      if constexpr (kPacked) {  // raw packed words in v[8..15] (inv_body_lazy PACKED)
        const uint4* src = reinterpret_cast<const uint4*>(stages + s * G::kStageBytes + G::poly_offset(warp, half)) + 2 * j;
        const uint4 a = src[0], b = src[1];
        v[8] = a.x, v[9] = a.y, v[10] = a.z, v[11] = a.w, v[12] = b.x, v[13] = b.y, v[14] = b.z, v[15] = b.w;
      } else if constexpr (inv_swz<IO>()) {
        load_contiguous_swz<IO, K::kSigned>(v, sbase + s * kStageBytes, soff);
      } else {
        load_contiguous<IO, K::kSigned>(
            v, reinterpret_cast<const IO*>(stages + s * G::kStageBytes + G::poly_offset(warp, half)), j);
      }
      release_stage(&empty[s], lane);
      constexpr int CM = MODE & 3;
      if constexpr (CM == 3) {  // partial: [0, 2p) without the conditional subtraction
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = v[r] + (v[r] >> A.cs_s) * A.negp;
      } else if (CM != 2) {
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = canon<IO, K::kSigned, CM == 1>(v[r], A);
      }
      if constexpr ((MODE & 64) != 0) {
        if constexpr (std::is_same<K, ImprovedN32>::value) inv_body_ct32(v, twl, A, X);
        else inv_body_ct<kPacked>(v, twl, A, X);
      }
      else if constexpr ((MODE & 32) != 0)
        inv_body_narrow<K, L>(v, twl, A, X);
      else
        inv_body<K, L, CM == 2, (MODE & 4) != 0, (MODE & 8) != 0, (MODE & 16) != 0, kPacked, CM == 3 ? 1 : 0>(
            v, twl, A, X);
      store_strided<IO>(optr, j, v, S, X, poly < nb);
      poly += pstep;
      optr += ostep;
      if (++s == G::kStages) {
        s = 0;
        phase ^= 1;
      }
    }
  };
  Tw twl[15];
  if constexpr ((MODE & 64) != 0 && !std::is_same<K, ImprovedN32>::value)
    ct_twiddles<K>(twl, A, j);
  else if constexpr ((MODE & 64) != 0)
    ct_twiddles32(twl, A, j);
  else
    inv_twiddles<K, L>(twl, A, j);
  run(twl);
}

// ---------------------------------------------------------------------------
// A/B switch while the F1 forward is measured (NTTK_FWD_F1=0 runs the umulhi form)
bool f1_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("NTTK_FWD_F1");
    return !(e && e[0] == '0');
  }();
  return v;
}

template <class Kern>
int grid_for(Kern kern, int threads, int tile, int smem, OccCache& occ, size_t batch) {
  const int o = occupancy_current(kern, threads, smem, occ);
  const int g_sms = sm_count_current();
  const size_t tiles = (batch + tile - 1) / tile;
  const size_t full = size_t(g_sms) * o;
  return static_cast<int>(tiles < full ? tiles : full);
}

template <class K, class IO, int L, bool PER_INDEX, bool W1, bool F1 = false>
cudaError_t fwd_launch_w(const void* in, void* out, size_t batch, const FastArgs& A,
                         cudaStream_t st) {
  static OccCache occ;
  auto kern = fwd256_tma_kernel<K, IO, L, PER_INDEX, W1, F1>;
  constexpr int smem = GeoK<K, IO, 0, L, W1>::kSmem;
  using G = GeoK<K, IO, 0, L, W1>;
  const int blocks = grid_for(kern, G::kThreadsP, G::kTileP, smem, occ, batch);
  return launch_pdl(kern, blocks, G::kThreadsP, smem, st, static_cast<const IO*>(in), static_cast<IO*>(out),
                    batch, A);
}

template <class K, class IO, int L, bool PER_INDEX>
cudaError_t fwd_launch(const void* in, void* out, size_t batch, const FastArgs& A, cudaStream_t st) {
  if constexpr (w1_of<K>::value && !PER_INDEX) {
    if constexpr (std::is_same<K, ImprovedN16<false>>::value && L == 8) {
      if ((A.flags & 1024) && f1_enabled())
        return fwd_launch_w<K, IO, L, PER_INDEX, true, true>(in, out, batch, A, st);
    }
    if constexpr (std::is_same<K, ImprovedN16<false>>::value && L == 7) {  // negacyclic: no W1
      if ((A.flags & 1024) && !(A.flags & 16) && f1_enabled())
        return fwd_launch_w<K, IO, L, PER_INDEX, false, true>(in, out, batch, A, st);
    }
    if (A.flags & 16) return fwd_launch_w<K, IO, L, PER_INDEX, true>(in, out, batch, A, st);
  }
  return fwd_launch_w<K, IO, L, PER_INDEX, false>(in, out, batch, A, st);
}

template <class K, class IO, int L, int MODE>
cudaError_t inv_launch_mode(const void* in, void* out, size_t batch, const FastArgs& A,
                            cudaStream_t st) {
  static OccCache occ;
  auto kern = inv256_tma_kernel<K, IO, L, MODE>;
  constexpr int smem = inv_swz<IO>() ? GeoSwzK<K, IO, 1>::kSmem : GeoK<K, IO, 1>::kSmem;
  CUtensorMap map{};
  if constexpr (inv_swz<IO>()) {
    const cudaError_t e = make_rows128_map(&map, in, uint64_t(batch) * GeoSwzK<K, IO, 1>::kRowsPerPoly,
                                           GeoSwzK<K, IO, 1>::kBoxRows);
    if (e != cudaSuccess) return e;
  }
  using G = GeoK<K, IO, 1>;
  const int blocks = grid_for(kern, G::kThreadsP, G::kTileP, smem, occ, batch);
  return launch_pdl(kern, blocks, G::kThreadsP, smem, st, static_cast<const IO*>(in), static_cast<IO*>(out),
                    batch, A, map);
}

template <class K, class IO, int L, int LZ>
cudaError_t inv_launch_canon(const void* in, void* out, size_t batch, const FastArgs& A,
                             cudaStream_t st) {
  constexpr bool kCanFuse = sizeof(IO) == 2 && std::is_same<K, ImprovedN16<false>>::value;
  const unsigned fast_bit = sizeof(IO) == 2 ? 1u : 2u;
  if (kCanFuse && (A.flags & 4)) return inv_launch_mode<K, IO, L, (kCanFuse ? 2 : 1) | LZ>(in, out, batch, A, st);
  // partial canonicalisation (lazy improved n = 32 on u32, A.flags bit 7)
  constexpr bool kPartial = sizeof(IO) == 4 && std::is_same<K, ImprovedN32>::value && (LZ & 4);
  if (kPartial && (A.flags & 128)) return inv_launch_mode<K, IO, L, (kPartial ? 3 : 1) | LZ>(in, out, batch, A, st);
  if (!K::kSigned && (A.flags & fast_bit)) return inv_launch_mode<K, IO, L, 1 | LZ>(in, out, batch, A, st);
  return inv_launch_mode<K, IO, L, 0 | LZ>(in, out, batch, A, st);
}

template <class K, class IO, int L>
cudaError_t inv_launch(const void* in, void* out, size_t batch, const FastArgs& A, cudaStream_t st) {
  if constexpr (std::is_same<K, ImprovedN16<false>>::value) {
    if (A.flags & 512)  // narrow image (n = 32 parameters on the n = 16 product)
      return (A.flags & (sizeof(IO) == 2 ? 1u : 2u)) ? inv_launch_mode<K, IO, L, 32 | 1>(in, out, batch, A, st)
                                                     : inv_launch_mode<K, IO, L, 32>(in, out, batch, A, st);
  }
  if constexpr (lazy_of<K>::value) {
    if (A.flags & 8) {
      if constexpr (L == 8) {
        // DEFER: u16 improved n = 16 with the fused first layer (flags 4 | 64)
        constexpr bool kDefer = sizeof(IO) == 2 && std::is_same<K, ImprovedN16<false>>::value;
        if (kDefer && (A.flags & 64) && (A.flags & 4))
          return (A.flags & 32) ? inv_launch_mode<K, IO, L, kDefer ? (2 | 4 | 8 | 16) : 4>(in, out, batch, A, st)
                                : inv_launch_mode<K, IO, L, kDefer ? (2 | 4 | 16) : 4>(in, out, batch, A, st);
        if (A.flags & 32) return inv_launch_canon<K, IO, L, 4 | 8>(in, out, batch, A, st);
      }
      return inv_launch_canon<K, IO, L, 4>(in, out, batch, A, st);
    }
  }
  if constexpr (inv_w1_of<K>::value && L == 8) {  // harvey / ntl: TW1 on the eager body
    if (A.flags & 32) return inv_launch_canon<K, IO, L, 8>(in, out, batch, A, st);
  }
  return inv_launch_canon<K, IO, L, 0>(in, out, batch, A, st);
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

cudaError_t fast256_tma_launch_one(const HostParams& P, int kind, int dir, const void* in,
                                   void* out, size_t batch, int elem_bytes, cudaStream_t st);

// the kernels count polynomials in 32 bits and the inverse addresses its input through a
// tensor map of at most kMaxMapRows 128-byte rows (8 per u32 polynomial): launches of at
// most 2^27 polynomials (more than any B200 holds at N = 256, kept for safety)
cudaError_t fast256_tma_launch(const HostParams& P, int kind, int dir, const void* in, void* out,
                               size_t batch, int elem_bytes, cudaStream_t st) {
  constexpr size_t kMax = size_t(1) << 27;
  const size_t bytes = size_t(256) * elem_bytes;
  for (size_t done = 0; done < batch;) {
    const size_t n = batch - done < kMax ? batch - done : kMax;
    const cudaError_t e = fast256_tma_launch_one(P, kind, dir, static_cast<const char*>(in) + done * bytes,
                                                 static_cast<char*>(out) + done * bytes, n, elem_bytes, st);
    if (e != cudaSuccess) return e;
    done += n;
  }
  return cudaSuccess;
}

cudaError_t fast256_tma_launch_one(const HostParams& P, int kind, int dir, const void* in,
                                   void* out, size_t batch, int elem_bytes, cudaStream_t st) {
  const FastArgs& A = P.fast[kind][dir];
  const int L = static_cast<int>(P.layers);
  const bool n16 = P.n_bits == 16;
  const bool cyclic = P.tree == NTTK_CYCLIC;
  if (batch == 0) return cudaSuccess;
  switch (kind) {
    case NTTK_IMPROVED:
      if (dir == 1 && P.ct_inv && ct_inverse_enabled()) {  // CT-form inverses (Kyber u16, Dilithium u32)
        if (n16 && elem_bytes == 2)
          return inv_launch_mode<ImprovedN16<false>, uint16_t, 8, 64 | 16 | 2>(in, out, batch, P.fast_ctinv, st);
        if (!n16 && elem_bytes == 4)
          return inv_launch_mode<ImprovedN32, uint32_t, 8, 64 | 3>(in, out, batch, P.fast_ctinv, st);
      }
      // canonicalised u32 words through the n = 16 CT body (n = 16 sets in u32 storage, and the
      // narrow image of an n = 32 set: the kyber256 preset)
      if (dir == 1 && P.ct_inv_c && elem_bytes == 4 && ct_inverse_enabled() &&
          (n16 || P.image(kind, dir) == kNarrow))
        return (P.fast_ctinv_c.flags & 2u)
                   ? inv_launch_mode<ImprovedN16<false>, uint32_t, 8, 64 | 1>(in, out, batch, P.fast_ctinv_c, st)
                   : inv_launch_mode<ImprovedN16<false>, uint32_t, 8, 64>(in, out, batch, P.fast_ctinv_c, st);
      if (P.image(kind, dir) == kNarrow)  // n = 32 parameters on the n = 16 product
        return by_io<ImprovedN16<false>, false>(dir, L, elem_bytes, in, out, batch,
                                                P.fast[kNarrow][dir], st);
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
    case NTTK_NTL:
      return n16 ? by_io<Ntl<16>, true>(dir, L, elem_bytes, in, out, batch, A, st)
                 : by_io<Ntl<32>, true>(dir, L, elem_bytes, in, out, batch, A, st);
    case NTTK_SCOTT:
      if (n16 || !cyclic) return cudaErrorInvalidValue;
      return by_io<Scott32, true>(dir, L, elem_bytes, in, out, batch, A, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace nttk_b200
