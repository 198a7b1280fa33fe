// polymul_tma.cu -- fused batched polynomial product for N = 256 (sm_100a).
//
// c = inverse(product(forward(a), forward(b))) in ONE kernel: the reference's
// cyclic_convolution_via_ntt (transform.hpp:372-379 = ntt_forward x2, pointwise_multiply,
// intt_inverse) and its Kyber-style twin (7-layer negacyclic forward, degree-2 basemul,
// inverse with 2^{-7}), SURVEY §8(f) item 1.  One HBM round trip per product (Kyber u16:
// 1 536 B instead of 4 608 B for the four-kernel pipeline).
//
// The forward transform ends in contiguous ownership (lane j holds spectrum slots
// 16 j .. 16 j + 15) and the inverse starts there, so the product stage needs no data
// movement: slotwise products and the 8 degree-2 pairs of a lane are lane-local.  The
// product is canonical, so every kind's own reduction (Plantard, Montgomery, signed
// Montgomery -- the per-variant runs of BASELINE config 2) is bit-identical with the
// reference's canonical result.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "arith.cuh"
#include "fast256.hpp"
#include "launch_cache.hpp"
#include "tma_common.cuh"

namespace nttk_b200 {
namespace {

using namespace tma;

// Consumer warps per CTA of the fused polymul, per storage width (shadow tma::kConsumers in
// this file).  Measured (B200, config 2, tools/polymul_probe.py): one CTA of 16 consumers
// per SM for u16 lifts improved 1.07 -> 1.12, harvey 0.68 -> 0.71, smont 0.73 -> 0.78 G
// products/s; u32 keeps 8 (16 would cap its registers at 60 and spill).
template <class IO>
constexpr int pm_cons() {
  return sizeof(IO) == 2 ? 16 : 8;
}

// stage = a-tile and b-tile, each two halves of 8 polynomials (one bulk copy per half)
template <class IO>
struct Geo2 {
  static constexpr int kPolyBytes = 256 * int(sizeof(IO));
  static constexpr int kPad = sizeof(IO) == 2 ? 32 : 64;
  static constexpr int kConsumers = pm_cons<IO>();
  static constexpr int kHalfBytes = kConsumers * kPolyBytes;
  static constexpr int kTileBytes = 2 * kHalfBytes + kPad + 64;
  static constexpr int kStages = sizeof(IO) == 2 ? 3 : 2;
  static constexpr int kStageBytes = 2 * kTileBytes;
  static constexpr int kSmem = kStages * kStageBytes + kConsumers * kScratchWords * 4 +
                               2 * kStages * 8;
  __device__ static constexpr int poly_offset(int w, int h, int which) {
    return which * kTileBytes + h * (kHalfBytes + kPad) + w * kPolyBytes;
  }
};

template <class IO>
__device__ __forceinline__ void produce2(const IO* a, const IO* b, size_t batch, uint8_t* stages,
                                         uint64_t* full, uint64_t* empty) {
  using G = Geo2<IO>;
  constexpr int kConsumers = G::kConsumers, kTile = 2 * kConsumers;
  const size_t ntiles = (batch + kTile - 1) / kTile;
  int k = 0;
  pdl_wait();
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int s = k % G::kStages;
    if (k >= G::kStages) mbar_wait(&empty[s], ((k / G::kStages) & 1) ^ 1);
    const size_t first = t * kTile;
    const int n = batch - first < size_t(kTile) ? int(batch - first) : kTile;
    const int n0 = n < kConsumers ? n : kConsumers, n1 = n - n0;
    mbar_expect_tx(&full[s], 2u * uint32_t(n) * G::kPolyBytes);
    uint8_t* base = stages + s * G::kStageBytes;
    const IO* src[2] = {a, b};
    for (int which = 0; which < 2; ++which) {
      bulk_g2s(base + G::poly_offset(0, 0, which), src[which] + first * 256,
               uint32_t(n0) * G::kPolyBytes, &full[s]);
      if (n1 > 0)
        bulk_g2s(base + G::poly_offset(0, 1, which), src[which] + (first + kConsumers) * 256,
                 uint32_t(n1) * G::kPolyBytes, &full[s]);
    }
  }
}

// Lane twiddles of both directions are read from shared memory (TwSmem) instead of 15
// pinned registers each.  Measured (B200, config 2, tools/polymul_probe.py): both tables in
// shared memory (96 -> 72 registers, no spills) lifts improved 1.05 -> 1.07, harvey 0.666 ->
// 0.680, smont 0.695 -> 0.726 G products/s; with the tables in registers a register cap
// spills (0.99 G).  u32 storage caps registers for 2 CTAs per SM (its stages admit 2).
template <class IO>
constexpr int pm_minb() {
  return sizeof(IO) == 4 ? 2 : 1;
}

template <class K, class IO, int L, bool PER_INDEX, bool LAZY, bool W1, bool F1 = false>
__global__ void __launch_bounds__((pm_cons<IO>() + 1) * 32, pm_minb<IO>())
    polymul256_tma_kernel(const IO* __restrict__ a, const IO* __restrict__ b, IO* __restrict__ out,
                          size_t batch, const __grid_constant__ PolymulArgs PA) {
  using G = Geo2<IO>;
  constexpr int kConsumers = G::kConsumers, kTile = 2 * kConsumers;
  using Enc = typename K::Enc;
  using Tw = typename K::Tw;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stages = smem;
  uint32_t* scratch = reinterpret_cast<uint32_t*>(smem + G::kStages * G::kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(scratch + kConsumers * kScratchWords);
  uint64_t* empty = full + G::kStages;
  Tw* tws = reinterpret_cast<Tw*>(empty + G::kStages);  // [2][240] lane twiddles
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < 16) {
    Tw t[15];
    fwd_twiddles<K, L, PER_INDEX>(t, PA.fwd, threadIdx.x);
#pragma unroll
    for (int i = 0; i < 15; ++i) tws[16 * i + threadIdx.x] = t[i];
    inv_twiddles<K, L>(t, PA.inv, threadIdx.x);
#pragma unroll
    for (int i = 0; i < 15; ++i) tws[240 + 16 * i + threadIdx.x] = t[i];
  }
  init_barriers(full, empty, G::kStages, kConsumers);  // __syncthreads: tables visible
  if (warp == kConsumers) {
    if (lane == 0) produce2<IO>(a, b, batch, stages, full, empty);
    return;
  }
  const FastArgs& AF = PA.fwd;
  const FastArgs& AI = PA.inv;
  const int j = lane & 15, half = lane >> 4;
  uint32_t* S = scratch + warp * kScratchWords + half * 272;
  Xpose X;
  X.init(S, j);
  const TwSmem<Tw> twf{tws + j}, twi{tws + 240 + j};
  // basemul moduli of this lane's 8 pairs (k = 8 j + q)
  Enc gam[8];
  if (PA.prod.basemul) {
#pragma unroll
    for (int q = 0; q < 8; ++q) gam[q] = pin(K::genc(8 * j + q, PA.prod));
  }

  // F1 forwards: surplus (L - 1) p (fwd_body_f1_free)
  const uint32_t sp = pin(uint32_t(L - 1) * AF.p), sp1 = sp + AF.p;
  // 32-bit counters, stride pointer, incremental stage/phase (launcher splits >= 2^30)
  const uint32_t ntiles = static_cast<uint32_t>((batch + kTile - 1) / kTile);
  const uint32_t nb = static_cast<uint32_t>(batch), pstep = gridDim.x * kTile;
  uint32_t poly = blockIdx.x * kTile + half * kConsumers + warp, s = 0, phase = 0;
  IO* optr = out + size_t(poly) * 256;
  const size_t ostep = size_t(pstep) * 256;
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    mbar_wait(&full[s], phase);
    const uint8_t* base = stages + s * G::kStageBytes;
    uint32_t va[16], vb[16];
    load_strided<IO, K::kSigned>(va, reinterpret_cast<const IO*>(base + G::poly_offset(warp, half, 0)), j);
    load_strided<IO, K::kSigned>(vb, reinterpret_cast<const IO*>(base + G::poly_offset(warp, half, 1)), j);
    release_stage(&empty[s], lane);
    if constexpr (F1) {
      fwd_body_f1_free<K, L, W1>(va, twf, AF, X, sp, sp1);
      fwd_body_f1_free<K, L, W1>(vb, twf, AF, X, sp, sp1);
    } else {
      fwd_body<K, L, PER_INDEX, W1>(va, twf, AF, X);
      fwd_body<K, L, PER_INDEX, W1>(vb, twf, AF, X);
    }
    // product stage (contiguous ownership, canonical results in va)
    if (PA.prod.basemul) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const Enc e0 = K::enc(va[2 * q], PA.prod, AF), e1 = K::enc(va[2 * q + 1], PA.prod, AF);
        const uint32_t b0 = vb[2 * q], b1 = vb[2 * q + 1];
        const uint32_t t11 = K::mulc(b1, e1, AF);
        uint32_t c0 = K::mulc(b0, e0, AF) + K::mulc(t11, gam[q], AF);
        uint32_t c1 = K::mulc(b1, e0, AF) + K::mulc(b0, e1, AF);
        va[2 * q] = umin32(c0, c0 - AF.p);
        va[2 * q + 1] = umin32(c1, c1 - AF.p);
      }
    } else {
#pragma unroll
      for (int r = 0; r < 16; ++r) va[r] = K::mulc(vb[r], K::enc(va[r], PA.prod, AF), AF);
    }
    inv_body<K, L, false, LAZY>(va, twi, AI, X);
    store_strided<IO>(optr, j, va, S, X, poly < nb);
    poly += pstep;
    optr += ostep;
    if (++s == G::kStages) {
      s = 0;
      phase ^= 1;
    }
  }
}


// NTTK_POLYMUL_EAGER=1 runs the standalone-transform policies of harvey / smont inside the
// fused kernel (the A/B of the lazy twins; tests check both against the oracle)
bool eager_kinds() {
  static const bool v = [] {
    const char* e = std::getenv("NTTK_POLYMUL_EAGER");
    return e && e[0] == '1';
  }();
  return v;
}

template <auto KERN, class K, class IO>
cudaError_t launch_k(const void* a, const void* b, void* out, size_t batch, const PolymulArgs& PA,
                     cudaStream_t st) {
  static OccCache occ;
  auto kern = KERN;
  constexpr int smem = Geo2<IO>::kSmem + 480 * int(sizeof(typename K::Tw));
  constexpr int kThreads = (Geo2<IO>::kConsumers + 1) * 32, kTile = 2 * Geo2<IO>::kConsumers;
  const int g_sms2 = sm_count_current();
  const int o = occupancy_current(kern, kThreads, smem, occ);
  const size_t tiles = (batch + kTile - 1) / kTile;
  const size_t full = size_t(g_sms2) * o;
  const int blocks = static_cast<int>(tiles < full ? tiles : full);
  return launch_pdl(kern, blocks, kThreads, smem, st, static_cast<const IO*>(a), static_cast<const IO*>(b),
                    static_cast<IO*>(out), batch, PA);
}

template <class K, class IO, int L, bool PER_INDEX, bool LAZY, bool W1>
cudaError_t launch_lz(const void* a, const void* b, void* out, size_t batch, const PolymulArgs& PA,
                      cudaStream_t st) {
  if constexpr (std::is_same<K, ImprovedN16<false>>::value && !PER_INDEX) {
    if (PA.prod.lazy && !eager_kinds())
      return launch_k<polymul256_tma_kernel<K, IO, L, PER_INDEX, LAZY, W1, true>, K, IO>(a, b, out, batch, PA, st);
  }
  return launch_k<polymul256_tma_kernel<K, IO, L, PER_INDEX, LAZY, W1, false>, K, IO>(a, b, out, batch, PA, st);
}

template <class K, class IO, int L, bool PER_INDEX>
cudaError_t launch(const void* a, const void* b, void* out, size_t batch, const PolymulArgs& PA,
                   cudaStream_t st) {
  if constexpr (w1_of<K>::value && !PER_INDEX) {
    if (PA.fwd.flags & 16) {
      if constexpr (lazy_of<K>::value) {
        if (PA.inv.flags & 8) return launch_lz<K, IO, L, PER_INDEX, true, true>(a, b, out, batch, PA, st);
      }
      return launch_lz<K, IO, L, PER_INDEX, false, true>(a, b, out, batch, PA, st);
    }
  }
  if constexpr (lazy_of<K>::value) {
    if (PA.inv.flags & 8) return launch_lz<K, IO, L, PER_INDEX, true, false>(a, b, out, batch, PA, st);
  }
  return launch_lz<K, IO, L, PER_INDEX, false, false>(a, b, out, batch, PA, st);
}

template <class K, bool PER_INDEX>
cudaError_t by_io(int L, int elem, const void* a, const void* b, void* out, size_t batch,
                  const PolymulArgs& PA, cudaStream_t st) {
  if (elem == 2) {
    if (L == 8) return launch<K, uint16_t, 8, PER_INDEX>(a, b, out, batch, PA, st);
    if (L == 7) return launch<K, uint16_t, 7, PER_INDEX>(a, b, out, batch, PA, st);
  } else if (elem == 4) {
    if (L == 8) return launch<K, uint32_t, 8, PER_INDEX>(a, b, out, batch, PA, st);
    if (L == 7) return launch<K, uint32_t, 7, PER_INDEX>(a, b, out, batch, PA, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t polymul256_launch_one(const HostParams& P, int kind, const void* a, const void* b,
                                  void* out, size_t batch, int elem_bytes, cudaStream_t st);

cudaError_t polymul256_launch(const HostParams& P, int kind, const void* a, const void* b,
                              void* out, size_t batch, int elem_bytes, cudaStream_t st) {
  constexpr size_t kMax = size_t(1) << 30;  // the kernel counts polynomials in 32 bits
  const size_t bytes = size_t(256) * elem_bytes;
  for (size_t done = 0; done < batch;) {
    const size_t n = batch - done < kMax ? batch - done : kMax;
    const cudaError_t e = polymul256_launch_one(
        P, kind, static_cast<const char*>(a) + done * bytes, static_cast<const char*>(b) + done * bytes,
        static_cast<char*>(out) + done * bytes, n, elem_bytes, st);
    if (e != cudaSuccess) return e;
    done += n;
  }
  return cudaSuccess;
}

cudaError_t polymul256_launch_one(const HostParams& P, int kind, const void* a, const void* b,
                                  void* out, size_t batch, int elem_bytes, cudaStream_t st) {
  if (batch == 0) return cudaSuccess;
  PolymulArgs PA;
  PA.fwd = P.fast[kind][0];
  PA.inv = P.fast[kind][1];
  PA.prod = P.prod[kind];
  const int L = static_cast<int>(P.layers);
  const bool n16 = P.n_bits == 16, cyclic = P.tree == NTTK_CYCLIC;
  switch (kind) {
    case NTTK_IMPROVED:
      return n16 ? by_io<ImprovedN16<false>, false>(L, elem_bytes, a, b, out, batch, PA, st)
                 : by_io<ImprovedN32, false>(L, elem_bytes, a, b, out, batch, PA, st);
    case NTTK_HARVEY:
      if (cyclic)
        return n16 ? by_io<Harvey<16, false>, true>(L, elem_bytes, a, b, out, batch, PA, st)
                   : by_io<Harvey<32, false>, true>(L, elem_bytes, a, b, out, batch, PA, st);
      if (n16 && PA.prod.lazy && elem_bytes == 2 && !eager_kinds())
        return by_io<HarveyLazy16, false>(L, elem_bytes, a, b, out, batch, PA, st);
      return n16 ? by_io<Harvey<16, true>, false>(L, elem_bytes, a, b, out, batch, PA, st)
                 : by_io<Harvey<32, true>, false>(L, elem_bytes, a, b, out, batch, PA, st);
    case NTTK_SMONT:
      if (n16 && PA.prod.lazy && elem_bytes == 2 && !eager_kinds())
        return by_io<SmontLazy16, false>(L, elem_bytes, a, b, out, batch, PA, st);
      return n16 ? by_io<Smont<16>, false>(L, elem_bytes, a, b, out, batch, PA, st)
                 : by_io<Smont<32>, false>(L, elem_bytes, a, b, out, batch, PA, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace nttk_b200
