// product.cu -- standalone slotwise product and degree-2 basemul of two spectra (sm_100a).
//
// pointwise_multiply (transform.hpp:349-370) and the basemul extension
// produce canonical slots, so any exact product is bit-identical with the reference.
// These kernels use each kind's own 32-bit reduction -- the same `enc` / `mulc` policy
// pair as the fused polymul's product stage (arith.cuh): modified Plantard for `improved`
// (the lhs is re-encoded like the reference's to_plantard_domain(lhs % p), then
// MP(w, rhs)), Montgomery for `harvey`, signed Montgomery for `smont` -- on u16 / u32
// storage with 128-bit vector loads and stores (8 or 4 slots per vector; a basemul pair
// never straddles a vector).  Inputs are canonicalised first (any storage word is
// accepted), so lazy forward spectra and arbitrary words give the canonical product.
//
// Algorithmic HBM bytes per slot: 3 x storage width (lhs + rhs in, product out); the
// kernels are HBM-bound (a few IMADs per slot), grid = SMs x resident CTAs, grid-stride.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "arith.cuh"
#include "launch_cache.hpp"
#include "product.hpp"
#include "tma_common.cuh"

namespace nttk_b200 {
namespace {

struct ProductArgs {
  FastArgs A;   // forward-direction constants of the kind (p, canonicalisation constants)
  ProdArgs Q;   // multiplier encodings and basemul moduli
};

template <class IO, bool SGN>
__device__ __forceinline__ uint32_t canon_word(uint32_t x, const FastArgs& A) {
  if (SGN) return mod_s32(x, A);
  if constexpr (sizeof(IO) == 2) return mod_u16(x, A);  // exact for every 16-bit word
  return mod_u32(x, A);
}

template <class IO>
struct Vec {
  static constexpr int kSlots = 16 / int(sizeof(IO));
};

// unpack one 16-byte vector into kSlots 32-bit words (sign-extended for signed kinds)
template <class IO, bool SGN>
__device__ __forceinline__ void unpack(const uint4& q, uint32_t (&v)[Vec<IO>::kSlots]) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
  if constexpr (sizeof(IO) == 2) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[2 * e] = tma::widen<uint16_t, SGN>(static_cast<uint16_t>(w[e] & 0xffffu));
      v[2 * e + 1] = tma::widen<uint16_t, SGN>(static_cast<uint16_t>(w[e] >> 16));
    }
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = w[e];
  }
}

template <class IO>
__device__ __forceinline__ uint4 pack(const uint32_t (&v)[Vec<IO>::kSlots]) {
  if constexpr (sizeof(IO) == 2)
    return make_uint4(__byte_perm(v[0], v[1], 0x5410), __byte_perm(v[2], v[3], 0x5410),
                      __byte_perm(v[4], v[5], 0x5410), __byte_perm(v[6], v[7], 0x5410));
  else
    return make_uint4(v[0], v[1], v[2], v[3]);
}

// Whether the storage words must be canonicalised before the kind's product.  The modified
// Plantard product is exact for every storage word (n = 16: w T < 2^32 for T < 2^16; n = 32:
// w T < 2^32 (2^32 - p) for T < 2^32), and so is the signed Montgomery product for 16-bit
// words (|w y| < p 2^15); the Montgomery (harvey) product and 32-bit signed words need
// canonical operands.
template <class K, class IO>
constexpr bool needs_canon() {
  if (std::is_same<K, ImprovedN16<false>>::value) return sizeof(IO) == 4;
  if (std::is_same<K, ImprovedN32>::value) return false;
  if (K::kSigned) return sizeof(IO) == 4;
  return true;
}

// one vector of slots; gam[q]: the basemul modulus of the vector's pair q (per thread:
// the grid stride is a multiple of N / 2 pairs, so a thread always sees the same pairs)
template <class K, class IO, bool BASEMUL>
__device__ __forceinline__ uint4 product_vec(const uint4& ql, const uint4& qr,
                                             const typename K::Enc (&gam)[Vec<IO>::kSlots / 2],
                                             const ProductArgs& P) {
  constexpr int S = Vec<IO>::kSlots;
  using Enc = typename K::Enc;
  uint32_t a[S], b[S];
  unpack<IO, K::kSigned>(ql, a);
  unpack<IO, K::kSigned>(qr, b);
  if constexpr (needs_canon<K, IO>()) {
#pragma unroll
    for (int i = 0; i < S; ++i) {
      a[i] = canon_word<IO, K::kSigned>(a[i], P.A);
      b[i] = canon_word<IO, K::kSigned>(b[i], P.A);
    }
  }
  if constexpr (BASEMUL) {
#pragma unroll
    for (int q = 0; q < S / 2; ++q) {
      const Enc e0 = K::enc(a[2 * q], P.Q, P.A), e1 = K::enc(a[2 * q + 1], P.Q, P.A);
      const uint32_t b0 = b[2 * q], b1 = b[2 * q + 1];
      const uint32_t t11 = K::mulc(b1, e1, P.A);
      uint32_t c0 = K::mulc(b0, e0, P.A) + K::mulc(t11, gam[q], P.A);
      uint32_t c1 = K::mulc(b1, e0, P.A) + K::mulc(b0, e1, P.A);
      a[2 * q] = umin32(c0, c0 - P.A.p);
      a[2 * q + 1] = umin32(c1, c1 - P.A.p);
    }
  } else {
#pragma unroll
    for (int i = 0; i < S; ++i) a[i] = K::mulc(b[i], K::enc(a[i], P.Q, P.A), P.A);
  }
  return pack<IO>(a);
}

// blockDim = kBlock; the grid stride (gridDim kBlock vectors, kBlock S / 2 pairs) is a
// multiple of N / 2 <= 512 pairs, so thread t always handles pairs (t S / 2 + q) mod N / 2
constexpr int kBlock = 256;

template <class K, class IO, bool BASEMUL>
__global__ void __launch_bounds__(kBlock) product_kernel(const uint4* __restrict__ l, const uint4* __restrict__ r,
                                                         uint4* __restrict__ out, size_t nvec,
                                                         uint32_t half_n_mask,
                                                         const __grid_constant__ ProductArgs P) {
  constexpr uint32_t S = Vec<IO>::kSlots;
  typename K::Enc gam[S / 2];
  if constexpr (BASEMUL) {
#pragma unroll
    for (uint32_t q = 0; q < S / 2; ++q)
      gam[q] = K::genc(static_cast<int>((threadIdx.x * (S / 2) + q) & half_n_mask), P.Q);
  }
  const size_t stride = size_t(gridDim.x) * kBlock;
  size_t i = blockIdx.x * size_t(kBlock) + threadIdx.x;
  // two vectors in flight per thread: 32 B of loads outstanding per operand
  for (; i + stride < nvec; i += 2 * stride) {
    const uint4 l0 = __ldcs(l + i), r0 = __ldcs(r + i);
    const uint4 l1 = __ldcs(l + i + stride), r1 = __ldcs(r + i + stride);
    __stcs(out + i, product_vec<K, IO, BASEMUL>(l0, r0, gam, P));
    __stcs(out + i + stride, product_vec<K, IO, BASEMUL>(l1, r1, gam, P));
  }
  if (i < nvec) __stcs(out + i, product_vec<K, IO, BASEMUL>(__ldcs(l + i), __ldcs(r + i), gam, P));
}

template <class K, class IO, bool BASEMUL>
cudaError_t launch(const void* l, const void* r, void* out, size_t slots, uint32_t N,
                   const ProductArgs& P, cudaStream_t st) {
  static OccCache occ;
  auto kern = product_kernel<K, IO, BASEMUL>;
  const size_t nvec = slots / Vec<IO>::kSlots;
  const int o = occupancy_current(kern, kBlock, 0, occ);
  const size_t full = size_t(sm_count_current()) * (o > 0 ? o : 1);
  const size_t want = (nvec + kBlock - 1) / kBlock;
  const int blocks = static_cast<int>(want < full ? (want ? want : 1) : full);
  kern<<<blocks, kBlock, 0, st>>>(static_cast<const uint4*>(l), static_cast<const uint4*>(r),
                               static_cast<uint4*>(out), nvec, (N / 2) - 1, P);
  return cudaGetLastError();
}

template <class K>
cudaError_t by_io(int elem, bool basemul, const void* l, const void* r, void* out, size_t slots,
                  uint32_t N, const ProductArgs& P, cudaStream_t st) {
  if (elem == 2)
    return basemul ? launch<K, uint16_t, true>(l, r, out, slots, N, P, st)
                   : launch<K, uint16_t, false>(l, r, out, slots, N, P, st);
  if (elem == 4)
    return basemul ? launch<K, uint32_t, true>(l, r, out, slots, N, P, st)
                   : launch<K, uint32_t, false>(l, r, out, slots, N, P, st);
  return cudaErrorInvalidValue;
}

}  // namespace

bool product_supports(const HostParams& P, int kind, bool basemul, int elem, const void* l,
                      const void* r, const void* out) {
  if (!((P.fast_mask >> kind) & 1u)) return false;  // encodings built by fill_fast
  if (kind != NTTK_IMPROVED && kind != NTTK_HARVEY && kind != NTTK_SMONT) return false;
  if (elem != 2 && elem != 4) return false;
  if (elem == 2 && P.p >= (1u << 16)) return false;
  if (basemul && ((P.N >> P.layers) != 2 || P.N / 2 > 128)) return false;  // 128 moduli
  const uintptr_t mis = reinterpret_cast<uintptr_t>(l) | reinterpret_cast<uintptr_t>(r) |
                        reinterpret_cast<uintptr_t>(out);
  return !(mis & 15) && P.N % 8 == 0;
}

cudaError_t product_launch(const HostParams& P, int kind, bool basemul, const void* l, const void* r,
                           void* out, size_t batch, int elem, cudaStream_t st) {
  if (batch == 0) return cudaSuccess;
  ProductArgs PA;
  PA.A = P.fast[kind][0];
  PA.Q = P.prod[kind];
  const bool n16 = P.n_bits == 16;
  // slot indices wrap mod 2^32 inside the kernel; N divides 2^32, so the basemul pair
  // index (slot / 2) mod (N / 2) stays exact for any batch
  const size_t slots = batch * P.N;
  switch (kind) {
    case NTTK_IMPROVED:
      return n16 ? by_io<ImprovedN16<false>>(elem, basemul, l, r, out, slots, P.N, PA, st)
                 : by_io<ImprovedN32>(elem, basemul, l, r, out, slots, P.N, PA, st);
    case NTTK_HARVEY:
      return n16 ? by_io<Harvey<16, false>>(elem, basemul, l, r, out, slots, P.N, PA, st)
                 : by_io<Harvey<32, false>>(elem, basemul, l, r, out, slots, P.N, PA, st);
    case NTTK_SMONT:
      return n16 ? by_io<Smont<16>>(elem, basemul, l, r, out, slots, P.N, PA, st)
                 : by_io<Smont<32>>(elem, basemul, l, r, out, slots, P.N, PA, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace nttk_b200
