// fast256.cu -- batched N = 256 NTT kernels for sm_100a (the hot path).
//
// Replaces the reference's per-polynomial drivers run_split_layers / run_merge_layers
// (proj/include/nttk/transform.hpp:77-116) and their callers ntt_forward /
// intt_inverse (transform.hpp:207-343) for N = 256, 5 <= layers <= 8, n in {16, 32}.
//
// Work decomposition (B200-first, no tensor cores: this is 32-bit integer work):
//   * a half-warp (16 lanes) owns one polynomial; every lane holds 16 coefficients
//     in registers, so 4 of the 8 butterfly layers are register-local per phase;
//   * layer schedule, pair mapping and per-block / per-index twiddle indices are the
//     reference's (bit-exact lazy outputs), baked in at compile time;
//   * phase 1 / phase 2 switch the register-index bits from index bits 7..4
//     ("strided" ownership: lane j holds a[j + 16 r]) to bits 3..0 ("contiguous":
//     lane j holds a[16 j + r]) through a per-warp shared-memory transpose with an
//     XOR swizzle on 16-byte chunks, conflict-free for both STS/LDS patterns and for
//     the two polynomials of a warp (second one offset by 16 banks);
//   * twiddles live in the kernel-parameter constant bank (FastArgs, by value,
//     __grid_constant__): the ones that are uniform across lanes are free IMAD
//     operands, the 15 lane-dependent ones per thread are loaded once at kernel start
//     and stay in registers for every polynomial the persistent warp processes;
//   * HBM traffic is one coalesced 128-bit read and one 128-bit write per
//     coefficient group; the next polynomial pair is prefetched into registers while
//     the current one is transformed.
#include <cuda_runtime.h>

#include <cstdint>

#include "arith.cuh"
#include "fast256.hpp"
#include "launch_cache.hpp"

namespace nttk_b200 {
namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int kPolyWords = 272;  // 256 coefficients + 16 words: second poly on the other 16 banks

// swizzled word position of coefficient i inside one polynomial's smem tile
__device__ __forceinline__ int swz(int i) {
  return (i & ~15) | ((((i >> 2) & 3) ^ ((i >> 5) & 3)) << 2) | (i & 3);
}

// ---------------------------------------------------------------------------
// global <-> register conversions
template <class IO>
struct Io;

template <>
struct Io<uint16_t> {
  static constexpr int kPerVec = 8;  // coefficients per 16-byte vector
  __device__ static uint32_t get(const uint4& v, int e, bool sgn) {
    const uint32_t w = (&v.x)[e >> 1];
    const uint32_t h = (e & 1) ? (w >> 16) : (w & 0xffffu);
    return sgn ? static_cast<uint32_t>(static_cast<int32_t>(static_cast<int16_t>(h))) : h;
  }
  __device__ static void put(uint4& v, int e, uint32_t x) {
    uint32_t& w = (&v.x)[e >> 1];
    w = (e & 1) ? ((w & 0xffffu) | (x << 16)) : ((w & 0xffff0000u) | (x & 0xffffu));
  }
};
template <>
struct Io<uint32_t> {
  static constexpr int kPerVec = 4;
  __device__ static uint32_t get(const uint4& v, int e, bool) { return (&v.x)[e]; }
  __device__ static void put(uint4& v, int e, uint32_t x) { (&v.x)[e] = x; }
};
template <>
struct Io<uint64_t> {
  static constexpr int kPerVec = 2;
  __device__ static uint64_t get64(const uint4& v, int e) {
    return e ? (uint64_t(v.w) << 32 | v.z) : (uint64_t(v.y) << 32 | v.x);
  }
  __device__ static uint32_t get(const uint4& v, int e, bool) {
    return static_cast<uint32_t>(get64(v, e));
  }
  __device__ static void put(uint4& v, int e, uint32_t x, bool sgn) {
    const uint64_t y = sgn ? static_cast<uint64_t>(static_cast<int64_t>(static_cast<int32_t>(x)))
                           : uint64_t(x);
    if (e) {
      v.z = static_cast<uint32_t>(y);
      v.w = static_cast<uint32_t>(y >> 32);
    } else {
      v.x = static_cast<uint32_t>(y);
      v.y = static_cast<uint32_t>(y >> 32);
    }
  }
};

template <class IO>
__device__ __forceinline__ void io_put(uint4& v, int e, uint32_t x, bool sgn) {
  if constexpr (sizeof(IO) == 8) Io<uint64_t>::put(v, e, x, sgn);
  else Io<IO>::put(v, e, x);
}

// Number of 16-byte vectors per thread for one polynomial (16 lanes share 512/1024/2048 B)
template <class IO>
constexpr int vecs_per_lane() { return 16 / Io<IO>::kPerVec; }

// canonical residue of one loaded coefficient (transform.hpp:38-40,243)
template <class IO, bool SGN>
__device__ __forceinline__ uint32_t canon_load(const uint4& v, int e, const FastArgs& A) {
  if constexpr (sizeof(IO) == 8) {
    const uint64_t x = Io<uint64_t>::get64(v, e);
    if (SGN) {
      const int64_t r = static_cast<int64_t>(x) % static_cast<int64_t>(A.p);
      return static_cast<uint32_t>(r < 0 ? r + A.p : r);
    }
    return static_cast<uint32_t>(x % A.p);
  } else if constexpr (sizeof(IO) == 2) {
    const uint32_t x = Io<uint16_t>::get(v, e, SGN);
    return SGN ? mod_s32(x, A) : mod_u16(x, A);
  } else {
    const uint32_t x = Io<uint32_t>::get(v, e, SGN);
    return SGN ? mod_s32(x, A) : mod_u32(x, A);
  }
}

// ---------------------------------------------------------------------------
// Forward transform.  K: arithmetic policy; PER_INDEX: DIF per-index twiddles
// (ntl/harvey/scott cyclic schedule, params.hpp:47-58) instead of CT per-block
// (params.hpp:60-72 and the negacyclic tree).
template <class K, class IO, int L, bool PER_INDEX>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    fwd256_kernel(const IO* __restrict__ in, IO* __restrict__ out, size_t batch,
                  const __grid_constant__ FastArgs A) {
  using Tw = typename K::Tw;
  constexpr int V = vecs_per_lane<IO>();
  constexpr int PV = Io<IO>::kPerVec;
  __shared__ __align__(16) uint32_t smem[kWarpsPerBlock][2 * kPolyWords];
  const int lane = threadIdx.x & 31, j = lane & 15, half = lane >> 4;
  uint32_t* S = smem[threadIdx.x >> 5] + half * kPolyWords;

  // lane-dependent twiddles, resident for the whole kernel
  Tw twl[15];
  if (PER_INDEX) {  // phase 1: j_index = j + 16 (r mod len/16)
#pragma unroll
    for (int r = 0; r < 8; ++r) twl[r] = K::tw(A, 0 + j + 16 * r);
#pragma unroll
    for (int r = 0; r < 4; ++r) twl[8 + r] = K::tw(A, 128 + j + 16 * r);
#pragma unroll
    for (int r = 0; r < 2; ++r) twl[12 + r] = K::tw(A, 192 + j + 16 * r);
    twl[14] = K::tw(A, 224 + j);
  } else {  // phase 2: block = j 2^{s-5} + (r >> (9 - s))
    twl[0] = K::tw(A, 15 + j);
#pragma unroll
    for (int q = 0; q < 2; ++q) twl[1 + q] = K::tw(A, 31 + 2 * j + q);
#pragma unroll
    for (int q = 0; q < 4; ++q) twl[3 + q] = K::tw(A, 63 + 4 * j + q);
    if (L >= 8) {
#pragma unroll
      for (int q = 0; q < 8; ++q) twl[7 + q] = K::tw(A, 127 + 8 * j + q);
    }
  }

  const size_t pairs = (batch + 1) / 2;
  const size_t warp0 = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = (size_t(gridDim.x) * blockDim.x) >> 5;

  uint4 pf[V];
  auto load = [&](size_t pair) {
    const size_t poly = 2 * pair + half;
    if (pair < pairs && poly < batch) {
      const uint4* src = reinterpret_cast<const uint4*>(in + poly * 256);
#pragma unroll
      for (int k = 0; k < V; ++k) pf[k] = __ldcs(src + j + 16 * k);  // streaming read
    }
  };
  size_t pair = warp0;
  load(pair);
  for (; pair < pairs; pair += nwarps) {
    const size_t poly = 2 * pair + half;
    // ---- stage coalesced vectors into smem (swizzled), read strided ownership
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int i0 = (j + 16 * k) * PV;  // first coefficient of this vector
#pragma unroll
      for (int c = 0; c < PV; c += 4) {
        if constexpr (PV >= 4) {
          uint4 w;
          w.x = Io<IO>::get(pf[k], c + 0, K::kSigned);
          w.y = Io<IO>::get(pf[k], c + 1, K::kSigned);
          w.z = Io<IO>::get(pf[k], c + 2, K::kSigned);
          w.w = Io<IO>::get(pf[k], c + 3, K::kSigned);
          *reinterpret_cast<uint4*>(S + swz(i0 + c)) = w;
        }
      }
      if constexpr (PV == 2) {
        uint2 w = make_uint2(Io<IO>::get(pf[k], 0, K::kSigned), Io<IO>::get(pf[k], 1, K::kSigned));
        *reinterpret_cast<uint2*>(S + swz(i0)) = w;
      }
    }
    __syncwarp();
    uint32_t v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = S[swz(j + 16 * r)];
    load(pair + nwarps);  // prefetch the next pair while this one is transformed

    // ---- phase 1: layers 1..4, index bits 7..4 = register bits 3..0
#pragma unroll
    for (int s = 1; s <= 4; ++s) {
      const int h = 8 >> (s - 1);
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r & h) continue;
        Tw w;
        if (PER_INDEX) {
          const int base = s == 1 ? 0 : s == 2 ? 8 : s == 3 ? 12 : 14;
          w = twl[base + (r & (h - 1))];
        } else {
          w = K::tw(A, (1 << (s - 1)) - 1 + (r >> (5 - s)));
        }
        K::fwd(v[r], v[r + h], w, A);
      }
    }
    // ---- transpose: strided -> contiguous ownership
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 16; ++r) S[swz(j + 16 * r)] = v[r];
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 w = *reinterpret_cast<const uint4*>(S + swz(16 * j + 4 * c));
      v[4 * c + 0] = w.x;
      v[4 * c + 1] = w.y;
      v[4 * c + 2] = w.z;
      v[4 * c + 3] = w.w;
    }
    // ---- phase 2: layers 5..L, index bits 3..0 = register bits 3..0
#pragma unroll
    for (int s = 5; s <= 8; ++s) {
      if (s > L) break;
      const int h = 1 << (8 - s);
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r & h) continue;
        Tw w;
        if (PER_INDEX) {
          const int cursor = 256 - (1 << (9 - s));
          w = K::tw(A, cursor + (r & (h - 1)));
        } else {
          const int base = s == 5 ? 0 : s == 6 ? 1 : s == 7 ? 3 : 7;
          w = twl[base + (r >> (9 - s))];
        }
        K::fwd(v[r], v[r + h], w, A);
      }
    }
    // ---- store the contiguous 16 coefficients of this lane
    if (poly < batch) {
      uint4* dst = reinterpret_cast<uint4*>(out + poly * 256) + j * V;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        uint4 w = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int e = 0; e < PV; ++e) io_put<IO>(w, e, v[k * PV + e], K::kSigned);
        __stcs(dst + k, w);
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Inverse transform: canonicalise, merge layers s = L..1 (GS, one twiddle per block,
// merge order tables params.hpp:74-88), final N^{-1} (or 2^{-L}) pass.
template <class K, class IO, int L>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    inv256_kernel(const IO* __restrict__ in, IO* __restrict__ out, size_t batch,
                  const __grid_constant__ FastArgs A) {
  using Tw = typename K::Tw;
  constexpr int V = vecs_per_lane<IO>();
  constexpr int PV = Io<IO>::kPerVec;
  constexpr int TL = (1 << L);  // 2^L; merge-order cursor of layer s is 2^L - 2^s
  __shared__ __align__(16) uint32_t smem[kWarpsPerBlock][2 * kPolyWords];
  const int lane = threadIdx.x & 31, j = lane & 15, half = lane >> 4;
  uint32_t* S = smem[threadIdx.x >> 5] + half * kPolyWords;

  // phase 1 (contiguous ownership) twiddles: block = j 2^{s-5} + (r >> (9 - s))
  Tw twl[15];
  twl[0] = K::tw(A, TL - 32 + j);  // s = 5
#pragma unroll
  for (int q = 0; q < 2; ++q) twl[1 + q] = K::tw(A, TL - 64 + 2 * j + q);  // s = 6
#pragma unroll
  for (int q = 0; q < 4; ++q) twl[3 + q] = K::tw(A, TL - 128 + 4 * j + q);  // s = 7
  if (L >= 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) twl[7 + q] = K::tw(A, TL - 256 + 8 * j + q);  // s = 8
  }

  const size_t pairs = (batch + 1) / 2;
  const size_t warp0 = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = (size_t(gridDim.x) * blockDim.x) >> 5;

  uint4 pf[V];
  auto load = [&](size_t pair) {
    const size_t poly = 2 * pair + half;
    if (pair < pairs && poly < batch) {
      const uint4* src = reinterpret_cast<const uint4*>(in + poly * 256) + j * V;
#pragma unroll
      for (int k = 0; k < V; ++k) pf[k] = __ldcs(src + k);
    }
  };
  size_t pair = warp0;
  load(pair);
  for (; pair < pairs; pair += nwarps) {
    const size_t poly = 2 * pair + half;
    uint32_t v[16];
#pragma unroll
    for (int k = 0; k < V; ++k)
#pragma unroll
      for (int e = 0; e < PV; ++e) v[k * PV + e] = canon_load<IO, K::kSigned>(pf[k], e, A);
    load(pair + nwarps);

    // ---- phase 1: merge layers s = L..5 (merge depth m = L - s + 1)
#pragma unroll
    for (int s = 8; s >= 5; --s) {
      if (s > L) continue;
      const int h = 1 << (8 - s);
      const uint32_t off = A.p << (L - s);  // 2^{m-1} p
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r & h) continue;
        const int base = s == 5 ? 0 : s == 6 ? 1 : s == 7 ? 3 : 7;
        K::inv(v[r], v[r + h], twl[base + (r >> (9 - s))], off, A);
      }
    }
    // ---- transpose: contiguous -> strided ownership
#pragma unroll
    for (int c = 0; c < 4; ++c)
      *reinterpret_cast<uint4*>(S + swz(16 * j + 4 * c)) =
          make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = S[swz(j + 16 * r)];
    // ---- phase 2: merge layers s = 4..1, uniform twiddles
#pragma unroll
    for (int s = 4; s >= 1; --s) {
      const int h = 1 << (4 - s);
      const uint32_t off = A.p << (L - s);
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r & h) continue;
        K::inv(v[r], v[r + h], K::tw(A, TL - (2 << (s - 1)) + (r >> (5 - s))), off, A);
      }
    }
    // ---- final scaling (canonical output), back through smem for coalesced stores
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = K::scale(v[r], A);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 16; ++r) S[swz(j + 16 * r)] = v[r];
    __syncwarp();
    if (poly < batch) {
      uint4* dst = reinterpret_cast<uint4*>(out + poly * 256);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const int i0 = (j + 16 * k) * PV;
        uint4 w = make_uint4(0, 0, 0, 0);
        if constexpr (PV >= 4) {
#pragma unroll
          for (int c = 0; c < PV; c += 4) {
            const uint4 q = *reinterpret_cast<const uint4*>(S + swz(i0 + c));
            io_put<IO>(w, c + 0, q.x, false);
            io_put<IO>(w, c + 1, q.y, false);
            io_put<IO>(w, c + 2, q.z, false);
            io_put<IO>(w, c + 3, q.w, false);
          }
        } else {
          const uint2 q = *reinterpret_cast<const uint2*>(S + swz(i0));
          io_put<IO>(w, 0, q.x, false);
          io_put<IO>(w, 1, q.y, false);
        }
        __stcs(dst + j + 16 * k, w);
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
template <class Kern>
int blocks_for(Kern kern, OccCache& occ, size_t batch) {  // occ: per kernel instantiation
  const size_t pairs = (batch + 1) / 2;
  const size_t need = (pairs + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const size_t full =
      size_t(sm_count_current()) * occupancy_current(kern, kWarpsPerBlock * 32, 0, occ);
  return static_cast<int>(need < full ? need : full);
}

template <class K, class IO, int L, bool PER_INDEX>
cudaError_t fwd_launch(const void* in, void* out, size_t batch, const FastArgs& A,
                       cudaStream_t st) {
  static OccCache occ;
  auto kern = fwd256_kernel<K, IO, L, PER_INDEX>;
  const int blocks = blocks_for(kern, occ, batch);
  kern<<<blocks, kWarpsPerBlock * 32, 0, st>>>(static_cast<const IO*>(in), static_cast<IO*>(out),
                                               batch, A);
  return cudaGetLastError();
}

template <class K, class IO, int L>
cudaError_t inv_launch(const void* in, void* out, size_t batch, const FastArgs& A,
                       cudaStream_t st) {
  static OccCache occ;
  auto kern = inv256_kernel<K, IO, L>;
  const int blocks = blocks_for(kern, occ, batch);
  kern<<<blocks, kWarpsPerBlock * 32, 0, st>>>(static_cast<const IO*>(in), static_cast<IO*>(out),
                                               batch, A);
  return cudaGetLastError();
}

template <class K, class IO, bool PER_INDEX>
cudaError_t dispatch_layers(int dir, int L, const void* in, void* out, size_t batch,
                            const FastArgs& A, cudaStream_t st) {
  switch (L) {
    case 8:
      return dir == 0 ? fwd_launch<K, IO, 8, PER_INDEX>(in, out, batch, A, st)
                      : inv_launch<K, IO, 8>(in, out, batch, A, st);
    case 7:
      return dir == 0 ? fwd_launch<K, IO, 7, PER_INDEX>(in, out, batch, A, st)
                      : inv_launch<K, IO, 7>(in, out, batch, A, st);
    default: return cudaErrorInvalidValue;
  }
}

template <class K, bool PER_INDEX>
cudaError_t dispatch_io(int dir, int L, int elem, const void* in, void* out, size_t batch,
                        const FastArgs& A, cudaStream_t st) {
  switch (elem) {
    case 2: return dispatch_layers<K, uint16_t, PER_INDEX>(dir, L, in, out, batch, A, st);
    case 4: return dispatch_layers<K, uint32_t, PER_INDEX>(dir, L, in, out, batch, A, st);
    case 8: return dispatch_layers<K, uint64_t, PER_INDEX>(dir, L, in, out, batch, A, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

bool fast256_supports(int kind, int layers, int n_bits) {
  if (layers != 7 && layers != 8) return false;
  if (n_bits != 16 && n_bits != 32) return false;
  if (kind == NTTK_SCOTT) return n_bits == 32;
  return kind == NTTK_IMPROVED || kind == NTTK_HARVEY || kind == NTTK_SMONT || kind == NTTK_NTL;
}

cudaError_t fast256_launch(const HostParams& P, int kind, int dir, const void* in, void* out,
                           size_t batch, int elem_bytes, cudaStream_t st, int variant) {
  const FastArgs& A = P.fast[kind][dir];
  const int L = static_cast<int>(P.layers);
  const bool n16 = P.n_bits == 16;
  const bool cyclic = P.tree == NTTK_CYCLIC;
  if (batch == 0) return cudaSuccess;
  switch (kind) {
    case NTTK_IMPROVED:
      if (n16) {
        if (variant == 1)
          return dispatch_io<ImprovedN16<true>, false>(dir, L, elem_bytes, in, out, batch, A, st);
        return dispatch_io<ImprovedN16<false>, false>(dir, L, elem_bytes, in, out, batch, A, st);
      }
      return dispatch_io<ImprovedN32, false>(dir, L, elem_bytes, in, out, batch, A, st);
    case NTTK_HARVEY:
      if (cyclic) {
        return n16 ? dispatch_io<Harvey<16, false>, true>(dir, L, elem_bytes, in, out, batch, A, st)
                   : dispatch_io<Harvey<32, false>, true>(dir, L, elem_bytes, in, out, batch, A, st);
      }
      return n16 ? dispatch_io<Harvey<16, true>, false>(dir, L, elem_bytes, in, out, batch, A, st)
                 : dispatch_io<Harvey<32, true>, false>(dir, L, elem_bytes, in, out, batch, A, st);
    case NTTK_SMONT:
      return n16 ? dispatch_io<Smont<16>, false>(dir, L, elem_bytes, in, out, batch, A, st)
                 : dispatch_io<Smont<32>, false>(dir, L, elem_bytes, in, out, batch, A, st);
    case NTTK_NTL:
      return n16 ? dispatch_io<Ntl<16>, true>(dir, L, elem_bytes, in, out, batch, A, st)
                 : dispatch_io<Ntl<32>, true>(dir, L, elem_bytes, in, out, batch, A, st);
    case NTTK_SCOTT:
      if (n16 || !cyclic) return cudaErrorInvalidValue;
      return dispatch_io<Scott32, true>(dir, L, elem_bytes, in, out, batch, A, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace nttk_b200
