// sweep.cu -- reduction sweep over an operand grid (BASELINE config 5).
//
// Runs one of the reference's word-level reductions (reduction.hpp:125-273) on every
// pair (A[i], B[j]) of an operand grid: mont_redc(a b), signed_mont_redc(a b),
// plantard_redc(a, b) and modified_plantard_mul(a, b).  Bit-exact with the reference
// bodies; the operand that plays the twiddle role (a) is premultiplied per row, so the
// per-pair cost is the reduction itself (IMAD + IMAD.HI for modified Plantard at n = 16).
// A block stages up to 256 premultiplied rows at a time in shared memory (read back as broadcasts),
// each thread keeps 16 columns in registers and walks the rows; results are optionally
// stored (int64, row-major) and always folded into a wrapping u64 checksum.
#include <cuda_runtime.h>

#include <cstdint>

#include "arith.cuh"
#include "launch_cache.hpp"
#include "sweep.hpp"

namespace nttk_b200 {
namespace {

constexpr int kCols = 16;                // columns per thread
constexpr int kThreads = 256;            // threads per block -> 4096 columns per block
constexpr int kRows = 256;               // rows staged per chunk
static_assert(kCols % 8 == 0 && kRows * kCols <= 16384, "sweep tile shape");

struct SweepArgs {
  uint64_t p, beta_mask, r2n_mask, p_inv_beta, neg_p_inv_beta, mu;
  uint32_t n_bits;
};

// per-row precompute + per-pair body, specialised for n = 16 / n = 32; NB = 0 is the
// any-n 64-bit form
template <int VAR, int NB>
struct Redc {
  struct Row {
    uint64_t a, am;  // a and its premultiplied form
  };
  __device__ static Row row(int64_t a, const SweepArgs& S) {
    Row r{static_cast<uint64_t>(a), 0};
    if (VAR == NTTK_REDC_PLANTARD || VAR == NTTK_REDC_MPLANTARD)
      r.am = static_cast<uint64_t>(a) * S.mu & S.r2n_mask;  // a mu mod 2^{2n}
    else if (VAR == NTTK_REDC_SMONT)
      r.am = static_cast<uint64_t>(a) * S.p_inv_beta & S.beta_mask;  // a p^{-1} mod 2^n
    else
      r.am = static_cast<uint64_t>(a) * S.neg_p_inv_beta & S.beta_mask;  // a k mod 2^n
    return r;
  }
  // The n = 16 / 32 bodies stay in 32-bit registers; each is exact against the
  // reference's 64-bit statement (reduction.hpp lines cited per variant).
  __device__ static int64_t pair(const Row& R, int64_t b, const SweepArgs& S) {
    const uint32_t p = static_cast<uint32_t>(S.p);
    const uint32_t b32 = static_cast<uint32_t>(b);
    const uint32_t lo = static_cast<uint32_t>(R.am), hi = static_cast<uint32_t>(R.am >> 32);
    if (VAR == NTTK_REDC_MPLANTARD) {  // reduction.hpp:252-258
      // r = ((h_hi + 1) p) >> 16 in the shift form with the +1 folded into the IMAD
      // addend (h + 2^16; the output is canonical, so h_hi + 1 never wraps): 2 IMAD + 2 SHF.
      // Alone in a sweep this beats the umulhi form (IMAD + IMAD.HI: the IMAD.HI holds the
      // fma-heavy pipe for 4 cycles); inside a butterfly the add/sub already load the ALU
      // pipe, which is why the NTT kernels keep the umulhi form (arith.cuh).
      if (NB == 16) return (((b32 * lo + 0x10000u) >> 16) * p) >> 16;
      // r = hi32((h_hi + 1) p); the output is canonical, so h_hi + 1 never wraps
      if (NB == 32) return __umulhi(hi * b32 + __umulhi(lo, b32) + 1u, p);
      const uint64_t h = (R.am * static_cast<uint64_t>(b)) & S.r2n_mask;
      return static_cast<int64_t>((((h >> S.n_bits) + 1) * S.p) >> S.n_bits);
    }
    if (VAR == NTTK_REDC_PLANTARD) {  // reduction.hpp:178-191: paper form + r == p corner
      // r == p exactly when h_hi = 2^n - 1; letting h_hi + 1 wrap to 0 in n bits returns
      // the reference's corrected 0 with no compare
      if (NB == 16) return (((b32 * lo + 0x10000u) >> 16) * p) >> 16;
      if (NB == 32) return __umulhi(hi * b32 + __umulhi(lo, b32) + 1u, p);
      const uint64_t h = (R.am * static_cast<uint64_t>(b)) & S.r2n_mask;
      const uint64_t r = (((h >> S.n_bits) + 1) * S.p) >> S.n_bits;
      return static_cast<int64_t>(r == S.p ? 0 : r);
    }
    if (VAR == NTTK_REDC_MONT) {  // reduction.hpp:125-135
      if (NB == 16) {
        const uint32_t T = static_cast<uint32_t>(R.a) * b32;
        const uint32_t m = (lo * b32) & 0xffffu;
        const uint32_t t = (T + m * p) >> 16;
        return umin32(t, t - p);
      }
      if (NB == 32) {  // t = hi32(m p + T): one IMAD.WIDE with the 64-bit addend T
        const uint64_t T = static_cast<uint64_t>(static_cast<uint32_t>(R.a)) * b32;
        const uint32_t m = lo * b32;
        const uint32_t t = static_cast<uint32_t>((static_cast<uint64_t>(m) * p + T) >> 32);
        return umin32(t, t - p);
      }
      const uint64_t T = R.a * static_cast<uint64_t>(b);
      const uint64_t m = (T & S.beta_mask) * S.neg_p_inv_beta & S.beta_mask;
      const unsigned __int128 s = (unsigned __int128)T + (unsigned __int128)m * S.p;
      uint64_t t = static_cast<uint64_t>(s >> S.n_bits);
      return static_cast<int64_t>(t >= S.p ? t - S.p : t);
    }
    // signed Montgomery, reduction.hpp:141-165: r = (A - m p) / 2^n
    if (NB == 16) {
      const int32_t A = static_cast<int32_t>(R.a) * static_cast<int32_t>(b);
      const int32_t m = static_cast<int32_t>((lo << 16) * b32) >> 16;
      return (A - m * static_cast<int32_t>(p)) >> 16;
    }
    if (NB == 32) {  // A and m p agree in their low words: r = hi(A) - hi(m p), signed
      const int32_t m = static_cast<int32_t>(lo * b32);
      return __mulhi(static_cast<int32_t>(R.a), static_cast<int32_t>(b32)) -
             __mulhi(m, static_cast<int32_t>(p));
    }
    const int64_t A = static_cast<int64_t>(R.a) * b;
    const int64_t a1 = A >> S.n_bits;
    const uint64_t mu = (static_cast<uint64_t>(A) & S.beta_mask) * S.p_inv_beta & S.beta_mask;
    const uint64_t half = (S.beta_mask + 1) >> 1;
    const int64_t m = mu >= half ? static_cast<int64_t>(mu) - static_cast<int64_t>(S.beta_mask + 1)
                                 : static_cast<int64_t>(mu);
    return a1 - ((m * static_cast<int64_t>(S.p)) >> S.n_bits);
  }
};

// plantard_redc's r == p corner (reduction.hpp:178-191) for the counting kernels: the
// 32-bit bodies fold it into an n-bit wrap of h_hi + 1, which is 0 exactly when it fires
template <int NB>
__device__ __forceinline__ bool plantard_fired(uint64_t am, int64_t b, const SweepArgs& S) {
  const uint32_t b32 = static_cast<uint32_t>(b);
  const uint32_t lo = static_cast<uint32_t>(am), hi = static_cast<uint32_t>(am >> 32);
  if (NB == 16) return ((b32 * lo + 0x10000u) >> 16) == 0;
  if (NB == 32) return hi * b32 + __umulhi(lo, b32) + 1u == 0;
  const uint64_t h = (am * static_cast<uint64_t>(b)) & S.r2n_mask;
  return (((h >> S.n_bits) + 1) * S.p) >> S.n_bits == S.p;
}

// Every variant maps b = 0 to 0 (all four bodies are linear in b before the final
// shift / reduction and the +1 Plantard offsets vanish under >> n for p < 2^n), so the
// out-of-range columns are zero-padded instead of masked per pair.
// COUNT (plantard_redc only): also count the r == p corner into *fires.
template <int VAR, int NB, bool STORE, bool COUNT = false>
__global__ void __launch_bounds__(kThreads)
    sweep_kernel(const int64_t* __restrict__ A, size_t na, const int64_t* __restrict__ B, size_t nb,
                 int64_t* __restrict__ r, unsigned long long* __restrict__ sum, SweepArgs S,
                 unsigned row_split, unsigned long long* __restrict__ fires) {
  using Row = typename Redc<VAR, NB>::Row;
  __shared__ Row rows[kRows];
  // work split: gridDim.x = col_tiles * row_split when the column tiles do not fill the
  // grid (each CTA owns one column tile and an even 1/row_split share of the rows, so the
  // last wave is never partial); otherwise row_split = 1 and CTAs stride over column tiles
  const size_t col_tiles = (nb + kThreads * kCols - 1) / (kThreads * kCols);
  const unsigned rs = blockIdx.x / static_cast<unsigned>(col_tiles < gridDim.x ? col_tiles : gridDim.x);
  const size_t ra = na * rs / row_split, rb = na * (rs + 1) / row_split;
  unsigned long long acc = 0;
  uint32_t nfired = 0;
  for (size_t ct = blockIdx.x % col_tiles; ct < col_tiles; ct += row_split == 1 ? gridDim.x : col_tiles)
   for (size_t r0 = ra; r0 < rb; r0 += kRows) {
    const size_t c0 = ct * kThreads * kCols + threadIdx.x;
    const int nrows = static_cast<int>(r0 + kRows < rb ? kRows : rb - r0);
    __syncthreads();  // previous chunk's rows consumed
    for (int i = threadIdx.x; i < nrows; i += kThreads) rows[i] = Redc<VAR, NB>::row(A[r0 + i], S);
    int64_t b[kCols];
#pragma unroll
    for (int k = 0; k < kCols; ++k) {
      const size_t c = c0 + size_t(k) * kThreads;
      b[k] = c < nb ? B[c] : 0;
    }
    __syncthreads();
    if (NB) {
      // |result| < p < 2^27: 8 results fit an int32 partial, 16-bit words a whole chunk.
      // Partials are summed as u32 bit patterns (two's complement) so ptxas sees plain
      // 32-bit adds, then sign-extended.
      uint32_t tile = 0;
#pragma unroll 2
      for (int i = 0; i < nrows; ++i) {
        const Row R = rows[i];
        uint32_t h[kCols / 8] = {};
#pragma unroll
        for (int k = 0; k < kCols; ++k) {
          const uint32_t v = static_cast<uint32_t>(Redc<VAR, NB>::pair(R, b[k], S));
          h[k / 8] += v;
          if (COUNT) nfired += plantard_fired<NB>(R.am, b[k], S) && (c0 + size_t(k) * kThreads < nb);
          if (STORE) {
            const size_t c = c0 + size_t(k) * kThreads;
            if (c < nb) r[(r0 + i) * nb + c] = static_cast<int32_t>(v);
          }
        }
#pragma unroll
        for (int j = 0; j < kCols / 8; ++j) {
          if (NB == 16) tile += h[j];
          else acc += static_cast<unsigned long long>(static_cast<int64_t>(static_cast<int32_t>(h[j])));
        }
      }
      if (NB == 16) acc += static_cast<unsigned long long>(static_cast<int64_t>(static_cast<int32_t>(tile)));
    } else {
      for (int i = 0; i < nrows; ++i) {
        const Row R = rows[i];
        int64_t part = 0;
#pragma unroll
        for (int k = 0; k < kCols; ++k) {
          const int64_t v = Redc<VAR, NB>::pair(R, b[k], S);
          part += v;
          if (COUNT) nfired += plantard_fired<NB>(R.am, b[k], S) && (c0 + size_t(k) * kThreads < nb);
          if (STORE) {
            const size_t c = c0 + size_t(k) * kThreads;
            if (c < nb) r[(r0 + i) * nb + c] = v;
          }
        }
        acc += static_cast<unsigned long long>(part);
      }
    }
  }
  // warp reduce, one atomic per warp
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(sum, acc);
  if (COUNT) {
#pragma unroll
    for (int o = 16; o; o >>= 1) nfired += __shfl_xor_sync(0xffffffffu, nfired, o);
    if ((threadIdx.x & 31) == 0 && nfired) atomicAdd(fires, static_cast<unsigned long long>(nfired));
  }
}

template <int VAR, int NB>
cudaError_t launch_var(const int64_t* A, size_t na, const int64_t* B, size_t nb, int64_t* r,
                       unsigned long long* sum, const SweepArgs& S, cudaStream_t st,
                       unsigned long long* fires) {
  static OccCache occ_store, occ_sum, occ_count;
  const int sms = sm_count_current();
  constexpr bool kCan = VAR == NTTK_REDC_PLANTARD;
  const bool count = kCan && fires;
  auto k = count ? (r ? sweep_kernel<VAR, NB, true, kCan> : sweep_kernel<VAR, NB, false, kCan>)
                 : (r ? sweep_kernel<VAR, NB, true> : sweep_kernel<VAR, NB, false>);
  const size_t cap = size_t(sms) * occupancy_current(k, kThreads, 0, count ? occ_count : r ? occ_store : occ_sum);
  const size_t col_tiles = (nb + kThreads * kCols - 1) / (kThreads * kCols);
  const size_t row_chunks = (na + kRows - 1) / kRows;
  size_t row_split = 1, g = col_tiles < cap ? col_tiles : cap;
  if (col_tiles < cap) {  // split the rows evenly across cap / col_tiles CTAs per column tile
    row_split = cap / col_tiles;
    if (row_split > row_chunks) row_split = row_chunks;
    g = col_tiles * row_split;
  }
  k<<<static_cast<unsigned>(g), kThreads, 0, st>>>(A, na, B, nb, r, sum, S,
                                                    static_cast<unsigned>(row_split), fires);
  return cudaGetLastError();
}

template <int NB>
cudaError_t launch_nb(int variant, const int64_t* A, size_t na, const int64_t* B, size_t nb,
                      int64_t* r, unsigned long long* sum, const SweepArgs& S, cudaStream_t st,
                      unsigned long long* f) {
  switch (variant) {
    case NTTK_REDC_MONT: return launch_var<NTTK_REDC_MONT, NB>(A, na, B, nb, r, sum, S, st, f);
    case NTTK_REDC_SMONT: return launch_var<NTTK_REDC_SMONT, NB>(A, na, B, nb, r, sum, S, st, f);
    case NTTK_REDC_PLANTARD: return launch_var<NTTK_REDC_PLANTARD, NB>(A, na, B, nb, r, sum, S, st, f);
    case NTTK_REDC_MPLANTARD: return launch_var<NTTK_REDC_MPLANTARD, NB>(A, na, B, nb, r, sum, S, st, f);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

cudaError_t sweep_launch(int variant, const Ctx& c, const int64_t* A, size_t na, const int64_t* B,
                         size_t nb, int64_t* r, unsigned long long* d_sum, cudaStream_t st,
                         unsigned long long* d_fires) {
  SweepArgs S{c.p, c.beta_mask, c.r2n_mask, c.p_inv_beta, c.neg_p_inv_beta, c.mu, c.n_bits};
  if (!na || !nb) return cudaSuccess;
  // the 32-bit forms need every intermediate inside 32 / 64 bits (checked host-side)
  const uint64_t p = c.p;
  if (c.n_bits == 16 && p * p + (p << 16) < (uint64_t(1) << 32))
    return launch_nb<16>(variant, A, na, B, nb, r, d_sum, S, st, d_fires);
  if (c.n_bits == 32 && p < (uint64_t(1) << 27))
    return launch_nb<32>(variant, A, na, B, nb, r, d_sum, S, st, d_fires);
  return launch_nb<0>(variant, A, na, B, nb, r, d_sum, S, st, d_fires);
}

}  // namespace nttk_b200
