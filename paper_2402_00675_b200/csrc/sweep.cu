// sweep.cu -- reduction sweep over an operand grid (BASELINE config 5).
//
// Runs one of the reference's word-level reductions (reduction.hpp:125-273) on every
// pair (A[i], B[j]) of an operand grid: mont_redc(a b), signed_mont_redc(a b),
// plantard_redc(a, b) and modified_plantard_mul(a, b).  Bit-exact with the reference
// bodies; the operand that plays the twiddle role (a) is premultiplied per row, so the
// per-pair cost is the reduction itself (2 IMAD for modified Plantard at n = 16).
// Each thread keeps 8 columns in registers and walks a block of rows; results are
// optionally stored (int64, row-major) and always folded into a wrapping u64 checksum.
#include <cuda_runtime.h>

#include <cstdint>

#include "arith.cuh"
#include "sweep.hpp"

namespace nttk_b200 {
namespace {

constexpr int kCols = 8;       // columns per thread
constexpr int kThreads = 256;  // threads per block -> 2048 columns per block
constexpr int kRows = 64;      // rows per block

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
  __device__ static int64_t pair(const Row& R, int64_t b, const SweepArgs& S) {
    const uint32_t p = static_cast<uint32_t>(S.p);
    if (VAR == NTTK_REDC_MPLANTARD) {  // reduction.hpp:252-258
      if (NB == 16) return mp_n16<false>(static_cast<uint32_t>(b), static_cast<uint32_t>(R.am), p);
      if (NB == 32)
        return mp_n32(static_cast<uint32_t>(b), static_cast<uint32_t>(R.am),
                      static_cast<uint32_t>(R.am >> 32), p);
      const uint64_t h = (R.am * static_cast<uint64_t>(b)) & S.r2n_mask;
      return static_cast<int64_t>((((h >> S.n_bits) + 1) * S.p) >> S.n_bits);
    }
    if (VAR == NTTK_REDC_PLANTARD) {  // reduction.hpp:178-191: paper form + r == p corner
      uint32_t r;
      if (NB == 16) {
        r = mp_n16<true>(static_cast<uint32_t>(b), static_cast<uint32_t>(R.am), p);
      } else if (NB == 32) {
        r = mp_n32(static_cast<uint32_t>(b), static_cast<uint32_t>(R.am),
                   static_cast<uint32_t>(R.am >> 32), p);
        // mp_n32 wraps h_hi + 1 = 2^32 to 0; the reference then returns p -> 0 as well
      } else {
        const uint64_t h = (R.am * static_cast<uint64_t>(b)) & S.r2n_mask;
        r = static_cast<uint32_t>((((h >> S.n_bits) + 1) * S.p) >> S.n_bits);
      }
      return r == p ? 0 : r;
    }
    if (VAR == NTTK_REDC_MONT) {  // reduction.hpp:125-135
      if (NB == 16) {
        const uint32_t T = static_cast<uint32_t>(R.a) * static_cast<uint32_t>(b);
        const uint32_t m = (static_cast<uint32_t>(R.am) * static_cast<uint32_t>(b)) & 0xffffu;
        const uint32_t t = (T + m * p) >> 16;
        return umin32(t, t - p);
      }
      if (NB == 32) {
        const uint64_t T = R.a * static_cast<uint64_t>(b);
        const uint32_t m = static_cast<uint32_t>(R.am) * static_cast<uint32_t>(b);
        const uint32_t t = static_cast<uint32_t>((T + static_cast<uint64_t>(m) * p) >> 32);
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
      const int32_t m =
          static_cast<int32_t>((static_cast<uint32_t>(R.am) << 16) * static_cast<uint32_t>(b)) >> 16;
      return (A - m * static_cast<int32_t>(p)) >> 16;
    }
    if (NB == 32) {
      const int64_t A = static_cast<int64_t>(R.a) * b;
      const int32_t m = static_cast<int32_t>(static_cast<uint32_t>(R.am) * static_cast<uint32_t>(b));
      return static_cast<int32_t>((A - static_cast<int64_t>(m) * p) >> 32);
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

template <int VAR, int NB, bool STORE>
__global__ void __launch_bounds__(kThreads)
    sweep_kernel(const int64_t* __restrict__ A, size_t na, const int64_t* __restrict__ B, size_t nb,
                 int64_t* __restrict__ r, unsigned long long* __restrict__ sum, SweepArgs S) {
  const size_t col_tiles = (nb + kThreads * kCols - 1) / (kThreads * kCols);
  const size_t row_tiles = (na + kRows - 1) / kRows;
  unsigned long long acc = 0;
  for (size_t t = blockIdx.x; t < col_tiles * row_tiles; t += gridDim.x) {
    const size_t ct = t % col_tiles, rt = t / col_tiles;
    const size_t c0 = ct * kThreads * kCols + threadIdx.x;
    int64_t b[kCols];
    bool ok[kCols];
#pragma unroll
    for (int k = 0; k < kCols; ++k) {
      const size_t c = c0 + size_t(k) * kThreads;
      ok[k] = c < nb;
      b[k] = ok[k] ? B[c] : 0;
    }
    const size_t r0 = rt * kRows, r1 = r0 + kRows < na ? r0 + kRows : na;
    for (size_t i = r0; i < r1; ++i) {
      const auto R = Redc<VAR, NB>::row(A[i], S);
      int32_t part = 0;  // |result| < p < 2^31 / kCols: no overflow inside one row
      int64_t part64 = 0;
#pragma unroll
      for (int k = 0; k < kCols; ++k) {
        const int64_t v = Redc<VAR, NB>::pair(R, b[k], S);
        if (NB) part += ok[k] ? static_cast<int32_t>(v) : 0;
        else part64 += ok[k] ? v : 0;
        if (STORE && ok[k]) r[i * nb + c0 + size_t(k) * kThreads] = v;
      }
      acc += static_cast<unsigned long long>(NB ? static_cast<int64_t>(part) : part64);
    }
  }
  // warp reduce, one atomic per warp
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(sum, acc);
}

template <int VAR, int NB>
cudaError_t launch_var(const int64_t* A, size_t na, const int64_t* B, size_t nb, int64_t* r,
                       unsigned long long* sum, const SweepArgs& S, cudaStream_t st) {
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t tiles = ((nb + kThreads * kCols - 1) / (kThreads * kCols)) * ((na + kRows - 1) / kRows);
  if (r) {
    auto k = sweep_kernel<VAR, NB, true>;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kThreads, 0);
    const size_t g = tiles < size_t(sms) * occ ? tiles : size_t(sms) * occ;
    k<<<static_cast<unsigned>(g ? g : 1), kThreads, 0, st>>>(A, na, B, nb, r, sum, S);
  } else {
    auto k = sweep_kernel<VAR, NB, false>;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kThreads, 0);
    const size_t g = tiles < size_t(sms) * occ ? tiles : size_t(sms) * occ;
    k<<<static_cast<unsigned>(g ? g : 1), kThreads, 0, st>>>(A, na, B, nb, r, sum, S);
  }
  return cudaGetLastError();
}

template <int NB>
cudaError_t launch_nb(int variant, const int64_t* A, size_t na, const int64_t* B, size_t nb,
                      int64_t* r, unsigned long long* sum, const SweepArgs& S, cudaStream_t st) {
  switch (variant) {
    case NTTK_REDC_MONT: return launch_var<NTTK_REDC_MONT, NB>(A, na, B, nb, r, sum, S, st);
    case NTTK_REDC_SMONT: return launch_var<NTTK_REDC_SMONT, NB>(A, na, B, nb, r, sum, S, st);
    case NTTK_REDC_PLANTARD: return launch_var<NTTK_REDC_PLANTARD, NB>(A, na, B, nb, r, sum, S, st);
    case NTTK_REDC_MPLANTARD: return launch_var<NTTK_REDC_MPLANTARD, NB>(A, na, B, nb, r, sum, S, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

cudaError_t sweep_launch(int variant, const Ctx& c, const int64_t* A, size_t na, const int64_t* B,
                         size_t nb, int64_t* r, unsigned long long* d_sum, cudaStream_t st) {
  SweepArgs S{c.p, c.beta_mask, c.r2n_mask, c.p_inv_beta, c.neg_p_inv_beta, c.mu, c.n_bits};
  if (!na || !nb) return cudaSuccess;
  // the 32-bit forms need every intermediate inside 32 / 64 bits (checked host-side)
  const uint64_t p = c.p;
  if (c.n_bits == 16 && p * p + (p << 16) < (uint64_t(1) << 32))
    return launch_nb<16>(variant, A, na, B, nb, r, d_sum, S, st);
  if (c.n_bits == 32 && p < (uint64_t(1) << 27))
    return launch_nb<32>(variant, A, na, B, nb, r, d_sum, S, st);
  return launch_nb<0>(variant, A, na, B, nb, r, d_sum, S, st);
}

}  // namespace nttk_b200
