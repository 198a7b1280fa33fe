// reduce.cu -- the reference's word-level reductions (reduction.hpp:125-291) applied
// elementwise to device arrays: the drop-in behind nttk::mont_redc & co.
//
// Each op restates the published formula in exact 64/128-bit arithmetic (bit-identical with
// the reference for every admitted input) and checks its operand range on the device like
// the reference's NTTK_REQUIRE; a violation sets a bit in *flag (the host turns it into the
// reference's message) and the element is left unwritten.
#include <cuda_runtime.h>

#include <cstdint>

#include "reduce.hpp"

namespace nttk_b200 {
namespace {

using u128 = unsigned __int128;

struct RArgs {
  uint64_t p, beta_mask, r2n_mask, p_inv_beta, neg_p_inv_beta, mu, beta, beta_mod_p, r2n_mod_p;
  uint32_t n_bits, ell;
};

template <int OP>
__global__ void reduce_kernel(const int64_t* __restrict__ x, const int64_t* __restrict__ y,
                              int64_t* __restrict__ out, size_t n, RArgs R, unsigned* flag) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const uint64_t p = R.p;
    if (OP == NTTK_OP_MONT_REDC) {  // reduction.hpp:125-135
      const uint64_t T = static_cast<uint64_t>(x[i]);
      if (!(T < p * p)) {
        atomicOr(flag, 1u);
        continue;
      }
      const uint64_t m = ((T & R.beta_mask) * R.neg_p_inv_beta) & R.beta_mask;
      uint64_t t = static_cast<uint64_t>((u128(T) + u128(m) * p) >> R.n_bits);
      if (t >= p) t -= p;
      out[i] = static_cast<int64_t>(t);
    } else if (OP == NTTK_OP_SIGNED_MONT_REDC) {  // reduction.hpp:141-165
      const int64_t A = x[i];
      const __int128 limit = (__int128(p) << R.n_bits) / 2;
      if (!(-limit < A && A < limit)) {
        atomicOr(flag, 1u);
        continue;
      }
      const int64_t a1 = A >> R.n_bits;
      const uint64_t a0 = static_cast<uint64_t>(A) & R.beta_mask;
      const uint64_t mu = (a0 * R.p_inv_beta) & R.beta_mask;
      const int64_t m = mu >= R.beta / 2 ? static_cast<int64_t>(mu) - static_cast<int64_t>(R.beta)
                                         : static_cast<int64_t>(mu);
      out[i] = a1 - ((m * static_cast<int64_t>(p)) >> R.n_bits);
    } else if (OP == NTTK_OP_PLANTARD_REDC || OP == NTTK_OP_MODIFIED_PLANTARD_MUL) {
      const uint64_t W = static_cast<uint64_t>(x[i]), T = static_cast<uint64_t>(y[i]);
      if (OP == NTTK_OP_PLANTARD_REDC) {  // reduction.hpp:178-191
        if (!(W <= p && T <= p)) {
          atomicOr(flag, 1u);
          continue;
        }
      } else {  // reduction.hpp:264-273: W checked first, then T
        if (!(W < p)) {
          atomicOr(flag, 1u);
          continue;
        }
        if (!(T < (p << R.ell))) {
          atomicOr(flag, 2u);
          continue;
        }
      }
      const uint64_t h = ((W * T) * R.mu) & R.r2n_mask;
      const uint64_t r = (((h >> R.n_bits) + 1) * p) >> R.n_bits;
      // the r == p corner counts into plantard_correction_fires (reduction.hpp:172-191):
      // flag[2..3] is the u64 counter of this launch
      if (OP == NTTK_OP_PLANTARD_REDC && r == p)
        atomicAdd(reinterpret_cast<unsigned long long*>(flag + 2), 1ull);
      out[i] = static_cast<int64_t>(OP == NTTK_OP_PLANTARD_REDC && r == p ? 0 : r);
    } else if (OP == NTTK_OP_MOD_P) {  // canonicalize, transform.hpp:38-40
      out[i] = static_cast<int64_t>(static_cast<uint64_t>(x[i]) % p);
    } else {  // domain encodings, reduction.hpp:279-291
      const uint64_t w = static_cast<uint64_t>(x[i]);
      if (!(w < p)) {
        atomicOr(flag, 1u);
        continue;
      }
      const uint64_t v = OP == NTTK_OP_TO_PLANTARD_DOMAIN
                             ? (p - static_cast<uint64_t>(u128(w) * R.r2n_mod_p % p)) % p
                             : static_cast<uint64_t>(u128(w) * R.beta_mod_p % p);
      out[i] = static_cast<int64_t>(v);
    }
  }
}

template <int OP>
cudaError_t launch(const int64_t* x, const int64_t* y, int64_t* out, size_t n, const RArgs& R,
                   unsigned* flag, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t want = (n + 255) / 256, cap = size_t(sms) * 8;
  reduce_kernel<OP><<<static_cast<unsigned>(want < cap ? (want ? want : 1) : cap), 256, 0, st>>>(
      x, y, out, n, R, flag);
  return cudaGetLastError();
}

// --- butterfly.hpp checked entry points, elementwise ---------------------------------
// aux0/aux1: scott N and L (offset (N/L) p); improved GS: layer.  Operand checks as in the
// reference's checked wrappers; flag bits: 1 = W out of range, 2 = stale W_quot (ntl),
// 4 = X/Y out of range.
template <int OP>
__global__ void butterfly_kernel(const int64_t* __restrict__ xs, const int64_t* __restrict__ ys,
                                 const int64_t* __restrict__ ws, const int64_t* __restrict__ wq,
                                 int64_t* __restrict__ xo, int64_t* __restrict__ yo, size_t n,
                                 RArgs R, uint32_t aux0, uint32_t aux1, unsigned* flag) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const uint64_t p = R.p, X = static_cast<uint64_t>(xs[i]), Y = static_cast<uint64_t>(ys[i]);
    const uint64_t W = static_cast<uint64_t>(ws[i]);
    uint64_t x1 = 0, y1 = 0;
    if (OP == NTTK_BF_NTL) {  // butterfly.hpp:60-86
      const uint64_t Wq = static_cast<uint64_t>(wq[i]);
      if (!(0 < W && W < p)) { atomicOr(flag, 1u); continue; }
      if (Wq != static_cast<uint64_t>((u128(W) << R.n_bits) / p)) { atomicOr(flag, 2u); continue; }
      if (!(X < p && Y < p)) { atomicOr(flag, 4u); continue; }
      x1 = X + Y;
      if (x1 >= p) x1 -= p;
      const uint64_t t = X >= Y ? X - Y : X + p - Y;
      const uint64_t q = (Wq * t) >> R.n_bits;
      y1 = (W * t - q * p) & R.beta_mask;
      if (y1 >= p) y1 -= p;
    } else if (OP == NTTK_BF_HARVEY) {  // butterfly.hpp:92-121
      if (!(0 < W && W < p)) { atomicOr(flag, 1u); continue; }
      if (!(X < 2 * p && Y < 2 * p)) { atomicOr(flag, 4u); continue; }
      x1 = X + Y;
      if (x1 >= 2 * p) x1 -= 2 * p;
      const uint64_t prod = W * (X + 2 * p - Y);
      const uint64_t q = (R.p_inv_beta * (prod & R.beta_mask)) & R.beta_mask;
      y1 = (prod >> R.n_bits) + p - ((q * p) >> R.n_bits);
    } else if (OP == NTTK_BF_SCOTT) {  // butterfly.hpp:172-212 (no guard)
      const uint64_t off = uint64_t(aux0 / aux1) * p;
      if (!(0 < W && W < p)) { atomicOr(flag, 1u); continue; }
      if (!(X < off && Y < off)) { atomicOr(flag, 4u); continue; }
      x1 = X + Y;
      const uint64_t wt = W * (X + off - Y);
      const uint64_t q = (R.neg_p_inv_beta * (wt & R.beta_mask)) & R.beta_mask;
      y1 = (wt + q * p) >> R.n_bits;  // uint64 like the reference (wraps identically)
    } else {  // improved CT / GS, butterfly.hpp:224-279
      const bool gs = OP == NTTK_BF_IMPROVED_GS;
      const uint64_t bound = gs ? (p << (aux0 - 1)) : ((p << R.ell) / 2);
      if (!(W < p)) { atomicOr(flag, 1u); continue; }
      if (!(X < bound && Y < bound)) { atomicOr(flag, 4u); continue; }
      auto mp = [&](uint64_t w, uint64_t t) {
        const uint64_t h = ((w * t) * R.mu) & R.r2n_mask;
        return (((h >> R.n_bits) + 1) * p) >> R.n_bits;
      };
      if (!gs) {
        const uint64_t r = mp(W, Y);
        x1 = X + r;
        y1 = X + p - r;
      } else {
        x1 = X + Y;
        y1 = mp(W, X + (p << (aux0 - 1)) - Y);
      }
    }
    xo[i] = static_cast<int64_t>(x1);
    yo[i] = static_cast<int64_t>(y1);
  }
}

template <int OP>
cudaError_t launch_bf(const int64_t* x, const int64_t* y, const int64_t* w, const int64_t* wq,
                      int64_t* xo, int64_t* yo, size_t n, const RArgs& R, uint32_t a0, uint32_t a1,
                      unsigned* flag, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t want = (n + 255) / 256, cap = size_t(sms) * 8;
  butterfly_kernel<OP><<<static_cast<unsigned>(want < cap ? (want ? want : 1) : cap), 256, 0, st>>>(
      x, y, w, wq, xo, yo, n, R, a0, a1, flag);
  return cudaGetLastError();
}

}  // namespace

cudaError_t butterfly_launch(int op, const nttk_reduction_ctx& c, uint32_t aux0, uint32_t aux1,
                             const int64_t* x, const int64_t* y, const int64_t* w,
                             const int64_t* wq, int64_t* xo, int64_t* yo, size_t n,
                             unsigned* d_flag, cudaStream_t st) {
  RArgs R{c.p,          c.beta_mask, c.r2n_mask,   c.p_inv_beta, c.neg_p_inv_beta, c.mu,
          c.beta,       c.beta_mod_p, c.r2n_mod_p, c.n_bits,     c.ell};
  switch (op) {
    case NTTK_BF_NTL: return launch_bf<NTTK_BF_NTL>(x, y, w, wq, xo, yo, n, R, aux0, aux1, d_flag, st);
    case NTTK_BF_HARVEY: return launch_bf<NTTK_BF_HARVEY>(x, y, w, wq, xo, yo, n, R, aux0, aux1, d_flag, st);
    case NTTK_BF_SCOTT: return launch_bf<NTTK_BF_SCOTT>(x, y, w, wq, xo, yo, n, R, aux0, aux1, d_flag, st);
    case NTTK_BF_IMPROVED_CT:
      return launch_bf<NTTK_BF_IMPROVED_CT>(x, y, w, wq, xo, yo, n, R, aux0, aux1, d_flag, st);
    case NTTK_BF_IMPROVED_GS:
      return launch_bf<NTTK_BF_IMPROVED_GS>(x, y, w, wq, xo, yo, n, R, aux0, aux1, d_flag, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t reduce_launch(int op, const nttk_reduction_ctx& c, const int64_t* x, const int64_t* y,
                          int64_t* out, size_t n, unsigned* d_flag, cudaStream_t st) {
  RArgs R{c.p,          c.beta_mask, c.r2n_mask,   c.p_inv_beta, c.neg_p_inv_beta, c.mu,
          c.beta,       c.beta_mod_p, c.r2n_mod_p, c.n_bits,     c.ell};
  switch (op) {
    case NTTK_OP_MONT_REDC: return launch<NTTK_OP_MONT_REDC>(x, y, out, n, R, d_flag, st);
    case NTTK_OP_SIGNED_MONT_REDC: return launch<NTTK_OP_SIGNED_MONT_REDC>(x, y, out, n, R, d_flag, st);
    case NTTK_OP_PLANTARD_REDC: return launch<NTTK_OP_PLANTARD_REDC>(x, y, out, n, R, d_flag, st);
    case NTTK_OP_MODIFIED_PLANTARD_MUL:
      return launch<NTTK_OP_MODIFIED_PLANTARD_MUL>(x, y, out, n, R, d_flag, st);
    case NTTK_OP_TO_PLANTARD_DOMAIN: return launch<NTTK_OP_TO_PLANTARD_DOMAIN>(x, y, out, n, R, d_flag, st);
    case NTTK_OP_TO_MONTGOMERY_DOMAIN:
      return launch<NTTK_OP_TO_MONTGOMERY_DOMAIN>(x, y, out, n, R, d_flag, st);
    case NTTK_OP_MOD_P: return launch<NTTK_OP_MOD_P>(x, y, out, n, R, d_flag, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace nttk_b200
