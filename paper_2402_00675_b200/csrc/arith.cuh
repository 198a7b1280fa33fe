// arith.cuh -- sm_100a modular arithmetic and butterfly policies (device).
//
// Each policy restates one reference butterfly family on the 32-bit integer datapath
// of Blackwell, bit-exact with the reference's u64 formulas (butterfly.hpp,
// reduction.hpp) for the parameter ranges the host admits to the fast path
// (params.cpp fast_eligible):
//
//   ImprovedN16 / ImprovedN32   Alg. 10-12 modified Plantard (reduction.hpp:252-258,
//                               butterfly.hpp:224-243) with n = 16 / n = 32
//   Harvey<16|32, CT>           Alg. 8 Montgomery lazy [0, 2p) (butterfly.hpp:92-106);
//                               CT = the CT-form twin used on the negacyclic tree
//   Smont<16|32>                signed Montgomery (reduction.hpp:141-165) in CT/GS form
//                               (extension)
//   Scott32, Ntl<16|32>         Alg. 9 / Alg. 7 (butterfly.hpp:172-184, 60-71)
//
// Issue-slot economy (measured on B200, profiles/r1a_imad_microbench.txt and
// r1b_bf_microbench*.txt): IMAD runs at 64 lanes/clk/SM on the fmaheavy pipe, IMAD.HI and
// IMAD.WIDE at half that, the ALU pipe at 64; mixed into a butterfly stream every non-FMA
// instruction costs about 0.8 cycles on top of the FMA cycles.  So:
//   * plain additions are written x + y + A.zero (A.zero == 0 at run time, opaque to
//     ptxas): a three-input add only exists as IADD3 on the ALU pipe, which stops
//     ptxas from moving the adds onto the fmaheavy pipe as IMAD.IADD;
//   * ALU work is removed where the algebra allows (lazy merge outputs instead of fence
//     ops, multiply-free twiddle-1 blocks), and the umulhi form is used everywhere by
//     default (the paper form trades 2 FMA cycles for 2 shifts, measured slower).
//
// SASS per Plantard multiply (census: profiles/r1b_sass_census.txt):
//   n=16: IMAD (h = t * w_hat mu) + IMAD.HI (r = hi32(h p))        [umulhi form]
//         IMAD + SHF + IMAD + SHF (r = (((h >> 16) + 1) p) >> 16)  [paper form]
//   n=32: IMAD + IMAD.HI (h_hi) + IMAD.HI/IMAD.WIDE (r = hi32(h_hi p + p))
#pragma once

#include <cstdint>

#include "params.hpp"

namespace nttk_b200 {

__device__ __forceinline__ uint32_t mad_hi(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

__device__ __forceinline__ uint32_t umin32(uint32_t a, uint32_t b) { return a < b ? a : b; }

// x mod p, exact for every 32-bit x: q = floor(x m / 2^32) with m = floor((2^32-1)/p)
// undershoots floor(x/p) by at most one, one min() fixes it.
__device__ __forceinline__ uint32_t mod_u32(uint32_t x, const FastArgs& A) {
  const uint32_t r = x - __umulhi(x, A.canon_m) * A.p;
  return umin32(r, r - A.p);
}
// x mod p for x < 2^16: m = ceil(2^32 / p) makes the quotient exact (two IMADs).
__device__ __forceinline__ uint32_t mod_u16(uint32_t x, const FastArgs& A) {
  return x - __umulhi(x, A.canon_m16) * A.p;
}
// x mod p for x < 2^17 with the host-validated Barrett pair (A.flags bit 0):
// IMAD + SHF + IMAD (x + q (-p): no negation op), no IMAD.HI
__device__ __forceinline__ uint32_t mod_cb(uint32_t x, const FastArgs& A) {
  return x + ((x * A.cb_m) >> A.cb_s) * A.negp;
}
// x mod p for any 32-bit x via the host-validated shift reduction (A.flags bit 1)
__device__ __forceinline__ uint32_t mod_cs(uint32_t x, const FastArgs& A) {
  const uint32_t r = x + (x >> A.cs_s) * A.negp;
  return umin32(r, r - A.p);
}
// Opaque identity (A.zero == 0): keeps ptxas from folding the following additions into
// the preceding IMAD.HI as an addend -- it then re-issues a second IMAD.HI for the other
// use of the same product, doubling the most expensive instruction.  One ALU op instead.
__device__ __forceinline__ uint32_t fence_val(uint32_t r, const FastArgs& A) {
  return r ^ A.zero;
}
// canonical residue of a two's complement 32-bit value
__device__ __forceinline__ uint32_t mod_s32(uint32_t x, const FastArgs& A) {
  // x + 2^31 is non-negative; subtract 2^31 mod p afterwards
  const uint32_t c = mod_u32(x ^ 0x80000000u, A);
  const uint32_t k = mod_u32(0x80000000u, A);
  const uint32_t t = c - k;
  return umin32(t, t + A.p);
}

// ---------------------------------------------------------------------------
// Modified Plantard multiply (Alg. 10), twiddle premultiplied by mu.
//   reference:  h = ((w t) mu) mod 2^{2n};  r = (((h >> n) + 1) p) >> n
// n = 16, umulhi form: on a 32-bit datapath the full 2n-bit product h p is one
// IMAD.HI away, and Prop. 4's exact-quotient identity r = (h p - w t) / 2^{2n}
// (asserted by reduction_test.cpp:166-170) with 0 <= w t < 2^{2n}
// gives r = floor(h p / 2^{2n}) = hi32(h p) exactly.
template <bool PAPER_FORM>
__device__ __forceinline__ uint32_t mp_n16(uint32_t t, uint32_t wm, uint32_t p) {
  const uint32_t h = t * wm;
  if (PAPER_FORM) return (((h >> 16) + 1u) * p) >> 16;
  return __umulhi(h, p);
}
// n = 32: only h_hi = hi32(h) is needed: h_hi = hi32(lo t) + hi t (mod 2^32), and
// r = hi32((h_hi + 1) p) = hi32(h_hi p + p): IMAD.HI + IMAD + IMAD.WIDE whose 64-bit
// addend {p, 0} is loop-invariant (a mad.hi with a register addend would need a zeroed
// register pair rebuilt with IMAD.MOV per butterfly).
__device__ __forceinline__ uint32_t mp_n32(uint32_t t, uint32_t lo, uint32_t hi, uint32_t p) {
  const uint32_t hh = hi * t + __umulhi(lo, t);
  return static_cast<uint32_t>((static_cast<uint64_t>(hh) * p + p) >> 32);
}

// ---------------------------------------------------------------------------
// Policies.  Values live in 32-bit registers (signed kinds: two's complement).
//   fwd(x, y, w)        forward butterfly (CT form unless noted)
//   inv(x, y, w, off)   GS form, off = 2^{layer-1} p
//   scale(v)            final N^{-1} pass (transform.hpp:323-335), canonical
//   inv_last(x, y, off) last merge layer with the N^{-1} pass folded in (kFold)

// The X-side product of the last (N^{-1}-folded) merge layer uses the paper form (IMAD + 2
// shifts, ALU-balanced); the umulhi form there (2 fewer instructions, +16 FMA cycles)
// measured neutral.
constexpr bool kLastPaper = true;

template <bool PAPER_FORM = false>
struct ImprovedN16 {
  using Tw = uint32_t;
  static constexpr bool kSigned = false;
  static constexpr bool kFold = true;
  __device__ static Tw tw(const FastArgs& A, int k) { return A.lo[k]; }
  // Alg. 11 (butterfly.hpp:224-230)
  __device__ static void fwd(uint32_t& x, uint32_t& y, Tw w, const FastArgs& A) {
    const uint32_t r = mp_n16<PAPER_FORM>(y, w, A.p);
    y = x + A.p - r;
    x = x + r + A.zero;
  }
  // twiddle w = omega^0 = 1: MP(w_hat, Y) is the canonical residue of Y -- no multiply.
  // Layer s inputs are < s p: r = Y (s = 1), min(Y, Y - p) (s = 2), and for s = 3, 4 first
  // min(Y, Y - 2p) < 2p, then min(., . - p)
  __device__ static void fwd_w1(uint32_t& x, uint32_t& y, int layer, const FastArgs& A) {
    uint32_t r = y;
    if (layer >= 3) r = umin32(r, r - A.two_p);
    if (layer >= 2) r = umin32(r, r - A.p);
    y = x + A.p - r;
    x = x + r + A.zero;
  }
  // Alg. 12 (butterfly.hpp:235-243)
  __device__ static void inv(uint32_t& x, uint32_t& y, Tw w, uint32_t off, const FastArgs& A) {
    const uint32_t t = x + off - y;
    x = x + y + A.zero;
    y = fence_val(mp_n16<PAPER_FORM>(t, w, A.p), A);
  }
  __device__ static uint32_t scale(uint32_t v, const FastArgs& A) {
    return mp_n16<PAPER_FORM>(v, A.scale_lo, A.p);
  }
  // MP(1^, v): canonical residue of any v inside Prop. 4's range (narrow inverse)
  __device__ static uint32_t canon1(uint32_t v, const FastArgs& A) {
    return mp_n16<false>(v, A.one_lo, A.p);
  }
  // (X, Y) -> (MP(n^, X + Y), MP((w n^{-1})^, X + off - Y)): both canonical, so the
  // result equals scale() applied after the last merge (canonical outputs are unique)
  __device__ static void inv_last(uint32_t& x, uint32_t& y, uint32_t off, const FastArgs& A) {
    const uint32_t t = x + off - y;
    x = mp_n16<kLastPaper>(x + y + A.zero, A.scale_lo, A.p);
    y = mp_n16<PAPER_FORM>(t, A.fold_lo, A.p);
  }
  // ---- lazy merge (inv_body_lazy, umulhi form only) ----
  // A merge output Y' = MP(w, T) = hi32(h p) is carried as h = T w_hat mu; the consumer
  // issues the IMAD.HI.  Lazy words only ever pair with lazy words (GS outputs at j + len
  // meet at the next layer), so the consumer computes X = hi(h_X p) and takes the sum
  // with Y's IMAD.HI as its addend: S = hi(h_Y p) + X, T = 2X + off - S.  Same words as
  // inv(); per butterfly IMAD + IMAD.HI + 2 ALU ops, no fence op, no re-issued IMAD.HI.
  static constexpr bool kLazy = !PAPER_FORM;
  __device__ static uint32_t materialize(uint32_t h, const FastArgs& A) { return __umulhi(h, A.p); }
  // materialised inputs -> (X + Y, lazy MP(w, X + off - Y))
  __device__ static void inv_h(uint32_t& x, uint32_t& y, Tw w, uint32_t off, const FastArgs& A) {
    const uint32_t t = x + off - y;
    x = x + y + A.zero;
    y = t * w;
  }
  // lazy inputs -> (X + Y, lazy MP(w, X + off - Y)).  The IMAD.HI addend is a 64-bit
  // register pair, so a 32-bit addend costs a zeroing move; instead X comes out of a
  // 64-bit product whose low word is w_X T_X (Prop. 4: h p = r 2^32 + w T exactly), and
  // that pair is the addend of Y's product: hi(h_Y p + {w_X T_X, X}) = X + Y whenever
  // w_X T_X + w_Y T_Y < 2^32 (host-validated, FastArgs flags bit 3).
  __device__ static uint32_t sum_hh(uint32_t hx, uint32_t hy, uint32_t& X, const FastArgs& A) {
    const uint64_t px = static_cast<uint64_t>(hx) * A.p;  // {w_X T_X, X}
    uint32_t xh = static_cast<uint32_t>(px >> 32);
    asm("mov.b32 %0, %0;" : "+r"(xh));  // opaque: keeps 2X from becoming a funnel shift
    X = xh;
    return static_cast<uint32_t>((static_cast<uint64_t>(hy) * A.p + px) >> 32);
  }
  __device__ static void inv_hh(uint32_t& x, uint32_t& y, Tw w, uint32_t off, const FastArgs& A) {
    uint32_t X;
    const uint32_t S = sum_hh(x, y, X, A);
    const uint32_t t = X + X + off - S + A.zero;
    x = S;
    y = t * w;
  }
  __device__ static void inv_last_hh(uint32_t& x, uint32_t& y, uint32_t off, const FastArgs& A) {
    uint32_t X;
    const uint32_t S = sum_hh(x, y, X, A);
    const uint32_t t = X + X + off - S + A.zero;
    x = mp_n16<kLastPaper>(S, A.scale_lo, A.p);
    y = mp_n16<PAPER_FORM>(t, A.fold_lo, A.p);
  }
  // product stage (fused polymul): x -> (x (-2^{2n}) mod p) mu, then MP(.., y) = x y mod p
  using Enc = uint32_t;
  __device__ static Enc enc(uint32_t x, const ProdArgs& Q, const FastArgs& A) {
    return mp_n16<false>(x, Q.enc_lo, A.p) * Q.mu_lo;
  }
  __device__ static Enc genc(int k, const ProdArgs& Q) { return Q.g_lo[k]; }
  __device__ static uint32_t mulc(uint32_t y, Enc e, const FastArgs& A) {
    return mp_n16<false>(y, e, A.p);
  }
};

struct ImprovedN32 {
  using Tw = uint2;
  static constexpr bool kSigned = false;
  static constexpr bool kFold = true;
  __device__ static Tw tw(const FastArgs& A, int k) { return make_uint2(A.lo[k], A.hi[k]); }
  __device__ static void fwd(uint32_t& x, uint32_t& y, Tw w, const FastArgs& A) {
    const uint32_t r = mp_n32(y, w.x, w.y, A.p);
    y = x + A.p - r;
    x = x + r + A.zero;
  }
  __device__ static void fwd_w1(uint32_t& x, uint32_t& y, int layer, const FastArgs& A) {
    uint32_t r = y;  // see ImprovedN16::fwd_w1
    if (layer >= 3) r = umin32(r, r - A.two_p);
    if (layer >= 2) r = umin32(r, r - A.p);
    y = x + A.p - r;
    x = x + r + A.zero;
  }
  __device__ static void inv(uint32_t& x, uint32_t& y, Tw w, uint32_t off, const FastArgs& A) {
    const uint32_t t = x + off - y;
    x = x + y + A.zero;
    y = fence_val(mp_n32(t, w.x, w.y, A.p), A);
  }
  __device__ static uint32_t scale(uint32_t v, const FastArgs& A) {
    return mp_n32(v, A.scale_lo, A.scale_hi, A.p);
  }
  // ---- lazy merge (see ImprovedN16) at n = 32 ----
  // The lazy word is h = h_hi (the first two multiplies of mp_n32); r = hi32(h p + p).
  // lo32(h p + p) = p + (W T - h_lo p) / 2^32 lies in (0, 2p) (Prop. 4 with 2n = 64), so
  // h_X p + 2p = {lo_X + p, X} (no carry) and hi(h_Y p + (h_X p + 2p)) = X + Y: both pair
  // addends are loop-invariant {p, 0} / {2p, 0} register pairs (flag bit 3, always valid on
  // the fast path).
  static constexpr bool kLazy = true;
  __device__ static uint32_t hprime(uint32_t t, Tw w) { return w.y * t + __umulhi(w.x, t); }
  __device__ static uint32_t materialize(uint32_t h, const FastArgs& A) {
    return static_cast<uint32_t>((static_cast<uint64_t>(h) * A.p + A.p) >> 32);
  }
  __device__ static uint32_t sum_hh(uint32_t hx, uint32_t hy, uint32_t& X, const FastArgs& A) {
    const uint64_t px = static_cast<uint64_t>(hx) * A.p + A.two_p;  // {lo_X + p, X}
    uint32_t xh = static_cast<uint32_t>(px >> 32);
    asm("mov.b32 %0, %0;" : "+r"(xh));  // opaque: keeps 2X from becoming a funnel shift
    X = xh;
    return static_cast<uint32_t>((static_cast<uint64_t>(hy) * A.p + px) >> 32);
  }
  __device__ static void inv_h(uint32_t& x, uint32_t& y, Tw w, uint32_t off, const FastArgs& A) {
    const uint32_t t = x + off - y;
    x = x + y + A.zero;
    y = hprime(t, w);
  }
  __device__ static void inv_hh(uint32_t& x, uint32_t& y, Tw w, uint32_t off, const FastArgs& A) {
    uint32_t X;
    const uint32_t S = sum_hh(x, y, X, A);
    const uint32_t t = X + X + off - S + A.zero;
    x = S;
    y = hprime(t, w);
  }
  __device__ static void inv_last_hh(uint32_t& x, uint32_t& y, uint32_t off, const FastArgs& A) {
    uint32_t X;
    const uint32_t S = sum_hh(x, y, X, A);
    const uint32_t t = X + X + off - S + A.zero;
    x = mp_n32(S, A.scale_lo, A.scale_hi, A.p);
    y = mp_n32(t, A.fold_lo, A.fold_hi, A.p);
  }
  __device__ static void inv_last(uint32_t& x, uint32_t& y, uint32_t off, const FastArgs& A) {
    const uint32_t t = x + off - y;
    x = mp_n32(x + y + A.zero, A.scale_lo, A.scale_hi, A.p);
    y = mp_n32(t, A.fold_lo, A.fold_hi, A.p);
  }
  using Enc = uint2;
  __device__ static Enc enc(uint32_t x, const ProdArgs& Q, const FastArgs& A) {
    const uint32_t xp = mp_n32(x, Q.enc_lo, Q.enc_hi, A.p);  // x (-2^{2n}) mod p
    return make_uint2(xp * Q.mu_lo, __umulhi(xp, Q.mu_lo) + xp * Q.mu_hi);  // xp mu mod 2^64
  }
  __device__ static Enc genc(int k, const ProdArgs& Q) { return make_uint2(Q.g_lo[k], Q.g_hi[k]); }
  __device__ static uint32_t mulc(uint32_t y, Enc e, const FastArgs& A) {
    return mp_n32(y, e.x, e.y, A.p);
  }
};

// Montgomery reduction of prod = w t with p^{-1} (harvey_core's Y path,
// butterfly.hpp:101-105):  r1 + p - ((q p) >> n), q = p^{-1} lo_n(prod) mod 2^n
template <int N_BITS>
__device__ __forceinline__ uint32_t harvey_mul(uint32_t t, uint32_t w, const FastArgs& A) {
  if (N_BITS == 16) {
    const uint32_t prod = w * t;        // < 4p^2 < 2^32
    const uint32_t q16 = prod * A.pinv; // (p^{-1} prod mod 2^16) << 16
    return (prod >> 16) + A.p - __umulhi(q16, A.p);
  } else {
    const uint64_t prod = static_cast<uint64_t>(w) * t;  // IMAD.WIDE
    const uint32_t q = static_cast<uint32_t>(prod) * A.pinv;
    return static_cast<uint32_t>(prod >> 32) + A.p - __umulhi(q, A.p);
  }
}

template <int N_BITS, bool CT_FORWARD>
struct Harvey {
  using Tw = uint32_t;
  static constexpr bool kSigned = false;
  static constexpr bool kFold = true;
  __device__ static Tw tw(const FastArgs& A, int k) { return A.lo[k]; }
  __device__ static void fwd(uint32_t& x, uint32_t& y, Tw w, const FastArgs& A) {
    if (CT_FORWARD) {
      // CT-form harvey (extension for the negacyclic tree): all values in [0, 2p)
      const uint32_t r = harvey_mul<N_BITS>(y, w, A);
      const uint32_t a = x + r + A.zero, b = x + A.two_p - r;
      x = umin32(a, a - A.two_p);
      y = umin32(b, b - A.two_p);
    } else {
      dif(x, y, w, A);
    }
  }
  // harvey_core (butterfly.hpp:92-106): X' = X + Y mod 2p (branchless), Y' lazy
  __device__ static void dif(uint32_t& x, uint32_t& y, Tw w, const FastArgs& A) {
    const uint32_t s = x + y + A.zero;
    const uint32_t t = x + A.two_p - y;
    x = umin32(s, s - A.two_p);
    y = harvey_mul<N_BITS>(t, w, A);
  }
  __device__ static void inv(uint32_t& x, uint32_t& y, Tw w, uint32_t, const FastArgs& A) {
    dif(x, y, w, A);
  }
  // merge butterfly whose twiddle is 1 (TW1): Y' = X - Y mod 2p, any representative in
  // [0, 2p) keeps the canonical inverse output bit-exact
  __device__ static void inv_w1(uint32_t& x, uint32_t& y, const FastArgs& A) {
    const uint32_t s = x + y + A.zero, t = x + A.two_p - y;
    x = umin32(s, s - A.two_p);
    y = umin32(t, t - A.two_p);
  }
  // v in [0, 2p) -> v n^{-1} mod p, canonical (the reference's mul_mod,
  // transform.hpp:331-335; any exact method is bit-identical)
  __device__ static uint32_t scale(uint32_t v, const FastArgs& A) {
    const uint32_t r = harvey_mul<N_BITS>(v, A.scale_lo, A);  // (0, 2p)
    return umin32(r, r - A.p);
  }
  __device__ static void inv_last(uint32_t& x, uint32_t& y, uint32_t, const FastArgs& A) {
    const uint32_t t = x + A.two_p - y;
    const uint32_t a = harvey_mul<N_BITS>(x + y + A.zero, A.scale_lo, A);  // X + Y < 4p
    const uint32_t b = harvey_mul<N_BITS>(t, A.fold_lo, A);
    x = umin32(a, a - A.p);
    y = umin32(b, b - A.p);
  }
  // product stage: x -> x 2^n mod p (lazy, via R^2), then Montgomery product, canonical
  using Enc = uint32_t;
  __device__ static Enc enc(uint32_t x, const ProdArgs& Q, const FastArgs& A) {
    return harvey_mul<N_BITS>(x, Q.enc_lo, A);
  }
  __device__ static Enc genc(int k, const ProdArgs& Q) { return Q.g_lo[k]; }
  __device__ static uint32_t mulc(uint32_t y, Enc e, const FastArgs& A) {
    const uint32_t r = harvey_mul<N_BITS>(y, e, A);
    return umin32(r, r - A.p);
  }
};

// scott_core's product at n = 32 (butterfly.hpp:172-184): (w t + q p) >> 32 with
// q = -p^{-1} lo(w t) mod 2^32 (A.pinv); w < p, t < 2^32 keep w t + q p < 2^64 and the
// result < 2p.  IMAD.WIDE + IMAD + IMAD.WIDE (64-bit accumulate), 10 fmaheavy cycles.
__device__ __forceinline__ uint32_t scott_mul(uint32_t t, uint32_t w, const FastArgs& A) {
  const uint64_t wt = static_cast<uint64_t>(w) * t;
  const uint32_t q = static_cast<uint32_t>(wt) * A.pinv;
  return static_cast<uint32_t>((wt + static_cast<uint64_t>(q) * A.p) >> 32);
}

// Alg. 9 (butterfly.hpp:172-184), n = 32: X' = X + Y unreduced, Y' = scott_mul(X + (N/L)p
// - Y) in [0, 2p).  The same core runs the DIF forward (per-index twiddles) and the GS
// merge layers (per-block), as in the reference.  Host-validated (fast_eligible): no T
// underflows or overflows 32 bits, so every word equals the reference's uint64 word.
struct Scott32 {
  using Tw = uint32_t;
  static constexpr bool kSigned = false;
  static constexpr bool kFold = true;
  __device__ static Tw tw(const FastArgs& A, int k) { return A.lo[k]; }
  __device__ static void fwd(uint32_t& x, uint32_t& y, Tw w, const FastArgs& A) {
    const uint32_t t = x + A.soff - y;
    x = x + y + A.zero;
    y = scott_mul(t, w, A);
  }
  __device__ static void inv(uint32_t& x, uint32_t& y, Tw w, uint32_t, const FastArgs& A) {
    fwd(x, y, w, A);
  }
  // twiddle 1 (TW1): canonical X - Y mod p without the Shoup product
  __device__ static void inv_w1(uint32_t& x, uint32_t& y, const FastArgs& A) {
    const uint32_t s = x + y + A.zero, t = x + A.p - y;
    x = umin32(s, s - A.p);
    y = umin32(t, t - A.p);
  }
  // canonical v n^{-1} mod p (transform.hpp:331-335; any exact method is bit-identical)
  __device__ static uint32_t scale(uint32_t v, const FastArgs& A) {
    const uint32_t r = scott_mul(v, A.scale_lo, A);
    return umin32(r, r - A.p);
  }
  __device__ static void inv_last(uint32_t& x, uint32_t& y, uint32_t, const FastArgs& A) {
    const uint32_t t = x + A.soff - y;
    const uint32_t a = scott_mul(x + y + A.zero, A.scale_lo, A);
    const uint32_t b = scott_mul(t, A.fold_lo, A);
    x = umin32(a, a - A.p);
    y = umin32(b, b - A.p);
  }
};

// ntl_core's Shoup product (butterfly.hpp:60-71): q = (w' t) >> n, w' = floor(w 2^n / p);
// w t - q p lies in [0, 2p) for every t < 2^n, then one conditional subtraction.  The
// result is the canonical residue, so feeding t + p for X - Y mod p changes nothing.
template <int N_BITS>
__device__ __forceinline__ uint32_t shoup_mul(uint32_t t, uint32_t w, uint32_t wq,
                                              const FastArgs& A) {
  const uint32_t q = N_BITS == 16 ? (wq * t) >> 16 : __umulhi(wq, t);
  const uint32_t r = w * t + q * A.negp;
  return umin32(r, r - A.p);
}

// Alg. 7 (butterfly.hpp:60-71): canonical in, canonical out; DIF forward per-index,
// GS merge per-block.  Outputs are unique residues, so these exact forms are bit-identical.
template <int N_BITS>
struct Ntl {
  using Tw = uint2;  // (w, floor(w 2^n / p))
  static constexpr bool kSigned = false;
  static constexpr bool kFold = true;
  __device__ static Tw tw(const FastArgs& A, int k) { return make_uint2(A.lo[k], A.hi[k]); }
  __device__ static void fwd(uint32_t& x, uint32_t& y, Tw w, const FastArgs& A) {
    const uint32_t t = x + A.p - y;  // (0, 2p)
    const uint32_t s = x + y + A.zero;
    x = umin32(s, s - A.p);
    y = shoup_mul<N_BITS>(t, w.x, w.y, A);
  }
  __device__ static void inv(uint32_t& x, uint32_t& y, Tw w, uint32_t, const FastArgs& A) {
    fwd(x, y, w, A);
  }
  __device__ static uint32_t scale(uint32_t v, const FastArgs& A) {
    return shoup_mul<N_BITS>(v, A.scale_lo, A.scale_hi, A);
  }
  __device__ static void inv_last(uint32_t& x, uint32_t& y, uint32_t, const FastArgs& A) {
    const uint32_t t = x + A.p - y;
    x = shoup_mul<N_BITS>(x + y + A.zero, A.scale_lo, A.scale_hi, A);
    y = shoup_mul<N_BITS>(t, A.fold_lo, A.fold_hi, A);
  }
};

// Signed Montgomery (reduction.hpp:141-165): r = (A - m p) / 2^n, m = centered
// lo_n(A p^{-1}); A = w y with the premultiplied quotient factor (w p^{-1} mod 2^n).
template <int N_BITS>
__device__ __forceinline__ int32_t smont_mul(int32_t y, int32_t w, uint32_t wq,
                                             const FastArgs& A) {
  if (N_BITS == 16) {
    const int32_t a = w * y;                                         // |a| < p 2^15
    const int32_t m = static_cast<int32_t>(wq * static_cast<uint32_t>(y)) >> 16;  // centered
    return (a - m * static_cast<int32_t>(A.p)) >> 16;
  } else {
    const int64_t a = static_cast<int64_t>(w) * y;
    const int32_t m = static_cast<int32_t>(wq * static_cast<uint32_t>(y));
    return static_cast<int32_t>((a - static_cast<int64_t>(m) * A.p) >> 32);
  }
}

// signed Barrett a - round(a V / 2^S) p, S = n + 10 (extension; oracle
// or_signed_barrett)
template <int N_BITS>
__device__ __forceinline__ int32_t sbarrett(int32_t a, const FastArgs& A) {
  if (N_BITS == 16) {
    const int32_t q = (a * static_cast<int32_t>(A.barrett_v) + (1 << 25)) >> 26;
    return a - q * static_cast<int32_t>(A.p);
  } else {
    const int64_t q = (static_cast<int64_t>(a) * A.barrett_v + (int64_t(1) << 41)) >> 42;
    return a - static_cast<int32_t>(q) * static_cast<int32_t>(A.p);
  }
}

template <int N_BITS>
struct Smont {
  using Tw = uint2;  // (w, w p^{-1} mod 2^n [n=16: << 16])
  static constexpr bool kSigned = true;
  static constexpr bool kFold = false;
  __device__ static Tw tw(const FastArgs& A, int k) { return make_uint2(A.lo[k], A.hi[k]); }
  __device__ static void fwd(uint32_t& x, uint32_t& y, Tw w, const FastArgs& A) {
    const int32_t t = smont_mul<N_BITS>(static_cast<int32_t>(y), static_cast<int32_t>(w.x), w.y, A);
    y = static_cast<uint32_t>(static_cast<int32_t>(x) - t);
    x = static_cast<uint32_t>(static_cast<int32_t>(x) + t) + A.zero;
  }
  __device__ static void inv(uint32_t& x, uint32_t& y, Tw w, uint32_t, const FastArgs& A) {
    const int32_t xs = static_cast<int32_t>(x), ys = static_cast<int32_t>(y);
    x = static_cast<uint32_t>(sbarrett<N_BITS>(xs + ys, A));
    y = static_cast<uint32_t>(smont_mul<N_BITS>(xs - ys, static_cast<int32_t>(w.x), w.y, A));
  }
  __device__ static uint32_t scale(uint32_t v, const FastArgs& A) {
    const int32_t r = smont_mul<N_BITS>(static_cast<int32_t>(v), static_cast<int32_t>(A.scale_lo),
                                        A.scale_hi, A);
    return static_cast<uint32_t>(r + (r < 0 ? static_cast<int32_t>(A.p) : 0));
  }
  __device__ static void inv_last(uint32_t& x, uint32_t& y, uint32_t off, const FastArgs& A) {
    (void)off;
    (void)x;
    (void)y;
  }
  // product stage: x -> x 2^n (signed Montgomery via R^2), then signed product
  using Enc = uint2;
  __device__ static Enc enc(uint32_t x, const ProdArgs& Q, const FastArgs& A) {
    const int32_t xs = smont_mul<N_BITS>(static_cast<int32_t>(x), static_cast<int32_t>(Q.enc_lo),
                                         Q.enc_hi, A);
    const uint32_t q = N_BITS == 16 ? static_cast<uint32_t>(xs) * (A.pinv << 16)
                                    : static_cast<uint32_t>(xs) * A.pinv;
    return make_uint2(static_cast<uint32_t>(xs), q);
  }
  __device__ static Enc genc(int k, const ProdArgs& Q) { return make_uint2(Q.g_lo[k], Q.g_hi[k]); }
  __device__ static uint32_t mulc(uint32_t y, Enc e, const FastArgs& A) {
    const int32_t r = smont_mul<N_BITS>(static_cast<int32_t>(y), static_cast<int32_t>(e.x), e.y, A);
    return static_cast<uint32_t>(r + (r < 0 ? static_cast<int32_t>(A.p) : 0));
  }
};

// ---------------------------------------------------------------------------
// Lazy twins of Harvey<16, true> and Smont<16> for the fused polymul (polymul_tma.cu).
// Inside fused fwd(a), fwd(b), product, inverse only the canonical output is pinned (it is
// unique), so -- exactly as the improved kernels carry lazy Plantard words -- the
// Montgomery kinds drop every intermediate normalisation that exists only to keep the
// standalone transform's words bit-exact:
//   HarveyLazy16  no [0, 2p) min-subtractions in the CT forward or the GS inverse; the
//                 inverse carries the improved kernel's offsets 2^{m-1} p, the last layer
//                 folds N^{-1} and ends with one exact Barrett reduction (mod_cb)
//   SmontLazy16   no signed Barrett on the GS sums; N^{-1} folded into the last layer,
//                 which canonicalises with one lift + mod_cb
// Host-validated bounds (params.cpp, ProdArgs::lazy; n = 16, u16):
//   harvey: (1 + 2L) p < 2^16 (every forward/product operand < 2^16, so each Montgomery
//           product r = d + p lies in (0, 2p)); (p - 1) 2^L p < 2^32 (inverse products);
//           final r < (p - 1) 2^L p / 2^16 + p < 2^17 (mod_cb exact)
//   smont:  (L + 1) p <= 2^16 (|r| < p in the forward and the product);
//           (p/2 + 1) 2^L p + 2^15 p < 2^31 (no int32 overflow in the inverse products);
//           final |r| + lzk < 2^17 with lzk = K p > max |r| (FastArgs::lzk)
// Montgomery difference: d = (w t >> 16) - hi(q p) with q = (p^{-1} w t mod 2^16) << 16;
// the Montgomery product is r = d + p (harvey_mul), so callers fold the + p into their adds.
__device__ __forceinline__ uint32_t mont_diff16(uint32_t t, uint32_t w, const FastArgs& A) {
  const uint32_t prod = w * t;
  const uint32_t q16 = prod * A.pinv;
  return (prod >> 16) - __umulhi(q16, A.p);
}

struct HarveyLazy16 {
  using Tw = uint32_t;
  static constexpr bool kSigned = false;
  static constexpr bool kFold = true;
  __device__ static Tw tw(const FastArgs& A, int k) { return A.lo[k]; }
  // CT: X' = X + r, Y' = X + 2p - r with r = d + p in (0, 2p)
  __device__ static void fwd(uint32_t& x, uint32_t& y, Tw w, const FastArgs& A) {
    const uint32_t d = mont_diff16(y, w, A);
    y = x + A.p - d;
    x = x + d + A.p;
  }
  // GS at merge depth m (off = 2^{m-1} p >= every Y input): X' = X + Y, Y' = r(X + off - Y)
  __device__ static void inv(uint32_t& x, uint32_t& y, Tw w, uint32_t off, const FastArgs& A) {
    const uint32_t t = x + off - y;
    x = x + y + A.zero;
    y = mont_diff16(t, w, A) + A.p;
  }
  __device__ static void inv_last(uint32_t& x, uint32_t& y, uint32_t off, const FastArgs& A) {
    const uint32_t t = x + off - y;
    const uint32_t a = mont_diff16(x + y + A.zero, A.scale_lo, A) + A.p;
    const uint32_t b = mont_diff16(t, A.fold_lo, A) + A.p;
    x = mod_cb(a, A);
    y = mod_cb(b, A);
  }
  __device__ static uint32_t scale(uint32_t v, const FastArgs& A) { return mod_cb(mont_diff16(v, A.scale_lo, A) + A.p, A); }
  // product stage: canonical encoding x R mod p (one min), canonical product
  using Enc = uint32_t;
  __device__ static Enc enc(uint32_t x, const ProdArgs& Q, const FastArgs& A) {
    const uint32_t r = mont_diff16(x, Q.enc_lo, A) + A.p;
    return umin32(r, r - A.p);
  }
  __device__ static Enc genc(int k, const ProdArgs& Q) { return Q.g_lo[k]; }
  __device__ static uint32_t mulc(uint32_t y, Enc e, const FastArgs& A) {
    const uint32_t r = mont_diff16(y, e, A) + A.p;
    return umin32(r, r - A.p);
  }
};

struct SmontLazy16 {
  using Tw = uint2;
  static constexpr bool kSigned = true;
  static constexpr bool kFold = true;
  __device__ static Tw tw(const FastArgs& A, int k) { return make_uint2(A.lo[k], A.hi[k]); }
  __device__ static void fwd(uint32_t& x, uint32_t& y, Tw w, const FastArgs& A) {
    Smont<16>::fwd(x, y, w, A);
  }
  __device__ static void inv(uint32_t& x, uint32_t& y, Tw w, uint32_t, const FastArgs& A) {
    const int32_t xs = static_cast<int32_t>(x), ys = static_cast<int32_t>(y);
    x = static_cast<uint32_t>(xs + ys) + A.zero;
    y = static_cast<uint32_t>(smont_mul<16>(xs - ys, static_cast<int32_t>(w.x), w.y, A));
  }
  // canonical residue of a signed |r| < lzk (lzk = K p): lift, then exact Barrett
  __device__ static uint32_t canon(int32_t r, const FastArgs& A) {
    return mod_cb(static_cast<uint32_t>(r) + A.lzk, A);
  }
  __device__ static void inv_last(uint32_t& x, uint32_t& y, uint32_t, const FastArgs& A) {
    const int32_t xs = static_cast<int32_t>(x), ys = static_cast<int32_t>(y);
    const int32_t a = smont_mul<16>(xs + ys, static_cast<int32_t>(A.scale_lo), A.scale_hi, A);
    const int32_t b = smont_mul<16>(xs - ys, static_cast<int32_t>(A.fold_lo), A.fold_hi, A);
    x = canon(a, A);
    y = canon(b, A);
  }
  __device__ static uint32_t scale(uint32_t v, const FastArgs& A) {
    return canon(smont_mul<16>(static_cast<int32_t>(v), static_cast<int32_t>(A.scale_lo), A.scale_hi, A), A);
  }
  using Enc = uint2;
  __device__ static Enc enc(uint32_t x, const ProdArgs& Q, const FastArgs& A) {
    return Smont<16>::enc(x, Q, A);
  }
  __device__ static Enc genc(int k, const ProdArgs& Q) { return Smont<16>::genc(k, Q); }
  __device__ static uint32_t mulc(uint32_t y, Enc e, const FastArgs& A) {
    return Smont<16>::mulc(y, e, A);
  }
};

}  // namespace nttk_b200
