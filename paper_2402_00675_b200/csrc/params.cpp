// params.cpp -- host-side parameter bundle of the B200 engine.
//
// Exact host precompute for one parameter set, the B200 counterpart of
// build_params (proj/include/nttk/params.hpp:137-268): validation with every fault
// collected into one message (same fault strings as the reference so callers that
// grep them keep working), the primitive root, the plain twiddle schedules and their
// per-kind encodings, plus the device-ready images for the N=256 fast kernels.
#include "params.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace nttk_b200 {

uint64_t pow_mod(uint64_t b, uint64_t e, uint64_t m) {
  uint64_t acc = 1 % m;
  b %= m;
  for (; e; e >>= 1) {
    if (e & 1) acc = static_cast<uint64_t>(u128(acc) * b % m);
    b = static_cast<uint64_t>(u128(b) * b % m);
  }
  return acc;
}

uint64_t bit_reverse(uint64_t x, unsigned bits) {
  uint64_t r = 0;
  for (unsigned i = 0; i < bits; ++i, x >>= 1) r = (r << 1) | (x & 1);
  return r;
}

// inverse of a modulo m (m up to 2^64 as u128), extended Euclid (crt.hpp:37-57)
u128 inverse(u128 a, u128 m) {
  a %= m;
  i128 r0 = static_cast<i128>(m), r1 = static_cast<i128>(a), t0 = 0, t1 = 1;
  while (r1 != 0) {
    const i128 q = r0 / r1;
    i128 tmp = r0 - q * r1;
    r0 = r1;
    r1 = tmp;
    tmp = t0 - q * t1;
    t0 = t1;
    t1 = tmp;
  }
  i128 v = t0 % static_cast<i128>(m);
  if (v < 0) v += static_cast<i128>(m);
  return static_cast<u128>(v);
}

// reduction.hpp:80-117
Ctx make_ctx(uint64_t p, unsigned n, unsigned ell) {
  Ctx c;
  c.p = static_cast<uint32_t>(p);
  c.n_bits = n;
  c.ell = ell;
  c.beta = uint64_t(1) << n;
  c.beta_mask = c.beta - 1;
  c.r2n_mask = 2 * n == 64 ? ~uint64_t(0) : (uint64_t(1) << (2 * n)) - 1;
  c.p_inv_beta = static_cast<uint64_t>(inverse(p, u128(1) << n));
  c.neg_p_inv_beta = (c.beta - c.p_inv_beta) & c.beta_mask;
  c.mu = static_cast<uint64_t>(inverse(p, u128(1) << (2 * n)));
  c.beta_mod_p = c.beta % p;
  c.r2n_mod_p = pow_mod(2, 2 * n, p);
  return c;
}

namespace {

unsigned log2_floor(uint64_t x) {
  unsigned r = 0;
  while (x >>= 1) ++r;
  return r;
}

bool pow2(uint64_t x) { return x && !(x & (x - 1)); }

bool prime(uint64_t x) {
  if (x < 2) return false;
  for (uint64_t d = 2; d * d <= x; ++d)
    if (x % d == 0) return false;
  return true;
}

uint64_t to_plantard(uint64_t w, const Ctx& c) {  // reduction.hpp:279-283
  return (c.p - static_cast<uint64_t>(u128(w) * c.r2n_mod_p % c.p)) % c.p;
}
uint64_t to_mont(uint64_t w, const Ctx& c) {  // reduction.hpp:287-291
  return static_cast<uint64_t>(u128(w) * c.beta_mod_p % c.p);
}
int64_t to_smont(uint64_t w, const Ctx& c) {  // centered Montgomery twiddle (extension)
  const uint64_t m = to_mont(w % c.p, c);
  return m > c.p / 2 ? static_cast<int64_t>(m) - static_cast<int64_t>(c.p)
                     : static_cast<int64_t>(m);
}

uint64_t smallest_root(uint64_t p, uint64_t order) {  // params.hpp:30-43
  if (order == 1) return 1;
  for (uint64_t w = 2; w < p; ++w)
    if (pow_mod(w, order, p) == 1 && pow_mod(w, order / 2, p) != 1) return w;
  return 0;
}

void add_fault(std::string& s, const std::string& f) { s += "\n  - " + f; }

// ---- device images for the N=256 fast kernels (fast256.cu) ----

bool fast_eligible(const HostParams& P, int kind) {
  if (!(P.n_bits == 16 || P.n_bits == 32)) return false;
  if (P.N == 256) {
    if (P.layers < 5) return false;
  } else if (!((P.N == 512 || P.N == 1024) && P.layers == P.log2N)) {
    return false;  // fastn_tma.cu: full trees only
  }
  const uint64_t p = P.p;
  switch (kind) {
    case NTTK_IMPROVED:  // every intermediate < 2^layers p must fit a 32-bit register
      return (uint64_t(P.layers) + 1) * p < (uint64_t(1) << 32) &&
             (p << P.layers) < (uint64_t(1) << 32);
    case NTTK_HARVEY: return 4 * p < (uint64_t(1) << 32);
    case NTTK_SMONT:  // signed values fit int32; Barrett constant fits 32 bits
      return (uint64_t(P.layers) + 2) * p < (uint64_t(1) << 31) &&
             (u128(1) << (P.n_bits + 10)) / p < (u128(1) << 32);
    case NTTK_NTL: return 2 * p < P.ctx.beta;  // Shoup products are exact for t < 2^n
    case NTTK_SCOTT: {
      // n = 32 only (n = 16 is the reference's underflowing configuration, SURVEY §0 item
      // 6; it stays on the 64-bit generic kernel).  Bit-exact on 32-bit registers when
      // no T = X + off - Y underflows (off >= 2^{L-1} p, the largest Y) and none
      // overflows (2^L p + off < 2^32); then w T + q p < 2^64 and Y' < 2p.
      if (P.n_bits != 32 || !P.scott_L) return false;
      const uint64_t off = uint64_t(P.N / P.scott_L) * p;
      return off >= (p << (P.layers - 1)) && (p << P.layers) + off < (uint64_t(1) << 32);
    }
    default: return false;
  }
}

void fill_fast(HostParams& P, int kind) {
  const Ctx& c = P.ctx;
  const bool n16 = P.n_bits == 16;
  for (int dir = 0; dir < 2; ++dir) {
    FastArgs& A = P.fast[kind][dir];
    A.p = P.p;
    A.two_p = 2 * P.p;
    A.negp = static_cast<uint32_t>(0u - P.p);
    for (unsigned m = 1; m < 12; ++m) A.off[m] = static_cast<uint32_t>(uint64_t(P.p) << (m - 1));
    A.layers = P.layers;
    A.canon_m = static_cast<uint32_t>(0xffffffffull / P.p);
    A.canon_m16 = static_cast<uint32_t>(((uint64_t(1) << 32) + P.p - 1) / P.p);
    // K p >= 2^{bits-1} (bits = 16 or 32 storage): lifts two's complement to unsigned
    {
      const uint64_t half = n16 ? (uint64_t(1) << 15) : (uint64_t(1) << 31);
      A.sgn_off = static_cast<uint32_t>((half + P.p - 1) / P.p * P.p);
    }
    A.barrett_v = static_cast<uint32_t>(((u128(1) << (P.n_bits + 10)) + (P.p >> 1)) / P.p);
    const uint64_t p = P.p;
    // exact Barrett floor(x M / 2^S) = floor(x / p) for every x < 2^17:
    // (2^17 - 1)(M p - 2^S) < 2^S, with the 32-bit product x M not wrapping
    for (uint32_t S = 16; S < 32; ++S) {
      const uint64_t M = ((uint64_t(1) << S) + p - 1) / p, xmax = (uint64_t(1) << 17) - 1;
      if (xmax * M < (uint64_t(1) << 32) && xmax * (M * p - (uint64_t(1) << S)) < (uint64_t(1) << S)) {
        A.cb_m = static_cast<uint32_t>(M);
        A.cb_s = S;
        A.flags |= 1;
        break;
      }
    }
    // shift reduction of a 32-bit x: r = x - (x >> s) p < 2^{32-s} (2^s - p) + 2^s, one
    // conditional subtraction is enough when that bound is <= 2p
    {
      uint32_t s = 0;
      while ((uint64_t(1) << s) < p) ++s;
      if ((uint64_t(1) << (32 - s)) * ((uint64_t(1) << s) - p) + (uint64_t(1) << s) <= 2 * p) {
        A.cs_s = s;
        A.flags |= 2;
      }
    }
    // fused first merge layer for u16 input (improved, n = 16): Y' = MP(w, X + K p - Y)
    // with every T = X + K p - Y inside Prop. 4's exact range, X' = (X + Y) mod p
    if (kind == NTTK_IMPROVED && n16 && (A.flags & 1)) {
      const uint64_t K = ((uint64_t(1) << 16) - 1 + p - 1) / p, kp = K * p;
      const uint64_t tmax = (uint64_t(1) << 16) - 1 + kp;
      if (u128(p - 1) * tmax < u128(c.beta) * (c.beta - p)) {
        A.kp = static_cast<uint32_t>(kp);
        A.flags |= 4;
      }
    }
    // lazy merge outputs (ImprovedN16::sum_hh): the two Plantard products w T of a lazy
    // pair must sum below 2^32.  Merge depth m has T < 2^m p (T < 2^16 + kp at depth 1
    // when fused); lazily consumed products come from depths 1..L-1.
    if (kind == NTTK_IMPROVED && n16) {
      u128 tmax = u128(p) << (P.layers - 1);
      if (A.flags & 4) tmax = std::max<u128>(tmax, (uint64_t(1) << 16) - 1 + A.kp);
      if (2 * u128(p - 1) * tmax < (u128(1) << 32)) A.flags |= 8;
    }
    // n = 32: lo32(h' p) < 2p for every fast-path operand (ImprovedN32 lazy merge)
    if (kind == NTTK_IMPROVED && !n16 && u128(4) * p < (u128(1) << 32)) A.flags |= 8;
    // inverse TW1 (inv_body_lazy): block 0 of merge layers len = 16, 32, 64 has twiddle
    // 1 (index 2^L - 2^s of the merge table, s = 4, 3, 2).  Every value of merge depth d
    // stays below 2^d p, the bound the lazy / exact-bound checks already assume.
    // N = 512 / 1024 (fastn_tma.cu, full trees): the phase-2 layers are s = 5..2, the same
    // table positions 2^L - 2^s.
    // harvey / ntl (eager merge, N = 256): inv_w1 keeps their [0, 2p) / canonical invariants
    const bool tw1_kind = (kind == NTTK_IMPROVED && (A.flags & 8)) ||
                          ((kind == NTTK_HARVEY || kind == NTTK_NTL) && P.N == 256);
    if (tw1_kind && dir == 1 &&
        ((P.N == 256 && P.layers == 8) || ((P.N == 512 || P.N == 1024) && (1u << P.layers) == P.N))) {
      const unsigned smax = P.N == 256 ? 4 : 5;
      bool ones = P.gs_plain.size() >= (size_t(1) << P.layers) - 4;
      for (unsigned st = 2; ones && st <= smax; ++st)
        ones = P.gs_plain[(size_t(1) << P.layers) - (size_t(1) << st)] == 1;
      if (ones) A.flags |= 32;
    }
    // inverse partial canonicalisation (u32, lazy improved n = 32): inputs reduced to [0, 2p)
    // by the shift reduction without its conditional subtraction; every merge bound doubles,
    // so the last layer's X + Y < 2^{L+1} p must fit 32 bits (Prop. 4's range at n = 32 is
    // far larger)
    if (kind == NTTK_IMPROVED && !n16 && dir == 1 && P.N == 256 && (A.flags & 2) && (A.flags & 8) &&
        (u128(p) << (P.layers + 1)) < (u128(1) << 32) &&
        u128(p - 1) * (u128(p) << (P.layers + 1)) < u128(c.beta) * (c.beta - p))
      A.flags |= 128;
    // inverse DEFER (u16 input, no canonicalisation): sum-chain products h K p + h (2^16 - 1)
    // for h <= 8 inside Prop. 4's range, lazily consumed ones (h <= 4) pairwise below 2^32,
    // and v0 < 16 (2^16 - 1) reducible by MP(1^, v0)
    if (kind == NTTK_IMPROVED && n16 && dir == 1 && P.layers == 8 && P.N == 256 &&
        (A.flags & 4) && (A.flags & 8)) {
      const u128 t1 = (uint64_t(1) << 16) - 1 + A.kp, lim = u128(c.beta) * (c.beta - p);
      const u128 tl = std::max<u128>(u128(p) << (P.layers - 1), 4 * t1);
      if (u128(p - 1) * 8 * t1 < lim && 2 * u128(p - 1) * tl < (u128(1) << 32) &&
          u128(p - 1) * 16 * ((uint64_t(1) << 16) - 1) < lim) {
        for (int m = 0; m < 4; ++m) A.skp[m] = A.kp << m;
        A.one_lo = static_cast<uint32_t>(to_plantard(1, c) * c.mu);
        A.flags |= 64;
      }
    }
    // forward block 0 of layers 1..4 has twiddle 1 (cyclic tree): multiply-free
    // Plantard products (fwd_body W1)
    if (kind == NTTK_IMPROVED && dir == 0 && P.layers >= 4 && P.ct_plain.size() >= 8 &&
        P.ct_plain[0] == 1 && P.ct_plain[1] == 1 && P.ct_plain[3] == 1 && P.ct_plain[7] == 1 &&
        uint64_t(4) * P.p < (uint64_t(1) << 32))
      A.flags |= 16;
    // F1 forward (tma_common.cuh fwd_body_f1 at N = 256, fastn_tma.cu fwd_body_n_f1 at N =
    // 512 / 1024; improved n = 16, cyclic full trees whose layer 1 has twiddle 1): every word
    // carries up to S = L - 2 extra multiples of p, so the largest operand is (2 L - 1) p;
    // Prop. 4 must hold for it
    {
      const uint64_t L = P.layers, S = L - 2;
      const bool full = (P.N == 256 && L == 8) || ((P.N == 512 || P.N == 1024) && L == P.log2N);
      // ... and the 7-layer negacyclic tree at N = 256 (fwd_body_f1_nega7: layer 1 multiplies)
      const bool nega7 = P.N == 256 && L == 7 && P.tree == NTTK_NEGACYCLIC && !(A.flags & 16);
      if (kind == NTTK_IMPROVED && n16 && dir == 0 && ((full && (A.flags & 16)) || nega7) &&
          u128(p - 1) * ((2 * L - 1) * p) < u128(c.beta) * (c.beta - p)) {
        A.f1_sp = static_cast<uint32_t>(S * p);
        A.f1_sp1 = static_cast<uint32_t>((S + 1) * p);
        A.flags |= 1024;
      }
    }
    // last merge twiddle times N^{-1} (the final scaling folded into the last layer)
    {
      const uint64_t wl = static_cast<uint64_t>(u128(P.gs_plain.back()) * P.n_inv % p);
      if (kind == NTTK_IMPROVED) {
        const uint64_t fm = to_plantard(wl, c) * c.mu & c.r2n_mask;
        A.fold_lo = static_cast<uint32_t>(fm);
        A.fold_hi = static_cast<uint32_t>(fm >> 32);
      } else if (kind == NTTK_HARVEY || kind == NTTK_SCOTT) {
        A.fold_lo = static_cast<uint32_t>(to_mont(wl, c));
      } else if (kind == NTTK_NTL) {
        A.fold_lo = static_cast<uint32_t>(wl);
        A.fold_hi = static_cast<uint32_t>((u128(wl) << P.n_bits) / p);
      } else if (kind == NTTK_SMONT) {  // SmontLazy16::inv_last (fused polymul)
        const int64_t ws = to_smont(wl, c);
        const uint64_t fq = static_cast<uint64_t>(ws) * c.p_inv_beta & c.beta_mask;
        A.fold_lo = static_cast<uint32_t>(ws);
        A.fold_hi = n16 ? static_cast<uint32_t>(fq << 16) : static_cast<uint32_t>(fq);
      }
    }
    // full per-direction twiddle words (reference table order) in the kind's encoding
    std::vector<uint32_t> tl(P.N, 0), th(P.N, 0);
    const std::vector<uint64_t>* tab = nullptr;
    switch (kind) {
      case NTTK_IMPROVED: {
        tab = dir == 0 ? &P.ct_plantard : &P.gs_plantard;
        const uint64_t mu = c.mu;  // p^{-1} mod 2^{2n}
        for (size_t k = 0; k < tab->size(); ++k) {
          const uint64_t wm = (*tab)[k] * mu & c.r2n_mask;  // w_hat mu mod 2^{2n}
          tl[k] = static_cast<uint32_t>(wm);
          th[k] = static_cast<uint32_t>(wm >> 32);
        }
        const uint64_t sm = P.n_inv_hat * mu & c.r2n_mask;
        A.scale_lo = static_cast<uint32_t>(sm);
        A.scale_hi = static_cast<uint32_t>(sm >> 32);
        break;
      }
      case NTTK_HARVEY: {
        if (dir == 0) tab = P.tree == NTTK_CYCLIC ? &P.dif_mont : &P.ct_mont;
        else tab = &P.gs_mont;
        for (size_t k = 0; k < tab->size(); ++k) tl[k] = static_cast<uint32_t>((*tab)[k]);
        A.pinv = n16 ? static_cast<uint32_t>(c.p_inv_beta << 16)
                     : static_cast<uint32_t>(c.p_inv_beta);
        A.scale_lo = static_cast<uint32_t>(P.n_inv_mont);
        break;
      }
      case NTTK_SCOTT: {  // forward: DIF per-index Montgomery twiddles; inverse: GS per-block
        tab = dir == 0 ? &P.dif_mont : &P.gs_mont;
        for (size_t k = 0; k < tab->size(); ++k) tl[k] = static_cast<uint32_t>((*tab)[k]);
        A.pinv = static_cast<uint32_t>(c.neg_p_inv_beta);
        A.scale_lo = static_cast<uint32_t>(P.n_inv_mont);
        A.soff = static_cast<uint32_t>(uint64_t(P.N / P.scott_L) * P.p);
        break;
      }
      case NTTK_NTL: {  // (w, floor(w 2^n / p)) pairs: dif_w/dif_wq forward, gs_w/gs_wq inverse
        const std::vector<uint64_t>& w = dir == 0 ? P.dif_w : P.gs_plain;
        const std::vector<uint64_t>& wq = dir == 0 ? P.dif_wq : P.gs_wq;
        for (size_t k = 0; k < w.size(); ++k) {
          tl[k] = static_cast<uint32_t>(w[k]);
          th[k] = static_cast<uint32_t>(wq[k]);
        }
        A.scale_lo = static_cast<uint32_t>(P.n_inv);
        A.scale_hi = static_cast<uint32_t>((u128(P.n_inv) << P.n_bits) / p);
        break;
      }
      case NTTK_SMONT: {
        const std::vector<int64_t>& st = dir == 0 ? P.ct_smont : P.gs_smont;
        for (size_t k = 0; k < st.size(); ++k) {
          const int64_t w = st[k];
          tl[k] = static_cast<uint32_t>(w);
          // premultiplied Montgomery quotient factor w p^{-1} mod 2^n (n=16: in the
          // high half so a 32-bit multiply leaves the n-bit product there)
          const uint64_t wp = static_cast<uint64_t>(w) * c.p_inv_beta & c.beta_mask;
          th[k] = n16 ? static_cast<uint32_t>(wp << 16) : static_cast<uint32_t>(wp);
        }
        const int64_t f = P.n_inv_smont;
        A.scale_lo = static_cast<uint32_t>(f);
        const uint64_t fp = static_cast<uint64_t>(f) * c.p_inv_beta & c.beta_mask;
        A.scale_hi = n16 ? static_cast<uint32_t>(fp << 16) : static_cast<uint32_t>(fp);
        A.pinv = static_cast<uint32_t>(c.p_inv_beta);
        break;
      }
    }
    const size_t tsize = kind == NTTK_SMONT ? (dir == 0 ? P.ct_smont.size() : P.gs_smont.size())
                         : kind == NTTK_NTL  ? (dir == 0 ? P.dif_w.size() : P.gs_plain.size())
                                             : tab->size();
    if (P.N == 256) {
      for (size_t k = 0; k < tsize && k < 256; ++k) {
        A.lo[k] = tl[k];
        A.hi[k] = th[k];
      }
    } else {
      // N = 512 / 1024 (fastn_tma.cu): the uniform twiddles become constant-bank words
      // in a compact order, the lane-dependent ones are read from a device copy of the
      // whole table (fastn_tab, staged into shared memory)
      const unsigned L = P.layers;
      const bool per_index = dir == 0 && P.tree == NTTK_CYCLIC &&
                             (kind == NTTK_NTL || kind == NTTK_HARVEY || kind == NTTK_SCOTT);
      auto put = [&](size_t dst, size_t src) {
        A.lo[dst] = tl[src];
        A.hi[dst] = th[src];
      };
      if (dir == 0 && !per_index) {  // CT per-block, layers 1..5 (strided phase)
        for (size_t k = 0; k < 31; ++k) put(k, k);
      } else if (dir == 0) {  // DIF per-index, layers 6..L (contiguous phase)
        for (unsigned st = 6; st <= L; ++st) {
          const size_t cur = P.N - (P.N >> (st - 1)), cnt = P.N >> st;
          for (size_t e = 0; e < cnt; ++e) put(32 - 2 * cnt + e, cur + e);
        }
      } else {  // GS merge order, layers 5..1 (strided phase)
        for (unsigned st = 1; st <= 5; ++st)
          for (size_t b = 0; b < (size_t(1) << (st - 1)); ++b)
            put(32 - (size_t(1) << st) + b, (size_t(1) << L) - (size_t(1) << st) + b);
      }
      std::vector<uint32_t>& F = P.fastn_tab[kind][dir];
      F.assign(2 * tsize, 0);
      for (size_t k = 0; k < tsize; ++k) {
        F[2 * k] = tl[k];
        F[2 * k + 1] = th[k];
      }
    }
  }
  // product stage of the fused polymul (ProdArgs): per-kind multiplier encodings
  ProdArgs& Q = P.prod[kind];
  const uint64_t p = P.p;
  Q.basemul = (P.N >> P.layers) == 2 ? 1u : 0u;
  const uint64_t r2 = static_cast<uint64_t>(u128(c.beta % p) * (c.beta % p) % p);  // 2^{2n} mod p
  auto smont_pair = [&](uint64_t w, uint32_t& lo, uint32_t& hi) {
    const int64_t ws = to_smont(w, c);  // centered w 2^n mod p
    const uint64_t q = static_cast<uint64_t>(ws) * c.p_inv_beta & c.beta_mask;
    lo = static_cast<uint32_t>(ws);
    hi = n16 ? static_cast<uint32_t>(q << 16) : static_cast<uint32_t>(q);
  };
  switch (kind) {
    case NTTK_IMPROVED: {
      const uint64_t c4 = static_cast<uint64_t>(u128(r2) * r2 % p);  // 2^{4n} mod p
      const uint64_t em = c4 * c.mu & c.r2n_mask;
      Q.enc_lo = static_cast<uint32_t>(em);
      Q.enc_hi = static_cast<uint32_t>(em >> 32);
      Q.mu_lo = static_cast<uint32_t>(c.mu);
      Q.mu_hi = static_cast<uint32_t>(c.mu >> 32);
      for (size_t k = 0; k < P.gamma.size() && k < 128; ++k) {
        const uint64_t gm = to_plantard(P.gamma[k], c) * c.mu & c.r2n_mask;
        Q.g_lo[k] = static_cast<uint32_t>(gm);
        Q.g_hi[k] = static_cast<uint32_t>(gm >> 32);
      }
      break;
    }
    case NTTK_HARVEY:
      Q.enc_lo = static_cast<uint32_t>(r2);  // harvey_mul(x, R^2) = x R mod p, lazy
      for (size_t k = 0; k < P.gamma.size() && k < 128; ++k)
        Q.g_lo[k] = static_cast<uint32_t>(to_mont(P.gamma[k], c));
      break;
    case NTTK_SMONT: {
      // multiplier R^2 in signed-Montgomery form: smont(x * R^2-encoding) = x R mod p
      smont_pair(static_cast<uint64_t>(u128(r2) * inverse(c.beta % p, p) % p), Q.enc_lo, Q.enc_hi);
      for (size_t k = 0; k < P.gamma.size() && k < 128; ++k)
        smont_pair(P.gamma[k], Q.g_lo[k], Q.g_hi[k]);
      break;
    }
  }
  // lazy twins of the Montgomery kinds for the fused polymul (arith.cuh HarveyLazy16 /
  // SmontLazy16): n = 16, CT forward (negacyclic tree), bounds stated there
  {
    const uint64_t L = P.layers, pL = p << L;
    FastArgs& AI = P.fast[kind][1];
    const bool cb = (AI.flags & 1) && (P.fast[kind][0].flags & 1);
    if (n16 && cb && P.tree == NTTK_NEGACYCLIC && kind == NTTK_HARVEY) {
      if ((1 + 2 * L) * p < (uint64_t(1) << 16) && u128(p - 1) * pL < (u128(1) << 32) &&
          ((u128(p - 1) * pL) >> 16) + 2 * p < (u128(1) << 17))
        Q.lazy = 1;
    }
    if (n16 && cb && kind == NTTK_SMONT) {
      const u128 half = p / 2 + 1;
      const uint64_t rmax = static_cast<uint64_t>((half * pL >> 16) + p / 2 + 1);  // final |r|
      const uint64_t lzk = (rmax / p + 1) * p;
      if ((L + 1) * p < (uint64_t(1) << 15) && half * pL + (u128(p) << 15) < (u128(1) << 31) &&
          2 * lzk < (uint64_t(1) << 17)) {
        AI.lzk = static_cast<uint32_t>(lzk);
        Q.lazy = 1;
      }
    }
    // improved: the free F1 forwards (tma_common.cuh fwd_body_f1_free) carry up to (L - 1) p
    // of surplus; every product operand stays below (2 L) p, inside Prop. 4's n = 16 range
    if (n16 && kind == NTTK_IMPROVED && (L == 7 || L == 8) &&
        u128(p - 1) * (2 * L * p) < u128(c.beta) * (c.beta - p))
      Q.lazy = 1;
    if (Q.lazy) AI.flags |= 256;  // introspection only (nttk_params_fast_flags)
  }
  P.fast_mask |= 1u << kind;
}

// Narrow image of an n = 32 improved parameter set (HostParams::narrow).  The improved
// butterflies' words do not depend on n: X' = X + r, Y' = X + p - r with r = w t mod p
// canonical, and the n = 16 modified Plantard product is exact for
// W T < 2^16 (2^16 - p) (Prop. 4).  The forward's operands are its lazy
// words, below (L + 1) p; so for small p (the paper's Table 2 presets: 7681, 12289) the
// whole forward runs on the cheaper n = 16 product, bit-exact with the reference's n = 32
// run.  The image is fill_fast's own output for the same tree at n = 16.
// CT-form inverse for the Kyber tree (improved n = 16, N = 256, cyclic L = 8, u16 input).  The
// inverse output is canonical, hence unique, so any exact algorithm gives the reference's bits
// (intt_inverse, transform.hpp:233-343).  inv_body_ct runs a radix-2 DIT on the bit-reversed
// spectrum with omega^{-1}: a[i+j] = u + w v, a[i+j+len] = u - w v, w = omega^{-(N/2len) j}.
// Those are CT butterflies, so the balanced F3 form applies (tma_common.cuh f1_bf), and the
// j = 0 butterfly of every block in the register-local layers len = 1..8 is multiply-free.
// Raw u16 words enter unreduced.  The host tracks the value interval of every register through
// the kernel's exact schedule and picks, per layer, the multiples of p that the multiply-free
// butterflies add to keep every F3 X input >= p (so X - r never underflows); the last layer
// folds N^{-1} into two Plantard products per butterfly.  Every product operand must stay
// inside Prop. 4's range, else the image is refused (the GS inverse stays).
// n = 32 (Dilithium, u32): the same DIT schedule with the umulhi-form Plantard products of
// ImprovedN32 (X' = X + r, Y' = X + p - r: never negative), inputs partially reduced to [0, 2p)
// on load (shift reduction, A.flags bit 1); the multiply-free butterflies add the multiple of p
// that covers their Y input.  Every word stays below 2^32 (host-checked); Prop. 4's n = 32 range
// holds for any 32-bit operand.
void fill_ct_inverse32(HostParams& P) {
  const Ctx& c = P.ctx;
  const uint64_t p = P.p;
  const FastArgs& G = P.fast[NTTK_IMPROVED][1];
  if (!(G.flags & 2) || (uint64_t(1) << G.cs_s) < p) return;  // the shift reduction of the load
  auto rup = [&](uint64_t x) { return (x + p - 1) / p * p; };
  uint64_t hi[16];
  for (int r = 0; r < 16; ++r) hi[r] = 2 * p - 1;  // after v + (v >> s) (-p): below 2p
  uint32_t consts[8] = {};
  for (int li = 0; li < 4; ++li) {
    const int len = 1 << li;
    uint64_t c2 = 0;
    for (int r = 0; r < 16; ++r)
      if (!(r & len) && (r & (len - 1)) == 0) c2 = std::max(c2, rup(hi[r + len]));
    consts[2 * li + 1] = static_cast<uint32_t>(c2);
    uint64_t nhi[16];
    std::copy(hi, hi + 16, nhi);
    for (int r = 0; r < 16; ++r) {
      if (r & len) continue;
      if ((r & (len - 1)) == 0) {
        nhi[r] = hi[r] + hi[r + len];
        nhi[r + len] = hi[r] + c2;
      } else {
        nhi[r] = hi[r] + p - 1;
        nhi[r + len] = hi[r] + p;
      }
    }
    std::copy(nhi, nhi + 16, hi);
  }
  uint64_t H = 0;
  for (int r = 0; r < 16; ++r) H = std::max(H, hi[r]);
  H += 3 * p;  // strided layers len 16, 32, 64: X' < X + p, Y' <= X + p
  if (H >= (uint64_t(1) << 32) || 2 * p >= (uint64_t(1) << 31)) return;
  FastArgs A = G;
  A.flags = (A.flags & 3u) | 2048u;
  std::copy(consts, consts + 8, A.ct_c);
  const uint64_t oi = static_cast<uint64_t>(inverse(P.omega, p));
  uint64_t w = 1;
  for (int e = 0; e < 128; ++e) {
    const uint64_t a = to_plantard(w, c) * c.mu & c.r2n_mask;
    const uint64_t b = to_plantard(static_cast<uint64_t>(u128(w) * P.n_inv % p), c) * c.mu & c.r2n_mask;
    A.lo[e] = static_cast<uint32_t>(a), A.hi[e] = static_cast<uint32_t>(a >> 32);
    A.lo[128 + e] = static_cast<uint32_t>(b), A.hi[128 + e] = static_cast<uint32_t>(b >> 32);
    w = static_cast<uint64_t>(u128(w) * oi % p);
  }
  const uint64_t sm = to_plantard(P.n_inv, c) * c.mu & c.r2n_mask;
  A.scale_lo = static_cast<uint32_t>(sm), A.scale_hi = static_cast<uint32_t>(sm >> 32);
  P.fast_ctinv = A;
  P.ct_inv = true;
}

// n = 16 image for input words in [0, in_hi] (65535: raw u16 words; p - 1: canonicalised words)
bool ct_image16(const HostParams& P, const Ctx& c, int64_t in_hi, const FastArgs& base, FastArgs& out) {
  const uint64_t p = P.p;
  const u128 lim = u128(c.beta) * (c.beta - p);
  // offsets are multiples of p, rounded up; the canonical-input image may also subtract (its
  // sums would otherwise outgrow Prop. 4's range for p = 7681), the raw-u16 image never needs to
  const bool neg = in_hi != 65535;
  auto rup = [&](int64_t x) -> int64_t {
    if (x <= 0) return neg ? -((-x) / int64_t(p)) * int64_t(p) : 0;
    return (x + int64_t(p) - 1) / int64_t(p) * int64_t(p);
  };
  auto prod_ok = [&](int64_t v) { return v >= 0 && u128(p - 1) * uint64_t(v) < lim; };
  int64_t lo[16], hi[16];
  for (int r = 0; r < 16; ++r) lo[r] = 0, hi[r] = in_hi;
  const int64_t P_ = int64_t(p);
  uint32_t consts[8];
  const int64_t floor_of[4] = {6 * P_, 5 * P_, 4 * P_, 3 * P_};  // remaining F3 layers + 3p
  for (int li = 0; li < 4; ++li) {  // register-local layers len = 1, 2, 4, 8
    const int len = 1 << li;
    int64_t c1 = neg ? INT64_MIN : 0, c2 = neg ? INT64_MIN : 0;
    for (int r = 0; r < 16; ++r)
      if (!(r & len) && (r & (len - 1)) == 0) {
        c1 = std::max(c1, rup(floor_of[li] - lo[r] - lo[r + len]));
        c2 = std::max(c2, rup(floor_of[li] - lo[r] + hi[r + len]));
      }
    consts[2 * li] = static_cast<uint32_t>(c1);
    consts[2 * li + 1] = static_cast<uint32_t>(c2);
    int64_t nlo[16], nhi[16];
    std::copy(lo, lo + 16, nlo);
    std::copy(hi, hi + 16, nhi);
    for (int r = 0; r < 16; ++r) {
      if (r & len) continue;
      const int u = r, v = r + len;
      if ((r & (len - 1)) == 0) {
        nlo[u] = lo[u] + lo[v] + c1, nhi[u] = hi[u] + hi[v] + c1;
        nlo[v] = lo[u] - hi[v] + c2, nhi[v] = hi[u] - lo[v] + c2;
      } else {
        if (lo[u] < P_ || !prod_ok(hi[v])) return false;
        nlo[u] = lo[u], nhi[u] = hi[u] + P_ - 1;
        nlo[v] = lo[u] - P_ + 1, nhi[v] = hi[u];
      }
    }
    std::copy(nlo, nlo + 16, lo);
    std::copy(nhi, nhi + 16, hi);
  }
  int64_t L0 = lo[0], H0 = hi[0];  // after the transpose a register may hold any position
  for (int r = 1; r < 16; ++r) L0 = std::min(L0, lo[r]), H0 = std::max(H0, hi[r]);
  if (L0 < 0 || H0 >= (int64_t(1) << 32)) return false;
  for (int r = 0; r < 16; ++r) lo[r] = L0, hi[r] = H0;
  for (int h = 1; h <= 4; h *= 2) {  // strided layers len = 16, 32, 64 (all F3)
    int64_t nlo[16], nhi[16];
    std::copy(lo, lo + 16, nlo);
    std::copy(hi, hi + 16, nhi);
    for (int r = 0; r < 16; ++r) {
      if (r & h) continue;
      if (lo[r] < P_ || !prod_ok(hi[r + h])) return false;
      nlo[r] = lo[r], nhi[r] = hi[r] + P_ - 1;
      nlo[r + h] = lo[r] - P_ + 1, nhi[r + h] = hi[r];
    }
    std::copy(nlo, nlo + 16, lo);
    std::copy(nhi, nhi + 16, hi);
  }
  for (int r = 0; r < 16; ++r)  // last layer: both operands are Plantard products
    if (!prod_ok(hi[r])) return false;
  FastArgs A = base;
  A.flags = (A.flags & 3u) | 2048u;
  std::copy(consts, consts + 8, A.ct_c);
  const uint64_t oi = static_cast<uint64_t>(inverse(P.omega, p));
  uint64_t w = 1;
  for (int e = 0; e < 128; ++e) {  // lo[e] = (omega^{-e})^ mu, lo[128 + e] = (N^{-1} omega^{-e})^ mu
    A.lo[e] = static_cast<uint32_t>(to_plantard(w, c) * c.mu & c.r2n_mask);
    A.lo[128 + e] = static_cast<uint32_t>(
        to_plantard(static_cast<uint64_t>(u128(w) * P.n_inv % p), c) * c.mu & c.r2n_mask);
    w = static_cast<uint64_t>(u128(w) * oi % p);
  }
  A.scale_lo = static_cast<uint32_t>(to_plantard(P.n_inv, c) * c.mu & c.r2n_mask);
  out = A;
  return true;
}

void fill_ct_inverse(HostParams& P) {
  if (P.N != 256 || P.layers != 8 || P.tree != NTTK_CYCLIC) return;
  if (!((P.fast_mask >> NTTK_IMPROVED) & 1u)) return;
  if (P.n_bits == 32) {
    fill_ct_inverse32(P);
    // the narrow image (kyber256 preset): canonicalised u32 words through the n = 16 body
    if (P.narrow[1])
      P.ct_inv_c = ct_image16(P, make_ctx(P.p, 16, P.log2N), int64_t(P.p) - 1, P.fast[kNarrow][1], P.fast_ctinv_c);
    return;
  }
  if (P.n_bits != 16) return;
  P.ct_inv = ct_image16(P, P.ctx, 65535, P.fast[NTTK_IMPROVED][1], P.fast_ctinv);
  P.ct_inv_c = ct_image16(P, P.ctx, int64_t(P.p) - 1, P.fast[NTTK_IMPROVED][1], P.fast_ctinv_c);
}

// CT-form inverse of the narrow image at N = 512 / 1024 (fastn_tma.cu inv_body_n_ct; the N = 256
// derivation above applies).  Lane j owns positions 32 j + k in the contiguous phase (len = 1..16,
// uniform twiddles omega^{-(N/32) e} in A.lo[e], e < 16, the jb = 0 butterflies multiply-free) and
// j + G k in the strided phase (len = G h; lane twiddles from the shared-memory table, segment
// (h - 1) G holds omega^{-(16/h)(j + G kk)} at kk G + j; the h = 16 segment carries N^{-1}).
// The kernel's schedule is fixed at compile time in units of p: canonical inputs, offsets
// A.pm[m] = m p, four canon1 reductions, every product operand below kCtLimN p -- so the image
// is valid exactly when kCtLimN p lies inside Prop. 4's n = 16 range.  The schedule itself is
// proven on the CPU against the reference inverse (tests/test_oracle.py).
void fill_ct_inverse_n(HostParams& P, const Ctx& c16) {
  const uint64_t p = P.p, N = P.N, G = N / 32;
  const u128 lim = u128(c16.beta) * (c16.beta - p);
  if (!(u128(p - 1) * (uint64_t(kCtLimN) * p - 1) < lim)) return;
  FastArgs A = P.fast[kNarrow][1];
  A.flags = (A.flags & 3u) | 2048u;
  for (uint32_t m = 0; m < 12; ++m) A.pm[m] = m * static_cast<uint32_t>(p);
  auto enc = [&](uint64_t w) { return static_cast<uint32_t>(to_plantard(w, c16) * c16.mu & c16.r2n_mask); };
  const uint64_t oi = static_cast<uint64_t>(inverse(P.omega, p));
  std::vector<uint64_t> pw(N / 2);  // omega^{-e}
  pw[0] = 1;
  for (size_t e = 1; e < pw.size(); ++e) pw[e] = static_cast<uint64_t>(u128(pw[e - 1]) * oi % p);
  for (int e = 0; e < 16; ++e) A.lo[e] = enc(pw[(N / 32) * e]);
  std::vector<uint32_t> tab(2 * N, 0);
  for (uint64_t h = 1; h <= 16; h *= 2)
    for (uint64_t kk = 0; kk < h; ++kk)
      for (uint64_t j = 0; j < G; ++j) {
        uint64_t w = pw[(16 / h) * (j + G * kk)];
        if (h == 16) w = static_cast<uint64_t>(u128(w) * P.n_inv % p);
        tab[(h - 1) * G + kk * G + j] = enc(w);
      }
  A.scale_lo = enc(P.n_inv);
  P.fast[kCtN][1] = A;
  P.fastn_tab[kCtN][1] = tab;
  P.ct_inv_n = true;
}

void fill_narrow(HostParams& P) {
  if (P.n_bits != 32 || P.p >= (1u << 15)) return;
  const uint64_t p = P.p;
  const Ctx c16 = make_ctx(p, 16, P.log2N);
  const u128 lim = u128(c16.beta) * (c16.beta - p);  // Prop. 4: W T < 2^16 (2^16 - p)
  if (!(u128(p - 1) * ((P.layers + 1) * p) < lim)) return;
  HostParams T;
  T.desc = P.desc;
  T.desc.n_bits = 16;
  T.p = P.p;
  T.N = P.N;
  T.log2N = P.log2N;
  T.n_bits = 16;
  T.tree = P.tree;
  T.layers = P.layers;
  T.kinds = 1u << NTTK_IMPROVED;
  T.ctx = c16;
  T.omega = P.omega;
  T.omega_inv = P.omega_inv;
  T.n_inv = P.n_inv;
  T.ct_plain = P.ct_plain;
  T.gs_plain = P.gs_plain;
  T.gamma = P.gamma;
  for (uint64_t w : T.ct_plain) T.ct_plantard.push_back(to_plantard(w, c16));
  for (uint64_t w : T.gs_plain) T.gs_plantard.push_back(to_plantard(w, c16));
  T.n_inv_hat = to_plantard(T.n_inv, c16);
  if (!fast_eligible(T, NTTK_IMPROVED)) return;
  fill_fast(T, NTTK_IMPROVED);
  P.fast[kNarrow][0] = T.fast[NTTK_IMPROVED][0];
  P.fastn_tab[kNarrow][0] = T.fastn_tab[NTTK_IMPROVED][0];
  P.narrow[0] = true;
  // inverse (tma_common.cuh inv_body_narrow): every GS operand below 2^kNarrowEmax p, kept
  // there by MP(1^, .) reductions; only the full trees of the fast kernels carry the body
  const bool full = (P.N == 256 && P.layers == 8) || ((P.N == 512 || P.N == 1024) && P.layers == P.log2N);
  if (full && u128(p - 1) * (p << kNarrowEmax) < lim) {
    FastArgs I = T.fast[NTTK_IMPROVED][1];
    I.flags = (I.flags & 3u) | 512u;  // canonicalisation bits only: no lazy / TW1 / DEFER
    I.one_lo = static_cast<uint32_t>(to_plantard(1, c16) * c16.mu);
    P.fast[kNarrow][1] = I;
    P.fastn_tab[kNarrow][1] = T.fastn_tab[NTTK_IMPROVED][1];
    P.narrow[1] = true;
    if ((P.N == 512 || P.N == 1024) && P.tree == NTTK_CYCLIC) fill_ct_inverse_n(P, c16);
  }
}

}  // namespace

bool ct_inverse_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("NTTK_INV_CT");
    return !(e && e[0] == '0');
  }();
  return v;
}

HostParams::~HostParams() {
  for (auto& d : dev)
    if (d.base) cudaFree(d.base);
  for (auto* d : fastn_dev)
    if (d) cudaFree(d);
}

// one allocation per device holding every (kind, dir) table, [kind][dir] at a fixed
// stride of 2N words
const uint32_t* HostParams::fastn_table(int device, int kind, int dir, std::string& err) const {
  if (device < 0 || device >= 64) {
    err = "device ordinal out of range";
    return nullptr;
  }
  std::lock_guard<std::mutex> lock(mu_dev);
  if (!fastn_dev[device]) {
    const size_t stride = 2 * size_t(N);
    std::vector<uint32_t> host(14 * stride, 0);
    for (int k = 0; k < 7; ++k)
      for (int d = 0; d < 2; ++d)
        std::copy(fastn_tab[k][d].begin(), fastn_tab[k][d].end(), host.begin() + (2 * k + d) * stride);
    uint32_t* buf = nullptr;
    cudaError_t e = cudaMalloc(&buf, host.size() * 4);
    if (e == cudaSuccess) e = cudaMemcpy(buf, host.data(), host.size() * 4, cudaMemcpyHostToDevice);
    // a pageable cudaMemcpy may return before the DMA lands, and the kernels that read the
    // table run on non-blocking streams: wait for the legacy stream that carries the copy
    if (e == cudaSuccess) e = cudaStreamSynchronize(cudaStreamLegacy);
    if (e != cudaSuccess) {
      if (buf) cudaFree(buf);
      err = std::string("fastn table upload: ") + cudaGetErrorString(e);
      return nullptr;
    }
    fastn_dev[device] = buf;
  }
  return fastn_dev[device] + (2 * kind + dir) * 2 * size_t(N);
}

const DeviceTables* HostParams::device_tables(int device, std::string& err) const {
  if (device < 0 || device >= 64) {
    err = "device ordinal out of range";
    return nullptr;
  }
  std::lock_guard<std::mutex> lock(mu_dev);
  DeviceTables& D = dev[device];
  if (D.base) return &D;
  const std::vector<const std::vector<uint64_t>*> tabs = {
      &dif_w, &dif_wq, &dif_mont, &ct_plantard, &ct_mont, &gs_plain, &gs_wq, &gs_mont,
      &gs_plantard};
  size_t total = 0;
  for (auto* t : tabs) total += t->size();
  total += ct_smont.size() + gs_smont.size() + gamma.size();
  std::vector<uint64_t> host;
  host.reserve(total);
  std::vector<size_t> off;
  for (auto* t : tabs) {
    off.push_back(host.size());
    host.insert(host.end(), t->begin(), t->end());
  }
  off.push_back(host.size());
  for (int64_t v : ct_smont) host.push_back(static_cast<uint64_t>(v));
  off.push_back(host.size());
  for (int64_t v : gs_smont) host.push_back(static_cast<uint64_t>(v));
  off.push_back(host.size());
  host.insert(host.end(), gamma.begin(), gamma.end());
  uint64_t* base = nullptr;
  cudaError_t e = cudaMalloc(&base, std::max<size_t>(host.size(), 1) * 8);
  if (e == cudaSuccess) e = cudaMemcpy(base, host.data(), host.size() * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cudaStreamLegacy);  // see fastn_table
  if (e != cudaSuccess) {
    err = std::string("device table upload: ") + cudaGetErrorString(e);
    if (base) cudaFree(base);
    return nullptr;
  }
  D.base = base;
  D.dif_w = base + off[0];
  D.dif_wq = base + off[1];
  D.dif_mont = base + off[2];
  D.ct_plantard = base + off[3];
  D.ct_mont = base + off[4];
  D.gs_w = base + off[5];
  D.gs_wq = base + off[6];
  D.gs_mont = base + off[7];
  D.gs_plantard = base + off[8];
  D.ct_smont = base + off[9];
  D.gs_smont = base + off[10];
  D.gamma = base + off[11];
  return &D;
}

int build_params(const nttk_params_desc& d, HostParams& P, std::string& err) {
  std::string faults = "build_params:";
  const size_t clean = faults.size();
  const uint64_t p = d.p;
  const uint32_t N = d.N, n = d.n_bits, kinds = d.kinds_mask;
  // structural faults (params.hpp:145-169)
  if (n < 2 || n > 32) add_fault(faults, "word size n must be in [2, 32]");
  if (p < 3 || !(p & 1)) add_fault(faults, "p must be odd and >= 3");
  else if (!prime(p)) add_fault(faults, "p must be prime");
  if (N < 2 || !pow2(N) || N > (1u << 20)) add_fault(faults, "N must be a power of two in [2, 2^20]");
  if (!kinds) add_fault(faults, "at least one butterfly kind must be requested");
  if (kinds & ~0x1fu) add_fault(faults, "unknown butterfly kind");
  if (d.tree > NTTK_NEGACYCLIC) add_fault(faults, "unknown transform tree");
  unsigned ell = 0, layers = 0;
  if (faults.size() == clean) {
    ell = log2_floor(N);
    layers = d.layers ? d.layers : ell;
    if (layers > ell || (d.tree == NTTK_CYCLIC && layers != ell))
      add_fault(faults, "layers must be log2(N) (cyclic) or <= log2(N) (negacyclic)");
    const uint64_t order = d.tree == NTTK_CYCLIC ? N : (uint64_t(2) << layers);
    if ((p - 1) % order != 0)
      add_fault(faults, "N must divide p - 1 (p=" + std::to_string(p) +
                            ", N=" + std::to_string(order) + ")");
    if (ell >= n) add_fault(faults, "word size n must exceed log2(N)");
    if (p >= (uint64_t(1) << n)) add_fault(faults, "p must be < 2^n");
  }
  if (faults.size() != clean) {
    err = faults;
    return NTTK_CONTRACT;
  }
  P.desc = d;
  P.p = static_cast<uint32_t>(p);
  P.N = N;
  P.log2N = ell;
  P.n_bits = n;
  P.tree = d.tree;
  P.layers = layers;
  P.kinds = kinds;
  P.ctx = make_ctx(p, n, ell);
  const Ctx& c = P.ctx;
  const uint64_t order = d.tree == NTTK_CYCLIC ? N : (uint64_t(2) << layers);
  if (d.root) {
    if (pow_mod(d.root, order, p) != 1 || pow_mod(d.root, order / 2, p) == 1) {
      err = "build_params:\n  - root does not have the required order";
      return NTTK_CONTRACT;
    }
    P.omega = d.root;
  } else {
    P.omega = smallest_root(p, order);
  }
  P.omega_inv = static_cast<uint64_t>(inverse(P.omega, p));
  P.n_inv = static_cast<uint64_t>(
      inverse((d.tree == NTTK_CYCLIC ? N : (uint64_t(1) << layers)) % p, p));

  // per-kind word-size faults (params.hpp:183-217)
  auto has = [&](int k) { return (kinds >> k) & 1u; };
  if (has(NTTK_NTL) && 2 * p >= c.beta)
    add_fault(faults, "ntl: p=" + std::to_string(p) + " violates 2p < 2^n (n=" +
                          std::to_string(n) + ")");
  if (has(NTTK_HARVEY) && 4 * p >= c.beta)
    add_fault(faults, "harvey: p=" + std::to_string(p) + " violates 4p < 2^n (n=" +
                          std::to_string(n) + ")");
  if (has(NTTK_SCOTT) && u128(4) * p >= c.beta)
    add_fault(faults, "scott: p=" + std::to_string(p) +
                          " violates 4*N*p < 2^n * L for every L <= N");
  if (has(NTTK_IMPROVED)) {
    bool ok;
    if (d.flags & NTTK_EXACT_BOUND) {
      // Prop. 4 exact requirement W T < 2^n (2^n - p), W <= p-1,
      // T <= 2^layers p - 1 (largest lazy operand: inverse merge and final scaling)
      const uint64_t T = (p << layers) - 1;
      ok = u128(p - 1) * T < u128(c.beta) * (c.beta - p);
    } else {
      ok = ell + 2 < n && u128(p) < (u128(1) << (n - ell - 2));  // reduction.hpp:72-74
    }
    if (!ok)
      add_fault(faults, "improved: p=" + std::to_string(p) + " violates p < 2^{n-ell-2} = " +
                            std::to_string(n >= ell + 2 ? (uint64_t(1) << (n - ell - 2)) : 0) +
                            " (n=" + std::to_string(n) + ", ell=" + std::to_string(ell) + ")");
  }
  if (has(NTTK_SMONT) && (2 * p >= c.beta || u128(layers + 1) * (p - 1) >= c.beta))
    add_fault(faults, "smont: p=" + std::to_string(p) + " violates (layers+1)(p-1) < 2^n (n=" +
                          std::to_string(n) + ")");
  if (d.tree == NTTK_NEGACYCLIC && (has(NTTK_NTL) || has(NTTK_SCOTT)))
    add_fault(faults, "ntl/scott are DIF kinds: cyclic tree only");
  if (faults.size() != clean) {
    err = faults;
    return NTTK_CONTRACT;
  }
  if (has(NTTK_SCOTT)) {  // butterfly.hpp:157-168
    for (uint64_t L = 1; L <= N; L *= 2)
      if (u128(4) * N * p < u128(c.beta) * L) {
        P.scott_L = static_cast<uint32_t>(L);
        break;
      }
  }

  // plain schedules and their encodings
  const size_t T = (size_t(1) << layers) - 1;
  if (d.tree == NTTK_CYCLIC && (has(NTTK_NTL) || has(NTTK_HARVEY) || has(NTTK_SCOTT))) {
    for (uint64_t len = N / 2; len >= 1; len /= 2) {  // params.hpp:47-58
      const uint64_t step = N / (2 * len);
      for (uint64_t j = 0; j < len; ++j) {
        const uint64_t w = pow_mod(P.omega, j * step, p);
        P.dif_w.push_back(w);
        P.dif_wq.push_back(static_cast<uint64_t>((u128(w) << n) / p));
        P.dif_mont.push_back(to_mont(w, c));
      }
    }
  }
  for (unsigned s = 1; s <= layers; ++s) {  // forward CT, one twiddle per block
    for (uint64_t b = 0; b < (uint64_t(1) << (s - 1)); ++b) {
      uint64_t w;
      if (d.tree == NTTK_CYCLIC)  // params.hpp:60-72
        w = pow_mod(P.omega, (uint64_t(N) >> s) * bit_reverse(b, s - 1), p);
      else  // zeta^{br_L(2^{s-1} + b)}
        w = pow_mod(P.omega, bit_reverse((uint64_t(1) << (s - 1)) + b, layers), p);
      P.ct_plain.push_back(w);
      P.ct_plantard.push_back(to_plantard(w, c));
      P.ct_mont.push_back(to_mont(w, c));
      P.ct_smont.push_back(to_smont(w, c));
    }
  }
  for (unsigned s = layers; s >= 1; --s) {  // inverse GS in merge order (params.hpp:74-88)
    for (uint64_t b = 0; b < (uint64_t(1) << (s - 1)); ++b) {
      uint64_t e, ord;
      if (d.tree == NTTK_CYCLIC) {
        ord = N;
        e = (uint64_t(N) >> s) * bit_reverse(b, s - 1) % N;
      } else {
        ord = uint64_t(2) << layers;
        e = bit_reverse((uint64_t(1) << (s - 1)) + b, layers) % ord;
      }
      const uint64_t w = pow_mod(P.omega, e == 0 ? 0 : ord - e, p);
      P.gs_plain.push_back(w);
      P.gs_wq.push_back(static_cast<uint64_t>((u128(w) << n) / p));
      P.gs_mont.push_back(to_mont(w, c));
      P.gs_plantard.push_back(to_plantard(w, c));
      P.gs_smont.push_back(to_smont(w, c));
    }
  }
  (void)T;
  if ((N >> layers) == 2) {  // degree-2 leaves: x^2 -/+ z_b for last-layer block b
    const size_t last = (size_t(1) << (layers - 1)) - 1;
    for (uint32_t k = 0; k < N / 2; ++k) {
      const uint64_t z = P.ct_plain[last + k / 2];
      P.gamma.push_back((k & 1) ? (p - z) % p : z);
    }
  }
  if (has(NTTK_IMPROVED)) P.n_inv_hat = to_plantard(P.n_inv, c);  // params.hpp:250
  P.n_inv_mont = to_mont(P.n_inv, c);
  P.n_inv_smont = to_smont(P.n_inv, c);

  for (int k : {NTTK_NTL, NTTK_HARVEY, NTTK_SCOTT, NTTK_IMPROVED, NTTK_SMONT})
    if (has(k) && fast_eligible(P, k)) fill_fast(P, k);
  if ((P.fast_mask >> NTTK_IMPROVED) & 1u) {
    fill_narrow(P);
    fill_ct_inverse(P);
  }
  return NTTK_OK;
}

// params.hpp:273-306
int preset_desc(const std::string& name, nttk_params_desc& d, std::string& err) {
  struct Spec {
    const char* name;
    uint32_t p, N, n;
  };
  static const Spec table[] = {
      {"kyber256", 7681, 256, 32},     {"kcl256", 7681, 256, 32},
      {"newhope512", 12289, 512, 32},  {"falcon512", 12289, 512, 32},
      {"remblem512", 12289, 512, 32},  {"newhope1024", 12289, 1024, 32},
      {"falcon1024", 12289, 1024, 32}, {"hila5-1024", 12289, 1024, 32},
      {"toy13", 13, 4, 8},
  };
  for (const auto& s : table)
    if (name == s.name) {
      std::memset(&d, 0, sizeof d);
      d.p = s.p;
      d.N = s.N;
      d.n_bits = s.n;
      d.kinds_mask = 0xf;  // all_butterfly_kinds()
      return NTTK_OK;
    }
  std::string known;
  for (const auto& s : table) known += known.empty() ? s.name : std::string(", ") + s.name;
  err = "unknown preset '" + name + "' (known: " + known + ")";
  return NTTK_CONTRACT;
}

}  // namespace nttk_b200
