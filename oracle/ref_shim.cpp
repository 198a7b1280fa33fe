// ref_shim.cpp -- C-ABI shim over the UNMODIFIED reference headers (TEST INFRASTRUCTURE ONLY).
//
// Built by oracle/Makefile (target `ref`) straight from /root/reference/proj/include
// into oracle/_ref/libnttk_ref.so.  No reference source is copied into this repo: the
// shim only #includes the reference headers where they lie.  It serves two purposes:
//   * pinning: tests/golden/make_golden.py and tests/test_oracle.py compare the C
//     restatement (oracle/nttk_oracle.c) against the reference itself;
//   * baseline: bench.py --impl reference and the cpu_baseline leg time the
//     reference's own CPU path (ntt_forward_inplace / intt_inverse,
//     transform.hpp:228-231, 339-343) on the GPU box's host cores.
// The product never loads this library.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#if __has_include("json.hpp")
#define NTTK_REF_HAS_BENCH 1
#include "nttk/bench.hpp"  // the reference's own timing harness (needs nlohmann json.hpp)
#endif
#include "nttk/oracle.hpp"
#include "nttk/verify.hpp"  // the reference's own property suites
#include "nttk/params.hpp"
#include "nttk/reduction.hpp"
#include "nttk/transform.hpp"

using namespace nttk;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

ButterflyKind to_kind(int k) { return static_cast<ButterflyKind>(k); }

struct Handle {
  NttParams P;
};

// Exact-bound params: the reference's build_params refuses
// `improved` when p >= 2^{n-ell-2}; assemble the bundle from the reference's own
// pieces (make_reduction_context, find_primitive_root, the plain twiddle schedules
// and to_plantard_domain), exactly as build_params does for admitted parameters.
NttParams assemble_exact(uint64_t p, uint32_t N, unsigned n_bits,
                         std::vector<ButterflyKind> kinds) {
  std::vector<ButterflyKind> others;
  for (auto k : kinds)
    if (k != ButterflyKind::improved) others.push_back(k);
  NttParams P;
  if (!others.empty()) {
    P = build_params(p, N, n_bits, others);
  } else {
    P.p = static_cast<uint32_t>(p);
    P.size = N;
    P.log2_size = floor_log2(N);
    P.n_bits = n_bits;
    P.ctx = make_reduction_context(p, n_bits, 0, P.log2_size);
    P.omega = find_primitive_root(p, N);
    P.omega_inv = static_cast<uint64_t>(mod_inverse(P.omega, p));
    P.n_inv = static_cast<uint64_t>(mod_inverse(N % p, p));
  }
  P.kinds = kinds;
  P.fwd.ct_plantard.clear();
  for (uint64_t w : ct_forward_plain_twiddles(N, P.omega, p))
    P.fwd.ct_plantard.push_back(to_plantard_domain(w, P.ctx));
  P.inv.gs_plantard.clear();
  for (uint64_t w : gs_inverse_plain_twiddles(N, P.omega, p))
    P.inv.gs_plantard.push_back(to_plantard_domain(w, P.ctx));
  P.n_inv_hat = to_plantard_domain(P.n_inv, P.ctx);
  return P;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_params_build(uint64_t p, uint32_t N, unsigned n_bits, uint32_t kinds_mask, int exact,
                     void** out) {
  return guarded([&] {
    std::vector<ButterflyKind> kinds;
    for (int k = 0; k < 4; ++k)
      if (kinds_mask & (1u << k)) kinds.push_back(to_kind(k));
    auto* h = new Handle;
    try {
      h->P = build_params(p, N, n_bits, kinds);
    } catch (const contract_violation&) {
      if (!exact || !(kinds_mask & (1u << 3))) {
        delete h;
        throw;
      }
      h->P = assemble_exact(p, N, n_bits, kinds);
    }
    *out = h;
  });
}

void ref_params_free(void* h) { delete static_cast<Handle*>(h); }

// scalar fields: omega, omega_inv, n_inv, n_inv_hat, mu, scott L
int ref_params_scalars(void* hv, uint64_t* out6) {
  const auto& P = static_cast<Handle*>(hv)->P;
  out6[0] = P.omega;
  out6[1] = P.omega_inv;
  out6[2] = P.n_inv;
  out6[3] = P.n_inv_hat;
  out6[4] = P.ctx.mu;
  out6[5] = P.scott.lazy_level;
  return 0;
}

size_t ref_params_table(void* hv, const char* name, uint64_t* out, size_t cap) {
  const auto& P = static_cast<Handle*>(hv)->P;
  std::vector<uint64_t> v;
  const std::string n = name;
  if (n == "dif_w") for (auto& t : P.fwd.dif_ntl) v.push_back(t.w);
  else if (n == "dif_wq") for (auto& t : P.fwd.dif_ntl) v.push_back(t.w_quot);
  else if (n == "dif_mont") v = P.fwd.dif_mont;
  else if (n == "ct_plantard") v = P.fwd.ct_plantard;
  else if (n == "gs_wq") for (auto& t : P.inv.gs_ntl) v.push_back(t.w_quot);
  else if (n == "gs_plain") for (auto& t : P.inv.gs_ntl) v.push_back(t.w);
  else if (n == "gs_mont") v = P.inv.gs_mont;
  else if (n == "gs_plantard") v = P.inv.gs_plantard;
  else if (n == "ct_plain") v = ct_forward_plain_twiddles(P.size, P.omega, P.p);
  if (out) std::memcpy(out, v.data(), std::min(v.size(), cap) * 8);
  return v.size();
}

// checked forward per poly (transform.hpp:220-224)
int ref_forward(void* hv, int kind, uint64_t* a, size_t batch) {
  return guarded([&] {
    const auto& P = static_cast<Handle*>(hv)->P;
    for (size_t i = 0; i < batch; ++i) {
      Polynomial f(a + i * P.size, a + (i + 1) * P.size);
      const Spectrum s = ntt_forward(f, P, to_kind(kind));
      std::memcpy(a + i * P.size, s.values.data(), P.size * 8);
    }
  });
}

// checked inverse per poly (transform.hpp:339-343)
int ref_inverse(void* hv, int kind, uint64_t* a, size_t batch) {
  return guarded([&] {
    const auto& P = static_cast<Handle*>(hv)->P;
    for (size_t i = 0; i < batch; ++i) {
      Spectrum s{std::vector<uint64_t>(a + i * P.size, a + (i + 1) * P.size),
                 Ordering::bit_reversed};
      const Polynomial f = intt_inverse(s, P, to_kind(kind));
      std::memcpy(a + i * P.size, f.data(), P.size * 8);
    }
  });
}

int ref_pointwise(void* hv, int kind, const uint64_t* l, const uint64_t* r, uint64_t* out,
                  size_t batch) {
  return guarded([&] {
    const auto& P = static_cast<Handle*>(hv)->P;
    for (size_t i = 0; i < batch; ++i) {
      Spectrum a{std::vector<uint64_t>(l + i * P.size, l + (i + 1) * P.size),
                 Ordering::bit_reversed};
      Spectrum b{std::vector<uint64_t>(r + i * P.size, r + (i + 1) * P.size),
                 Ordering::bit_reversed};
      const Spectrum c = pointwise_multiply(a, b, P, to_kind(kind));
      std::memcpy(out + i * P.size, c.values.data(), P.size * 8);
    }
  });
}

int ref_convolution(void* hv, int kind, const uint64_t* x, const uint64_t* y, uint64_t* out,
                    size_t batch) {
  return guarded([&] {
    const auto& P = static_cast<Handle*>(hv)->P;
    for (size_t i = 0; i < batch; ++i) {
      Polynomial a(x + i * P.size, x + (i + 1) * P.size);
      Polynomial b(y + i * P.size, y + (i + 1) * P.size);
      const Polynomial c = cyclic_convolution_via_ntt(a, b, P, to_kind(kind));
      std::memcpy(out + i * P.size, c.data(), P.size * 8);
    }
  });
}

// ---- reductions (checked entry points, reduction.hpp:125-291) ----
int ref_mont_redc(uint64_t p, unsigned n, uint64_t T, uint64_t* out) {
  return guarded([&] { *out = mont_redc(T, make_reduction_context(p, n)); });
}
int ref_signed_mont_redc(uint64_t p, unsigned n, int64_t A, int64_t* out) {
  return guarded([&] { *out = signed_mont_redc(A, make_reduction_context(p, n)); });
}
int ref_plantard_redc(uint64_t p, unsigned n, uint64_t W, uint64_t T, uint64_t* out) {
  return guarded([&] { *out = plantard_redc(W, T, make_reduction_context(p, n)); });
}
int ref_modified_plantard_mul(uint64_t p, unsigned n, unsigned ell, uint64_t W, uint64_t T,
                              uint64_t* out) {
  return guarded(
      [&] { *out = modified_plantard_mul(W, T, make_reduction_context(p, n, 0, ell)); });
}
int ref_to_plantard_domain(uint64_t p, unsigned n, uint64_t w, uint64_t* out) {
  return guarded([&] { *out = to_plantard_domain(w, make_reduction_context(p, n)); });
}

// reduction sweep through the reference's checked entry points over a pair grid
int ref_sweep(int variant, uint64_t p, unsigned n, unsigned ell, const int64_t* A, size_t na,
              const int64_t* B, size_t nb, int64_t* r, uint64_t* checksum) {
  return guarded([&] {
    const auto ctx = make_reduction_context(p, n, 0, ell);
    uint64_t s = 0;
    for (size_t i = 0; i < na; ++i)
      for (size_t j = 0; j < nb; ++j) {
        int64_t v = 0;
        switch (variant) {
          case 0: v = static_cast<int64_t>(mont_redc(uint64_t(A[i]) * uint64_t(B[j]), ctx)); break;
          case 1: v = signed_mont_redc(A[i] * B[j], ctx); break;
          case 2: v = static_cast<int64_t>(plantard_redc(uint64_t(A[i]), uint64_t(B[j]), ctx)); break;
          default:
            v = static_cast<int64_t>(modified_plantard_mul(uint64_t(A[i]), uint64_t(B[j]), ctx));
        }
        s += uint64_t(v);
        if (r) r[i * nb + j] = v;
      }
    *checksum = s;
  });
}

uint64_t ref_plantard_fires() { return plantard_correction_fires().load(); }

void ref_rng_fill(uint64_t seed, uint64_t bound, uint64_t* out, size_t count) {
  Rng rng(seed);
  for (size_t i = 0; i < count; ++i) out[i] = rng.below(bound);
}

void ref_naive_dft(const uint64_t* f, size_t N, uint64_t omega, uint64_t p, uint64_t* out) {
  const auto v = naive_dft(std::vector<uint64_t>(f, f + N), omega, p);
  std::memcpy(out, v.data(), N * 8);
}

// ---- CPU baseline: the reference's own batch loop, sharded over host threads ----
// mode 0: forward only (ntt_forward_inplace, the reference bench path,
// bench.hpp:198-230); mode 1: forward then intt_inverse (round trip); mode 2: intt_inverse
// only (`a` holds spectra in butterfly order).
// `a` holds batch canonical polys; each thread works on its own contiguous shard.
// Returns elapsed wall nanoseconds in *ns.
int ref_time_batch(void* hv, int kind, int mode, uint64_t* a, size_t batch, int threads,
                   uint64_t* ns) {
  return guarded([&] {
    const auto& P = static_cast<Handle*>(hv)->P;
    const ButterflyKind k = to_kind(kind);
    if (threads < 1) threads = 1;
    std::atomic<int> failed{0};
    auto work = [&](size_t lo, size_t hi) {
      try {
        std::vector<uint64_t> buf(P.size);
        for (size_t i = lo; i < hi; ++i) {
          uint64_t* poly = a + i * P.size;
          std::memcpy(buf.data(), poly, P.size * 8);
          if (mode == 2) {
            const Polynomial f = intt_inverse(Spectrum{buf, Ordering::bit_reversed}, P, k);
            std::memcpy(poly, f.data(), P.size * 8);
            continue;
          }
          ntt_forward_inplace(buf, P, k);
          if (mode == 1) {
            const Polynomial f = intt_inverse(Spectrum{buf, Ordering::bit_reversed}, P, k);
            std::memcpy(poly, f.data(), P.size * 8);
          } else {
            std::memcpy(poly, buf.data(), P.size * 8);
          }
        }
      } catch (...) {
        failed = 1;
      }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back(work, batch * t / threads, batch * (t + 1) / threads);
    for (auto& th : pool) th.join();
    const auto t1 = std::chrono::steady_clock::now();
    *ns = static_cast<uint64_t>(
        std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
    if (failed) throw contract_violation("ref_time_batch: a worker failed");
  });
}

// ntt_forward_observed / intt_inverse_observed of the reference (transform.hpp:207-337):
// one polynomial; states[(layer - 1) * N ...] receives the state after each layer
int ref_observed(void* hv, int kind, int dir, const uint64_t* in, uint64_t* states, uint64_t* out) {
  return guarded([&] {
    const auto& P = static_cast<Handle*>(hv)->P;
    const size_t N = P.size;
    auto obs = [&](unsigned layer, const std::vector<uint64_t>& v) {
      std::memcpy(states + size_t(layer - 1) * N, v.data(), N * 8);
    };
    if (dir == 0) {
      const Spectrum s = ntt_forward_observed(Polynomial(in, in + N), P, to_kind(kind), obs);
      std::memcpy(out, s.values.data(), N * 8);
    } else {
      const Polynomial f = intt_inverse_observed(
          Spectrum{std::vector<uint64_t>(in, in + N), Ordering::bit_reversed}, P, to_kind(kind), obs);
      std::memcpy(out, f.data(), N * 8);
    }
  });
}

// ---- extension trees driven by the reference's UNMODIFIED cores ----
// The reference has no negacyclic / 7-layer driver, basemul or signed-Montgomery transform.
// These drivers reproduce the split/merge loop shape of run_split_layers / run_merge_layers
// (transform.hpp:77-116) on the a22 schedule -- layer s, block b uses zeta^{br_L(2^{s-1}+b)}
// (negacyclic) or omega^{(N >> s) br_{s-1}(b)} (cyclic, params.hpp:60-88) -- and compute
// every product with the reference's own functions:
//   improved  improved_ct_core / improved_gs_core (butterfly.hpp:224-243) on twiddles
//             encoded by to_plantard_domain (reduction.hpp:279-283), final scale by
//             modified_plantard_core with the encoded 2^{-L} (transform.hpp:323-330 pattern)
//   harvey    the Montgomery product of harvey_core (butterfly.hpp:92-106, its Y output with
//             X = Y, Y = 2p, i.e. t = Y) on to_montgomery_domain twiddles; the CT-form sums
//             (X + t, X + 2p - t) mod 2p are the extension's own
//   smont     signed_mont_redc (reduction.hpp:141-165, checked entry) on centered
//             Montgomery twiddles; the GS sum uses the extension's signed Barrett
// Words of the forward transform are the reference-run words the GPU kernels must equal;
// the inverse and basemul outputs are canonical.
namespace tree {

enum { kNtl = 0, kHarvey = 1, kScott = 2, kImproved = 3, kSmont = 4 };

struct Sched {
  ReductionContext ctx;
  uint32_t N = 0, L = 0;
  int nega = 0;
  uint64_t root = 0, order = 0, scale = 0;  // scale = N^{-1} (cyclic) or 2^{-L} (nega)
  std::vector<uint64_t> ct, gs;             // plain twiddles, driver order (layer, block)
};

Sched make(uint64_t p, uint32_t N, unsigned n_bits, int nega, uint32_t L) {
  Sched S;
  S.ctx = make_reduction_context(p, n_bits);
  S.N = N;
  S.L = L;
  S.nega = nega;
  S.order = nega ? (uint64_t(2) << L) : N;
  S.root = find_primitive_root(p, static_cast<uint32_t>(S.order));
  for (unsigned s = 1; s <= L; ++s)
    for (uint64_t b = 0; b < (uint64_t(1) << (s - 1)); ++b) {
      const uint64_t e = nega ? bit_reverse((uint64_t(1) << (s - 1)) + b, L) % S.order
                              : (uint64_t(N >> s) * bit_reverse(b, s - 1)) % S.order;
      S.ct.push_back(pow_mod(S.root, e, p));
    }
  for (unsigned s = L; s >= 1; --s)
    for (uint64_t b = 0; b < (uint64_t(1) << (s - 1)); ++b) {
      const uint64_t e = nega ? bit_reverse((uint64_t(1) << (s - 1)) + b, L) % S.order
                              : (uint64_t(N >> s) * bit_reverse(b, s - 1)) % S.order;
      S.gs.push_back(pow_mod(S.root, e == 0 ? 0 : S.order - e, p));
    }
  S.scale = static_cast<uint64_t>(mod_inverse((nega ? (uint64_t(1) << L) : N) % p, p));
  return S;
}

int64_t signed_twiddle(uint64_t w, const ReductionContext& c) {  // centered w 2^n mod p
  const uint64_t m = to_montgomery_domain(w, c);
  return m > c.p / 2 ? int64_t(m) - int64_t(c.p) : int64_t(m);
}

int64_t signed_barrett(int64_t a, const ReductionContext& c) {  // extension, S = n + 10
  const unsigned S = c.n_bits + 10;
  const int64_t V = static_cast<int64_t>(((u128(1) << S) + (c.p >> 1)) / c.p);
  const int64_t q = static_cast<int64_t>((i128(a) * V + (i128(1) << (S - 1))) >> S);
  return a - q * int64_t(c.p);
}

uint64_t harvey_mul(uint64_t t, uint64_t w_mont, const ReductionContext& c) {
  return harvey_core(t, 2 * uint64_t(c.p), w_mont, c.p_inv_beta, c.p, c.n_bits, c.beta_mask).y;
}

void forward(const Sched& S, int kind, uint64_t* a) {
  const auto& c = S.ctx;
  const uint64_t p = c.p;
  size_t cursor = 0;
  for (unsigned s = 1; s <= S.L; ++s) {
    const uint32_t len = S.N >> s, blocks = 1u << (s - 1);
    for (uint32_t b = 0; b < blocks; ++b) {
      const uint64_t w = S.ct[cursor + b];
      const uint64_t w_hat = kind == kImproved ? to_plantard_domain(w, c) : 0;
      const uint64_t w_mont = kind == kHarvey ? to_montgomery_domain(w, c) : 0;
      const int64_t w_s = kind == kSmont ? signed_twiddle(w, c) : 0;
      for (uint32_t j = 0; j < len; ++j) {
        uint64_t& X = a[size_t(b) * 2 * len + j];
        uint64_t& Y = a[size_t(b) * 2 * len + j + len];
        if (kind == kImproved) {
          const auto o = improved_ct_core<uint64_t>(X, Y, w_hat, c.mu, p, c.n_bits, c.r2n_mask);
          X = o.x, Y = o.y;
        } else if (kind == kHarvey) {
          const uint64_t r = harvey_mul(Y, w_mont, c);
          uint64_t u = X + r, v = X + 2 * p - r;
          if (u >= 2 * p) u -= 2 * p;
          if (v >= 2 * p) v -= 2 * p;
          X = u, Y = v;
        } else {
          const int64_t t = signed_mont_redc(w_s * int64_t(Y), c);
          const int64_t x = int64_t(X);
          X = uint64_t(x + t), Y = uint64_t(x - t);
        }
      }
    }
    cursor += blocks;
  }
}

void inverse(const Sched& S, int kind, uint64_t* a) {
  const auto& c = S.ctx;
  const uint64_t p = c.p;
  for (uint32_t i = 0; i < S.N; ++i) {  // canonicalize (transform.hpp:243)
    if (kind == kSmont) {
      const int64_t v = int64_t(a[i]) % int64_t(p);
      a[i] = uint64_t(v < 0 ? v + int64_t(p) : v);
    } else {
      a[i] %= p;
    }
  }
  size_t cursor = 0;
  unsigned m = 0;
  for (unsigned s = S.L; s >= 1; --s) {
    ++m;
    const uint32_t len = S.N >> s, blocks = 1u << (s - 1);
    for (uint32_t b = 0; b < blocks; ++b) {
      const uint64_t w = S.gs[cursor + b];
      const uint64_t w_hat = kind == kImproved ? to_plantard_domain(w, c) : 0;
      const uint64_t w_mont = kind == kHarvey ? to_montgomery_domain(w, c) : 0;
      const int64_t w_s = kind == kSmont ? signed_twiddle(w, c) : 0;
      for (uint32_t j = 0; j < len; ++j) {
        uint64_t& X = a[size_t(b) * 2 * len + j];
        uint64_t& Y = a[size_t(b) * 2 * len + j + len];
        if (kind == kImproved) {
          const auto o = improved_gs_core<uint64_t>(X, Y, p << (m - 1), w_hat, c.mu, p, c.n_bits,
                                                    c.r2n_mask);
          X = o.x, Y = o.y;
        } else if (kind == kHarvey) {
          const auto o = harvey_core(X, Y, w_mont, c.p_inv_beta, p, c.n_bits, c.beta_mask);
          X = o.x, Y = o.y;
        } else {
          const int64_t x = int64_t(X), y = int64_t(Y);
          X = uint64_t(signed_barrett(x + y, c));
          Y = uint64_t(signed_mont_redc(w_s * (x - y), c));
        }
      }
    }
    cursor += blocks;
  }
  const uint64_t s_hat = kind == kImproved ? to_plantard_domain(S.scale, c) : 0;
  const int64_t s_s = kind == kSmont ? signed_twiddle(S.scale, c) : 0;
  for (uint32_t i = 0; i < S.N; ++i) {
    if (kind == kImproved) {
      a[i] = modified_plantard_core<uint64_t>(s_hat, a[i], c.mu, p, c.n_bits, c.r2n_mask);
    } else if (kind == kSmont) {
      const int64_t v = signed_mont_redc(s_s * int64_t(a[i]), c);
      a[i] = uint64_t(v < 0 ? v + int64_t(p) : v);
    } else {
      a[i] = static_cast<uint64_t>(u128(a[i] % p) * S.scale % p);
    }
  }
}

// canonical product of canonical a, b: modified_plantard_core(to_plantard_domain(a), b)
uint64_t mulc(uint64_t a, uint64_t b, const ReductionContext& c) {
  return modified_plantard_core<uint64_t>(to_plantard_domain(a, c), b, c.mu, c.p, c.n_bits,
                                          c.r2n_mask);
}

// degree-2 basemul mod (x^2 - gamma), gamma = +-(last-layer twiddle), canonical output
void basemul(const Sched& S, int kind, const uint64_t* l, const uint64_t* r, uint64_t* o) {
  const auto& c = S.ctx;
  const uint64_t p = c.p;
  auto canon = [&](uint64_t v) {
    if (kind == kSmont) {
      const int64_t s = int64_t(v) % int64_t(p);
      return uint64_t(s < 0 ? s + int64_t(p) : s);
    }
    return v % p;
  };
  const size_t last = (size_t(1) << (S.L - 1)) - 1;
  for (uint32_t k = 0; k < S.N / 2; ++k) {
    const uint64_t z = S.ct[last + k / 2];
    const uint64_t g = (k & 1) ? (p - z) % p : z;
    const uint64_t a0 = canon(l[2 * k]), a1 = canon(l[2 * k + 1]);
    const uint64_t b0 = canon(r[2 * k]), b1 = canon(r[2 * k + 1]);
    o[2 * k] = (mulc(a0, b0, c) + mulc(mulc(a1, b1, c), g, c)) % p;
    o[2 * k + 1] = (mulc(a0, b1, c) + mulc(a1, b0, c)) % p;
  }
}

}  // namespace tree

// dir 0 forward, 1 inverse, 2 polymul (forward a, forward b, basemul, inverse; `b` used)
int ref_tree_run(uint64_t p, uint32_t N, unsigned n_bits, int nega, uint32_t layers, int kind,
                 int dir, uint64_t* a, const uint64_t* b, size_t batch) {
  return guarded([&] {
    NTTK_REQUIRE(kind == tree::kImproved || kind == tree::kHarvey || kind == tree::kSmont,
                 "ref_tree_run: kind must be improved, harvey or smont");
    NTTK_REQUIRE(layers >= 1 && (N >> layers) >= 1, "ref_tree_run: bad layer count");
    const tree::Sched S = tree::make(p, N, n_bits, nega, layers);
    std::vector<uint64_t> fb(N), prod(N);
    for (size_t i = 0; i < batch; ++i) {
      uint64_t* x = a + i * N;
      if (dir == 0) {
        tree::forward(S, kind, x);
      } else if (dir == 1) {
        tree::inverse(S, kind, x);
      } else {
        NTTK_REQUIRE((N >> layers) == 2, "ref_tree_run: polymul needs degree-2 leaves");
        std::memcpy(fb.data(), b + i * N, N * 8);
        tree::forward(S, kind, x);
        tree::forward(S, kind, fb.data());
        tree::basemul(S, kind, x, fb.data(), prod.data());
        tree::inverse(S, kind, prod.data());
        std::memcpy(x, prod.data(), N * 8);
      }
    }
  });
}

// CPU baselines of the extension configs: ref_tree_run over `batch` polys split across
// `threads` host threads (each shard independent); elapsed wall ns in *ns
int ref_time_tree(uint64_t p, uint32_t N, unsigned n_bits, int nega, uint32_t layers, int kind,
                  int dir, uint64_t* a, const uint64_t* b, size_t batch, int threads, uint64_t* ns) {
  return guarded([&] {
    if (threads < 1) threads = 1;
    std::atomic<int> failed{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
      const size_t lo = batch * t / threads, hi = batch * (t + 1) / threads;
      pool.emplace_back([&, lo, hi] {
        if (ref_tree_run(p, N, n_bits, nega, layers, kind, dir, a + lo * N, b ? b + lo * N : nullptr,
                         hi - lo) != 0)
          failed = 1;
      });
    }
    for (auto& th : pool) th.join();
    const auto t1 = std::chrono::steady_clock::now();
    *ns = static_cast<uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
    if (failed) throw contract_violation("ref_time_tree: a worker failed");
  });
}

// cyclic_convolution_via_ntt (transform.hpp:372-379) over host threads, wall ns in *ns
int ref_time_convolution(void* hv, int kind, const uint64_t* x, const uint64_t* y, uint64_t* out,
                         size_t batch, int threads, uint64_t* ns) {
  return guarded([&] {
    if (threads < 1) threads = 1;
    std::atomic<int> failed{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
      const size_t lo = batch * t / threads, hi = batch * (t + 1) / threads;
      const size_t N = static_cast<Handle*>(hv)->P.size;
      pool.emplace_back([&, lo, hi, N] {
        if (ref_convolution(hv, kind, x + lo * N, y + lo * N, out + lo * N, hi - lo) != 0) failed = 1;
      });
    }
    for (auto& th : pool) th.join();
    const auto t1 = std::chrono::steady_clock::now();
    *ns = static_cast<uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
    if (failed) throw contract_violation("ref_time_convolution: a worker failed");
  });
}

// The reference's own property suites (verify.hpp:576-584 run_all_suites): writes one line
// "name cases failures" per suite into out; returns the total failure count in *failures.
int ref_run_all_suites(uint64_t random_cases, char* out, size_t cap, uint64_t* failures) {
  return guarded([&] {
    VerifyOptions opt;
    opt.random_cases = random_cases;
    std::string txt;
    uint64_t f = 0;
    for (const auto& r : run_all_suites(opt)) {
      txt += r.name + " " + std::to_string(r.cases) + " " + std::to_string(r.failures) + "\n";
      f += r.failures;
    }
    *failures = f;
    if (out && cap) {
      const size_t n = txt.size() < cap - 1 ? txt.size() : cap - 1;
      std::memcpy(out, txt.data(), n);
      out[n] = 0;
    }
  });
}

// The reference's own run_bench (bench.hpp:334-361) at the given presets, serialised by
// its own to_json (schema 1, bench.hpp:365-424) -- the CPU rows of the paper's Table 2.
// Writes at most cap bytes of JSON into out; *need = full length.  Status 3 when this
// shim was built without json.hpp.
int ref_run_bench(const char* presets_csv, uint64_t iters, uint64_t seed, int micro, char* out,
                  size_t cap, size_t* need) {
#ifdef NTTK_REF_HAS_BENCH
  return guarded([&] {
    BenchOptions opt;
    opt.presets.clear();
    std::string cur;
    for (const char* c = presets_csv;; ++c) {
      if (*c == ',' || *c == 0) {
        if (!cur.empty()) opt.presets.push_back(cur);
        cur.clear();
        if (*c == 0) break;
      } else {
        cur += *c;
      }
    }
    opt.iters = iters;
    opt.seed = seed;
    opt.micro = micro != 0;
    const BenchReport rep = run_bench(opt);
    nlohmann::json j = rep;
    const std::string txt = j.dump();
    *need = txt.size();
    if (out && cap) {
      const size_t n = txt.size() < cap - 1 ? txt.size() : cap - 1;
      std::memcpy(out, txt.data(), n);
      out[n] = 0;
    }
  });
#else
  (void)presets_csv, (void)iters, (void)seed, (void)micro, (void)out, (void)cap, (void)need;
  g_err = "ref_run_bench: shim built without json.hpp";
  return 3;
#endif
}

}  // extern "C"
