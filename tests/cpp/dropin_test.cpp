// dropin_test.cpp -- the reference's transform/params test cases, run against the B200
// engine through the C++ drop-in header (paper_2402_00675_b200/include/nttk_gpu/nttk.hpp).
//
// Mirrors proj/tests/transform_test.cpp and params_test.cpp case by case (hand-evaluated
// spectra, every-kind round trips, convolution vs schoolbook, contract messages) with
// plain checks instead of GoogleTest (absent in this image).  Exit code 0 = all passed.
// Built and run by tests/test_cpp_dropin.py (-m gpu).
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>

#include "nttk_gpu/nttk.hpp"

using namespace nttk;

static int g_fail = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (!(cond)) {                                                         \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
      ++g_fail;                                                            \
    }                                                                      \
  } while (0)

template <class F>
static bool throws_with(F&& f, const char* needle) {
  try {
    f();
  } catch (const contract_violation& e) {
    return std::string(e.what()).find(needle) != std::string::npos;
  }
  return false;
}

static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t p) {
  return static_cast<uint64_t>((unsigned __int128)a * b % p);
}

static std::vector<uint64_t> natural(const Spectrum& s, uint64_t p) {  // bit-reversal + canon
  const size_t N = s.values.size();
  unsigned bits = 0;
  while ((size_t(1) << bits) < N) ++bits;
  std::vector<uint64_t> v(N);
  for (size_t i = 0; i < N; ++i) {
    size_t r = 0;
    for (unsigned b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
    v[r] = s.values[i] % p;
  }
  return v;
}

static std::vector<uint64_t> naive_dft(const Polynomial& f, uint64_t w, uint64_t p) {
  std::vector<uint64_t> out(f.size());
  uint64_t x = 1;
  for (size_t i = 0; i < f.size(); ++i, x = mulmod(x, w, p)) {
    uint64_t acc = 0;
    for (size_t j = f.size(); j-- > 0;) acc = (mulmod(acc, x, p) + f[j]) % p;
    out[i] = acc;
  }
  return out;
}

static Polynomial schoolbook(const Polynomial& a, const Polynomial& b, uint64_t p) {
  Polynomial c(a.size(), 0);
  for (size_t i = 0; i < a.size(); ++i)
    for (size_t j = 0; j < a.size(); ++j) {
      const size_t k = (i + j) % a.size();
      c[k] = (c[k] + mulmod(a[i], b[j], p)) % p;
    }
  return c;
}

static Polynomial random_poly(uint32_t N, uint64_t p, std::mt19937_64& rng) {
  std::uniform_int_distribution<uint64_t> d(0, p - 1);
  Polynomial f(N);
  for (auto& c : f) c = d(rng);
  return f;
}

int main() {
  // params_test.cpp:56-69 -- toy13 bundle scalars
  {
    const auto P = preset("toy13");
    CHECK(P.p == 13 && P.size == 4 && P.log2_size == 2);
    CHECK(P.omega == 5 && P.omega_inv == 8 && P.n_inv == 10);
    for (auto k : all_butterfly_kinds()) CHECK(P.has(k));
  }
  // params_test.cpp:71-110 -- fault collection and messages
  CHECK(throws_with([] { (void)build_params(15, 4, 8); }, "p must be prime"));
  CHECK(throws_with([] { (void)build_params(13, 8, 8); }, "N must divide p - 1"));
  CHECK(throws_with([] { (void)build_params(15, 6, 40); }, "[2, 32]"));
  CHECK(throws_with([] { (void)build_params(7681, 256, 16); }, "p < 2^{n-ell-2}"));
  CHECK(throws_with([] { (void)preset("nope"); }, "unknown preset"));
  CHECK(throws_with([] { (void)butterfly_kind_from_string("fancy"); }, "unknown butterfly kind"));
  // transform_test.cpp:39-48 -- hand-evaluated DFT, every kind
  {
    const auto P = build_params(17, 4, 16);
    const Polynomial f{1, 2, 3, 4};
    const std::vector<uint64_t> want{10, 7, 15, 6};
    CHECK(naive_dft(f, P.omega, P.p) == want);
    for (auto k : all_butterfly_kinds()) CHECK(natural(ntt_forward(f, P, k), P.p) == want);
  }
  // transform_test.cpp:50-59 -- delta in slot one lists the root powers
  {
    const auto P = preset("toy13");
    const std::vector<uint64_t> want{1, 5, 12, 8};
    for (auto k : all_butterfly_kinds())
      CHECK(natural(ntt_forward({0, 1, 0, 0}, P, k), P.p) == want);
  }
  // transform_test.cpp:61-93 -- kinds agree; every kind pair inverts every other
  for (const char* name : {"toy13", "kyber256", "falcon512"}) {
    const auto P = preset(name);
    std::mt19937_64 rng(7);
    const auto f = random_poly(P.size, P.p, rng);
    const auto base = natural(ntt_forward(f, P, ButterflyKind::ntl), P.p);
    CHECK(base == naive_dft(f, P.omega, P.p));
    for (auto fk : all_butterfly_kinds()) {
      const auto spec = ntt_forward(f, P, fk);
      CHECK(natural(spec, P.p) == base);
      for (auto ik : all_butterfly_kinds()) CHECK(intt_inverse(spec, P, ik) == f);
    }
  }
  // transform_test.cpp:373-400 -- convolution vs schoolbook
  {
    const auto P = build_params(17, 4, 16);
    for (auto k : all_butterfly_kinds())
      CHECK(cyclic_convolution_via_ntt({1, 2, 3, 4}, {1, 0, 0, 1}, P, k) ==
            (Polynomial{3, 5, 7, 5}));
    const auto K = preset("kyber256");
    std::mt19937_64 rng(31337);
    for (int t = 0; t < 3; ++t) {
      const auto a = random_poly(K.size, K.p, rng), b = random_poly(K.size, K.p, rng);
      const auto want = schoolbook(a, b, K.p);
      for (auto k : all_butterfly_kinds()) CHECK(cyclic_convolution_via_ntt(a, b, K, k) == want);
    }
  }
  // transform_test.cpp:402-420 -- improved pointwise takes a lazy right operand
  {
    const auto P = preset("toy13");
    const Spectrum lhs{{1, 2, 3, 4}}, rhs{{51, 40, 27, 14}};
    const auto out = pointwise_multiply(lhs, rhs, P, ButterflyKind::improved);
    for (int i = 0; i < 4; ++i) CHECK(out.values[i] == lhs.values[i] * (rhs.values[i] % 13) % 13);
    CHECK(pointwise_multiply(lhs, rhs, P, ButterflyKind::harvey).values == out.values);
    CHECK(throws_with(
        [&] { (void)pointwise_multiply(lhs, Spectrum{{1, 2, 3, 4}, Ordering::natural}, P,
                                       ButterflyKind::ntl); },
        "mixed orderings"));
  }
  // transform_test.cpp:440-463 -- entry points validate their inputs
  {
    const auto P = preset("toy13");
    CHECK(throws_with([&] { (void)ntt_forward({1, 2}, P, ButterflyKind::ntl); }, "wrong input length"));
    CHECK(throws_with([&] { (void)ntt_forward({13, 0, 0, 0}, P, ButterflyKind::ntl); },
                      "coefficients must be canonical"));
    CHECK(throws_with(
        [&] { (void)intt_inverse(Spectrum{{1, 2, 3, 4}, Ordering::natural}, P, ButterflyKind::ntl); },
        "butterfly order"));
    const auto only = build_params(13, 4, 8, {ButterflyKind::ntl});
    CHECK(throws_with([&] { (void)ntt_forward({1, 2, 3, 4}, only, ButterflyKind::harvey); },
                      "kind not built"));
  }
  // BASELINE moduli through the fast path: Kyber (n=16) and Dilithium (n=32) round trips
  {
    BuildOptions o;
    o.exact_bound = true;
    for (auto [p, n] : {std::pair<uint64_t, unsigned>{3329, 16}, {8380417, 32}}) {
      const auto P = build_params(p, 256, n, {ButterflyKind::improved, ButterflyKind::harvey}, o);
      std::mt19937_64 rng(p);
      std::vector<uint64_t> batch(64 * 256);
      for (auto& c : batch) c = rng() % p;
      std::vector<uint64_t> spec(batch.size()), back(batch.size());
      for (auto k : {ButterflyKind::improved, ButterflyKind::harvey}) {
        ntt_forward_batch(batch.data(), spec.data(), 64, P, k);
        intt_inverse_batch(spec.data(), back.data(), 64, P, k);
        CHECK(back == batch);
        const Polynomial f0(batch.begin(), batch.begin() + 256);
        CHECK(natural(Spectrum{std::vector<uint64_t>(spec.begin(), spec.begin() + 256)}, p) ==
              naive_dft(f0, P.omega, p));
      }
    }
  }
  // reduction.hpp through the GPU: the reference's known answers (reduction_test.cpp:11-190)
  {
    const ReductionContext c = make_reduction_context(13, 8, 0, 2);
    CHECK(c.mu == 20165 && c.fits_plantard_bound() && c.fits_lazy_plantard_bound());
    CHECK(mont_redc(100, make_reduction_context(17, 5)) == 1);
    const ReductionContext s = make_reduction_context(17, 6);
    CHECK(signed_mont_redc(100, s) == 9 && signed_mont_redc(-100, s) == -9);
    CHECK(plantard_redc(5, 12, make_reduction_context(13, 8)) == 6);
    CHECK(modified_plantard_mul(5, 20, c) == 10 && modified_plantard_mul(1, 1, c) == 4);
    CHECK(to_plantard_domain(7, c) == 5);
    for (uint64_t w = 0; w < 13; ++w) {
      CHECK(to_montgomery_domain(w, c) == w * 256 % 13);
      CHECK(modified_plantard_mul(to_plantard_domain(w, c), 1, c) == w);
    }
    // batched: the exhaustive Montgomery range of (17, n=5) in one call
    const ReductionContext m = make_reduction_context(17, 5);
    std::vector<uint64_t> T(17 * 17);
    for (uint64_t t = 0; t < T.size(); ++t) T[t] = t;
    const auto r = mont_redc(T, m);
    uint64_t inv32 = 0;  // 2^{-5} mod 17
    for (uint64_t v = 1; v < 17; ++v)
      if (v * 32 % 17 == 1) inv32 = v;
    bool all = true;
    for (uint64_t t = 0; t < T.size(); ++t) all = all && r[t] == t * inv32 % 17;
    CHECK(all);
    // contract messages of the reference
    CHECK(throws_with([&] { (void)mont_redc(17 * 17, m); }, "mont_redc: T must be < p^2"));
    CHECK(throws_with([&] { (void)modified_plantard_mul(13, 0, c); }, "W must be < p"));
    CHECK(throws_with([&] { (void)modified_plantard_mul(0, 52, c); }, "T must be < 2^ell * p"));
    CHECK(throws_with([&] { (void)plantard_redc(14, 0, make_reduction_context(13, 8)); },
                      "inputs exceed p"));
    CHECK(throws_with([] { (void)make_reduction_context(12, 8); }, "p must be odd"));
    CHECK(throws_with([] { (void)modified_plantard_mul(1, 1, make_reduction_context(17, 8, 0, 2)); },
                      "requires p < 2^{n-ell-2}"));
  }
  // butterfly.hpp through the GPU: the reference's hand cases (butterfly_test.cpp:31-197)
  {
    const ReductionContext c8 = make_reduction_context(13, 8);
    CHECK((ntl_butterfly(5, 9, 3, 59, c8) == ButterflyOut{1, 1}));
    CHECK((harvey_butterfly(100, 4000, 4583, make_reduction_context(7681, 16)) ==
           ButterflyOut{4100, 3662}));
    CHECK((harvey_butterfly_ref(100, 4000, 4583, make_reduction_context(7681, 16)) ==
           ButterflyOut{4100, 3662}));
    const ScottConfig cfg = make_scott_config(4, c8);
    CHECK(cfg.lazy_level == 1);
    CHECK((scott_butterfly(5, 9, 3, c8, cfg) == ButterflyOut{14, 3}));
    const ReductionContext c = make_reduction_context(13, 8, 0, 2);
    CHECK((improved_ct_butterfly(3, 20, 5, c) == ButterflyOut{13, 6}));
    CHECK((improved_gs_butterfly(5, 9, 5, c, 1) == ButterflyOut{14, 11}));
    CHECK(throws_with([&] { (void)ntl_butterfly(5, 9, 3, 58, c8); }, "stale W_quot"));
    CHECK(throws_with([&] { (void)harvey_butterfly(0, 0, 0, make_reduction_context(7681, 16)); },
                      "W out of (0, p)"));
    CHECK(throws_with([&] { (void)improved_gs_butterfly(5, 9, 5, c, 3); }, "layer out of [1, ell]"));
    CHECK(throws_with([&] { (void)improved_ct_butterfly(26, 0, 5, c); }, "inputs must be < 2^ell * p / 2"));
  }
  // params.hpp / transform.hpp helpers and the NttParams tables (params_test.cpp patterns)
  {
    const auto P = preset("kyber256");
    CHECK(find_primitive_root(7681, 256) == P.omega && P.omega == 198);
    CHECK(ct_forward_plain_twiddles(256, P.omega, P.p) == P.table("ct_plain"));
    CHECK(gs_inverse_plain_twiddles(256, P.omega, P.p) == P.table("gs_plain"));
    const auto dif = dif_forward_plain_twiddles(256, P.omega, P.p);
    CHECK(dif.size() == P.fwd.dif_ntl.size() && P.fwd.dif_ntl[5].w == dif[5]);
    CHECK(P.fwd.ct_plantard.size() == 255 && P.inv.gs_plantard.size() == 255);
    CHECK(P.ctx.p == 7681 && P.ctx.ell == 8 && P.scott.lazy_level >= 1);
    // decode the encoded tables back against the plain schedules (on the device)
    const auto ct = P.table("ct_plain");
    bool ok = true;
    for (size_t i = 0; i < ct.size(); ++i)
      ok = ok && P.fwd.ct_plantard[i] == to_plantard_domain(ct[i], P.ctx) &&
           P.fwd.dif_mont[i] == to_montgomery_domain(dif[i], P.ctx);
    CHECK(ok);
    CHECK(spectrum_value_bound(P, ButterflyKind::improved) == 9 * 7681ull);
    CHECK(spectrum_value_bound(P, ButterflyKind::scott) == 256 * 7681ull);
    std::vector<uint64_t> v{7681, 7682, 15363, ~0ull};
    canonicalize(v, 7681);
    CHECK((v == std::vector<uint64_t>{0, 1, 1, ~0ull % 7681}));
    const Spectrum sp{{0, 1, 2, 3, 4, 5, 6, 7}};
    CHECK((to_natural_order(sp) == std::vector<uint64_t>{0, 4, 2, 6, 1, 5, 3, 7}));
    CHECK(preset_spec("falcon1024").size == 1024);
    CHECK(throws_with([] { (void)preset_spec("nope"); }, "unknown preset"));
  }
  // observed transforms: one callback per layer, the last forward state is the spectrum,
  // the inverse's states end in the scaled polynomial's pre-scaling sums
  {
    const auto P = preset("toy13");
    const Polynomial f{1, 2, 3, 4};
    for (auto k : all_butterfly_kinds()) {
      std::vector<std::vector<uint64_t>> states;
      const auto s = ntt_forward_observed(f, P, k, [&](unsigned layer, const std::vector<uint64_t>& v) {
        CHECK(layer == states.size() + 1);
        states.push_back(v);
      });
      CHECK(states.size() == 2 && states.back() == s.values && s.values == ntt_forward(f, P, k).values);
      unsigned layers = 0;
      const auto g = intt_inverse_observed(s, P, k, [&](unsigned, const std::vector<uint64_t>&) { ++layers; });
      CHECK(layers == 2 && g == f);
    }
    CHECK(throws_with([&] { (void)ntt_forward_observed({13, 0, 0, 0}, P, ButterflyKind::ntl, nullptr); },
                      "coefficients must be canonical"));
  }
  std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "OK", g_fail);
  return g_fail ? 1 : 0;
}
