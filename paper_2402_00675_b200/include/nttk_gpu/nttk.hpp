// nttk_gpu/nttk.hpp -- header-only C++ drop-in for the reference's nttk hot path.
//
// Same namespace, names, signatures and error behaviour as the reference library
// (/root/reference/proj/include/nttk): swap
//     #include "nttk/transform.hpp"      ->   #include "nttk_gpu/nttk.hpp"
// and link libnttk_gpu.so.  Every call runs on the B200 through the C ABI
// (include/nttk_gpu.h); contract violations throw nttk::contract_violation with the
// reference's messages.  Batched overloads take many polynomials per call, which is
// how the engine should be driven.
//
//   reference                                   here
//   params.hpp:137  build_params(p,N,n,kinds)   build_params(p,N,n,kinds [, opts])
//   params.hpp:303  preset(name)                preset(name)
//   transform.hpp:220  ntt_forward              ntt_forward (+ batch overload)
//   transform.hpp:228  ntt_forward_inplace      ntt_forward_inplace
//   transform.hpp:339  intt_inverse             intt_inverse (+ batch overload)
//   transform.hpp:349  pointwise_multiply       pointwise_multiply
//   transform.hpp:372  cyclic_convolution_via_ntt  cyclic_convolution_via_ntt
//   transform.hpp:38-70 canonicalize / to_natural_order / spectrum_value_bound (same names)
//   reduction.hpp:44-291 make_reduction_context, mont_redc, signed_mont_redc, plantard_redc,
//                    modified_plantard_mul, to_plantard_domain, to_montgomery_domain (GPU)
//   butterfly.hpp:52-279 ntl_/harvey_/scott_/improved_ct_/improved_gs_butterfly,
//                    make_scott_config (GPU)
//   params.hpp:30-128 NttParams fields (ctx, scott, fwd, inv tables), find_primitive_root,
//                    *_plain_twiddles, preset_table, preset_spec
#pragma once

#include <cstdint>
#include <exception>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "nttk_gpu.h"

namespace nttk {

class contract_violation : public std::invalid_argument {  // int_util.hpp:17-21
 public:
  explicit contract_violation(const std::string& what) : std::invalid_argument(what) {}
};

class device_error : public std::runtime_error {
 public:
  explicit device_error(const std::string& what) : std::runtime_error(what) {}
};

enum class ButterflyKind { ntl, harvey, scott, improved, smont };  // butterfly.hpp:30 (+smont)
enum class Ordering { natural, bit_reversed };                   // transform.hpp:26
enum class Tree { cyclic = NTTK_CYCLIC, negacyclic = NTTK_NEGACYCLIC };

using Polynomial = std::vector<uint64_t>;  // transform.hpp:28

struct Spectrum {  // transform.hpp:30-33
  std::vector<uint64_t> values;
  Ordering ordering = Ordering::bit_reversed;
};

[[nodiscard]] constexpr const char* to_string(ButterflyKind k) {  // butterfly.hpp:32-40
  switch (k) {
    case ButterflyKind::ntl: return "ntl";
    case ButterflyKind::harvey: return "harvey";
    case ButterflyKind::scott: return "scott";
    case ButterflyKind::improved: return "improved";
    case ButterflyKind::smont: return "smont";
  }
  return "?";
}

[[nodiscard]] inline ButterflyKind butterfly_kind_from_string(std::string_view name) {
  if (name == "ntl") return ButterflyKind::ntl;
  if (name == "harvey") return ButterflyKind::harvey;
  if (name == "scott") return ButterflyKind::scott;
  if (name == "improved") return ButterflyKind::improved;
  if (name == "smont") return ButterflyKind::smont;
  throw contract_violation("unknown butterfly kind \"" + std::string(name) +
                           "\" (ntl, harvey, scott, improved)");
}

[[nodiscard]] inline std::vector<ButterflyKind> all_butterfly_kinds() {
  return {ButterflyKind::ntl, ButterflyKind::harvey, ButterflyKind::scott,
          ButterflyKind::improved};
}

namespace detail {
inline void check(int status) {
  if (status == NTTK_OK) return;
  const std::string msg = nttk_last_error();
  if (status == NTTK_CONTRACT) throw contract_violation(msg);
  throw device_error(msg);
}
struct HandleDeleter {
  void operator()(nttk_params_s* h) const { nttk_params_destroy(h); }
};
}  // namespace detail

struct BuildOptions {
  Tree tree = Tree::cyclic;
  uint32_t layers = 0;     // 0 = log2 N
  uint64_t root = 0;       // 0 = smallest root of the required order
  bool exact_bound = false;  // admit `improved` under Prop. 4's exact bound
};

// ---- reductions (reduction.hpp:44-291), executed on the GPU ------------------------
// Same names, arguments, results and contract messages as the reference; every call runs
// the device kernel (reduce.cu).  The scalar overloads are for drop-in compatibility; the
// std::vector overloads amortise the launch over many operands.

struct ReductionContext {  // reduction.hpp:44-78
  uint32_t p = 0;
  unsigned n_bits = 0, alpha = 0, ell = 0;
  uint64_t beta = 0, beta_mask = 0, r2n_mask = 0;
  uint64_t p_inv_beta = 0, neg_p_inv_beta = 0, mu = 0;
  int64_t mu_centered = 0;
  uint64_t beta_mod_p = 0, r2n_mod_p = 0;

  [[nodiscard]] unsigned two_n() const { return 2 * n_bits; }
  [[nodiscard]] bool fits_plantard_bound() const {
    const unsigned __int128 lhs = (unsigned __int128)5 * p * p;
    const unsigned __int128 d = ((unsigned __int128)1 << (n_bits + 1)) - p;
    return lhs < d * d;
  }
  [[nodiscard]] bool fits_signed_plantard_bound() const {
    return alpha + 1 < n_bits && (unsigned __int128)p < ((unsigned __int128)1 << (n_bits - alpha - 1));
  }
  [[nodiscard]] bool fits_lazy_plantard_bound() const {
    return ell + 2 < n_bits && (unsigned __int128)p < ((unsigned __int128)1 << (n_bits - ell - 2));
  }
  [[nodiscard]] bool fits_signed_montgomery_bound() const {
    return (unsigned __int128)2 * p < ((unsigned __int128)1 << n_bits);
  }
  [[nodiscard]] nttk_reduction_ctx raw() const {
    nttk_reduction_ctx c{};
    c.p = p;
    c.n_bits = n_bits;
    c.alpha = alpha;
    c.ell = ell;
    c.beta = beta;
    c.beta_mask = beta_mask;
    c.r2n_mask = r2n_mask;
    c.p_inv_beta = p_inv_beta;
    c.neg_p_inv_beta = neg_p_inv_beta;
    c.mu = mu;
    c.mu_centered = mu_centered;
    c.beta_mod_p = beta_mod_p;
    c.r2n_mod_p = r2n_mod_p;
    return c;
  }
};

[[nodiscard]] inline ReductionContext make_reduction_context(uint64_t p, unsigned n_bits,
                                                             unsigned alpha = 0, unsigned ell = 0) {
  nttk_reduction_ctx c{};
  detail::check(nttk_make_reduction_context(p, n_bits, alpha, ell, &c));
  ReductionContext r;
  r.p = static_cast<uint32_t>(c.p);
  r.n_bits = c.n_bits;
  r.alpha = c.alpha;
  r.ell = c.ell;
  r.beta = c.beta;
  r.beta_mask = c.beta_mask;
  r.r2n_mask = c.r2n_mask;
  r.p_inv_beta = c.p_inv_beta;
  r.neg_p_inv_beta = c.neg_p_inv_beta;
  r.mu = c.mu;
  r.mu_centered = c.mu_centered;
  r.beta_mod_p = c.beta_mod_p;
  r.r2n_mod_p = c.r2n_mod_p;
  return r;
}

namespace detail {
template <class Out, class In>
inline std::vector<Out> reduce(int op, const ReductionContext& ctx, const std::vector<In>& x,
                               const std::vector<In>* y = nullptr) {
  if (y && y->size() != x.size()) throw contract_violation("reduce: operand lengths differ");
  const nttk_reduction_ctx c = ctx.raw();
  std::vector<int64_t> out(x.size());
  check(nttk_reduce_host(op, &c, reinterpret_cast<const int64_t*>(x.data()),
                         y ? reinterpret_cast<const int64_t*>(y->data()) : nullptr, out.data(),
                         x.size()));
  return std::vector<Out>(out.begin(), out.end());
}
}  // namespace detail

[[nodiscard]] inline std::vector<uint64_t> mont_redc(const std::vector<uint64_t>& T,
                                                     const ReductionContext& ctx) {
  return detail::reduce<uint64_t>(NTTK_OP_MONT_REDC, ctx, T);
}
[[nodiscard]] inline std::vector<int64_t> signed_mont_redc(const std::vector<int64_t>& A,
                                                           const ReductionContext& ctx) {
  return detail::reduce<int64_t>(NTTK_OP_SIGNED_MONT_REDC, ctx, A);
}
[[nodiscard]] inline std::vector<uint64_t> plantard_redc(const std::vector<uint64_t>& W,
                                                         const std::vector<uint64_t>& T,
                                                         const ReductionContext& ctx) {
  return detail::reduce<uint64_t>(NTTK_OP_PLANTARD_REDC, ctx, W, &T);
}
[[nodiscard]] inline std::vector<uint64_t> modified_plantard_mul(const std::vector<uint64_t>& W,
                                                                 const std::vector<uint64_t>& T,
                                                                 const ReductionContext& ctx) {
  return detail::reduce<uint64_t>(NTTK_OP_MODIFIED_PLANTARD_MUL, ctx, W, &T);
}
[[nodiscard]] inline std::vector<uint64_t> to_plantard_domain(const std::vector<uint64_t>& w,
                                                              const ReductionContext& ctx) {
  return detail::reduce<uint64_t>(NTTK_OP_TO_PLANTARD_DOMAIN, ctx, w);
}
[[nodiscard]] inline std::vector<uint64_t> to_montgomery_domain(const std::vector<uint64_t>& w,
                                                                const ReductionContext& ctx) {
  return detail::reduce<uint64_t>(NTTK_OP_TO_MONTGOMERY_DOMAIN, ctx, w);
}

// reduction.hpp:172-175 returns the std::atomic<uint64_t>& the corner bumps; here the count
// lives in the engine (device-counted, nttk_plantard_correction_fires), so the drop-in hands
// back a view with the atomic's read API: plantard_correction_fires().load() as in
// verify.hpp:132,156.
struct PlantardFiresView {
  [[nodiscard]] uint64_t load() const { return nttk_plantard_correction_fires(); }
  operator uint64_t() const { return load(); }
};
[[nodiscard]] inline PlantardFiresView plantard_correction_fires() { return {}; }

// scalar signatures of reduction.hpp
[[nodiscard]] inline uint64_t mont_redc(uint64_t T, const ReductionContext& ctx) {
  return mont_redc(std::vector<uint64_t>{T}, ctx)[0];
}
[[nodiscard]] inline int64_t signed_mont_redc(int64_t A, const ReductionContext& ctx) {
  return signed_mont_redc(std::vector<int64_t>{A}, ctx)[0];
}
[[nodiscard]] inline uint64_t plantard_redc(uint64_t W, uint64_t T, const ReductionContext& ctx) {
  return plantard_redc(std::vector<uint64_t>{W}, std::vector<uint64_t>{T}, ctx)[0];
}
[[nodiscard]] inline uint64_t modified_plantard_mul(uint64_t W, uint64_t T,
                                                    const ReductionContext& ctx) {
  return modified_plantard_mul(std::vector<uint64_t>{W}, std::vector<uint64_t>{T}, ctx)[0];
}
[[nodiscard]] inline uint64_t to_plantard_domain(uint64_t w, const ReductionContext& ctx) {
  return to_plantard_domain(std::vector<uint64_t>{w}, ctx)[0];
}
[[nodiscard]] inline uint64_t to_montgomery_domain(uint64_t w, const ReductionContext& ctx) {
  return to_montgomery_domain(std::vector<uint64_t>{w}, ctx)[0];
}

// ---- butterfly.hpp checked entry points, executed on the GPU ------------------------

struct ButterflyOut {  // butterfly.hpp:52-55
  uint64_t x = 0;
  uint64_t y = 0;
  bool operator==(const ButterflyOut& o) const { return x == o.x && y == o.y; }
};

struct ScottConfig {  // butterfly.hpp:151-155 (the guard hook is not carried to the device)
  uint32_t transform_size = 0;  // N
  uint32_t lazy_level = 0;      // L
};

// butterfly.hpp:157-168: smallest power-of-two L with 4 N p < 2^n L
[[nodiscard]] inline ScottConfig make_scott_config(uint32_t N, const ReductionContext& ctx) {
  if (N == 0 || (N & (N - 1))) throw contract_violation("scott config: N must be a power of two");
  for (uint32_t L = 1; L <= N; L *= 2)
    if ((unsigned __int128)4 * N * ctx.p < (unsigned __int128)ctx.beta * L) return ScottConfig{N, L};
  throw contract_violation("scott config: no lazy level satisfies 4*N*p/L < 2^n for p=" +
                           std::to_string(ctx.p));
}

namespace detail {
inline std::vector<ButterflyOut> butterflies(int op, const ReductionContext& ctx, uint32_t a0,
                                             uint32_t a1, const std::vector<uint64_t>& X,
                                             const std::vector<uint64_t>& Y,
                                             const std::vector<uint64_t>& W,
                                             const std::vector<uint64_t>* Wq = nullptr) {
  const size_t n = X.size();
  if (Y.size() != n || W.size() != n || (Wq && Wq->size() != n))
    throw contract_violation("butterfly: operand lengths differ");
  const nttk_reduction_ctx c = ctx.raw();
  std::vector<int64_t> xo(n), yo(n);
  check(nttk_butterfly_host(op, &c, a0, a1, reinterpret_cast<const int64_t*>(X.data()),
                            reinterpret_cast<const int64_t*>(Y.data()),
                            reinterpret_cast<const int64_t*>(W.data()),
                            Wq ? reinterpret_cast<const int64_t*>(Wq->data()) : nullptr, xo.data(),
                            yo.data(), n));
  std::vector<ButterflyOut> out(n);
  for (size_t i = 0; i < n; ++i)
    out[i] = {static_cast<uint64_t>(xo[i]), static_cast<uint64_t>(yo[i])};
  return out;
}
}  // namespace detail

// batched forms (one launch)
[[nodiscard]] inline std::vector<ButterflyOut> ntl_butterfly(
    const std::vector<uint64_t>& X, const std::vector<uint64_t>& Y, const std::vector<uint64_t>& W,
    const std::vector<uint64_t>& W_quot, const ReductionContext& ctx) {
  return detail::butterflies(NTTK_BF_NTL, ctx, 0, 0, X, Y, W, &W_quot);
}
[[nodiscard]] inline std::vector<ButterflyOut> harvey_butterfly(const std::vector<uint64_t>& X,
                                                                const std::vector<uint64_t>& Y,
                                                                const std::vector<uint64_t>& W_mont,
                                                                const ReductionContext& ctx) {
  return detail::butterflies(NTTK_BF_HARVEY, ctx, 0, 0, X, Y, W_mont);
}
[[nodiscard]] inline std::vector<ButterflyOut> scott_butterfly(
    const std::vector<uint64_t>& X, const std::vector<uint64_t>& Y,
    const std::vector<uint64_t>& W_mont, const ReductionContext& ctx, const ScottConfig& cfg) {
  return detail::butterflies(NTTK_BF_SCOTT, ctx, cfg.transform_size, cfg.lazy_level, X, Y, W_mont);
}
[[nodiscard]] inline std::vector<ButterflyOut> improved_ct_butterfly(
    const std::vector<uint64_t>& X, const std::vector<uint64_t>& Y,
    const std::vector<uint64_t>& W_hat, const ReductionContext& ctx) {
  return detail::butterflies(NTTK_BF_IMPROVED_CT, ctx, 0, 0, X, Y, W_hat);
}
[[nodiscard]] inline std::vector<ButterflyOut> improved_gs_butterfly(
    const std::vector<uint64_t>& X, const std::vector<uint64_t>& Y,
    const std::vector<uint64_t>& W_hat, const ReductionContext& ctx, unsigned layer) {
  return detail::butterflies(NTTK_BF_IMPROVED_GS, ctx, layer, 0, X, Y, W_hat);
}

// scalar signatures of butterfly.hpp
[[nodiscard]] inline ButterflyOut ntl_butterfly(uint64_t X, uint64_t Y, uint64_t W, uint64_t W_quot,
                                                const ReductionContext& ctx) {
  return ntl_butterfly(std::vector<uint64_t>{X}, {Y}, {W}, {W_quot}, ctx)[0];
}
[[nodiscard]] inline ButterflyOut harvey_butterfly(uint64_t X, uint64_t Y, uint64_t W_mont,
                                                   const ReductionContext& ctx) {
  return harvey_butterfly(std::vector<uint64_t>{X}, {Y}, {W_mont}, ctx)[0];
}
// branch-based twin in the reference (butterfly.hpp:124-142): bit-identical by contract
[[nodiscard]] inline ButterflyOut harvey_butterfly_ref(uint64_t X, uint64_t Y, uint64_t W_mont,
                                                       const ReductionContext& ctx) {
  return harvey_butterfly(X, Y, W_mont, ctx);
}
[[nodiscard]] inline ButterflyOut scott_butterfly(uint64_t X, uint64_t Y, uint64_t W_mont,
                                                  const ReductionContext& ctx, const ScottConfig& cfg) {
  return scott_butterfly(std::vector<uint64_t>{X}, {Y}, {W_mont}, ctx, cfg)[0];
}
[[nodiscard]] inline ButterflyOut improved_ct_butterfly(uint64_t X, uint64_t Y, uint64_t W_hat,
                                                        const ReductionContext& ctx) {
  return improved_ct_butterfly(std::vector<uint64_t>{X}, {Y}, {W_hat}, ctx)[0];
}
[[nodiscard]] inline ButterflyOut improved_gs_butterfly(uint64_t X, uint64_t Y, uint64_t W_hat,
                                                        const ReductionContext& ctx, unsigned layer) {
  return improved_gs_butterfly(std::vector<uint64_t>{X}, {Y}, {W_hat}, ctx, layer)[0];
}

struct NtlTwiddle {  // params.hpp:90-93
  uint64_t w = 0;       // plain twiddle in (0, p)
  uint64_t w_quot = 0;  // floor(w * 2^n / p)
};
struct ForwardTables {  // params.hpp:95-99
  std::vector<NtlTwiddle> dif_ntl;
  std::vector<uint64_t> dif_mont;
  std::vector<uint64_t> ct_plantard;
};
struct InverseTables {  // params.hpp:101-105
  std::vector<NtlTwiddle> gs_ntl;
  std::vector<uint64_t> gs_mont;
  std::vector<uint64_t> gs_plantard;
};

// params.hpp:107-128: the reference bundle (scalars, context, Scott config, host copies of
// the encoded tables) plus the engine handle the calls run on
struct NttParams {
  uint32_t p = 0, size = 0;
  unsigned log2_size = 0, n_bits = 0, layers = 0;
  uint64_t omega = 0, omega_inv = 0, n_inv = 0, n_inv_hat = 0;
  ReductionContext ctx;  // alpha = 0, ell = log2_size
  ScottConfig scott;
  ForwardTables fwd;
  InverseTables inv;
  std::vector<ButterflyKind> kinds;
  std::shared_ptr<nttk_params_s> handle;

  [[nodiscard]] bool has(ButterflyKind k) const {
    for (auto x : kinds)
      if (x == k) return true;
    return false;
  }
  [[nodiscard]] std::vector<uint64_t> table(const char* name) const {
    std::vector<uint64_t> v(nttk_params_table(handle.get(), name, nullptr, 0));
    nttk_params_table(handle.get(), name, v.data(), v.size());
    return v;
  }
};

namespace detail {
inline NttParams wrap(nttk_params_t h) {
  NttParams P;
  P.handle.reset(h, HandleDeleter{});
  nttk_params_info info{};
  check(nttk_params_get_info(h, &info));
  P.p = static_cast<uint32_t>(info.p);
  P.size = info.N;
  P.log2_size = info.log2N;
  P.n_bits = info.n_bits;
  P.layers = info.layers;
  P.omega = info.omega;
  P.omega_inv = info.omega_inv;
  P.n_inv = info.n_inv;
  P.n_inv_hat = info.n_inv_hat;
  for (int k = 0; k < 5; ++k)
    if ((info.kinds_mask >> k) & 1u) P.kinds.push_back(static_cast<ButterflyKind>(k));
  if (P.log2_size < P.n_bits) P.ctx = make_reduction_context(P.p, P.n_bits, 0, P.log2_size);
  P.scott = ScottConfig{P.size, info.scott_L};
  const auto w = P.table("dif_w"), wq = P.table("dif_wq"), gw = P.table("gs_plain"),
             gq = P.table("gs_wq");
  for (size_t i = 0; i < w.size() && i < wq.size(); ++i) P.fwd.dif_ntl.push_back({w[i], wq[i]});
  for (size_t i = 0; i < gw.size() && i < gq.size(); ++i) P.inv.gs_ntl.push_back({gw[i], gq[i]});
  P.fwd.dif_mont = P.table("dif_mont");
  P.fwd.ct_plantard = P.table("ct_plantard");
  P.inv.gs_mont = P.table("gs_mont");
  P.inv.gs_plantard = P.table("gs_plantard");
  return P;
}
}  // namespace detail

[[nodiscard]] inline NttParams build_params(uint64_t p, uint32_t N, unsigned n_bits,
                                            std::vector<ButterflyKind> kinds = all_butterfly_kinds(),
                                            const BuildOptions& opt = {}) {
  nttk_params_desc d{};
  d.p = p;
  d.N = N;
  d.n_bits = n_bits;
  for (auto k : kinds) d.kinds_mask |= 1u << static_cast<int>(k);
  d.tree = static_cast<uint32_t>(opt.tree);
  d.layers = opt.layers;
  d.root = opt.root;
  d.flags = opt.exact_bound ? NTTK_EXACT_BOUND : 0;
  nttk_params_t h = nullptr;
  detail::check(nttk_build_params(&d, &h));
  return detail::wrap(h);
}

[[nodiscard]] inline NttParams preset(const std::string& name) {
  nttk_params_t h = nullptr;
  detail::check(nttk_preset(name.c_str(), &h));
  return detail::wrap(h);
}

// ---- batched host-memory calls (polys contiguous, P.size words each) ----------

inline void ntt_forward_batch(const uint64_t* in, uint64_t* out, size_t batch, const NttParams& P,
                              ButterflyKind kind) {
  detail::check(nttk_ntt_forward_host(P.handle.get(), static_cast<int>(kind), in, out, batch, 8));
}
inline void intt_inverse_batch(const uint64_t* in, uint64_t* out, size_t batch, const NttParams& P,
                               ButterflyKind kind) {
  detail::check(nttk_intt_inverse_host(P.handle.get(), static_cast<int>(kind), in, out, batch, 8));
}

// ---- reference-shaped single-polynomial calls ------------------------------------

[[nodiscard]] inline Spectrum ntt_forward(const Polynomial& f, const NttParams& P,
                                          ButterflyKind kind) {
  if (!P.has(kind)) throw contract_violation("ntt_forward: kind not built into these params");
  if (f.size() != P.size) throw contract_violation("ntt_forward: wrong input length");
  Spectrum s{std::vector<uint64_t>(P.size), Ordering::bit_reversed};
  ntt_forward_batch(f.data(), s.values.data(), 1, P, kind);
  return s;
}

inline void ntt_forward_inplace(std::vector<uint64_t>& a, const NttParams& P, ButterflyKind kind) {
  ntt_forward_batch(a.data(), a.data(), a.size() / P.size, P, kind);
}

[[nodiscard]] inline Polynomial intt_inverse(const Spectrum& s, const NttParams& P,
                                             ButterflyKind kind) {
  if (!P.has(kind)) throw contract_violation("intt_inverse: kind not built into these params");
  if (s.values.size() != P.size) throw contract_violation("intt_inverse: wrong input length");
  if (s.ordering != Ordering::bit_reversed)
    throw contract_violation("intt_inverse: spectrum must be in butterfly order");
  Polynomial f(P.size);
  intt_inverse_batch(s.values.data(), f.data(), 1, P, kind);
  return f;
}

[[nodiscard]] inline Spectrum pointwise_multiply(const Spectrum& lhs, const Spectrum& rhs,
                                                 const NttParams& P, ButterflyKind kind) {
  if (lhs.values.size() != P.size || rhs.values.size() != P.size)
    throw contract_violation("pointwise_multiply: wrong spectrum length");
  if (lhs.ordering != rhs.ordering)
    throw contract_violation("pointwise_multiply: mixed orderings");
  Spectrum out{std::vector<uint64_t>(P.size), lhs.ordering};
  detail::check(nttk_pointwise_multiply_host(P.handle.get(), static_cast<int>(kind),
                                             lhs.values.data(), rhs.values.data(),
                                             out.values.data(), 1, 8));
  return out;
}

[[nodiscard]] inline Polynomial cyclic_convolution_via_ntt(
    const Polynomial& x, const Polynomial& y, const NttParams& P,
    ButterflyKind kind = ButterflyKind::improved) {
  if (x.size() != P.size || y.size() != P.size)
    throw contract_violation("ntt_forward: wrong input length");
  Polynomial out(P.size);
  detail::check(nttk_polymul_host(P.handle.get(), static_cast<int>(kind), x.data(), y.data(),
                                  out.data(), 1, 8));
  return out;
}

// ---- observed transforms (transform.hpp:207-217, 233-337) -------------------------
using LayerObserver = std::function<void(unsigned layer, const std::vector<uint64_t>& state)>;

namespace detail {
struct ObserverCtx {
  const LayerObserver* fn;
  std::exception_ptr error;
};
inline void observer_trampoline(unsigned layer, const uint64_t* state, size_t n, void* user) {
  auto* c = static_cast<ObserverCtx*>(user);
  if (c->error || !*c->fn) return;
  try {
    (*c->fn)(layer, std::vector<uint64_t>(state, state + n));
  } catch (...) {  // never unwind through the C ABI: rethrown after the call returns
    c->error = std::current_exception();
  }
}
}  // namespace detail

[[nodiscard]] inline Spectrum ntt_forward_observed(const Polynomial& f, const NttParams& P,
                                                   ButterflyKind kind, const LayerObserver& observer) {
  if (!P.has(kind)) throw contract_violation("ntt_forward: kind not built into these params");
  if (f.size() != P.size) throw contract_violation("ntt_forward: wrong input length");
  Spectrum s{std::vector<uint64_t>(P.size), Ordering::bit_reversed};
  detail::ObserverCtx c{&observer, nullptr};
  const int st = nttk_ntt_forward_observed(P.handle.get(), static_cast<int>(kind), f.data(),
                                           s.values.data(), detail::observer_trampoline, &c);
  if (c.error) std::rethrow_exception(c.error);
  detail::check(st);
  return s;
}

[[nodiscard]] inline Polynomial intt_inverse_observed(const Spectrum& s, const NttParams& P,
                                                      ButterflyKind kind,
                                                      const LayerObserver& observer) {
  if (!P.has(kind)) throw contract_violation("intt_inverse: kind not built into these params");
  if (s.values.size() != P.size) throw contract_violation("intt_inverse: wrong input length");
  if (s.ordering != Ordering::bit_reversed)
    throw contract_violation("intt_inverse: spectrum must be in butterfly order");
  Polynomial f(P.size);
  detail::ObserverCtx c{&observer, nullptr};
  const int st = nttk_intt_inverse_observed(P.handle.get(), static_cast<int>(kind), s.values.data(),
                                            f.data(), detail::observer_trampoline, &c);
  if (c.error) std::rethrow_exception(c.error);
  detail::check(st);
  return f;
}

// ---- device-pointer batched calls (asynchronous on `stream`) ----------------------

inline void ntt_forward_device(const NttParams& P, ButterflyKind kind, const void* d_in, void* d_out,
                               size_t batch, int elem_bytes, void* stream = nullptr) {
  detail::check(nttk_ntt_forward(P.handle.get(), static_cast<int>(kind), d_in, d_out, batch,
                                 elem_bytes, stream));
}
inline void intt_inverse_device(const NttParams& P, ButterflyKind kind, const void* d_in,
                                void* d_out, size_t batch, int elem_bytes, void* stream = nullptr) {
  detail::check(nttk_intt_inverse(P.handle.get(), static_cast<int>(kind), d_in, d_out, batch,
                                  elem_bytes, stream));
}

// ---- transform.hpp / params.hpp helpers ----------------------------------------------

// transform.hpp:61-70
[[nodiscard]] inline uint64_t spectrum_value_bound(const NttParams& P, ButterflyKind kind) {
  switch (kind) {
    case ButterflyKind::ntl: return P.p;
    case ButterflyKind::harvey: return uint64_t(2) * P.p;
    case ButterflyKind::scott: return uint64_t(P.size) * P.p;
    case ButterflyKind::improved: return uint64_t(P.log2_size + 1) * P.p;
    case ButterflyKind::smont: return uint64_t(P.log2_size + 2) * P.p;  // |value| bound
  }
  return 0;
}

// transform.hpp:38-40: v[i] mod p, on the device
inline void canonicalize(std::vector<uint64_t>& v, uint64_t p) {
  if (v.empty()) return;
  nttk_reduction_ctx c{};
  c.p = p;  // the mod-p op reads only p
  c.n_bits = 32;
  detail::check(nttk_reduce_host(NTTK_OP_MOD_P, &c, reinterpret_cast<const int64_t*>(v.data()),
                                 nullptr, reinterpret_cast<int64_t*>(v.data()), v.size()));
}

// transform.hpp:42-59: index permutations (data layout, no arithmetic)
[[nodiscard]] inline std::vector<uint64_t> bit_reverse_permutation(const std::vector<uint64_t>& v) {
  if (v.empty() || (v.size() & (v.size() - 1)))
    throw contract_violation("bit_reverse_permutation: size must be a power of two");
  unsigned bits = 0;
  while ((size_t(1) << bits) < v.size()) ++bits;
  std::vector<uint64_t> out(v.size());
  for (size_t i = 0; i < v.size(); ++i) {
    size_t r = 0;
    for (unsigned b = 0; b < bits; ++b) r |= ((i >> b) & 1u) << (bits - 1 - b);
    out[r] = v[i];
  }
  return out;
}
[[nodiscard]] inline std::vector<uint64_t> to_natural_order(const Spectrum& s) {
  return s.ordering == Ordering::natural ? s.values : bit_reverse_permutation(s.values);
}

// params.hpp:273-301 (the preset table the engine builds from)
struct PresetSpec {
  const char* name;
  uint32_t p;
  uint32_t size;
  unsigned n_bits;
};
[[nodiscard]] inline const std::vector<PresetSpec>& preset_table() {
  static const std::vector<PresetSpec> table = {
      {"kyber256", 7681, 256, 32},     {"kcl256", 7681, 256, 32},
      {"newhope512", 12289, 512, 32},  {"falcon512", 12289, 512, 32},
      {"remblem512", 12289, 512, 32},  {"newhope1024", 12289, 1024, 32},
      {"falcon1024", 12289, 1024, 32}, {"hila5-1024", 12289, 1024, 32},
      {"toy13", 13, 4, 8},
  };
  return table;
}
[[nodiscard]] inline const PresetSpec& preset_spec(const std::string& name) {
  for (const auto& s : preset_table())
    if (name == s.name) return s;
  (void)preset(name);  // throws the engine's "unknown preset ... (known: ...)" message
  throw contract_violation("unknown preset '" + name + "'");
}

// params.hpp:30-88: root search and the plain twiddle schedules (host parameter precompute,
// the same arithmetic build_params runs; exposed for callers that build their own tables)
namespace detail {
inline uint64_t pow_mod(uint64_t b, uint64_t e, uint64_t m) {
  unsigned __int128 acc = 1 % m, x = b % m;
  for (; e; e >>= 1) {
    if (e & 1) acc = acc * x % m;
    x = x * x % m;
  }
  return static_cast<uint64_t>(acc);
}
inline uint64_t bitrev(uint64_t i, unsigned bits) {
  uint64_t r = 0;
  for (unsigned b = 0; b < bits; ++b) r |= ((i >> b) & 1u) << (bits - 1 - b);
  return r;
}
}  // namespace detail
[[nodiscard]] inline uint64_t find_primitive_root(uint64_t p, uint32_t N) {
  if (N == 0 || (N & (N - 1))) throw contract_violation("find_primitive_root: N must be a power of two");
  if ((p - 1) % N) throw contract_violation("find_primitive_root: N must divide p - 1");
  if (N == 1) return 1;
  for (uint64_t w = 2; w < p; ++w)
    if (detail::pow_mod(w, N, p) == 1 && detail::pow_mod(w, N / 2, p) != 1) return w;
  throw contract_violation("find_primitive_root: no root found");
}
[[nodiscard]] inline std::vector<uint64_t> dif_forward_plain_twiddles(uint32_t N, uint64_t omega,
                                                                      uint64_t p) {
  std::vector<uint64_t> out;
  for (uint64_t len = N / 2; len >= 1; len /= 2)
    for (uint64_t j = 0; j < len; ++j) out.push_back(detail::pow_mod(omega, j * (N / (2 * len)), p));
  return out;
}
[[nodiscard]] inline std::vector<uint64_t> ct_forward_plain_twiddles(uint32_t N, uint64_t omega,
                                                                     uint64_t p) {
  std::vector<uint64_t> out;
  unsigned L = 0;
  while ((uint64_t(1) << L) < N) ++L;
  for (unsigned s = 1; s <= L; ++s)
    for (uint64_t b = 0; b < (uint64_t(1) << (s - 1)); ++b)
      out.push_back(detail::pow_mod(omega, (uint64_t(N) >> s) * detail::bitrev(b, s - 1), p));
  return out;
}
[[nodiscard]] inline std::vector<uint64_t> gs_inverse_plain_twiddles(uint32_t N, uint64_t omega,
                                                                     uint64_t p) {
  const uint64_t inv = detail::pow_mod(omega, N - 1, p);  // omega^{-1}
  std::vector<uint64_t> out;
  unsigned L = 0;
  while ((uint64_t(1) << L) < N) ++L;
  for (unsigned s = L; s >= 1; --s)
    for (uint64_t b = 0; b < (uint64_t(1) << (s - 1)); ++b)
      out.push_back(detail::pow_mod(inv, (uint64_t(N) >> s) * detail::bitrev(b, s - 1), p));
  return out;
}

}  // namespace nttk
