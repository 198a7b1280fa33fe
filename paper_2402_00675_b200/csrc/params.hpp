// params.hpp -- host-side parameter bundle of the B200 engine (internal).
//
// B200 counterpart of the reference's NttParams / build_params
// (proj/include/nttk/params.hpp:107-268) and ReductionContext
// (reduction.hpp:44-117).  Everything here is exact host integer precompute done once
// per parameter set; the compute runs in the CUDA kernels of fast256.cu / generic.cu.
// On top of the reference's encoded tables, the bundle carries the device-ready forms:
//   * mu-premultiplied Plantard twiddles  w_hat * mu mod 2^{2n}  (the product
//     (w_hat * t) * mu mod 2^{2n} of reduction.hpp:256 is associative mod 2^{2n}, so
//     premultiplying is bit-exact and saves one multiply per butterfly);
//   * per-device copies of every table for the generic kernel (uploaded lazily).
#pragma once

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/nttk_gpu.h"

namespace nttk_b200 {

using u128 = unsigned __int128;
using i128 = __int128;

// reduction.hpp:44-78
struct Ctx {
  uint32_t p = 0;
  unsigned n_bits = 0, ell = 0;
  uint64_t beta = 0, beta_mask = 0, r2n_mask = 0;
  uint64_t p_inv_beta = 0, neg_p_inv_beta = 0, mu = 0;
  uint64_t beta_mod_p = 0, r2n_mod_p = 0;
};

// Device copies of the tables used by the generic kernel (u64, reference order).
struct DeviceTables {
  uint64_t* base = nullptr;  // one allocation holding every table below
  const uint64_t *dif_w = nullptr, *dif_wq = nullptr, *dif_mont = nullptr;
  const uint64_t *ct_plantard = nullptr, *ct_mont = nullptr, *ct_smont = nullptr;
  const uint64_t *gs_w = nullptr, *gs_wq = nullptr, *gs_mont = nullptr, *gs_plantard = nullptr,
                 *gs_smont = nullptr;
  const uint64_t* gamma = nullptr;  // basemul moduli (trees ending in degree-2 factors)
};

// Kernel-parameter image of one N=256 transform direction for the fast kernels.
// Passed by value (lives in the constant bank): uniform twiddle reads are free
// operands of IMAD; lane-dependent ones are loaded once per thread at kernel start.
struct FastArgs {
  uint32_t p = 0, two_p = 0;
  uint32_t pinv = 0;       // harvey/smont: p^{-1} mod 2^n (n=16: shifted left by 16); scott: -p^{-1}
  uint32_t canon_m = 0;    // floor((2^32 - 1) / p): inverse-input canonicalisation
  uint32_t canon_m16 = 0;  // ceil(2^32 / p): exact floor(x / p) for x < 2^16
  uint32_t sgn_off = 0;    // K p >= 2^{bits-1}: lifts signed inputs to unsigned
  uint32_t scale_lo = 0, scale_hi = 0;  // inverse final multiplier (per kind encoding)
  uint32_t barrett_v = 0;  // smont signed Barrett constant V (S = n + 10)
  uint32_t layers = 0;
  // --- issue-slot economy (all host-validated, see params.cpp fill_fast) ---
  uint32_t zero = 0;       // always 0: x + y + zero forces a 3-input IADD3 (ALU pipe)
  uint32_t two = 2;        // always 2: 2 X - X' as one IMAD (fmaheavy pipe, f1_bf)
  uint32_t one = 1;        // always 1: X + Y as one IMAD (fmaheavy pipe, narrow_bf)
  uint32_t negp = 0;       // -p mod 2^32 (x - q p as one IMAD)
  uint32_t off[12] = {};   // off[m] = 2^{m-1} p: GS offset of merge depth m (constant operand)
  uint32_t cb_m = 0, cb_s = 0;  // x mod p = x - ((x cb_m) >> cb_s) p, exact for x < 2^17
  uint32_t cs_s = 0;       // x mod p = min(r, r - p), r = x - (x >> cs_s) p, exact for x < 2^32
  uint32_t kp = 0;         // K p >= 2^16 - 1: fused first inverse layer offset (u16 input)
  uint32_t skp[4] = {};    // kp << m: inverse sum-chain offsets without canonicalisation
  uint32_t one_lo = 0;     // Plantard encoding of 1 times mu mod 2^32 (n = 16)
  uint32_t flags = 0;      // bit0: cb valid; bit1: cs valid; bit2: fused first layer valid;
                           // bit3: lazy merge valid (improved n = 16);
                           // bit4: forward block-0 twiddles are 1 (cyclic, improved);
                           // bit5: inverse phase-2 block-0 twiddles are 1 (TW1, L = 8);
                           // bit6: u16 inverse without canonicalisation (DEFER);
                           // bit7: u32 inverse with partial canonicalisation to [0, 2p);
                           // bit10: F1 forward (paper-form products, fwd_body_f1);
                           // bit11: CT-form inverse image (HostParams::fast_ctinv)
  uint32_t fold_lo = 0, fold_hi = 0;  // last merge twiddle times N^{-1}, kind encoding
  uint32_t soff = 0;       // scott: butterfly offset (N/L) p (butterfly.hpp:172-184)
  uint32_t lzk = 0;        // SmontLazy16: K p > every final |r| (lift before mod_cb)
  uint32_t f1_sp = 0, f1_sp1 = 0;  // F1 forward surplus S p and (S + 1) p (fwd_body_f1)
  uint32_t ct_c[8] = {};   // CT-form inverse: (X, Y) offsets of the twiddle-1 butterflies per layer
  uint32_t pm[12] = {};    // pm[m] = m p: offsets of the N = 512 / 1024 CT-form inverse (inv_body_n_ct)
  uint32_t lo[256] = {};   // twiddle words in reference table order
  uint32_t hi[256] = {};   // high words of 64-bit premultiplied Plantard twiddles
};

// Product stage of the fused polymul kernel (slotwise product or degree-2 basemul of two
// forward spectra).  The product is canonical, so any exact method is bit-identical with
// the reference's pointwise_multiply (transform.hpp:349-370); each kind uses its own
// reduction: `enc` turns a runtime operand into that kind's multiplier encoding.
struct ProdArgs {
  uint32_t enc_lo = 0, enc_hi = 0;  // improved: (2^{4n} mod p) mu; harvey: 2^{2n} mod p; smont: centered R^2 + quotient factor
  uint32_t mu_lo = 0, mu_hi = 0;    // improved: p^{-1} mod 2^{2n}
  uint32_t basemul = 0;             // 1: degree-2 leaves (x^2 - gamma), 0: slotwise
  uint32_t lazy = 0;                // 1: the fused polymul may run the kind's lazy twin
                                    // (HarveyLazy16 / SmontLazy16, bounds in params.cpp)
  uint32_t g_lo[128] = {}, g_hi[128] = {};  // gamma per pair, kind encoding (basemul)
};

struct PolymulArgs {
  FastArgs fwd, inv;
  ProdArgs prod;
};

constexpr int kNarrow = 5;  // pseudo-kind index of the narrow improved image
constexpr int kCtN = 6;     // pseudo-kind index of the N = 512 / 1024 CT-form inverse image
// CT-form inverse at N = 512 / 1024 (fastn_tma.cu inv_body_n_ct): every product operand stays
// below kCtLimN p, which must lie inside the n = 16 Prop. 4 range (params.cpp fill_ct_inverse_n)
constexpr int kCtLimN = 20;
// NTTK_INV_CT=0 keeps the GS-form inverses (the A/B of the CT-form ones)
bool ct_inverse_enabled();
// narrow inverse: every GS operand below 2^kNarrowEmax p (tma_common.cuh inv_body_narrow)
constexpr int kNarrowEmax = 4;
// F1 forward at N = 256: surplus multiples of p injected by layer 1 (= L - 2, fwd_body_f1)
constexpr uint32_t kF1Surplus = 6;
// F1 forward of the 7-layer negacyclic tree: surplus L - 2 (tma_common.cuh fwd_body_f1_nega7)
constexpr uint32_t kF1SurplusNega7 = 5;

struct HostParams {
  nttk_params_desc desc{};
  uint32_t p = 0, N = 0, log2N = 0, n_bits = 0, tree = 0, layers = 0, kinds = 0;
  uint32_t scott_L = 0;
  uint64_t omega = 0, omega_inv = 0, n_inv = 0, n_inv_hat = 0, n_inv_mont = 0;
  int64_t n_inv_smont = 0;
  Ctx ctx;
  // tables, reference order (params.hpp:47-88, 226-266)
  std::vector<uint64_t> dif_w, dif_wq, dif_mont;
  std::vector<uint64_t> ct_plain, ct_plantard, ct_mont;
  std::vector<int64_t> ct_smont;
  std::vector<uint64_t> gs_plain, gs_wq, gs_mont, gs_plantard;
  std::vector<int64_t> gs_smont;
  // basemul: pair k of a degree-2-leaf tree is a mod (x^2 - gamma[k])
  std::vector<uint64_t> gamma;
  // fast-path images, indexed [kind][dir] (dir 0 forward, 1 inverse)
  uint32_t fast_mask = 0;
  FastArgs fast[7][2];  // [5] = kNarrow, [6] = kCtN
  ProdArgs prod[5];
  // n = 16 evaluation of an n = 32 improved parameter set (params.cpp fill_narrow): the
  // improved words do not depend on n, so when every operand of a
  // direction lies inside the n = 16 Prop. 4 range the kernels run ImprovedN16 on the
  // image fast[kNarrow][dir] (IMAD + IMAD.HI per product instead of IMAD.HI + IMAD +
  // IMAD.WIDE)
  bool narrow[2] = {};
  // CT-form inverse of the Kyber u16 tree (params.cpp fill_ct_inverse, tma_common.cuh
  // inv_body_ct): DIT butterflies on the bit-reversed spectrum with per-index twiddles
  bool ct_inv = false;
  FastArgs fast_ctinv;
  // the same CT-form inverse for canonicalised (unpacked) input words: u32 storage of an n = 16
  // improved set, or the narrow image of an n = 32 set (the kyber256 preset)
  bool ct_inv_c = false;
  FastArgs fast_ctinv_c;
  // CT-form inverse of the narrow image at N = 512 / 1024 (params.cpp fill_ct_inverse_n)
  bool ct_inv_n = false;
  // fast-image index of (kind, dir): kNarrow where the narrow image applies, kCtN where its
  // inverse runs in CT form
  int image(int kind, int dir) const {
    if (!(kind == NTTK_IMPROVED && n_bits == 32 && narrow[dir])) return kind;
    return dir == 1 && ct_inv_n && ct_inverse_enabled() ? kCtN : kNarrow;
  }
  // N = 512 / 1024 fast kernels: whole per-direction tables, interleaved (lo, hi) words,
  // uploaded once per device on first use
  std::vector<uint32_t> fastn_tab[7][2];
  mutable uint32_t* fastn_dev[64] = {};
  const uint32_t* fastn_table(int device, int kind, int dir, std::string& err) const;

  mutable std::mutex mu_dev;
  mutable DeviceTables dev[64];

  const DeviceTables* device_tables(int device, std::string& err) const;
  ~HostParams();
};

int build_params(const nttk_params_desc& d, HostParams& P, std::string& err);
int preset_desc(const std::string& name, nttk_params_desc& d, std::string& err);

// exact integer helpers shared with the host code
Ctx make_ctx(uint64_t p, unsigned n_bits, unsigned ell);
u128 inverse(u128 a, u128 m);
uint64_t pow_mod(uint64_t b, uint64_t e, uint64_t m);
uint64_t bit_reverse(uint64_t x, unsigned bits);

}  // namespace nttk_b200
