/*
 * nttk_oracle.h -- CPU restatement of the reference NTT path (TEST INFRASTRUCTURE ONLY).
 *
 * This library is the parity checker for the B200 engine.  It is imported only by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs.
 * The product (paper_2402_00675_b200/, libnttk_gpu.so) never links or calls it.
 *
 * Every function restates an algorithm of the reference header-only library `nttk`
 * (/root/reference/proj/include/nttk/ headers) in plain C with exact 64/128-bit integer
 * arithmetic; each definition cites the reference file:line it follows.  Parity of
 * this restatement is pinned in tests/test_oracle.py against (a) the known-answer
 * values of the reference's own GoogleTest suites and (b) golden vectors produced by
 * running the unmodified reference code (oracle/_ref, tests/golden/make_golden.py).
 *
 * Extension paths that have no reference implementation (negacyclic / incomplete
 * trees, degree-2 basemul, signed-Montgomery and Montgomery-CT butterflies) are
 * restated from SURVEY.md §8(a) row a22 and validated against naive evaluation
 * (or_naive_nega_eval / or_schoolbook_negacyclic): "parity unpinned" by any
 * reference test for those rows.
 */
#ifndef NTTK_ORACLE_H
#define NTTK_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror the reference CLI contract (ntt_kernel_cli.cpp:17-18) */
enum { OR_OK = 0, OR_PROPERTY = 1, OR_CONTRACT = 2 };

/* butterfly kinds: the reference enum (butterfly.hpp:30) plus two extension kinds */
enum { OR_NTL = 0, OR_HARVEY = 1, OR_SCOTT = 2, OR_IMPROVED = 3, OR_SMONT = 4 };

/* transform trees: the reference cyclic tree plus the extension negacyclic tree */
enum { OR_TREE_CYCLIC = 0, OR_TREE_NEGA = 1 };

const char* or_last_error(void);

/* ---------------- integer plumbing (int_util.hpp, crt.hpp) ---------------- */
uint64_t or_pow_mod(uint64_t b, uint64_t e, uint64_t m);
uint64_t or_bit_reverse(uint64_t x, unsigned bits);
int or_is_prime(uint64_t x);
/* inverse of a mod m (m <= 2^64 passed as log2 when m is a power of two > 2^63) */
int or_mod_inverse_u64(uint64_t a, uint64_t m, uint64_t* out);

/* reference Rng (xoshiro256** seeded by splitmix64), int_util.hpp:90-138 */
typedef struct { uint64_t s[4]; } or_rng;
void or_rng_seed(or_rng* r, uint64_t seed);
uint64_t or_rng_next(or_rng* r);
uint64_t or_rng_below(or_rng* r, uint64_t bound);
/* convenience: count values of Rng(seed).below(bound) */
void or_rng_fill(uint64_t seed, uint64_t bound, uint64_t* out, size_t count);

/* ---------------- reductions (reduction.hpp) ---------------- */
typedef struct {
  uint32_t p;
  unsigned n_bits, alpha, ell;
  uint64_t beta, beta_mask, r2n_mask;
  uint64_t p_inv_beta, neg_p_inv_beta, mu;
  int64_t mu_centered;
  uint64_t beta_mod_p, r2n_mod_p;
} or_ctx;

int or_make_ctx(uint64_t p, unsigned n_bits, unsigned alpha, unsigned ell, or_ctx* out);
int or_ctx_fits_plantard(const or_ctx* c);
int or_ctx_fits_lazy_plantard(const or_ctx* c);
int or_ctx_fits_signed_montgomery(const or_ctx* c);

int or_mont_redc(uint64_t T, const or_ctx* c, uint64_t* out);
int or_signed_mont_redc(int64_t A, const or_ctx* c, int64_t* out);
int or_plantard_redc(uint64_t W, uint64_t T, const or_ctx* c, uint64_t* out);
uint64_t or_plantard_fires(void);
uint64_t or_modified_plantard_core(uint64_t w, uint64_t t, uint64_t mu, uint64_t p,
                                   unsigned n_bits, uint64_t r2n_mask);
int or_modified_plantard_mul(uint64_t W, uint64_t T, const or_ctx* c, uint64_t* out);
int or_to_plantard_domain(uint64_t w, const or_ctx* c, uint64_t* out);
int or_to_montgomery_domain(uint64_t w, const or_ctx* c, uint64_t* out);
/* extension: centered Montgomery twiddle, w*2^n mod p mapped to (-p/2, p/2] */
int64_t or_to_signed_montgomery_domain(uint64_t w, const or_ctx* c);
/* extension: signed Barrett used by the signed-Montgomery inverse */
int64_t or_signed_barrett(int64_t a, const or_ctx* c);

/* ---------------- butterflies (butterfly.hpp) ---------------- */
void or_ntl_core(uint64_t X, uint64_t Y, uint64_t W, uint64_t Wq, const or_ctx* c,
                 uint64_t* x1, uint64_t* y1);
void or_harvey_core(uint64_t X, uint64_t Y, uint64_t Wm, const or_ctx* c,
                    uint64_t* x1, uint64_t* y1);
void or_scott_core(uint64_t X, uint64_t Y, uint64_t Wm, uint64_t offset,
                   const or_ctx* c, uint64_t* x1, uint64_t* y1);
void or_improved_ct_core(uint64_t X, uint64_t Y, uint64_t What, const or_ctx* c,
                         uint64_t* x1, uint64_t* y1);
void or_improved_gs_core(uint64_t X, uint64_t Y, uint64_t offset, uint64_t What,
                         const or_ctx* c, uint64_t* x1, uint64_t* y1);
/* extension CT-form butterflies (negacyclic tree / ext kinds) */
void or_harvey_ct_core(uint64_t X, uint64_t Y, uint64_t Wm, const or_ctx* c,
                       uint64_t* x1, uint64_t* y1);
void or_smont_ct_core(int64_t X, int64_t Y, int64_t Ws, const or_ctx* c,
                      int64_t* x1, int64_t* y1);
void or_smont_gs_core(int64_t X, int64_t Y, int64_t Ws, const or_ctx* c,
                      int64_t* x1, int64_t* y1);
/* smallest power-of-two lazy level (butterfly.hpp:157-168); 0 when none exists */
uint32_t or_scott_lazy_level(uint32_t N, const or_ctx* c);

/* ---------------- params (params.hpp) ---------------- */
uint64_t or_find_primitive_root(uint64_t p, uint64_t order);

typedef struct {
  uint32_t p, N, log2N, n_bits, tree, layers;
  uint32_t kinds_mask;          /* bit k set = kind k built */
  uint32_t scott_L;             /* scott lazy level (0 = not built) */
  uint64_t omega, omega_inv;    /* cyclic: order-N root; nega: order-2^{layers+1} root */
  uint64_t n_inv;               /* cyclic: N^{-1}; nega: 2^{-layers} */
  uint64_t n_inv_hat;           /* n_inv in the Plantard encoding (improved only) */
  uint64_t n_inv_mont;          /* n_inv * 2^n mod p (harvey/scott/ext)      */
  int64_t n_inv_smont;          /* centered n_inv * 2^n mod p (smont)         */
  or_ctx ctx;
  /* forward tables, all of length T = number of butterflies groups (see below) */
  size_t fwd_len, inv_len;
  uint64_t *dif_w, *dif_wq, *dif_mont;      /* per-index DIF (cyclic, ntl/harvey/scott) */
  uint64_t *ct_plain, *ct_plantard, *ct_mont;/* per-block CT (improved + ext)           */
  int64_t *ct_smont;
  uint64_t *gs_plain, *gs_w, *gs_wq, *gs_mont, *gs_plantard; /* per-block GS inverse */
  int64_t *gs_smont;
} or_params;

/* Builds params.  tree=OR_TREE_CYCLIC with layers=log2 N is the reference path
 * (build_params, params.hpp:137-268).  exact_bound=1 replaces the paper's
 * p < 2^{n-ell-2} check for `improved` by the exact Prop. 4 requirement
 * (SURVEY §0 item 3); root=0 picks the smallest root like find_primitive_root. */
int or_params_build(uint64_t p, uint32_t N, unsigned n_bits, uint32_t kinds_mask,
                    uint32_t tree, uint32_t layers, uint64_t root, int exact_bound,
                    or_params** out);
void or_params_free(or_params* P);
size_t or_params_table(const or_params* P, const char* name, uint64_t* out, size_t cap);

/* ---------------- transforms (transform.hpp) ---------------- */
/* in-place on `batch` contiguous polys of length N stored as u64 (signed kinds
 * store two's complement int64 in the same words) */
int or_forward(const or_params* P, int kind, uint64_t* a, size_t batch);
int or_inverse(const or_params* P, int kind, uint64_t* a, size_t batch);
int or_pointwise(const or_params* P, int kind, const uint64_t* lhs, const uint64_t* rhs,
                 uint64_t* out, size_t batch);
/* degree-2 basemul for trees whose last layer leaves len=2 blocks (Kyber-style) */
int or_basemul(const or_params* P, int kind, const uint64_t* lhs, const uint64_t* rhs,
               uint64_t* out, size_t batch);
/* product via NTT: fwd(a), fwd(b), pointwise/basemul, inverse */
int or_polymul(const or_params* P, int kind, const uint64_t* a, const uint64_t* b,
               uint64_t* out, size_t batch);

/* ---------------- oracle.hpp ---------------- */
void or_naive_dft(const uint64_t* f, size_t N, uint64_t omega, uint64_t p, uint64_t* out);
void or_schoolbook_cyclic(const uint64_t* a, const uint64_t* b, size_t N, uint64_t p,
                          uint64_t* out);
void or_schoolbook_negacyclic(const uint64_t* a, const uint64_t* b, size_t N, uint64_t p,
                              uint64_t* out);
/* naive evaluation of the negacyclic/incomplete tree: out in butterfly (bit-reversed) order */
int or_naive_nega_eval(const or_params* P, const uint64_t* f, uint64_t* out);

/* ---------------- reduction sweep (config 5) ---------------- */
enum { OR_SW_MONT = 0, OR_SW_SMONT = 1, OR_SW_PLANTARD = 2, OR_SW_MPLANTARD = 3 };
/* operand grid: pair (i, j) = (A[i], B[j]); results row-major r[i*nb + j] (may be NULL);
 * returns the wrapping u64 sum of results (signed results as two's complement) */
int or_sweep(int variant, const or_ctx* c, const int64_t* A, size_t na, const int64_t* B,
             size_t nb, int64_t* r, uint64_t* checksum, int threads);

/* ---------------- hashing helper for golden vectors ---------------- */
uint64_t or_fnv1a_u32(const uint64_t* v, size_t n);

#ifdef __cplusplus
}
#endif
#endif
