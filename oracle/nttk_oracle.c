/*
 * nttk_oracle.c -- CPU restatement of the reference NTT path (TEST INFRASTRUCTURE ONLY).
 *
 * See nttk_oracle.h for the contract.  Nothing in the product links this file: it is
 * loaded by tests/, __graft_entry__.smoke() and the CPU legs of bench.py as the
 * checker.  All arithmetic is exact (u64 with explicit masks, unsigned __int128 where
 * the reference uses u128), so outputs are the reference's bit for bit; the pinning
 * tests in tests/test_oracle.py prove it against the reference's known answers and
 * against golden vectors produced by the unmodified reference (oracle/_ref).
 */
#include "nttk_oracle.h"

#include <pthread.h>
#include <stdatomic.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
typedef __int128 i128;

static _Thread_local char g_err[512];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* or_last_error(void) { return g_err; }

/* ----------------------------------------------------------------------------
 * integer plumbing -- int_util.hpp:38-86, crt.hpp:37-57
 * ------------------------------------------------------------------------- */

/* square-and-multiply with u128 products (int_util.hpp:47-57) */
uint64_t or_pow_mod(uint64_t b, uint64_t e, uint64_t m) {
  uint64_t acc = 1 % m, base = b % m;
  for (; e; e >>= 1) {
    if (e & 1) acc = (uint64_t)(((u128)acc * base) % m);
    base = (uint64_t)(((u128)base * base) % m);
  }
  return acc;
}

static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) {
  return (uint64_t)(((u128)a * b) % m);
}

/* low `bits` bits reversed (int_util.hpp:72-78) */
uint64_t or_bit_reverse(uint64_t x, unsigned bits) {
  uint64_t r = 0;
  for (unsigned i = 0; i < bits; ++i) r |= ((x >> i) & 1u) << (bits - 1 - i);
  return r;
}

/* trial division (int_util.hpp:80-86) */
int or_is_prime(uint64_t x) {
  if (x < 2) return 0;
  for (uint64_t d = 2; d * d <= x; ++d)
    if (x % d == 0) return 0;
  return 1;
}

static unsigned ilog2(uint64_t x) {
  unsigned r = 0;
  while (x >>= 1) ++r;
  return r;
}

static int is_pow2(uint64_t x) { return x && !(x & (x - 1)); }

/* extended Euclid over i128, positive representative (crt.hpp:37-57) */
static int mod_inverse128(u128 a, u128 m, u128* out) {
  if (m < 2) return fail(OR_CONTRACT, "mod_inverse: modulus must be >= 2");
  a %= m;
  if (a == 0) return fail(OR_CONTRACT, "mod_inverse: inputs share a factor");
  i128 r0 = (i128)m, r1 = (i128)a, t0 = 0, t1 = 1;
  while (r1 != 0) {
    i128 q = r0 / r1, tmp = r0 - q * r1;
    r0 = r1;
    r1 = tmp;
    tmp = t0 - q * t1;
    t0 = t1;
    t1 = tmp;
  }
  if (r0 != 1) return fail(OR_CONTRACT, "mod_inverse: inputs share a factor");
  i128 v = t0 % (i128)m;
  if (v < 0) v += (i128)m;
  *out = (u128)v;
  return OR_OK;
}

int or_mod_inverse_u64(uint64_t a, uint64_t m, uint64_t* out) {
  u128 v;
  int st = mod_inverse128(a, m, &v);
  if (st == OR_OK) *out = (uint64_t)v;
  return st;
}

/* ----------------------------------------------------------------------------
 * Rng -- xoshiro256** seeded through splitmix64 (int_util.hpp:90-138)
 * ------------------------------------------------------------------------- */
static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

void or_rng_seed(or_rng* r, uint64_t seed) {
  uint64_t z = seed;
  for (int i = 0; i < 4; ++i) {
    z += 0x9e3779b97f4a7c15ull;
    uint64_t w = z;
    w = (w ^ (w >> 30)) * 0xbf58476d1ce4e5b9ull;
    w = (w ^ (w >> 27)) * 0x94d049bb133111ebull;
    r->s[i] = w ^ (w >> 31);
  }
}

uint64_t or_rng_next(or_rng* r) {
  uint64_t* s = r->s;
  const uint64_t out = rotl64(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return out;
}

/* masked rejection sampling (int_util.hpp:117-125) */
uint64_t or_rng_below(or_rng* r, uint64_t bound) {
  if (bound <= 1) return 0;
  const unsigned bits = ilog2(bound - 1) + 1;
  const uint64_t mask = bits >= 64 ? ~0ull : ((1ull << bits) - 1);
  for (;;) {
    uint64_t v = or_rng_next(r) & mask;
    if (v < bound) return v;
  }
}

void or_rng_fill(uint64_t seed, uint64_t bound, uint64_t* out, size_t count) {
  or_rng r;
  or_rng_seed(&r, seed);
  for (size_t i = 0; i < count; ++i) out[i] = or_rng_below(&r, bound);
}

/* ----------------------------------------------------------------------------
 * ReductionContext -- reduction.hpp:44-117
 * ------------------------------------------------------------------------- */
int or_make_ctx(uint64_t p, unsigned n_bits, unsigned alpha, unsigned ell, or_ctx* c) {
  if (n_bits < 2 || n_bits > 32)
    return fail(OR_CONTRACT, "reduction context: word size n must be in [2, 32]");
  if (p < 3 || !(p & 1)) return fail(OR_CONTRACT, "reduction context: p must be odd and >= 3");
  if (p >= (1ull << n_bits)) return fail(OR_CONTRACT, "reduction context: p must be < 2^n");
  if (alpha >= n_bits) return fail(OR_CONTRACT, "reduction context: alpha must be < n");
  if (ell >= n_bits) return fail(OR_CONTRACT, "reduction context: ell must be < n");
  memset(c, 0, sizeof *c);
  c->p = (uint32_t)p;
  c->n_bits = n_bits;
  c->alpha = alpha;
  c->ell = ell;
  c->beta = 1ull << n_bits;
  c->beta_mask = c->beta - 1;
  const unsigned two_n = 2 * n_bits;
  c->r2n_mask = two_n == 64 ? ~0ull : (1ull << two_n) - 1;
  u128 v;
  mod_inverse128(p, (u128)1 << n_bits, &v);
  c->p_inv_beta = (uint64_t)v;
  c->neg_p_inv_beta = (c->beta - c->p_inv_beta) & c->beta_mask;
  mod_inverse128(p, (u128)1 << two_n, &v);
  c->mu = (uint64_t)v;
  if (two_n == 64) {
    c->mu_centered = (int64_t)c->mu;
  } else {
    const uint64_t half = 1ull << (two_n - 1);
    c->mu_centered = c->mu >= half ? (int64_t)c->mu - (int64_t)(1ull << two_n) : (int64_t)c->mu;
  }
  c->beta_mod_p = c->beta % p;
  c->r2n_mod_p = or_pow_mod(2, two_n, p);
  return OR_OK;
}

/* bound predicates, reduction.hpp:64-77 */
int or_ctx_fits_plantard(const or_ctx* c) {
  const u128 lhs = (u128)5 * c->p * c->p;
  const u128 d = ((u128)1 << (c->n_bits + 1)) - c->p;
  return lhs < d * d;
}
int or_ctx_fits_lazy_plantard(const or_ctx* c) {
  return c->ell + 2 < c->n_bits && (u128)c->p < ((u128)1 << (c->n_bits - c->ell - 2));
}
int or_ctx_fits_signed_montgomery(const or_ctx* c) {
  return (u128)2 * c->p < ((u128)1 << c->n_bits);
}

/* Alg. 3, canonical output with the inclusive correction (reduction.hpp:125-135) */
int or_mont_redc(uint64_t T, const or_ctx* c, uint64_t* out) {
  if (!(T < (uint64_t)c->p * c->p)) return fail(OR_CONTRACT, "mont_redc: T must be < p^2");
  const uint64_t m = ((T & c->beta_mask) * c->neg_p_inv_beta) & c->beta_mask;
  const u128 s = (u128)T + (u128)m * c->p;
  if ((uint64_t)(s & c->beta_mask)) return fail(OR_PROPERTY, "mont_redc: inexact division");
  uint64_t t = (uint64_t)(s >> c->n_bits);
  if (t >= c->p) t -= c->p;
  *out = t;
  return OR_OK;
}

/* Alg. 4, Seiler signed Montgomery with floor split (reduction.hpp:141-165) */
static int64_t smont_core(int64_t A, const or_ctx* c) {
  const int64_t a1 = A >> c->n_bits;
  const uint64_t a0 = (uint64_t)A & c->beta_mask;
  const uint64_t mu = (a0 * c->p_inv_beta) & c->beta_mask;
  const int64_t m = mu >= c->beta / 2 ? (int64_t)mu - (int64_t)c->beta : (int64_t)mu;
  const int64_t t = (m * (int64_t)c->p) >> c->n_bits;
  return a1 - t;
}

int or_signed_mont_redc(int64_t A, const or_ctx* c, int64_t* out) {
  if (!or_ctx_fits_signed_montgomery(c))
    return fail(OR_CONTRACT, "signed_mont_redc: requires 2p < 2^n");
  const i128 limit = ((i128)c->p << c->n_bits) / 2;
  if (!(-limit < A && A < limit))
    return fail(OR_CONTRACT, "signed_mont_redc: A out of (-p*2^{n-1}, p*2^{n-1})");
  const int64_t r = smont_core(A, c);
  if (!(-(int64_t)c->p < r && r < (int64_t)c->p))
    return fail(OR_PROPERTY, "signed_mont_redc: result escaped (-p, p)");
  *out = r;
  return OR_OK;
}

/* Alg. 5 with the rarely-taken r == p corner (reduction.hpp:172-191) */
static _Atomic uint64_t g_plantard_fires;
uint64_t or_plantard_fires(void) { return atomic_load(&g_plantard_fires); }

static uint64_t plantard_core(uint64_t W, uint64_t T, const or_ctx* c) {
  const uint64_t h = ((W * T) * c->mu) & c->r2n_mask;
  const uint64_t r = (((h >> c->n_bits) + 1) * c->p) >> c->n_bits;
  if (r == c->p) {
    atomic_fetch_add(&g_plantard_fires, 1);
    return 0;
  }
  return r;
}

int or_plantard_redc(uint64_t W, uint64_t T, const or_ctx* c, uint64_t* out) {
  if (!or_ctx_fits_plantard(c)) return fail(OR_CONTRACT, "plantard_redc: requires p*phi < 2^n");
  if (!(W <= c->p && T <= c->p)) return fail(OR_CONTRACT, "plantard_redc: inputs exceed p");
  *out = plantard_core(W, T, c);
  return OR_OK;
}

/* Alg. 10 straight-line core: h = w t mu mod 2^{2n}; r = ((h >> n) + 1) p >> n
 * (reduction.hpp:252-258) */
uint64_t or_modified_plantard_core(uint64_t w, uint64_t t, uint64_t mu, uint64_t p,
                                   unsigned n_bits, uint64_t r2n_mask) {
  const uint64_t h = ((w * t) * mu) & r2n_mask;
  return (((h >> n_bits) + 1) * p) >> n_bits;
}

static inline uint64_t mp(uint64_t w, uint64_t t, const or_ctx* c) {
  return or_modified_plantard_core(w, t, c->mu, c->p, c->n_bits, c->r2n_mask);
}

/* checked Alg. 10 (reduction.hpp:264-273) */
int or_modified_plantard_mul(uint64_t W, uint64_t T, const or_ctx* c, uint64_t* out) {
  if (!or_ctx_fits_lazy_plantard(c))
    return fail(OR_CONTRACT, "modified_plantard_mul: requires p < 2^{n-ell-2}");
  if (!(W < c->p)) return fail(OR_CONTRACT, "modified_plantard_mul: W must be < p");
  if (!(T < ((uint64_t)c->p << c->ell)))
    return fail(OR_CONTRACT, "modified_plantard_mul: T must be < 2^ell * p");
  *out = mp(W, T, c);
  return OR_OK;
}

/* w -> w (-2^{2n}) mod p  (reduction.hpp:279-283) */
int or_to_plantard_domain(uint64_t w, const or_ctx* c, uint64_t* out) {
  if (!(w < c->p)) return fail(OR_CONTRACT, "to_plantard_domain: w must be < p");
  *out = (c->p - mulmod(w, c->r2n_mod_p, c->p)) % c->p;
  return OR_OK;
}

/* w -> w 2^n mod p  (reduction.hpp:287-291) */
int or_to_montgomery_domain(uint64_t w, const or_ctx* c, uint64_t* out) {
  if (!(w < c->p)) return fail(OR_CONTRACT, "to_montgomery_domain: w must be < p");
  *out = mulmod(w, c->beta_mod_p, c->p);
  return OR_OK;
}

/* extension: centered Montgomery twiddle for the signed butterflies */
int64_t or_to_signed_montgomery_domain(uint64_t w, const or_ctx* c) {
  const uint64_t m = mulmod(w % c->p, c->beta_mod_p, c->p);
  return m > c->p / 2 ? (int64_t)m - (int64_t)c->p : (int64_t)m;
}

/* extension: signed Barrett a - round(a V / 2^S) p with S = n + 10,
 * V = floor((2^S + floor(p/2)) / p); for (p, n) = (3329, 16) this is the usual
 * V = 20159, S = 26 pair.  Output lies in (-p, p) for |a| < 2^{S-1}. */
int64_t or_signed_barrett(int64_t a, const or_ctx* c) {
  const unsigned S = c->n_bits + 10;
  const int64_t V = (int64_t)((((u128)1 << S) + (c->p >> 1)) / c->p);
  const int64_t q = (int64_t)(((i128)a * V + ((i128)1 << (S - 1))) >> S);
  return a - q * (int64_t)c->p;
}

/* ----------------------------------------------------------------------------
 * butterflies -- butterfly.hpp
 * ------------------------------------------------------------------------- */

/* Alg. 7 canonical Shoup-style butterfly (butterfly.hpp:60-71) */
void or_ntl_core(uint64_t X, uint64_t Y, uint64_t W, uint64_t Wq, const or_ctx* c,
                 uint64_t* x1, uint64_t* y1) {
  const uint64_t p = c->p;
  uint64_t s = X + Y;
  if (s >= p) s -= p;
  const uint64_t t = X >= Y ? X - Y : X + p - Y;
  const uint64_t q = (Wq * t) >> c->n_bits;
  uint64_t y = (W * t - q * p) & c->beta_mask;
  if (y >= p) y -= p;
  *x1 = s;
  *y1 = y;
}

/* Alg. 8 lazy [0,2p) DIF butterfly with a branchless X fix (butterfly.hpp:92-106) */
void or_harvey_core(uint64_t X, uint64_t Y, uint64_t Wm, const or_ctx* c, uint64_t* x1,
                    uint64_t* y1) {
  const uint64_t p = c->p, p2 = 2 * p;
  uint64_t s = X + Y;
  if (s >= p2) s -= p2;
  const uint64_t t = X + p2 - Y;
  const uint64_t prod = Wm * t;
  const uint64_t q = (c->p_inv_beta * (prod & c->beta_mask)) & c->beta_mask;
  *x1 = s;
  *y1 = (prod >> c->n_bits) + p - ((q * p) >> c->n_bits);
}

/* Alg. 9 unreduced-sum butterfly (butterfly.hpp:172-184) */
void or_scott_core(uint64_t X, uint64_t Y, uint64_t Wm, uint64_t offset, const or_ctx* c,
                   uint64_t* x1, uint64_t* y1) {
  const uint64_t t = X + offset - Y;
  const uint64_t wt = Wm * t;
  const uint64_t q = (c->neg_p_inv_beta * (wt & c->beta_mask)) & c->beta_mask;
  *x1 = X + Y;
  *y1 = (wt + q * c->p) >> c->n_bits;
}

/* Alg. 11 CT butterfly (butterfly.hpp:224-230) */
void or_improved_ct_core(uint64_t X, uint64_t Y, uint64_t What, const or_ctx* c,
                         uint64_t* x1, uint64_t* y1) {
  const uint64_t r = mp(What, Y, c);
  *x1 = X + r;
  *y1 = X + c->p - r;
}

/* Alg. 12 GS butterfly (butterfly.hpp:235-243) */
void or_improved_gs_core(uint64_t X, uint64_t Y, uint64_t offset, uint64_t What,
                         const or_ctx* c, uint64_t* x1, uint64_t* y1) {
  const uint64_t t = X + offset - Y;
  *x1 = X + Y;
  *y1 = mp(What, t, c);
}

/* extension: CT-form Montgomery butterfly, everything lazy in [0, 2p).
 * r = W*Y*2^{-n} + {0,p} computed exactly like harvey_core's Y output; requires
 * W*Y < 2^n p, which holds for W < p, Y < 2p, 4p < 2^n. */
void or_harvey_ct_core(uint64_t X, uint64_t Y, uint64_t Wm, const or_ctx* c, uint64_t* x1,
                       uint64_t* y1) {
  const uint64_t p = c->p, p2 = 2 * p;
  const uint64_t prod = Wm * Y;
  const uint64_t q = (c->p_inv_beta * (prod & c->beta_mask)) & c->beta_mask;
  const uint64_t r = (prod >> c->n_bits) + p - ((q * p) >> c->n_bits);
  uint64_t a = X + r;
  if (a >= p2) a -= p2;
  uint64_t b = X + p2 - r;
  if (b >= p2) b -= p2;
  *x1 = a;
  *y1 = b;
}

/* extension: signed-Montgomery CT butterfly (X + t, X - t), t = smont(Ws Y) */
void or_smont_ct_core(int64_t X, int64_t Y, int64_t Ws, const or_ctx* c, int64_t* x1,
                      int64_t* y1) {
  const int64_t t = smont_core(Ws * Y, c);
  *x1 = X + t;
  *y1 = X - t;
}

/* extension: signed-Montgomery GS butterfly (sbarrett(X + Y), smont(Ws (X - Y))) */
void or_smont_gs_core(int64_t X, int64_t Y, int64_t Ws, const or_ctx* c, int64_t* x1,
                      int64_t* y1) {
  *x1 = or_signed_barrett(X + Y, c);
  *y1 = smont_core(Ws * (X - Y), c);
}

/* smallest power-of-two L with 4 N p < 2^n L (butterfly.hpp:157-168) */
uint32_t or_scott_lazy_level(uint32_t N, const or_ctx* c) {
  for (uint64_t L = 1; L <= N; L *= 2)
    if ((u128)4 * N * c->p < (u128)c->beta * L) return (uint32_t)L;
  return 0;
}

/* ----------------------------------------------------------------------------
 * params -- params.hpp:30-268 (+ the extension trees of SURVEY a22)
 * ------------------------------------------------------------------------- */

/* smallest element of exact order `order` (a power of two), params.hpp:30-43 */
uint64_t or_find_primitive_root(uint64_t p, uint64_t order) {
  if (order == 1) return 1;
  for (uint64_t w = 2; w < p; ++w)
    if (or_pow_mod(w, order, p) == 1 && or_pow_mod(w, order / 2, p) != 1) return w;
  return 0;
}

/* plain twiddle of forward CT block b at layer s (1-based) */
static uint64_t ct_plain(const or_params* P, unsigned s, uint64_t b) {
  if (P->tree == OR_TREE_CYCLIC) {
    const uint64_t len = (uint64_t)P->N >> s; /* params.hpp:60-72 */
    return or_pow_mod(P->omega, len * or_bit_reverse(b, s - 1), P->p);
  }
  /* negacyclic: zeta^{br_L(2^{s-1} + b)} */
  return or_pow_mod(P->omega, or_bit_reverse((1ull << (s - 1)) + b, P->layers), P->p);
}

/* plain twiddle of inverse GS block b at forward layer s: the inverse of ct_plain */
static uint64_t gs_plain(const or_params* P, unsigned s, uint64_t b) {
  if (P->tree == OR_TREE_CYCLIC) {
    /* w^{-e} as w^{N-e}, exponent 0 stays 0 (params.hpp:74-88) */
    const uint64_t len = (uint64_t)P->N >> s;
    const uint64_t e = len * or_bit_reverse(b, s - 1) % P->N;
    return or_pow_mod(P->omega, e == 0 ? 0 : P->N - e, P->p);
  }
  const uint64_t order = 2ull << P->layers;
  const uint64_t e = or_bit_reverse((1ull << (s - 1)) + b, P->layers) % order;
  return or_pow_mod(P->omega, e == 0 ? 0 : order - e, P->p);
}

void or_params_free(or_params* P) {
  if (!P) return;
  free(P->dif_w);
  free(P->dif_wq);
  free(P->dif_mont);
  free(P->ct_plain);
  free(P->ct_plantard);
  free(P->ct_mont);
  free(P->ct_smont);
  free(P->gs_plain);
  free(P->gs_w);
  free(P->gs_wq);
  free(P->gs_mont);
  free(P->gs_plantard);
  free(P->gs_smont);
  free(P);
}

#define KIND(k) (1u << (k))

static int append_fault(char* buf, size_t cap, const char* msg) {
  size_t n = strlen(buf);
  snprintf(buf + n, cap - n, "\n  - %s", msg);
  return 1;
}

int or_params_build(uint64_t p, uint32_t N, unsigned n_bits, uint32_t kinds, uint32_t tree,
                    uint32_t layers, uint64_t root, int exact_bound, or_params** out) {
  char faults[2048] = "build_params:";
  char msg[256];
  int nf = 0;
  *out = NULL;
  /* structural faults, collected together (params.hpp:145-169) */
  if (n_bits < 2 || n_bits > 32) nf += append_fault(faults, sizeof faults, "word size n must be in [2, 32]");
  if (p < 3 || !(p & 1)) nf += append_fault(faults, sizeof faults, "p must be odd and >= 3");
  else if (!or_is_prime(p)) nf += append_fault(faults, sizeof faults, "p must be prime");
  if (N < 2 || !is_pow2(N) || N > (1u << 20))
    nf += append_fault(faults, sizeof faults, "N must be a power of two in [2, 2^20]");
  if (!kinds) nf += append_fault(faults, sizeof faults, "at least one butterfly kind must be requested");
  if (tree > OR_TREE_NEGA) nf += append_fault(faults, sizeof faults, "unknown transform tree");
  unsigned ell = 0;
  if (!nf) {
    ell = ilog2(N);
    if (layers == 0) layers = ell;
    if (layers > ell || (tree == OR_TREE_CYCLIC && layers != ell))
      nf += append_fault(faults, sizeof faults, "layers must be log2(N) (cyclic) or <= log2(N) (negacyclic)");
    const uint64_t order = tree == OR_TREE_CYCLIC ? N : (2ull << layers);
    if ((p - 1) % order != 0) {
      snprintf(msg, sizeof msg, "N must divide p - 1 (p=%llu, N=%llu)", (unsigned long long)p,
               (unsigned long long)order);
      nf += append_fault(faults, sizeof faults, msg);
    }
    if (ell >= n_bits) nf += append_fault(faults, sizeof faults, "word size n must exceed log2(N)");
    if (n_bits <= 32 && p >= (1ull << n_bits)) nf += append_fault(faults, sizeof faults, "p must be < 2^n");
  }
  if (nf) return fail(OR_CONTRACT, faults);

  or_params* P = (or_params*)calloc(1, sizeof *P);
  P->p = (uint32_t)p;
  P->N = N;
  P->log2N = ell;
  P->n_bits = n_bits;
  P->tree = tree;
  P->layers = layers;
  P->kinds_mask = kinds;
  or_make_ctx(p, n_bits, 0, ell, &P->ctx);
  const or_ctx* c = &P->ctx;
  const uint64_t order = tree == OR_TREE_CYCLIC ? N : (2ull << layers);
  if (root) {
    if (or_pow_mod(root, order, p) != 1 || or_pow_mod(root, order / 2, p) == 1) {
      or_params_free(P);
      return fail(OR_CONTRACT, "build_params:\n  - root does not have the required order");
    }
    P->omega = root;
  } else {
    P->omega = or_find_primitive_root(p, order);
  }
  or_mod_inverse_u64(P->omega, p, &P->omega_inv);
  /* cyclic scale N^{-1}; negacyclic scale 2^{-layers} */
  or_mod_inverse_u64(tree == OR_TREE_CYCLIC ? N % p : (1ull << layers) % p, p, &P->n_inv);

  /* per-kind word-size faults (params.hpp:183-217) */
  const uint64_t exact_T = ((uint64_t)p << layers); /* largest lazy multiplicand */
  if ((kinds & KIND(OR_NTL)) && 2ull * p >= c->beta) {
    snprintf(msg, sizeof msg, "ntl: p=%llu violates 2p < 2^n (n=%u)", (unsigned long long)p, n_bits);
    nf += append_fault(faults, sizeof faults, msg);
  }
  if ((kinds & KIND(OR_HARVEY)) && 4ull * p >= c->beta) {
    snprintf(msg, sizeof msg, "harvey: p=%llu violates 4p < 2^n (n=%u)", (unsigned long long)p, n_bits);
    nf += append_fault(faults, sizeof faults, msg);
  }
  if ((kinds & KIND(OR_SCOTT)) && (u128)4 * p >= c->beta) {
    snprintf(msg, sizeof msg, "scott: p=%llu violates 4*N*p < 2^n * L for every L <= N",
             (unsigned long long)p);
    nf += append_fault(faults, sizeof faults, msg);
  }
  if (kinds & KIND(OR_IMPROVED)) {
    int ok;
    if (exact_bound) {
      /* Prop. 4 exact requirement W T < 2^n (2^n - p) with
       * W <= p-1 and T <= 2^layers p - 1 */
      ok = (u128)(p - 1) * (exact_T - 1) < ((u128)c->beta) * (c->beta - p);
    } else {
      ok = or_ctx_fits_lazy_plantard(c);
    }
    if (!ok) {
      snprintf(msg, sizeof msg, "improved: p=%llu violates p < 2^{n-ell-2} = %llu (n=%u, ell=%u)",
               (unsigned long long)p,
               (unsigned long long)(n_bits >= ell + 2 ? (1ull << (n_bits - ell - 2)) : 0), n_bits,
               ell);
      nf += append_fault(faults, sizeof faults, msg);
    }
  }
  if (kinds & KIND(OR_SMONT)) {
    /* extension bound: (layers+1) (p-1) < 2^n keeps every smont input in range */
    if (!or_ctx_fits_signed_montgomery(c) || (u128)(layers + 1) * (p - 1) >= c->beta) {
      snprintf(msg, sizeof msg, "smont: p=%llu violates (layers+1)(p-1) < 2^n (n=%u)",
               (unsigned long long)p, n_bits);
      nf += append_fault(faults, sizeof faults, msg);
    }
  }
  if (tree == OR_TREE_NEGA && (kinds & (KIND(OR_NTL) | KIND(OR_SCOTT)))) {
    nf += append_fault(faults, sizeof faults, "ntl/scott are DIF kinds: cyclic tree only");
  }
  if (nf) {
    or_params_free(P);
    return fail(OR_CONTRACT, faults);
  }
  if (kinds & KIND(OR_SCOTT)) P->scott_L = or_scott_lazy_level(N, c);

  /* tables.  Forward tables hold one entry per (layer, block) [CT] or per
   * (layer, index) [DIF], layers in driver order; N-1 entries for complete trees. */
  const size_t T = (1ull << layers) - 1;
  P->fwd_len = T;
  P->inv_len = T;
  const int want_dif = tree == OR_TREE_CYCLIC &&
                       (kinds & (KIND(OR_NTL) | KIND(OR_HARVEY) | KIND(OR_SCOTT)));
  if (want_dif) {
    P->dif_w = (uint64_t*)calloc(T, 8);
    P->dif_wq = (uint64_t*)calloc(T, 8);
    P->dif_mont = (uint64_t*)calloc(T, 8);
    size_t k = 0;
    for (uint64_t len = N / 2; len >= 1; len /= 2) { /* params.hpp:47-58 */
      const uint64_t step = N / (2 * len);
      for (uint64_t j = 0; j < len; ++j, ++k) {
        const uint64_t w = or_pow_mod(P->omega, j * step, p);
        P->dif_w[k] = w;
        P->dif_wq[k] = (uint64_t)(((u128)w << n_bits) / p);
        or_to_montgomery_domain(w, c, &P->dif_mont[k]);
      }
    }
  }
  P->ct_plain = (uint64_t*)calloc(T, 8);
  P->ct_plantard = (uint64_t*)calloc(T, 8);
  P->ct_mont = (uint64_t*)calloc(T, 8);
  P->ct_smont = (int64_t*)calloc(T, 8);
  P->gs_plain = (uint64_t*)calloc(T, 8);
  P->gs_w = (uint64_t*)calloc(T, 8);
  P->gs_wq = (uint64_t*)calloc(T, 8);
  P->gs_mont = (uint64_t*)calloc(T, 8);
  P->gs_plantard = (uint64_t*)calloc(T, 8);
  P->gs_smont = (int64_t*)calloc(T, 8);
  {
    size_t k = 0;
    for (unsigned s = 1; s <= layers; ++s) /* forward layer order */
      for (uint64_t b = 0; b < (1ull << (s - 1)); ++b, ++k) {
        const uint64_t w = ct_plain(P, s, b);
        P->ct_plain[k] = w;
        or_to_plantard_domain(w, c, &P->ct_plantard[k]);
        or_to_montgomery_domain(w, c, &P->ct_mont[k]);
        P->ct_smont[k] = or_to_signed_montgomery_domain(w, c);
      }
    k = 0;
    for (unsigned s = layers; s >= 1; --s) /* merge order: last forward layer first */
      for (uint64_t b = 0; b < (1ull << (s - 1)); ++b, ++k) {
        const uint64_t w = gs_plain(P, s, b);
        P->gs_plain[k] = w;
        P->gs_w[k] = w;
        P->gs_wq[k] = (uint64_t)(((u128)w << n_bits) / p);
        or_to_plantard_domain(w, c, &P->gs_plantard[k]);
        or_to_montgomery_domain(w, c, &P->gs_mont[k]);
        P->gs_smont[k] = or_to_signed_montgomery_domain(w, c);
      }
  }
  if (kinds & KIND(OR_IMPROVED)) or_to_plantard_domain(P->n_inv, c, &P->n_inv_hat); /* params.hpp:250 */
  or_to_montgomery_domain(P->n_inv, c, &P->n_inv_mont);
  P->n_inv_smont = or_to_signed_montgomery_domain(P->n_inv, c);
  *out = P;
  return OR_OK;
}

size_t or_params_table(const or_params* P, const char* name, uint64_t* out, size_t cap) {
  const uint64_t* src = NULL;
  size_t n = P->fwd_len;
  if (!strcmp(name, "dif_w")) src = P->dif_w;
  else if (!strcmp(name, "dif_wq")) src = P->dif_wq;
  else if (!strcmp(name, "dif_mont")) src = P->dif_mont;
  else if (!strcmp(name, "ct_plain")) src = P->ct_plain;
  else if (!strcmp(name, "ct_plantard")) src = P->ct_plantard;
  else if (!strcmp(name, "ct_mont")) src = P->ct_mont;
  else if (!strcmp(name, "ct_smont")) src = (const uint64_t*)P->ct_smont;
  else if (!strcmp(name, "gs_plain")) src = P->gs_plain, n = P->inv_len;
  else if (!strcmp(name, "gs_wq")) src = P->gs_wq, n = P->inv_len;
  else if (!strcmp(name, "gs_mont")) src = P->gs_mont, n = P->inv_len;
  else if (!strcmp(name, "gs_plantard")) src = P->gs_plantard, n = P->inv_len;
  else if (!strcmp(name, "gs_smont")) src = (const uint64_t*)P->gs_smont, n = P->inv_len;
  if (!src) return 0;
  if (out) memcpy(out, src, (n < cap ? n : cap) * 8);
  return n;
}

/* ----------------------------------------------------------------------------
 * transforms -- transform.hpp:77-379
 * ------------------------------------------------------------------------- */

static int kind_ok(const or_params* P, int kind) {
  if (kind < 0 || kind > OR_SMONT || !(P->kinds_mask & KIND(kind)))
    return fail(OR_CONTRACT, "ntt: kind not built into these params");
  return OR_OK;
}

/* forward: splitting passes, len = N/2 down to N >> layers (transform.hpp:77-96,125-203) */
static void forward_one(const or_params* P, int kind, uint64_t* a) {
  const or_ctx* c = &P->ctx;
  const uint32_t N = P->N;
  size_t cursor = 0;
  const uint64_t scott_off = P->scott_L ? (uint64_t)(N / P->scott_L) * c->p : 0;
  for (unsigned s = 1; s <= P->layers; ++s) {
    const uint32_t len = N >> s, blocks = 1u << (s - 1);
    for (uint32_t b = 0; b < blocks; ++b) {
      uint64_t* x = a + (size_t)b * 2 * len;
      for (uint32_t j = 0; j < len; ++j) {
        uint64_t* X = x + j;
        uint64_t* Y = x + j + len;
        switch (kind) {
          case OR_NTL:
            or_ntl_core(*X, *Y, P->dif_w[cursor + j], P->dif_wq[cursor + j], c, X, Y);
            break;
          case OR_HARVEY:
            if (P->tree == OR_TREE_CYCLIC)
              or_harvey_core(*X, *Y, P->dif_mont[cursor + j], c, X, Y);
            else
              or_harvey_ct_core(*X, *Y, P->ct_mont[cursor + b], c, X, Y);
            break;
          case OR_SCOTT:
            or_scott_core(*X, *Y, P->dif_mont[cursor + j], scott_off, c, X, Y);
            break;
          case OR_IMPROVED:
            or_improved_ct_core(*X, *Y, P->ct_plantard[cursor + b], c, X, Y);
            break;
          case OR_SMONT: {
            int64_t xs, ys;
            or_smont_ct_core((int64_t)*X, (int64_t)*Y, P->ct_smont[cursor + b], c, &xs, &ys);
            *X = (uint64_t)xs;
            *Y = (uint64_t)ys;
            break;
          }
        }
      }
    }
    const int per_index = P->tree == OR_TREE_CYCLIC && kind != OR_IMPROVED && kind != OR_SMONT;
    cursor += per_index ? len : blocks;
  }
}

int or_forward(const or_params* P, int kind, uint64_t* a, size_t batch) {
  int st = kind_ok(P, kind);
  if (st) return st;
  for (size_t i = 0; i < batch * P->N; ++i)
    if (a[i] >= P->p) return fail(OR_CONTRACT, "ntt_forward: coefficients must be canonical");
  for (size_t i = 0; i < batch; ++i) forward_one(P, kind, a + i * P->N);
  return OR_OK;
}

/* inverse: canonicalize, merging passes, final scale (transform.hpp:233-337) */
static void inverse_one(const or_params* P, int kind, uint64_t* a) {
  const or_ctx* c = &P->ctx;
  const uint32_t N = P->N;
  const uint64_t p = c->p;
  for (uint32_t i = 0; i < N; ++i) {
    if (kind == OR_SMONT) {
      int64_t v = (int64_t)a[i] % (int64_t)p;
      a[i] = (uint64_t)(v < 0 ? v + (int64_t)p : v);
    } else {
      a[i] %= p; /* transform.hpp:38-40,243 */
    }
  }
  const uint64_t scott_off = P->scott_L ? (uint64_t)(N / P->scott_L) * p : 0;
  size_t cursor = 0;
  unsigned m = 0; /* merge depth, 1-based */
  for (unsigned s = P->layers; s >= 1; --s) {
    ++m;
    const uint32_t len = N >> s, blocks = 1u << (s - 1);
    for (uint32_t b = 0; b < blocks; ++b) {
      uint64_t* x = a + (size_t)b * 2 * len;
      const size_t ti = cursor + b;
      for (uint32_t j = 0; j < len; ++j) {
        uint64_t* X = x + j;
        uint64_t* Y = x + j + len;
        switch (kind) {
          case OR_NTL: or_ntl_core(*X, *Y, P->gs_w[ti], P->gs_wq[ti], c, X, Y); break;
          case OR_HARVEY: or_harvey_core(*X, *Y, P->gs_mont[ti], c, X, Y); break;
          case OR_SCOTT: or_scott_core(*X, *Y, P->gs_mont[ti], scott_off, c, X, Y); break;
          case OR_IMPROVED:
            or_improved_gs_core(*X, *Y, p << (m - 1), P->gs_plantard[ti], c, X, Y);
            break;
          case OR_SMONT: {
            int64_t xs, ys;
            or_smont_gs_core((int64_t)*X, (int64_t)*Y, P->gs_smont[ti], c, &xs, &ys);
            *X = (uint64_t)xs;
            *Y = (uint64_t)ys;
            break;
          }
        }
      }
    }
    cursor += blocks;
  }
  for (uint32_t i = 0; i < N; ++i) {
    if (kind == OR_IMPROVED) {
      a[i] = mp(P->n_inv_hat, a[i], c); /* transform.hpp:323-330 */
    } else if (kind == OR_SMONT) {
      int64_t v = smont_core(P->n_inv_smont * (int64_t)a[i], c);
      a[i] = (uint64_t)(v < 0 ? v + (int64_t)p : v);
    } else {
      a[i] = mulmod(a[i], P->n_inv, p); /* transform.hpp:331-335 */
    }
  }
}

int or_inverse(const or_params* P, int kind, uint64_t* a, size_t batch) {
  int st = kind_ok(P, kind);
  if (st) return st;
  for (size_t i = 0; i < batch; ++i) inverse_one(P, kind, a + i * P->N);
  return OR_OK;
}

static uint64_t canon(uint64_t v, int kind, uint64_t p) {
  if (kind == OR_SMONT) {
    int64_t s = (int64_t)v % (int64_t)p;
    return (uint64_t)(s < 0 ? s + (int64_t)p : s);
  }
  return v % p;
}

/* slotwise product, canonical output (transform.hpp:349-370) */
int or_pointwise(const or_params* P, int kind, const uint64_t* lhs, const uint64_t* rhs,
                 uint64_t* out, size_t batch) {
  int st = kind_ok(P, kind);
  if (st) return st;
  const or_ctx* c = &P->ctx;
  const uint64_t p = c->p;
  for (size_t i = 0; i < batch * P->N; ++i) {
    if (kind == OR_IMPROVED) {
      uint64_t w;
      or_to_plantard_domain(lhs[i] % p, c, &w);
      if (rhs[i] >= ((uint64_t)p << P->log2N))
        return fail(OR_CONTRACT, "modified_plantard_mul: T must be < 2^ell * p");
      out[i] = mp(w, rhs[i], c);
    } else {
      out[i] = mulmod(canon(lhs[i], kind, p), canon(rhs[i], kind, p), p);
    }
  }
  return OR_OK;
}

/* extension: degree-2 basemul mod (x^2 - gamma), gamma = +-(last-layer twiddle) */
int or_basemul(const or_params* P, int kind, const uint64_t* lhs, const uint64_t* rhs,
               uint64_t* out, size_t batch) {
  int st = kind_ok(P, kind);
  if (st) return st;
  if ((P->N >> P->layers) != 2) return fail(OR_CONTRACT, "basemul: tree must end in degree-2 factors");
  const uint64_t p = P->p;
  const size_t last = ((size_t)1 << (P->layers - 1)) - 1; /* first block of the last layer */
  for (size_t i = 0; i < batch; ++i) {
    const uint64_t* a = lhs + i * P->N;
    const uint64_t* b = rhs + i * P->N;
    uint64_t* o = out + i * P->N;
    for (uint32_t k = 0; k < P->N / 2; ++k) {
      const uint64_t z = P->ct_plain[last + k / 2];
      const uint64_t g = (k & 1) ? (p - z) % p : z;
      const uint64_t a0 = canon(a[2 * k], kind, p), a1 = canon(a[2 * k + 1], kind, p);
      const uint64_t b0 = canon(b[2 * k], kind, p), b1 = canon(b[2 * k + 1], kind, p);
      o[2 * k] = (mulmod(a0, b0, p) + mulmod(mulmod(a1, b1, p), g, p)) % p;
      o[2 * k + 1] = (mulmod(a0, b1, p) + mulmod(a1, b0, p)) % p;
    }
  }
  return OR_OK;
}

/* transform.hpp:372-379 (and the Kyber-style basemul pipeline) */
int or_polymul(const or_params* P, int kind, const uint64_t* a, const uint64_t* b,
               uint64_t* out, size_t batch) {
  const size_t n = batch * P->N;
  uint64_t* fa = (uint64_t*)malloc(n * 8);
  uint64_t* fb = (uint64_t*)malloc(n * 8);
  memcpy(fa, a, n * 8);
  memcpy(fb, b, n * 8);
  int st = or_forward(P, kind, fa, batch);
  if (!st) st = or_forward(P, kind, fb, batch);
  if (!st) {
    if ((P->N >> P->layers) == 2) st = or_basemul(P, kind, fa, fb, out, batch);
    else st = or_pointwise(P, kind, fa, fb, out, batch);
  }
  if (!st) st = or_inverse(P, kind, out, batch);
  free(fa);
  free(fb);
  return st;
}

/* ----------------------------------------------------------------------------
 * naive references -- oracle.hpp:49-102 (plus the negacyclic counterparts)
 * ------------------------------------------------------------------------- */

/* Horner evaluation at omega^i, natural order (oracle.hpp:49-63) */
void or_naive_dft(const uint64_t* f, size_t N, uint64_t omega, uint64_t p, uint64_t* out) {
  uint64_t x = 1 % p;
  for (size_t i = 0; i < N; ++i) {
    uint64_t acc = 0;
    for (size_t j = N; j-- > 0;) acc = (mulmod(acc, x, p) + f[j] % p) % p;
    out[i] = acc;
    x = mulmod(x, omega, p);
  }
}

/* oracle.hpp:88-102 */
void or_schoolbook_cyclic(const uint64_t* a, const uint64_t* b, size_t N, uint64_t p,
                          uint64_t* out) {
  memset(out, 0, N * 8);
  for (size_t i = 0; i < N; ++i)
    for (size_t j = 0; j < N; ++j) {
      const size_t k = (i + j) % N;
      out[k] = (out[k] + mulmod(a[i] % p, b[j] % p, p)) % p;
    }
}

void or_schoolbook_negacyclic(const uint64_t* a, const uint64_t* b, size_t N, uint64_t p,
                              uint64_t* out) {
  memset(out, 0, N * 8);
  for (size_t i = 0; i < N; ++i)
    for (size_t j = 0; j < N; ++j) {
      const uint64_t t = mulmod(a[i] % p, b[j] % p, p);
      const size_t k = i + j;
      if (k < N) out[k] = (out[k] + t) % p;
      else out[k - N] = (out[k - N] + p - t) % p;
    }
}

/* Residues of f modulo the leaves of the tree, in butterfly order: block b of
 * the last layer with twiddle z splits into (x^len - z, x^len + z). */
int or_naive_nega_eval(const or_params* P, const uint64_t* f, uint64_t* out) {
  const uint64_t p = P->p;
  const uint32_t N = P->N, len = N >> P->layers, blocks = 1u << (P->layers - 1);
  const size_t last = (size_t)blocks - 1;
  for (uint32_t b = 0; b < blocks; ++b) {
    for (int half = 0; half < 2; ++half) {
      uint64_t z = P->tree == OR_TREE_CYCLIC ? ct_plain(P, P->layers, b) : P->ct_plain[last + b];
      if (half) z = (p - z) % p;
      /* f mod (x^len - z): fold coefficient k into slot k % len times z^{k / len} */
      uint64_t* o = out + (size_t)(2 * b + half) * len;
      for (uint32_t r = 0; r < len; ++r) o[r] = 0;
      uint64_t zp = 1;
      for (uint32_t k = 0; k < N; k += len) {
        for (uint32_t r = 0; r < len; ++r) o[r] = (o[r] + mulmod(f[k + r] % p, zp, p)) % p;
        zp = mulmod(zp, z, p);
      }
    }
  }
  return OR_OK;
}

/* ----------------------------------------------------------------------------
 * reduction sweep (config 5): grid of operand pairs through one reduction
 * ------------------------------------------------------------------------- */
typedef struct {
  int variant;
  const or_ctx* c;
  const int64_t *A, *B;
  size_t na, nb, i0, i1;
  int64_t* r;
  uint64_t sum;
} sweep_job;

static int64_t sweep_one(int variant, const or_ctx* c, int64_t a, int64_t b) {
  switch (variant) {
    case OR_SW_MONT: { /* reduction.hpp:125-135 (unchecked body) */
      const uint64_t T = (uint64_t)a * (uint64_t)b;
      const uint64_t m = ((T & c->beta_mask) * c->neg_p_inv_beta) & c->beta_mask;
      uint64_t t = (uint64_t)(((u128)T + (u128)m * c->p) >> c->n_bits);
      if (t >= c->p) t -= c->p;
      return (int64_t)t;
    }
    case OR_SW_SMONT: return smont_core(a * b, c); /* reduction.hpp:141-165 */
    case OR_SW_PLANTARD: return (int64_t)plantard_core((uint64_t)a, (uint64_t)b, c);
    default: return (int64_t)mp((uint64_t)a, (uint64_t)b, c); /* reduction.hpp:252-258 */
  }
}

static void* sweep_worker(void* arg) {
  sweep_job* j = (sweep_job*)arg;
  uint64_t s = 0;
  for (size_t i = j->i0; i < j->i1; ++i)
    for (size_t k = 0; k < j->nb; ++k) {
      const int64_t v = sweep_one(j->variant, j->c, j->A[i], j->B[k]);
      s += (uint64_t)v;
      if (j->r) j->r[i * j->nb + k] = v;
    }
  j->sum = s;
  return NULL;
}

int or_sweep(int variant, const or_ctx* c, const int64_t* A, size_t na, const int64_t* B,
             size_t nb, int64_t* r, uint64_t* checksum, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  sweep_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (sweep_job){variant, c, A, B, na, nb, na * t / threads, na * (t + 1) / threads, r, 0};
    if (threads > 1) pthread_create(&tid[t], NULL, sweep_worker, &jobs[t]);
    else sweep_worker(&jobs[t]);
  }
  uint64_t s = 0;
  for (int t = 0; t < threads; ++t) {
    if (threads > 1) pthread_join(tid[t], NULL);
    s += jobs[t].sum;
  }
  *checksum = s;
  return OR_OK;
}

/* FNV-1a-64 over values serialized as little-endian u32 */
uint64_t or_fnv1a_u32(const uint64_t* v, size_t n) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < n; ++i) {
    const uint32_t x = (uint32_t)v[i];
    for (int k = 0; k < 4; ++k) {
      h ^= (x >> (8 * k)) & 0xff;
      h *= 0x100000001b3ull;
    }
  }
  return h;
}
