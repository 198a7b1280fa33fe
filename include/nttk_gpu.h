/*
 * nttk_gpu.h -- C ABI of the B200-native batched NTT engine (libnttk_gpu.so).
 *
 * This is the drop-in boundary for the reference's hot path, the header-only C++20
 * library `nttk` (/root/reference/proj/include/nttk).  Each entry point names the
 * reference interface it replaces (file:line under proj/include/nttk/).  The
 * reference works on one std::vector<uint64_t> polynomial per call; every entry
 * point here is batched: `batch` contiguous polynomials of P.size coefficients.
 *
 * Conventions
 *   - plain pointers and sizes only; no C++ or torch types cross this boundary;
 *   - status codes mirror the reference CLI contract (tools/ntt_kernel_cli.cpp:17-18):
 *       0 ok, 1 property violation, 2 contract violation (the reference throws
 *       nttk::contract_violation there, with the message returned by
 *       nttk_last_error()), 3 CUDA error;
 *   - `d_*` pointers are device memory on the current CUDA device; `h_*` pointers are
 *     host memory (pinned memory makes the copies asynchronous and overlapped);
 *   - `elem_bytes` is the storage width of one coefficient: 2 (uint16 / int16, valid
 *     when the kind's spectrum bound is < 2^16, e.g. Kyber), 4 (uint32 / int32) or 8
 *     (uint64, the reference's own width).  Signed kinds store two's complement;
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Device entry points
 *     are asynchronous and validate nothing on the device data (like
 *     ntt_forward_inplace, transform.hpp:228-231); host entry points synchronise and
 *     perform the reference's checked-path validation (transform.hpp:207-218).
 *   - parameter handles are immutable after creation and may be shared by host
 *     threads working on distinct buffers/streams.
 *   - there is no CPU fallback: without a usable CUDA device every compute entry
 *     point returns 3.
 */
#ifndef NTTK_GPU_H
#define NTTK_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum nttk_status { NTTK_OK = 0, NTTK_PROPERTY = 1, NTTK_CONTRACT = 2, NTTK_CUDA = 3 };

/* butterfly.hpp:30 ButterflyKind {ntl, harvey, scott, improved}, plus the signed-
 * Montgomery CT/GS kind (extension: the reference has only signed_mont_redc,
 * reduction.hpp:141-165). */
enum nttk_kind {
  NTTK_NTL = 0,
  NTTK_HARVEY = 1,
  NTTK_SCOTT = 2,
  NTTK_IMPROVED = 3,
  NTTK_SMONT = 4
};

/* transform tree: the reference's complete cyclic tree (x^N - 1), or the extension
 * negacyclic tree (x^N + 1) with `layers` <= log2 N splitting layers (layers =
 * log2 N - 1 ends in degree-2 factors, Kyber-style). */
enum nttk_tree { NTTK_CYCLIC = 0, NTTK_NEGACYCLIC = 1 };

/* flags for nttk_params_desc.flags */
enum nttk_flags {
  /* admit `improved` whenever Prop. 4's exact requirement W*T < 2^n (2^n - p) holds
   * instead of the paper's sufficient p < 2^{n-ell-2}
   * (params.hpp:204-214); needed for Kyber at n=16 and Dilithium at n=32. */
  NTTK_EXACT_BOUND = 1u << 0
};

typedef struct nttk_params_s* nttk_params_t;

typedef struct {
  uint64_t p;          /* prime modulus */
  uint32_t N;          /* transform size (power of two, 2..2^20) */
  uint32_t n_bits;     /* radix exponent n of 2^n, 2..32 */
  uint32_t kinds_mask; /* bit k set = kind k built (build_params `kinds`) */
  uint32_t tree;       /* enum nttk_tree */
  uint32_t layers;     /* 0 = log2 N */
  uint64_t root;       /* 0 = smallest root of the required order */
  uint32_t flags;      /* enum nttk_flags */
} nttk_params_desc;

typedef struct {
  uint64_t p, omega, omega_inv, n_inv, n_inv_hat, mu;
  uint32_t N, log2N, n_bits, layers, tree, kinds_mask, scott_L;
  uint32_t fast_path; /* bit k set = kind k runs on the specialised N=256 kernels */
} nttk_params_info;

/* ---- parameters (params.hpp) -------------------------------------------- */

/* replaces build_params (params.hpp:137-268): validates, collecting every fault into
 * one message; builds every encoded twiddle table on the host and keeps the
 * per-device copies (uploaded lazily, once per device). */
int nttk_build_params(const nttk_params_desc* desc, nttk_params_t* out);
/* replaces preset()/preset_spec() (params.hpp:273-306) */
int nttk_preset(const char* name, nttk_params_t* out);
int nttk_params_destroy(nttk_params_t P);
int nttk_params_get_info(nttk_params_t P, nttk_params_info* out);
/* extension (introspection): the host-validated fast-kernel option bits of (kind, dir)
 * (dir 0 forward, 1 inverse): 1/2 fast canonicalisation (u16 Barrett / u32 shift), 4 fused
 * u16 first merge layer, 8 lazy merge, 16 forward twiddle-1 blocks, 32 inverse twiddle-1
 * blocks (TW1), 64 u16 inverse without canonicalisation (DEFER), 128 u32 inverse partial
 * canonicalisation, 256 (dir 1) the fused polymul runs the kind's lazy Montgomery twin
 * (harvey / smont, n = 16), 512 the direction runs the n = 16 product on an n = 32 improved
 * parameter set (narrow image), 1024 (dir 0) the F1 forward, 2048 (dir 1) the inverse runs the
 * CT-form body (N = 256: Kyber u16 / Dilithium u32 trees; N = 512 / 1024: the narrow image when
 * 20 p lies inside the n = 16 Prop. 4 range).  Status 2 if the kind is not built into P.
 * Process-wide A/B switches read once from the environment (results never change):
 * NTTK_INV_CT=0 keeps the GS-form inverses, NTTK_FWD_F1=0 the umulhi-form Kyber forward,
 * NTTK_POLYMUL_EAGER=1 the standalone policies inside the fused polymul. */
int nttk_params_fast_flags(nttk_params_t P, int kind, int dir, uint32_t* flags);
/* read back a host table (names: dif_w dif_wq dif_mont ct_plain ct_plantard ct_mont
 * ct_smont gs_plain gs_wq gs_mont gs_plantard gs_smont); returns its length */
size_t nttk_params_table(nttk_params_t P, const char* name, uint64_t* out, size_t cap);

/* ---- device entry points (asynchronous on `stream`) ------------------------- */

/* ntt_forward / ntt_forward_inplace (transform.hpp:207-231): natural-order
 * coefficients in, butterfly-order (bit-reversed) lazy spectrum out.  d_in may equal
 * d_out. */
int nttk_ntt_forward(nttk_params_t P, int kind, const void* d_in, void* d_out, size_t batch,
                     int elem_bytes, void* stream);
/* intt_inverse (transform.hpp:233-343): any representative in, canonical natural-
 * order coefficients out (input canonicalised first, N^{-1} / 2^{-layers} last). */
int nttk_intt_inverse(nttk_params_t P, int kind, const void* d_in, void* d_out, size_t batch,
                      int elem_bytes, void* stream);
/* pointwise_multiply (transform.hpp:349-370): slotwise product, canonical output. */
int nttk_pointwise_multiply(nttk_params_t P, int kind, const void* d_lhs, const void* d_rhs,
                            void* d_out, size_t batch, int elem_bytes, void* stream);
/* extension: degree-2 basemul mod (x^2 - gamma_i) for trees ending in degree-2
 * factors (Kyber-style); canonical output. */
int nttk_basemul(nttk_params_t P, int kind, const void* d_lhs, const void* d_rhs, void* d_out,
                 size_t batch, int elem_bytes, void* stream);
/* cyclic_convolution_via_ntt (transform.hpp:372-379) and its negacyclic twin:
 * forward(a), forward(b), pointwise/basemul, inverse.  d_out may alias d_a or d_b. */
int nttk_polymul(nttk_params_t P, int kind, const void* d_a, const void* d_b, void* d_out,
                 size_t batch, int elem_bytes, void* stream);

/* ---- captured plans (small batches) ------------------------------------------
 * Engine extension, no reference counterpart: the reference transforms one polynomial per
 * call (transform.hpp:207-379); a batch of a few thousand polynomials finishes on the B200
 * in microseconds, where the per-call host work (argument checks, launch) dominates.  A plan
 * fixes one operation on fixed device buffers, runs it once (table uploads, checks), and
 * records `repeat` back-to-back copies into a CUDA graph; nttk_plan_launch replays the graph
 * on `stream` (one host call per `repeat` operations).  op: NTTK_PLAN_FORWARD / _INVERSE
 * (d_b unused) or NTTK_PLAN_POLYMUL; same contracts as the device entry points above. */
typedef struct nttk_plan* nttk_plan_t;
enum { NTTK_PLAN_FORWARD = 0, NTTK_PLAN_INVERSE = 1, NTTK_PLAN_POLYMUL = 2 };
int nttk_plan_create(nttk_params_t P, int kind, int op, const void* d_a, const void* d_b,
                     void* d_out, size_t batch, int elem_bytes, int repeat, nttk_plan_t* plan);
int nttk_plan_launch(nttk_plan_t plan, void* stream);
void nttk_plan_destroy(nttk_plan_t plan);

/* ---- host entry points (checked, synchronous) ------------------------------ */

/* ntt_forward (transform.hpp:207-224) on host buffers: rejects non-canonical
 * coefficients with "ntt_forward: coefficients must be canonical". */
int nttk_ntt_forward_host(nttk_params_t P, int kind, const void* h_in, void* h_out,
                          size_t batch, int elem_bytes);
int nttk_intt_inverse_host(nttk_params_t P, int kind, const void* h_in, void* h_out,
                           size_t batch, int elem_bytes);
/* forward then inverse (the bench round trip), one pipelined pass over host memory */
int nttk_roundtrip_host(nttk_params_t P, int kind, const void* h_in, void* h_spec,
                        void* h_out, size_t batch, int elem_bytes);
int nttk_pointwise_multiply_host(nttk_params_t P, int kind, const void* h_lhs,
                                 const void* h_rhs, void* h_out, size_t batch, int elem_bytes);
int nttk_polymul_host(nttk_params_t P, int kind, const void* h_a, const void* h_b, void* h_out,
                      size_t batch, int elem_bytes);

/* ---- reductions (reduction.hpp:125-273) ------------------------------------- */

enum nttk_redc {
  NTTK_REDC_MONT = 0,      /* mont_redc(a*b), a,b in [0,p)           reduction.hpp:125-135 */
  NTTK_REDC_SMONT = 1,     /* signed_mont_redc(a*b)                  reduction.hpp:141-165 */
  NTTK_REDC_PLANTARD = 2,  /* plantard_redc(a, b), a,b in [0,p]      reduction.hpp:178-191 */
  NTTK_REDC_MPLANTARD = 3  /* modified_plantard_mul(a, b)            reduction.hpp:264-273 */
};

/* Sweep one reduction over the operand grid (A[i], B[j]), i < na, j < nb.  Results
 * go to d_r[i*nb + j] (int64, may be NULL to skip the store); *h_checksum receives
 * the wrapping u64 sum of all results (synchronises `stream`).  Operands must lie in
 * the variant's contract range (the reference's checked entry points throw there);
 * the device trusts them.  A scalar reduction is the 1x1 grid. */
int nttk_modmul_sweep(int variant, uint64_t p, uint32_t n_bits, uint32_t ell, const int64_t* d_A,
                      size_t na, const int64_t* d_B, size_t nb, int64_t* d_r,
                      uint64_t* h_checksum, void* stream);
/* Device form of nttk_modmul_sweep: atomically ADDS the wrapping sum into the device
 * word *d_checksum (the caller zeroes it) and returns without synchronising, so sweeps
 * can be queued back to back or captured in a CUDA graph. */
int nttk_modmul_sweep_device(int variant, uint64_t p, uint32_t n_bits, uint32_t ell,
                             const int64_t* d_A, size_t na, const int64_t* d_B, size_t nb,
                             int64_t* d_r, uint64_t* d_checksum, void* stream);
/* ---- observed transforms (transform.hpp:207-217, 233-337) ------------------------ */
/* One polynomial (u64 words), run one layer per launch; after every layer the state is
 * copied back and observer(layer, state, N, user) runs on the calling thread, with layers
 * numbered as the reference's run_split_layers / run_merge_layers number them.  The
 * forward checks its input is canonical ("ntt_forward: coefficients must be canonical"). */
typedef void (*nttk_layer_observer)(unsigned layer, const uint64_t* state, size_t n, void* user);
int nttk_ntt_forward_observed(nttk_params_t P, int kind, const uint64_t* h_in, uint64_t* h_out,
                              nttk_layer_observer observer, void* user);
int nttk_intt_inverse_observed(nttk_params_t P, int kind, const uint64_t* h_in, uint64_t* h_out,
                               nttk_layer_observer observer, void* user);

/* ---- reduction.hpp on arrays (the drop-in behind nttk::mont_redc & co.) ---------- */

/* ReductionContext (reduction.hpp:44-78): every precomputed constant of (p, n, alpha, ell) */
typedef struct nttk_reduction_ctx {
  uint64_t p;
  uint32_t n_bits, alpha, ell, pad_;
  uint64_t beta, beta_mask, r2n_mask;
  uint64_t p_inv_beta, neg_p_inv_beta, mu;
  int64_t mu_centered;
  uint64_t beta_mod_p, r2n_mod_p;
} nttk_reduction_ctx;

/* make_reduction_context (reduction.hpp:80-117): same validation, same messages */
int nttk_make_reduction_context(uint64_t p, uint32_t n_bits, uint32_t alpha, uint32_t ell,
                                nttk_reduction_ctx* out);

enum nttk_reduce_op {
  NTTK_OP_MONT_REDC = 0,              /* x = T in [0, p^2)          reduction.hpp:125-135 */
  NTTK_OP_SIGNED_MONT_REDC = 1,       /* x = A, |A| < p 2^{n-1}     reduction.hpp:141-165 */
  NTTK_OP_PLANTARD_REDC = 2,          /* x = W, y = T in [0, p]     reduction.hpp:178-191 */
  NTTK_OP_MODIFIED_PLANTARD_MUL = 3,  /* x = W < p, y = T < 2^ell p reduction.hpp:264-273 */
  NTTK_OP_TO_PLANTARD_DOMAIN = 4,     /* x = w < p                  reduction.hpp:279-283 */
  NTTK_OP_TO_MONTGOMERY_DOMAIN = 5,   /* x = w < p                  reduction.hpp:287-291 */
  NTTK_OP_MOD_P = 6                   /* x mod p, any 64-bit word   transform.hpp:38-40   */
};

/* out[i] = op(x[i] [, y[i]]) for i < n on device arrays of int64 words (the unsigned ops
 * read them as uint64).  The context bound of the op and every operand are checked like the
 * reference's NTTK_REQUIRE; a violation returns NTTK_CONTRACT with the reference's message
 * (operands are checked on the device: the call synchronises `stream`). */
int nttk_reduce(int op, const nttk_reduction_ctx* ctx, const int64_t* d_x, const int64_t* d_y,
                int64_t* d_out, size_t n, void* stream);
/* same on host arrays (staged through the device; synchronous) */
int nttk_reduce_host(int op, const nttk_reduction_ctx* ctx, const int64_t* h_x, const int64_t* h_y,
                     int64_t* h_out, size_t n);

/* ---- butterfly.hpp checked entry points on arrays ------------------------------ */
enum nttk_butterfly_op {
  NTTK_BF_NTL = 0,          /* ntl_butterfly(X, Y, W, W_quot)        butterfly.hpp:60-86   */
  NTTK_BF_HARVEY = 1,       /* harvey_butterfly(X, Y, W_mont)        butterfly.hpp:92-121  */
  NTTK_BF_SCOTT = 2,        /* scott_butterfly(X, Y, W_mont, cfg)    butterfly.hpp:172-212 */
  NTTK_BF_IMPROVED_CT = 3,  /* improved_ct_butterfly(X, Y, W_hat)    butterfly.hpp:247-260 */
  NTTK_BF_IMPROVED_GS = 4   /* improved_gs_butterfly(X, Y, W_hat, l) butterfly.hpp:263-279 */
};
/* (xo[i], yo[i]) = op(x[i], y[i], w[i] [, wq[i] for ntl]) on device arrays.  aux0/aux1:
 * scott transform_size N and lazy_level L (ScottConfig); improved GS: layer (aux0).  The
 * reference's context and operand checks are applied (operands on the device; the call
 * synchronises `stream`), with its messages. */
int nttk_butterfly(int op, const nttk_reduction_ctx* ctx, uint32_t aux0, uint32_t aux1,
                   const int64_t* d_x, const int64_t* d_y, const int64_t* d_w, const int64_t* d_wq,
                   int64_t* d_xo, int64_t* d_yo, size_t n, void* stream);
/* same on host arrays (synchronous) */
int nttk_butterfly_host(int op, const nttk_reduction_ctx* ctx, uint32_t aux0, uint32_t aux1,
                        const int64_t* h_x, const int64_t* h_y, const int64_t* h_w,
                        const int64_t* h_wq, int64_t* h_xo, int64_t* h_yo, size_t n);

/* ---- diagnostics ------------------------------------------------------------ */

/* message of the last failing call on this host thread ("" when none) */
const char* nttk_last_error(void);
/* number of kernel launches issued by this process so far (bench gpu_launches) */
uint64_t nttk_launch_count(void);
/* replaces plantard_correction_fires() (reduction.hpp:172-175): how often plantard_redc's
 * r == p corner (reduction.hpp:186-189) has fired in this process, counted on the device by
 * nttk_reduce / nttk_reduce_host (NTTK_OP_PLANTARD_REDC) and the synchronous
 * nttk_modmul_sweep (NTTK_REDC_PLANTARD); the throughput form nttk_modmul_sweep_device does
 * not count */
uint64_t nttk_plantard_correction_fires(void);
/* 1 when a CUDA device is usable, else 0 (the engine has no CPU fallback) */
int nttk_device_available(void);
/* version string of the engine */
const char* nttk_version(void);

#ifdef __cplusplus
}
#endif
#endif
