// abi.cpp -- the extern "C" boundary of libnttk_gpu.so (include/nttk_gpu.h).
//
// Dispatches every entry point to the sm_100a kernels: the specialised N = 256
// kernels (fast256.cu) when the parameter set qualifies, the any-parameter kernels
// (generic.cu) otherwise.  No exception crosses this boundary; the reference's
// contract_violation messages (transform.hpp / params.hpp / reduction.hpp) come back
// through nttk_last_error() with status 2.  There is no CPU compute path: every
// transform, product and reduction runs on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/nttk_gpu.h"
#include "fast256.hpp"
#include "fastn.hpp"
#include "generic.hpp"
#include "product.hpp"
#include "params.hpp"
#include "reduce.hpp"
#include "sweep.hpp"

struct nttk_params_s {
  nttk_b200::HostParams P;
};

using nttk_b200::HostParams;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};
// plantard_redc's r == p corner, as the reference counts it (reduction.hpp:172-191)
std::atomic<uint64_t> g_plantard_fires{0};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(NTTK_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

int device_count() {  // probed once per process (the device set does not change)
  static const int n = [] {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    return c;
  }();
  return n;
}

int need_device(const char* who) {
  if (device_count() <= 0)
    return fail(NTTK_CUDA, std::string(who) + ": no CUDA device (the engine has no CPU path)");
  return NTTK_OK;
}

const char* kind_name(int k) {
  static const char* names[] = {"ntl", "harvey", "scott", "improved", "smont"};
  return (k >= 0 && k < 5) ? names[k] : "?";
}

int check_kind(const HostParams& P, int kind, const char* who) {
  if (kind < 0 || kind > NTTK_SMONT || !((P.kinds >> kind) & 1u))
    return fail(NTTK_CONTRACT, std::string(who) + ": kind not built into these params");
  return NTTK_OK;
}

// Forward spectrum range per kind (transform.hpp:61-70, plus the extension kinds):
// values lie in [lo, hi).
void spectrum_range(const HostParams& P, int kind, int64_t& lo, uint64_t& hi) {
  lo = 0;
  switch (kind) {
    case NTTK_NTL: hi = P.p; break;
    case NTTK_HARVEY: hi = 2ull * P.p; break;
    case NTTK_SCOTT:
      // N p when no T = X + (N/L) p - Y underflows (offset >= 2^{layers-1} p); otherwise the
      // reference's uint64 words wrap (e.g. Kyber at n = 16) and only
      // 64-bit storage holds them
      hi = P.scott_L && uint64_t(P.N / P.scott_L) * P.p >= (uint64_t(P.p) << (P.layers - 1))
               ? uint64_t(P.N) * P.p
               : ~uint64_t(0);
      break;
    case NTTK_IMPROVED: hi = uint64_t(P.layers + 1) * P.p; break;
    default:  // smont: X + t / X - t growth from [0, p)
      hi = uint64_t(P.layers + 1) * P.p;
      lo = -static_cast<int64_t>(P.layers) * static_cast<int64_t>(P.p);
  }
}

int check_storage(const HostParams& P, int kind, int elem, const char* who) {
  if (elem != 2 && elem != 4 && elem != 8)
    return fail(NTTK_CONTRACT, std::string(who) + ": elem_bytes must be 2, 4 or 8");
  if (elem == 8) return NTTK_OK;
  int64_t lo;
  uint64_t hi;
  spectrum_range(P, kind, lo, hi);
  const bool sgn = kind == NTTK_SMONT;
  const unsigned bits = 8 * elem;
  const bool ok = sgn ? (lo >= -(int64_t(1) << (bits - 1)) && hi <= (uint64_t(1) << (bits - 1)))
                      : hi <= (uint64_t(1) << bits);
  if (!ok)
    return fail(NTTK_CONTRACT, std::string(who) + ": elem_bytes=" + std::to_string(elem) +
                                   " cannot hold the " + kind_name(kind) + " spectrum bound");
  return NTTK_OK;
}

// canonical outputs (inverse, products) must fit the storage width
int check_canonical_storage(const HostParams& P, int elem, const char* who) {
  if (elem != 2 && elem != 4 && elem != 8)
    return fail(NTTK_CONTRACT, std::string(who) + ": elem_bytes must be 2, 4 or 8");
  if (elem < 8 && uint64_t(P.p) > (uint64_t(1) << (8 * elem)))
    return fail(NTTK_CONTRACT, std::string(who) + ": elem_bytes=" + std::to_string(elem) +
                                   " cannot hold canonical coefficients of p=" + std::to_string(P.p));
  return NTTK_OK;
}

bool aligned16(const void* p) { return !(reinterpret_cast<uintptr_t>(p) & 15); }

bool use_fast(const HostParams& P, int kind) {
  if (!((P.fast_mask >> kind) & 1u)) return false;
  if (P.N != 256) return true;  // fastn_tma.cu (N = 512 / 1024, full trees; fast_eligible)
  return nttk_b200::fast256_supports(kind, P.layers, P.n_bits);
}

// one fused kernel for fwd(a), fwd(b), product, inverse (polymul_tma.cu); NTTK_KERNEL=v1
// keeps the four-kernel composition for A/B runs
bool use_fused_polymul(const HostParams& P, int kind, int elem, const void* a, const void* b,
                       const void* out) {
  static const bool v1 = [] {
    const char* k = std::getenv("NTTK_KERNEL");
    return k && std::string(k) == "v1";
  }();
  // ntl / scott: no fused product stage (config 2 compares improved, harvey, smont); their
  // polymul runs fwd, fwd, pointwise, inv as four kernels
  if (v1 || P.N != 256 || !use_fast(P, kind) || kind == NTTK_NTL || kind == NTTK_SCOTT) return false;
  return nttk_b200::fast256_tma_supports(elem, a, out) && !(reinterpret_cast<uintptr_t>(b) & 15);
}

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

// one transform pass on device buffers
int run_transform(const HostParams& P, int kind, int dir, const void* in, void* out, size_t batch,
                  int elem, cudaStream_t st) {
  cudaError_t e;
  if (P.N != 256 && use_fast(P, kind) && nttk_b200::fastn_supports(P, elem, in, out)) {
    std::string err;
    const uint32_t* tab = P.fastn_table(current_device(), P.image(kind, dir), dir, err);
    if (!tab) return fail(NTTK_CUDA, err);
    e = nttk_b200::fastn_launch(P, kind, dir, in, out, batch, elem, tab, st);
    g_launches += batch ? 1 : 0;
  } else if (P.N == 256 && use_fast(P, kind) && aligned16(in) && aligned16(out)) {
    // both N = 256 kernels read and write 16-byte vectors: misaligned buffers take the
    // generic kernel
    // NTTK_KERNEL=v1 selects the register-prefetch kernels (A/B comparisons)
    static const bool v1 = [] {
      const char* k = std::getenv("NTTK_KERNEL");
      return k && std::string(k) == "v1";
    }();
    if (!v1 && nttk_b200::fast256_tma_supports(elem, in, out))
      e = nttk_b200::fast256_tma_launch(P, kind, dir, in, out, batch, elem, st);
    else
      e = nttk_b200::fast256_launch(P, kind, dir, in, out, batch, elem, st);
    g_launches += batch ? 1 : 0;
  } else {
    std::string err;
    const nttk_b200::DeviceTables* T = P.device_tables(current_device(), err);
    if (!T) return fail(NTTK_CUDA, err);
    e = nttk_b200::generic_transform(P, *T, kind, dir, in, out, batch, elem, st);
    if (batch) g_launches += P.N <= 4096 ? 1 : P.layers + 2;
  }
  if (e != cudaSuccess) return cuda_fail(e, dir ? "intt_inverse" : "ntt_forward");
  return NTTK_OK;
}

int run_product(const HostParams& P, int kind, const void* l, const void* r, void* out,
                size_t batch, int elem, cudaStream_t st) {
  cudaError_t e;
  const bool basemul = (P.N >> P.layers) == 2;
  if (nttk_b200::product_supports(P, kind, basemul, elem, l, r, out)) {
    e = nttk_b200::product_launch(P, kind, basemul, l, r, out, batch, elem, st);
  } else if (basemul) {
    std::string err;
    const nttk_b200::DeviceTables* T = P.device_tables(current_device(), err);
    if (!T) return fail(NTTK_CUDA, err);
    e = nttk_b200::generic_basemul(P, T->gamma, kind, l, r, out, batch, elem, st);
  } else {
    e = nttk_b200::generic_pointwise(P, kind, l, r, out, batch, elem, st);
  }
  if (batch) ++g_launches;
  if (e != cudaSuccess) return cuda_fail(e, "pointwise_multiply");
  return NTTK_OK;
}

// ---- host pipeline: chunked H2D -> kernels -> D2H over three streams ----------

struct Workspace {
  std::mutex mu;
  int device = -1;
  cudaStream_t st[3] = {};
  cudaEvent_t ev[3] = {};  // stream joins (no timing)
  void* buf[3][3] = {};
  size_t cap = 0;  // bytes per buffer
  unsigned* d_flag = nullptr;
  unsigned* h_flag = nullptr;  // pinned: the flag read stays asynchronous until the one sync
};

Workspace* workspace(int dev) {
  static std::mutex m;
  static std::unique_ptr<Workspace> ws[64];
  std::lock_guard<std::mutex> lock(m);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!ws[dev]) {
    auto w = std::make_unique<Workspace>();
    w->device = dev;
    for (auto& s : w->st)
      if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    for (auto& e : w->ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    if (cudaMalloc(&w->d_flag, sizeof(unsigned)) != cudaSuccess) return nullptr;
    if (cudaMallocHost(&w->h_flag, sizeof(unsigned)) != cudaSuccess) return nullptr;
    ws[dev] = std::move(w);
  }
  return ws[dev].get();
}

int ensure_cap(Workspace& W, size_t bytes) {
  if (W.cap >= bytes) return NTTK_OK;
  cudaDeviceSynchronize();
  for (auto& row : W.buf)
    for (auto& b : row)
      if (b) {
        cudaFree(b);
        b = nullptr;
      }
  W.cap = 0;
  for (auto& row : W.buf)
    for (auto& b : row) {
      cudaError_t e = cudaMalloc(&b, bytes);
      if (e != cudaSuccess) return cuda_fail(e, "workspace");
    }
  W.cap = bytes;
  return NTTK_OK;
}

constexpr size_t kChunkBytes = size_t(64) << 20;

// compute(stream, dev bufs[3], chunk polys) issues the kernels for one chunk;
// inputs land in bufs[0..n_in), outputs are read from out_slot[i]; input i is checked
// against `bound` on the device when bit i of check_mask is set
template <class F>
int host_pipeline(const HostParams& P, int elem, size_t batch, const std::vector<const void*>& h_in,
                  const std::vector<std::pair<void*, int>>& h_out, F compute, const char* who,
                  unsigned check_mask, uint64_t bound) {
  if (int s = need_device(who)) return s;
  Workspace* W = workspace(current_device());
  if (!W) return fail(NTTK_CUDA, std::string(who) + ": workspace setup failed");
  std::lock_guard<std::mutex> lock(W->mu);
  const size_t poly_bytes = size_t(P.N) * elem;
  size_t chunk = std::max<size_t>(1, kChunkBytes / poly_bytes);
  if (chunk > batch) chunk = batch ? batch : 1;
  if (int s = ensure_cap(*W, chunk * poly_bytes)) return s;
  // only as many streams as chunks; stream 0 clears the flag, the others wait for it
  const size_t nchunks = (batch + chunk - 1) / chunk;
  const int nst = nchunks < 3 ? static_cast<int>(nchunks ? nchunks : 1) : 3;
  cudaError_t e = cudaMemsetAsync(W->d_flag, 0, sizeof(unsigned), W->st[0]);
  if (e == cudaSuccess && nst > 1) e = cudaEventRecord(W->ev[0], W->st[0]);
  for (int i = 1; i < nst && e == cudaSuccess; ++i) e = cudaStreamWaitEvent(W->st[i], W->ev[0], 0);
  if (e != cudaSuccess) return cuda_fail(e, who);
  size_t k = 0;
  for (size_t done = 0; done < batch; done += chunk, ++k) {
    const size_t n = std::min(chunk, batch - done);
    const int s = static_cast<int>(k % nst);
    cudaStream_t st = W->st[s];
    for (size_t i = 0; i < h_in.size(); ++i) {
      e = cudaMemcpyAsync(W->buf[s][i], static_cast<const char*>(h_in[i]) + done * poly_bytes,
                          n * poly_bytes, cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return cuda_fail(e, who);
      if ((check_mask >> i) & 1) {  // bound-checked inputs (check_mask bit i = input i)
        e = nttk_b200::check_canonical(W->buf[s][i], n * P.N, elem, bound, W->d_flag, st);
        ++g_launches;
        if (e != cudaSuccess) return cuda_fail(e, who);
      }
    }
    if (int rc = compute(st, W->buf[s], n)) return rc;
    for (const auto& o : h_out) {
      if (!o.first) continue;
      e = cudaMemcpyAsync(static_cast<char*>(o.first) + done * poly_bytes, W->buf[s][o.second],
                          n * poly_bytes, cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return cuda_fail(e, who);
    }
  }
  // join the other streams into stream 0, read the flag there, one host sync
  for (int i = 1; i < nst && e == cudaSuccess; ++i) {
    e = cudaEventRecord(W->ev[i], W->st[i]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(W->st[0], W->ev[i], 0);
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(W->h_flag, W->d_flag, sizeof(unsigned), cudaMemcpyDeviceToHost, W->st[0]);
  if (e == cudaSuccess) e = cudaStreamSynchronize(W->st[0]);
  if (e != cudaSuccess) return cuda_fail(e, who);
  if (*W->h_flag) return NTTK_PROPERTY;  // caller turns it into its contract message
  return NTTK_OK;
}

}  // namespace

extern "C" {

const char* nttk_last_error(void) { return g_err.c_str(); }
uint64_t nttk_launch_count(void) { return g_launches.load(); }
uint64_t nttk_plantard_correction_fires(void) { return g_plantard_fires.load(); }
int nttk_device_available(void) { return device_count() > 0 ? 1 : 0; }
const char* nttk_version(void) { return "nttk-b200 0.1 (sm_100a)"; }

int nttk_build_params(const nttk_params_desc* desc, nttk_params_t* out) {
  if (!desc || !out) return fail(NTTK_CONTRACT, "build_params: null argument");
  try {
    auto h = std::make_unique<nttk_params_s>();
    std::string err;
    const int st = nttk_b200::build_params(*desc, h->P, err);
    if (st != NTTK_OK) return fail(st, err);
    *out = h.release();
    return NTTK_OK;
  } catch (const std::exception& e) {
    return fail(NTTK_CONTRACT, e.what());
  }
}

int nttk_preset(const char* name, nttk_params_t* out) {
  nttk_params_desc d;
  std::string err;
  if (nttk_b200::preset_desc(name ? name : "", d, err) != NTTK_OK) return fail(NTTK_CONTRACT, err);
  return nttk_build_params(&d, out);
}

int nttk_params_destroy(nttk_params_t P) {
  delete P;
  return NTTK_OK;
}

int nttk_params_get_info(nttk_params_t h, nttk_params_info* o) {
  if (!h || !o) return fail(NTTK_CONTRACT, "params_get_info: null argument");
  const HostParams& P = h->P;
  o->p = P.p;
  o->omega = P.omega;
  o->omega_inv = P.omega_inv;
  o->n_inv = P.n_inv;
  o->n_inv_hat = P.n_inv_hat;
  o->mu = P.ctx.mu;
  o->N = P.N;
  o->log2N = P.log2N;
  o->n_bits = P.n_bits;
  o->layers = P.layers;
  o->tree = P.tree;
  o->kinds_mask = P.kinds;
  o->scott_L = P.scott_L;
  o->fast_path = 0;
  for (int k = 0; k < 5; ++k)
    if (((P.kinds >> k) & 1u) && use_fast(P, k)) o->fast_path |= 1u << k;
  return NTTK_OK;
}

int nttk_params_fast_flags(nttk_params_t h, int kind, int dir, uint32_t* flags) {
  if (!h || !flags) return fail(NTTK_CONTRACT, "params_fast_flags: null argument");
  if (dir != 0 && dir != 1) return fail(NTTK_CONTRACT, "params_fast_flags: dir must be 0 or 1");
  if (int s = check_kind(h->P, kind, "params_fast_flags")) return s;
  const int img = h->P.image(kind, dir);
  *flags = h->P.fast[kind][dir].flags | (img == nttk_b200::kNarrow ? 512u : 0u) |
           (img == nttk_b200::kCtN ? 512u | 2048u : 0u) |
           (kind == NTTK_IMPROVED && dir == 1 && (h->P.ct_inv || h->P.ct_inv_c) ? 2048u : 0u);
  return NTTK_OK;
}

size_t nttk_params_table(nttk_params_t h, const char* name, uint64_t* out, size_t cap) {
  if (!h || !name) return 0;
  const HostParams& P = h->P;
  const std::string n = name;
  std::vector<uint64_t> tmp;
  const std::vector<uint64_t>* v = nullptr;
  if (n == "dif_w") v = &P.dif_w;
  else if (n == "dif_wq") v = &P.dif_wq;
  else if (n == "dif_mont") v = &P.dif_mont;
  else if (n == "ct_plain") v = &P.ct_plain;
  else if (n == "ct_plantard") v = &P.ct_plantard;
  else if (n == "ct_mont") v = &P.ct_mont;
  else if (n == "gs_plain") v = &P.gs_plain;
  else if (n == "gs_wq") v = &P.gs_wq;
  else if (n == "gs_mont") v = &P.gs_mont;
  else if (n == "gs_plantard") v = &P.gs_plantard;
  else if (n == "gamma") v = &P.gamma;
  else if (n == "ct_smont" || n == "gs_smont") {
    for (int64_t x : (n == "ct_smont" ? P.ct_smont : P.gs_smont))
      tmp.push_back(static_cast<uint64_t>(x));
    v = &tmp;
  }
  if (!v) return 0;
  if (out) std::memcpy(out, v->data(), std::min(cap, v->size()) * 8);
  return v->size();
}

// ---- device entry points ---------------------------------------------------

int nttk_ntt_forward(nttk_params_t h, int kind, const void* d_in, void* d_out, size_t batch,
                     int elem, void* stream) {
  if (!h) return fail(NTTK_CONTRACT, "ntt_forward: null params");
  if (int s = check_kind(h->P, kind, "ntt_forward")) return s;
  if (int s = check_storage(h->P, kind, elem, "ntt_forward")) return s;
  if (int s = need_device("ntt_forward")) return s;
  return run_transform(h->P, kind, 0, d_in, d_out, batch, elem, static_cast<cudaStream_t>(stream));
}

int nttk_intt_inverse(nttk_params_t h, int kind, const void* d_in, void* d_out, size_t batch,
                      int elem, void* stream) {
  if (!h) return fail(NTTK_CONTRACT, "intt_inverse: null params");
  if (int s = check_kind(h->P, kind, "intt_inverse")) return s;
  if (int s = check_canonical_storage(h->P, elem, "intt_inverse")) return s;
  if (int s = need_device("intt_inverse")) return s;
  return run_transform(h->P, kind, 1, d_in, d_out, batch, elem, static_cast<cudaStream_t>(stream));
}

int nttk_pointwise_multiply(nttk_params_t h, int kind, const void* d_l, const void* d_r,
                            void* d_out, size_t batch, int elem, void* stream) {
  if (!h) return fail(NTTK_CONTRACT, "pointwise_multiply: null params");
  if (int s = check_kind(h->P, kind, "pointwise_multiply")) return s;
  if (int s = check_canonical_storage(h->P, elem, "pointwise_multiply")) return s;
  if (int s = need_device("pointwise_multiply")) return s;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = nttk_b200::product_supports(h->P, kind, false, elem, d_l, d_r, d_out)
                      ? nttk_b200::product_launch(h->P, kind, false, d_l, d_r, d_out, batch, elem, st)
                      : nttk_b200::generic_pointwise(h->P, kind, d_l, d_r, d_out, batch, elem, st);
  if (batch) ++g_launches;
  if (e != cudaSuccess) return cuda_fail(e, "pointwise_multiply");
  return NTTK_OK;
}

int nttk_basemul(nttk_params_t h, int kind, const void* d_l, const void* d_r, void* d_out,
                 size_t batch, int elem, void* stream) {
  if (!h) return fail(NTTK_CONTRACT, "basemul: null params");
  if (int s = check_kind(h->P, kind, "basemul")) return s;
  if ((h->P.N >> h->P.layers) != 2)
    return fail(NTTK_CONTRACT, "basemul: tree must end in degree-2 factors");
  if (int s = check_canonical_storage(h->P, elem, "basemul")) return s;
  if (int s = need_device("basemul")) return s;
  return run_product(h->P, kind, d_l, d_r, d_out, batch, elem, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

namespace {
// forward(a), forward(b), product, inverse: the fused kernel when eligible, else four
// passes at the storage width, else -- when only canonical words fit the width (e.g. the
// improved spectrum of q = 12289 in 16 bits) -- the same passes on u64 copies
int run_polymul(const HostParams& P, int kind, const void* a, const void* b, void* out,
                size_t batch, int elem, cudaStream_t st) {
  if (use_fused_polymul(P, kind, elem, a, b, out)) {
    cudaError_t e = nttk_b200::polymul256_launch(P, kind, a, b, out, batch, elem, st);
    ++g_launches;
    return e == cudaSuccess ? int(NTTK_OK) : cuda_fail(e, "polymul");
  }
  const std::string keep = g_err;
  const bool narrow_ok = check_storage(P, kind, elem, "polymul") == NTTK_OK;
  g_err = keep;  // a failed width probe is not an error of this call
  const int w = narrow_ok ? elem : 8;
  const size_t n = batch * P.N;
  char* tmp = nullptr;
  cudaError_t e = cudaMallocAsync(&tmp, n * size_t(w) * (narrow_ok ? 1 : 3), st);
  if (e != cudaSuccess) return cuda_fail(e, "polymul");
  const void* A = a;
  const void* Bv = b;
  void* O = out;
  void* T = tmp;
  if (!narrow_ok) {  // u64 copies: a -> O (in place), b -> B64, temp
    uint64_t* o64 = reinterpret_cast<uint64_t*>(tmp);
    uint64_t* b64 = o64 + n;
    e = nttk_b200::widen_to_u64(a, elem, o64, n, st);
    if (e == cudaSuccess) e = nttk_b200::widen_to_u64(b, elem, b64, n, st);
    g_launches += 2;
    if (e != cudaSuccess) {
      cudaFreeAsync(tmp, st);
      return cuda_fail(e, "polymul");
    }
    A = o64;
    Bv = b64;
    O = o64;
    T = b64 + n;
  }
  int rc = run_transform(P, kind, 0, Bv, T, batch, w, st);
  if (!rc) rc = run_transform(P, kind, 0, A, O, batch, w, st);
  if (!rc) rc = run_product(P, kind, O, T, O, batch, w, st);
  if (!rc) rc = run_transform(P, kind, 1, O, O, batch, w, st);
  if (!rc && !narrow_ok) {
    e = nttk_b200::narrow_from_u64(reinterpret_cast<const uint64_t*>(O), out, elem, n, st);
    ++g_launches;
    if (e != cudaSuccess) rc = cuda_fail(e, "polymul");
  }
  cudaFreeAsync(tmp, st);
  return rc;
}
}  // namespace

extern "C" {

int nttk_polymul(nttk_params_t h, int kind, const void* d_a, const void* d_b, void* d_out,
                 size_t batch, int elem, void* stream) {
  if (!h) return fail(NTTK_CONTRACT, "polymul: null params");
  const HostParams& P = h->P;
  if (int s = check_kind(P, kind, "polymul")) return s;
  if (elem != 2 && elem != 4 && elem != 8)
    return fail(NTTK_CONTRACT, "polymul: elem_bytes must be 2, 4 or 8");
  if (int s = check_canonical_storage(P, elem, "polymul")) return s;
  if (int s = need_device("polymul")) return s;
  if (!batch) return NTTK_OK;
  return run_polymul(P, kind, d_a, d_b, d_out, batch, elem, static_cast<cudaStream_t>(stream));
}

// ---- host entry points ----------------------------------------------------------

int nttk_ntt_forward_host(nttk_params_t h, int kind, const void* h_in, void* h_out, size_t batch,
                          int elem) {
  if (!h) return fail(NTTK_CONTRACT, "ntt_forward: null params");
  const HostParams& P = h->P;
  if (int s = check_kind(P, kind, "ntt_forward")) return s;
  if (int s = check_storage(P, kind, elem, "ntt_forward")) return s;
  const int rc = host_pipeline(
      P, elem, batch, {h_in}, {{h_out, 1}},
      [&](cudaStream_t st, void** b, size_t n) { return run_transform(P, kind, 0, b[0], b[1], n, elem, st); },
      "ntt_forward", 1u, P.p);
  if (rc == NTTK_PROPERTY) return fail(NTTK_CONTRACT, "ntt_forward: coefficients must be canonical");
  return rc;
}

int nttk_intt_inverse_host(nttk_params_t h, int kind, const void* h_in, void* h_out, size_t batch,
                           int elem) {
  if (!h) return fail(NTTK_CONTRACT, "intt_inverse: null params");
  const HostParams& P = h->P;
  if (int s = check_kind(P, kind, "intt_inverse")) return s;
  if (int s = check_canonical_storage(P, elem, "intt_inverse")) return s;
  return host_pipeline(
      P, elem, batch, {h_in}, {{h_out, 1}},
      [&](cudaStream_t st, void** b, size_t n) { return run_transform(P, kind, 1, b[0], b[1], n, elem, st); },
      "intt_inverse", 0u, 0);
}

int nttk_roundtrip_host(nttk_params_t h, int kind, const void* h_in, void* h_spec, void* h_out,
                        size_t batch, int elem) {
  if (!h) return fail(NTTK_CONTRACT, "roundtrip: null params");
  const HostParams& P = h->P;
  if (int s = check_kind(P, kind, "ntt_forward")) return s;
  if (int s = check_storage(P, kind, elem, "ntt_forward")) return s;
  const int rc = host_pipeline(
      P, elem, batch, {h_in}, {{h_spec, 1}, {h_out, 2}},
      [&](cudaStream_t st, void** b, size_t n) {
        int r = run_transform(P, kind, 0, b[0], b[1], n, elem, st);
        if (!r) r = run_transform(P, kind, 1, b[1], b[2], n, elem, st);
        return r;
      },
      "roundtrip", 1u, P.p);
  if (rc == NTTK_PROPERTY) return fail(NTTK_CONTRACT, "ntt_forward: coefficients must be canonical");
  return rc;
}

int nttk_pointwise_multiply_host(nttk_params_t h, int kind, const void* h_l, const void* h_r,
                                 void* h_out, size_t batch, int elem) {
  if (!h) return fail(NTTK_CONTRACT, "pointwise_multiply: null params");
  const HostParams& P = h->P;
  if (int s = check_kind(P, kind, "pointwise_multiply")) return s;
  if (int s = check_canonical_storage(P, elem, "pointwise_multiply")) return s;
  // the improved product consumes a lazy right operand below 2^ell p
  // (modified_plantard_mul's contract, reduction.hpp:264-273); the left operand is reduced
  // mod p first (transform.hpp:362-365), so only the right one (input 0) is bound-checked
  const unsigned chk = kind == NTTK_IMPROVED ? 1u : 0u;
  const uint64_t bound = uint64_t(P.p) << P.log2N;
  const int rc = host_pipeline(
      P, elem, batch, {h_r, h_l}, {{h_out, 2}},
      [&](cudaStream_t st, void** b, size_t n) { return run_product(P, kind, b[1], b[0], b[2], n, elem, st); },
      "pointwise_multiply", chk, bound);
  if (rc == NTTK_PROPERTY)
    return fail(NTTK_CONTRACT, "modified_plantard_mul: T must be < 2^ell * p");
  return rc;
}

int nttk_polymul_host(nttk_params_t h, int kind, const void* h_a, const void* h_b, void* h_out,
                      size_t batch, int elem) {
  if (!h) return fail(NTTK_CONTRACT, "polymul: null params");
  const HostParams& P = h->P;
  if (int s = check_kind(P, kind, "polymul")) return s;
  if (elem != 2 && elem != 4 && elem != 8)
    return fail(NTTK_CONTRACT, "polymul: elem_bytes must be 2, 4 or 8");
  if (int s = check_canonical_storage(P, elem, "polymul")) return s;
  const int rc = host_pipeline(
      P, elem, batch, {h_a, h_b}, {{h_out, 2}},
      [&](cudaStream_t st, void** b, size_t n) {
        return run_polymul(P, kind, b[0], b[1], b[2], n, elem, st);
      },
      "polymul", 3u, P.p);
  if (rc == NTTK_PROPERTY) return fail(NTTK_CONTRACT, "ntt_forward: coefficients must be canonical");
  return rc;
}

// ---- reductions -------------------------------------------------------------------

static int sweep_check(int variant, uint64_t p, uint32_t n_bits, uint32_t ell) {
  if (variant < NTTK_REDC_MONT || variant > NTTK_REDC_MPLANTARD)
    return fail(NTTK_CONTRACT, "modmul_sweep: unknown reduction variant");
  if (n_bits < 2 || n_bits > 32)
    return fail(NTTK_CONTRACT, "reduction context: word size n must be in [2, 32]");
  if (p < 3 || !(p & 1)) return fail(NTTK_CONTRACT, "reduction context: p must be odd and >= 3");
  if (p >= (uint64_t(1) << n_bits)) return fail(NTTK_CONTRACT, "reduction context: p must be < 2^n");
  if (ell >= n_bits) return fail(NTTK_CONTRACT, "reduction context: ell must be < n");
  using nttk_b200::u128;
  // per-variant context bounds (reduction.hpp:64-77)
  if (variant == NTTK_REDC_SMONT && !(u128(2) * p < (u128(1) << n_bits)))
    return fail(NTTK_CONTRACT, "signed_mont_redc: requires 2p < 2^n");
  if (variant == NTTK_REDC_PLANTARD) {
    const u128 d = (u128(1) << (n_bits + 1)) - p;
    if (!(u128(5) * p * p < d * d)) return fail(NTTK_CONTRACT, "plantard_redc: requires p*phi < 2^n");
  }
  if (variant == NTTK_REDC_MPLANTARD &&
      !(ell + 2 < n_bits && u128(p) < (u128(1) << (n_bits - ell - 2))))
    return fail(NTTK_CONTRACT, "modified_plantard_mul: requires p < 2^{n-ell-2}");
  return need_device("modmul_sweep");
}

int nttk_modmul_sweep_device(int variant, uint64_t p, uint32_t n_bits, uint32_t ell,
                             const int64_t* d_A, size_t na, const int64_t* d_B, size_t nb,
                             int64_t* d_r, uint64_t* d_checksum, void* stream) {
  if (int s = sweep_check(variant, p, n_bits, ell)) return s;
  if (!d_checksum) return fail(NTTK_CONTRACT, "modmul_sweep: null checksum accumulator");
  const nttk_b200::Ctx c = nttk_b200::make_ctx(p, n_bits, ell);
  cudaError_t e = nttk_b200::sweep_launch(variant, c, d_A, na, d_B, nb, d_r,
                                          reinterpret_cast<unsigned long long*>(d_checksum),
                                          static_cast<cudaStream_t>(stream));
  ++g_launches;
  if (e != cudaSuccess) return cuda_fail(e, "modmul_sweep");
  return NTTK_OK;
}

int nttk_modmul_sweep(int variant, uint64_t p, uint32_t n_bits, uint32_t ell, const int64_t* d_A,
                      size_t na, const int64_t* d_B, size_t nb, int64_t* d_r,
                      uint64_t* h_checksum, void* stream) {
  if (int s = sweep_check(variant, p, n_bits, ell)) return s;
  const nttk_b200::Ctx c = nttk_b200::make_ctx(p, n_bits, ell);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long* d_sum = nullptr;  // [0] checksum, [1] plantard corner count
  cudaError_t e = cudaMallocAsync(&d_sum, 2 * sizeof(unsigned long long), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_sum, 0, 2 * sizeof(unsigned long long), st);
  // the synchronous form counts plantard_redc's r == p corner (plantard_correction_fires,
  // reduction.hpp:172-191); the throughput form nttk_modmul_sweep_device does not
  if (e == cudaSuccess)
    e = nttk_b200::sweep_launch(variant, c, d_A, na, d_B, nb, d_r, d_sum, st,
                                variant == NTTK_REDC_PLANTARD ? d_sum + 1 : nullptr);
  ++g_launches;
  unsigned long long sum[2] = {};
  if (e == cudaSuccess) e = cudaMemcpyAsync(sum, d_sum, sizeof sum, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (d_sum) cudaFreeAsync(d_sum, st);
  if (e != cudaSuccess) return cuda_fail(e, "modmul_sweep");
  g_plantard_fires += sum[1];
  if (h_checksum) *h_checksum = sum[0];
  return NTTK_OK;
}

// transform.hpp:207-217, 233-337 (observed transforms): one polynomial through the
// generic per-layer kernel, observer called after every layer
static int observed(nttk_params_t h, int kind, int dir, const uint64_t* h_in, uint64_t* h_out,
                    nttk_layer_observer obs, void* user) {
  const char* who = dir ? "intt_inverse" : "ntt_forward";
  if (!h) return fail(NTTK_CONTRACT, std::string(who) + ": null params");
  if (int s = check_kind(h->P, kind, who)) return s;
  if (!h_in || !h_out) return fail(NTTK_CONTRACT, std::string(who) + ": null buffer");
  const HostParams& P = h->P;
  if (dir == 0)
    for (uint32_t i = 0; i < P.N; ++i)  // contract check of the reference (input words)
      if (h_in[i] >= P.p) return fail(NTTK_CONTRACT, "ntt_forward: coefficients must be canonical");
  if (int s = need_device(who)) return s;
  std::string err;
  const nttk_b200::DeviceTables* T = P.device_tables(current_device(), err);
  if (!T) return fail(NTTK_CUDA, err);
  cudaStream_t st = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  uint64_t* d = nullptr;
  uint64_t* hs = nullptr;
  const size_t bytes = size_t(P.N) * 8;
  if (e == cudaSuccess) e = cudaMallocAsync(&d, bytes, st);
  if (e == cudaSuccess) e = cudaMallocHost(&hs, bytes);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d, h_in, bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = nttk_b200::generic_transform_observed(
        P, *T, kind, dir, d, hs,
        [&](unsigned layer) {
          if (obs) obs(layer, hs, P.N, user);
        },
        st);
  g_launches += P.layers + 2;
  if (e == cudaSuccess) e = cudaMemcpyAsync(h_out, d, bytes, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (d) cudaFreeAsync(d, st);
  if (st) {
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  }
  if (hs) cudaFreeHost(hs);
  if (e != cudaSuccess) return cuda_fail(e, who);
  return NTTK_OK;
}

int nttk_ntt_forward_observed(nttk_params_t h, int kind, const uint64_t* h_in, uint64_t* h_out,
                              nttk_layer_observer obs, void* user) {
  return observed(h, kind, 0, h_in, h_out, obs, user);
}

int nttk_intt_inverse_observed(nttk_params_t h, int kind, const uint64_t* h_in, uint64_t* h_out,
                               nttk_layer_observer obs, void* user) {
  return observed(h, kind, 1, h_in, h_out, obs, user);
}

// reduction.hpp:80-117
int nttk_make_reduction_context(uint64_t p, uint32_t n_bits, uint32_t alpha, uint32_t ell,
                                nttk_reduction_ctx* out) {
  if (!out) return fail(NTTK_CONTRACT, "reduction context: null output");
  if (n_bits < 2 || n_bits > 32)
    return fail(NTTK_CONTRACT, "reduction context: word size n must be in [2, 32]");
  if (p < 3 || !(p & 1)) return fail(NTTK_CONTRACT, "reduction context: p must be odd and >= 3");
  if (p >= (uint64_t(1) << n_bits)) return fail(NTTK_CONTRACT, "reduction context: p must be < 2^n");
  if (alpha >= n_bits) return fail(NTTK_CONTRACT, "reduction context: alpha must be < n");
  if (ell >= n_bits) return fail(NTTK_CONTRACT, "reduction context: ell must be < n");
  const nttk_b200::Ctx c = nttk_b200::make_ctx(p, n_bits, ell);
  std::memset(out, 0, sizeof *out);
  out->p = p;
  out->n_bits = n_bits;
  out->alpha = alpha;
  out->ell = ell;
  out->beta = c.beta;
  out->beta_mask = c.beta_mask;
  out->r2n_mask = c.r2n_mask;
  out->p_inv_beta = c.p_inv_beta;
  out->neg_p_inv_beta = c.neg_p_inv_beta;
  out->mu = c.mu;
  if (2 * n_bits == 64) {
    out->mu_centered = static_cast<int64_t>(c.mu);
  } else {
    const uint64_t half = uint64_t(1) << (2 * n_bits - 1);
    out->mu_centered = c.mu >= half ? static_cast<int64_t>(c.mu) -
                                          static_cast<int64_t>(uint64_t(1) << (2 * n_bits))
                                    : static_cast<int64_t>(c.mu);
  }
  out->beta_mod_p = c.beta_mod_p;
  out->r2n_mod_p = c.r2n_mod_p;
  return NTTK_OK;
}

namespace {
// per-op context bound and the operand-range messages (reduction.hpp:64-77, 125-291)
int reduce_precheck(int op, const nttk_reduction_ctx* c) {
  using nttk_b200::u128;
  if (!c) return fail(NTTK_CONTRACT, "reduce: null context");
  if (op < NTTK_OP_MONT_REDC || op > NTTK_OP_MOD_P)
    return fail(NTTK_CONTRACT, "reduce: unknown operation");
  const uint64_t p = c->p;
  const unsigned n = c->n_bits;
  if (op == NTTK_OP_SIGNED_MONT_REDC && !(u128(2) * p < (u128(1) << n)))
    return fail(NTTK_CONTRACT, "signed_mont_redc: requires 2p < 2^n");
  if (op == NTTK_OP_PLANTARD_REDC) {
    const u128 d = (u128(1) << (n + 1)) - p;
    if (!(u128(5) * p * p < d * d)) return fail(NTTK_CONTRACT, "plantard_redc: requires p*phi < 2^n");
  }
  if (op == NTTK_OP_MODIFIED_PLANTARD_MUL &&
      !(c->ell + 2 < n && u128(p) < (u128(1) << (n - c->ell - 2))))
    return fail(NTTK_CONTRACT, "modified_plantard_mul: requires p < 2^{n-ell-2}");
  return NTTK_OK;
}

int reduce_flag_message(int op, unsigned flag) {
  static const char* const first[] = {
      "mont_redc: T must be < p^2", "signed_mont_redc: A out of (-p*2^{n-1}, p*2^{n-1})",
      "plantard_redc: inputs exceed p", "modified_plantard_mul: W must be < p",
      "to_plantard_domain: w must be < p", "to_montgomery_domain: w must be < p"};
  if (flag & 1u) return fail(NTTK_CONTRACT, first[op]);
  return fail(NTTK_CONTRACT, "modified_plantard_mul: T must be < 2^ell * p");
}
}  // namespace

int nttk_reduce(int op, const nttk_reduction_ctx* ctx, const int64_t* d_x, const int64_t* d_y,
                int64_t* d_out, size_t n, void* stream) {
  if (int s = reduce_precheck(op, ctx)) return s;
  const bool binary = op == NTTK_OP_PLANTARD_REDC || op == NTTK_OP_MODIFIED_PLANTARD_MUL;
  if (n && (!d_x || !d_out || (binary && !d_y))) return fail(NTTK_CONTRACT, "reduce: null buffer");
  if (int s = need_device("reduce")) return s;
  if (!n) return NTTK_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned* d_flag = nullptr;  // [0] violation bits, [2..3] plantard corner count
  cudaError_t e = cudaMallocAsync(&d_flag, 16, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_flag, 0, 16, st);
  if (e == cudaSuccess) e = nttk_b200::reduce_launch(op, *ctx, d_x, d_y, d_out, n, d_flag, st);
  ++g_launches;
  unsigned flag[4] = {};
  if (e == cudaSuccess) e = cudaMemcpyAsync(flag, d_flag, sizeof flag, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (d_flag) cudaFreeAsync(d_flag, st);
  if (e != cudaSuccess) return cuda_fail(e, "reduce");
  uint64_t fires;
  std::memcpy(&fires, flag + 2, sizeof fires);
  g_plantard_fires += fires;
  if (flag[0]) return reduce_flag_message(op, flag[0]);
  return NTTK_OK;
}

namespace {
// butterfly.hpp checked wrappers: context/config checks (host) and operand messages
int butterfly_precheck(int op, const nttk_reduction_ctx* c, uint32_t aux0, uint32_t aux1) {
  using nttk_b200::u128;
  if (!c) return fail(NTTK_CONTRACT, "butterfly: null context");
  const uint64_t p = c->p;
  const unsigned n = c->n_bits;
  const bool lazy = c->ell + 2 < n && u128(p) < (u128(1) << (n - c->ell - 2));
  switch (op) {
    case NTTK_BF_NTL:
      if (!(2 * p < c->beta)) return fail(NTTK_CONTRACT, "ntl_butterfly: requires 2p < 2^n");
      return NTTK_OK;
    case NTTK_BF_HARVEY:
      if (!(4 * p < c->beta)) return fail(NTTK_CONTRACT, "harvey_butterfly: requires 4p < 2^n");
      return NTTK_OK;
    case NTTK_BF_SCOTT:
      if (!(aux1 >= 1 && aux0 >= aux1)) return fail(NTTK_CONTRACT, "scott_butterfly: malformed config");
      if (!(u128(4) * aux0 * p < u128(c->beta) * aux1))
        return fail(NTTK_CONTRACT, "scott_butterfly: requires 4*N*p/L < 2^n");
      return NTTK_OK;
    case NTTK_BF_IMPROVED_CT:
      if (!lazy) return fail(NTTK_CONTRACT, "improved_ct_butterfly: requires p < 2^{n-ell-2}");
      return NTTK_OK;
    case NTTK_BF_IMPROVED_GS:
      if (!lazy) return fail(NTTK_CONTRACT, "improved_gs_butterfly: requires p < 2^{n-ell-2}");
      if (!(aux0 >= 1 && aux0 <= c->ell))
        return fail(NTTK_CONTRACT, "improved_gs_butterfly: layer out of [1, ell]");
      return NTTK_OK;
    default: return fail(NTTK_CONTRACT, "butterfly: unknown kind");
  }
}

int butterfly_flag_message(int op, unsigned flag) {
  static const char* const wmsg[] = {"ntl_butterfly: W out of (0, p)", "harvey_butterfly: W out of (0, p)",
                                     "scott_butterfly: W out of (0, p)",
                                     "improved_ct_butterfly: W_hat must be < p",
                                     "improved_gs_butterfly: W_hat must be < p"};
  static const char* const xmsg[] = {"ntl_butterfly: inputs must be canonical",
                                     "harvey_butterfly: inputs must be < 2p",
                                     "scott_butterfly: inputs must be < (N/L)*p",
                                     "improved_ct_butterfly: inputs must be < 2^ell * p / 2",
                                     "improved_gs_butterfly: inputs must be < 2^{layer-1} * p"};
  if (flag & 1u) return fail(NTTK_CONTRACT, wmsg[op]);
  if (flag & 2u) return fail(NTTK_CONTRACT, "ntl_butterfly: stale W_quot");
  return fail(NTTK_CONTRACT, xmsg[op]);
}
}  // namespace

int nttk_butterfly(int op, const nttk_reduction_ctx* ctx, uint32_t aux0, uint32_t aux1,
                   const int64_t* d_x, const int64_t* d_y, const int64_t* d_w, const int64_t* d_wq,
                   int64_t* d_xo, int64_t* d_yo, size_t n, void* stream) {
  if (int s = butterfly_precheck(op, ctx, aux0, aux1)) return s;
  if (n && (!d_x || !d_y || !d_w || !d_xo || !d_yo || (op == NTTK_BF_NTL && !d_wq)))
    return fail(NTTK_CONTRACT, "butterfly: null buffer");
  if (int s = need_device("butterfly")) return s;
  if (!n) return NTTK_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned* d_flag = nullptr;
  cudaError_t e = cudaMallocAsync(&d_flag, sizeof(unsigned), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_flag, 0, sizeof(unsigned), st);
  if (e == cudaSuccess)
    e = nttk_b200::butterfly_launch(op, *ctx, aux0, aux1, d_x, d_y, d_w, d_wq, d_xo, d_yo, n, d_flag, st);
  ++g_launches;
  unsigned flag = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&flag, d_flag, sizeof flag, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (d_flag) cudaFreeAsync(d_flag, st);
  if (e != cudaSuccess) return cuda_fail(e, "butterfly");
  if (flag) return butterfly_flag_message(op, flag);
  return NTTK_OK;
}

int nttk_butterfly_host(int op, const nttk_reduction_ctx* ctx, uint32_t aux0, uint32_t aux1,
                        const int64_t* h_x, const int64_t* h_y, const int64_t* h_w,
                        const int64_t* h_wq, int64_t* h_xo, int64_t* h_yo, size_t n) {
  if (int s = butterfly_precheck(op, ctx, aux0, aux1)) return s;
  if (n && (!h_x || !h_y || !h_w || !h_xo || !h_yo || (op == NTTK_BF_NTL && !h_wq)))
    return fail(NTTK_CONTRACT, "butterfly: null buffer");
  if (int s = need_device("butterfly")) return s;
  if (!n) return NTTK_OK;
  cudaStream_t st = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  int64_t* d = nullptr;
  const size_t bytes = n * sizeof(int64_t);
  if (e == cudaSuccess) e = cudaMallocAsync(&d, 6 * bytes, st);
  const int64_t* src[4] = {h_x, h_y, h_w, h_wq};
  for (int k = 0; k < 4 && e == cudaSuccess; ++k)
    if (src[k]) e = cudaMemcpyAsync(d + k * n, src[k], bytes, cudaMemcpyHostToDevice, st);
  int rc = NTTK_OK;
  if (e == cudaSuccess) {
    rc = nttk_butterfly(op, ctx, aux0, aux1, d, d + n, d + 2 * n, d + 3 * n, d + 4 * n, d + 5 * n, n, st);
    if (rc == NTTK_OK) e = cudaMemcpyAsync(h_xo, d + 4 * n, bytes, cudaMemcpyDeviceToHost, st);
    if (rc == NTTK_OK && e == cudaSuccess)
      e = cudaMemcpyAsync(h_yo, d + 5 * n, bytes, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  if (d) cudaFreeAsync(d, st);
  if (st) {
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  }
  if (rc != NTTK_OK) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "butterfly");
  return NTTK_OK;
}

int nttk_reduce_host(int op, const nttk_reduction_ctx* ctx, const int64_t* h_x, const int64_t* h_y,
                     int64_t* h_out, size_t n) {
  if (int s = reduce_precheck(op, ctx)) return s;
  const bool binary = op == NTTK_OP_PLANTARD_REDC || op == NTTK_OP_MODIFIED_PLANTARD_MUL;
  if (n && (!h_x || !h_out || (binary && !h_y))) return fail(NTTK_CONTRACT, "reduce: null buffer");
  if (int s = need_device("reduce")) return s;
  if (!n) return NTTK_OK;
  cudaStream_t st = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  int64_t* d = nullptr;
  const size_t bytes = n * sizeof(int64_t);
  if (e == cudaSuccess) e = cudaMallocAsync(&d, 3 * bytes, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d, h_x, bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && binary) e = cudaMemcpyAsync(d + n, h_y, bytes, cudaMemcpyHostToDevice, st);
  int rc = NTTK_OK;
  if (e == cudaSuccess) {
    rc = nttk_reduce(op, ctx, d, d + n, d + 2 * n, n, st);
    if (rc == NTTK_OK) e = cudaMemcpyAsync(h_out, d + 2 * n, bytes, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  if (d) cudaFreeAsync(d, st);
  if (st) {
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  }
  if (rc != NTTK_OK) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "reduce");
  return NTTK_OK;
}

}  // extern "C"

// ---- captured plans (include/nttk_gpu.h) ----------------------------------------
struct nttk_plan {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  uint64_t kernels = 0;  // kernel launches per replay (launch count diagnostics)
};

extern "C" {

int nttk_plan_create(nttk_params_t h, int kind, int op, const void* d_a, const void* d_b,
                     void* d_out, size_t batch, int elem, int repeat, nttk_plan_t* plan) {
  if (!h || !plan) return fail(NTTK_CONTRACT, "plan_create: null argument");
  if (op < NTTK_PLAN_FORWARD || op > NTTK_PLAN_POLYMUL)
    return fail(NTTK_CONTRACT, "plan_create: unknown op");
  if (repeat < 1) return fail(NTTK_CONTRACT, "plan_create: repeat must be >= 1");
  *plan = nullptr;
  if (int s = check_kind(h->P, kind, "plan_create")) return s;
  if (int s = need_device("plan_create")) return s;
  // the synchronous first-use uploads happen here, outside the capture (nothing runs: the
  // buffers are untouched until the first nttk_plan_launch)
  const HostParams& P = h->P;
  std::string err;
  const int dev = current_device();
  if (!P.device_tables(dev, err)) return fail(NTTK_CUDA, "plan_create: " + err);
  if (P.N != 256 && use_fast(P, kind))
    for (int dir = 0; dir < 2; ++dir)
      if (!P.fastn_table(dev, P.image(kind, dir), dir, err)) return fail(NTTK_CUDA, "plan_create: " + err);
  cudaStream_t st = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cuda_fail(e, "plan_create");
  nttk_plan* p = new nttk_plan;
  int rc = NTTK_OK;
  const uint64_t before = g_launches.load();
  e = cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed);
  for (int i = 0; e == cudaSuccess && rc == NTTK_OK && i < repeat; ++i) {
    switch (op) {
      case NTTK_PLAN_FORWARD: rc = nttk_ntt_forward(h, kind, d_a, d_out, batch, elem, st); break;
      case NTTK_PLAN_INVERSE: rc = nttk_intt_inverse(h, kind, d_a, d_out, batch, elem, st); break;
      default: rc = nttk_polymul(h, kind, d_a, d_b, d_out, batch, elem, st);
    }
  }
  p->kernels = (g_launches.load() - before) / uint64_t(repeat);
  const std::string keep = g_err;
  const cudaError_t ec = e == cudaSuccess ? cudaStreamEndCapture(st, &p->graph) : e;
  if (e == cudaSuccess) e = ec;
  if (e == cudaSuccess && rc == NTTK_OK) e = cudaGraphInstantiate(&p->exec, p->graph, 0);
  cudaStreamDestroy(st);
  if (rc != NTTK_OK) {
    g_err = keep;  // the failing call's message, not the capture teardown's
  } else if (e != cudaSuccess) {
    rc = cuda_fail(e, "plan_create");
  }
  if (rc != NTTK_OK) {
    nttk_plan_destroy(p);
    return rc;
  }
  *plan = p;
  return NTTK_OK;
}

int nttk_plan_launch(nttk_plan_t plan, void* stream) {
  if (!plan || !plan->exec) return fail(NTTK_CONTRACT, "plan_launch: null plan");
  const cudaError_t e = cudaGraphLaunch(plan->exec, static_cast<cudaStream_t>(stream));
  g_launches += plan->kernels;
  return e == cudaSuccess ? int(NTTK_OK) : cuda_fail(e, "plan_launch");
}

void nttk_plan_destroy(nttk_plan_t plan) {
  if (!plan) return;
  if (plan->exec) cudaGraphExecDestroy(plan->exec);
  if (plan->graph) cudaGraphDestroy(plan->graph);
  delete plan;
}

}  // extern "C"
