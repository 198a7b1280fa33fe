// generic.cu -- sm_100a kernels for every parameter set the reference admits.
//
// The fast N = 256 kernels (fast256.cu) cover the hot configurations.  Everything else
// build_params accepts (params.hpp:137-268: any prime p, N = 2..2^20, n = 2..32, every
// ButterflyKind, toy radices included) runs here, so every drop-in ntt_forward /
// intt_inverse / pointwise_multiply call executes on the GPU.  Arithmetic is 64-bit
// with the reference's masks, bit-exact with transform.hpp:77-337 for any n:
//   * N <= 4096: one CTA per polynomial, the whole transform in shared memory;
//   * larger N: one launch per layer over a u64 device buffer.
// Also here: the pointwise / basemul kernels (canonical outputs) and the device-side
// canonical-input check behind the host entry points.
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>

#include "generic.hpp"

namespace nttk_b200 {
namespace {

struct GCtx {  // reduction.hpp:44-78, device copy
  uint64_t p, beta_mask, r2n_mask, p_inv_beta, neg_p_inv_beta, mu, n_inv, n_inv_hat;
  int64_t n_inv_smont;
  uint32_t n_bits, N, log2N, layers, tree, scott_off_mult;
  uint64_t scott_off;
  // signed Barrett (extension): S = n + 10
  int64_t barrett_v;
};

__device__ __forceinline__ uint64_t mulmod64(uint64_t a, uint64_t b, uint64_t p) {
  // p < 2^32, a, b < 2^32: exact product fits 64 bits
  return (a * b) % p;
}

__device__ __forceinline__ uint64_t mp64(uint64_t w, uint64_t t, const GCtx& c) {
  // reduction.hpp:252-258
  const uint64_t h = ((w * t) * c.mu) & c.r2n_mask;
  return (((h >> c.n_bits) + 1) * c.p) >> c.n_bits;
}

__device__ __forceinline__ int64_t smont64(int64_t A, const GCtx& c) {
  // reduction.hpp:141-165 (unchecked body)
  const int64_t a1 = A >> c.n_bits;
  const uint64_t a0 = static_cast<uint64_t>(A) & c.beta_mask;
  const uint64_t mu = (a0 * c.p_inv_beta) & c.beta_mask;
  const uint64_t half = (c.beta_mask + 1) >> 1;
  const int64_t m = mu >= half ? static_cast<int64_t>(mu) - static_cast<int64_t>(c.beta_mask + 1)
                               : static_cast<int64_t>(mu);
  return a1 - ((m * static_cast<int64_t>(c.p)) >> c.n_bits);
}

__device__ __forceinline__ int64_t sbarrett64(int64_t a, const GCtx& c) {
  const unsigned S = c.n_bits + 10;
  const __int128 q = (static_cast<__int128>(a) * c.barrett_v + (static_cast<__int128>(1) << (S - 1))) >> S;
  return a - static_cast<int64_t>(q) * static_cast<int64_t>(c.p);
}

// forward butterfly of `kind` on (x, y); `ti` indexes the table of that kind
__device__ __forceinline__ void fwd_bf(int kind, uint64_t& X, uint64_t& Y, size_t ti,
                                       const GCtx& c, const DeviceTables& T) {
  const uint64_t p = c.p;
  switch (kind) {
    case NTTK_NTL: {  // butterfly.hpp:60-71
      const uint64_t W = T.dif_w[ti], Wq = T.dif_wq[ti];
      uint64_t s = X + Y;
      if (s >= p) s -= p;
      const uint64_t t = X >= Y ? X - Y : X + p - Y;
      const uint64_t q = (Wq * t) >> c.n_bits;
      uint64_t y = (W * t - q * p) & c.beta_mask;
      if (y >= p) y -= p;
      X = s;
      Y = y;
      break;
    }
    case NTTK_HARVEY: {
      if (c.tree == NTTK_CYCLIC) {  // butterfly.hpp:92-106
        const uint64_t p2 = 2 * p;
        uint64_t s = X + Y;
        if (s >= p2) s -= p2;
        const uint64_t t = X + p2 - Y;
        const uint64_t prod = T.dif_mont[ti] * t;
        const uint64_t q = (c.p_inv_beta * (prod & c.beta_mask)) & c.beta_mask;
        X = s;
        Y = (prod >> c.n_bits) + p - ((q * p) >> c.n_bits);
      } else {  // CT-form harvey (extension)
        const uint64_t p2 = 2 * p;
        const uint64_t prod = T.ct_mont[ti] * Y;
        const uint64_t q = (c.p_inv_beta * (prod & c.beta_mask)) & c.beta_mask;
        const uint64_t r = (prod >> c.n_bits) + p - ((q * p) >> c.n_bits);
        uint64_t a = X + r;
        if (a >= p2) a -= p2;
        uint64_t b = X + p2 - r;
        if (b >= p2) b -= p2;
        X = a;
        Y = b;
      }
      break;
    }
    case NTTK_SCOTT: {  // butterfly.hpp:172-184
      const uint64_t t = X + c.scott_off - Y;
      const uint64_t wt = T.dif_mont[ti] * t;
      const uint64_t q = (c.neg_p_inv_beta * (wt & c.beta_mask)) & c.beta_mask;
      X = X + Y;
      Y = (wt + q * p) >> c.n_bits;
      break;
    }
    case NTTK_IMPROVED: {  // butterfly.hpp:224-230
      const uint64_t r = mp64(T.ct_plantard[ti], Y, c);
      Y = X + p - r;
      X = X + r;
      break;
    }
    case NTTK_SMONT: {  // extension
      const int64_t t = smont64(static_cast<int64_t>(T.ct_smont[ti]) * static_cast<int64_t>(Y), c);
      const int64_t x = static_cast<int64_t>(X);
      X = static_cast<uint64_t>(x + t);
      Y = static_cast<uint64_t>(x - t);
      break;
    }
  }
}

__device__ __forceinline__ void inv_bf(int kind, uint64_t& X, uint64_t& Y, size_t ti,
                                       unsigned m, const GCtx& c, const DeviceTables& T) {
  const uint64_t p = c.p;
  switch (kind) {
    case NTTK_NTL: {
      const uint64_t W = T.gs_w[ti], Wq = T.gs_wq[ti];
      uint64_t s = X + Y;
      if (s >= p) s -= p;
      const uint64_t t = X >= Y ? X - Y : X + p - Y;
      const uint64_t q = (Wq * t) >> c.n_bits;
      uint64_t y = (W * t - q * p) & c.beta_mask;
      if (y >= p) y -= p;
      X = s;
      Y = y;
      break;
    }
    case NTTK_HARVEY: {
      const uint64_t p2 = 2 * p;
      uint64_t s = X + Y;
      if (s >= p2) s -= p2;
      const uint64_t t = X + p2 - Y;
      const uint64_t prod = T.gs_mont[ti] * t;
      const uint64_t q = (c.p_inv_beta * (prod & c.beta_mask)) & c.beta_mask;
      X = s;
      Y = (prod >> c.n_bits) + p - ((q * p) >> c.n_bits);
      break;
    }
    case NTTK_SCOTT: {
      const uint64_t t = X + c.scott_off - Y;
      const uint64_t wt = T.gs_mont[ti] * t;
      const uint64_t q = (c.neg_p_inv_beta * (wt & c.beta_mask)) & c.beta_mask;
      X = X + Y;
      Y = (wt + q * p) >> c.n_bits;
      break;
    }
    case NTTK_IMPROVED: {  // butterfly.hpp:235-243
      const uint64_t t = X + (p << (m - 1)) - Y;
      X = X + Y;
      Y = mp64(T.gs_plantard[ti], t, c);
      break;
    }
    case NTTK_SMONT: {
      const int64_t x = static_cast<int64_t>(X), y = static_cast<int64_t>(Y);
      X = static_cast<uint64_t>(sbarrett64(x + y, c));
      Y = static_cast<uint64_t>(smont64(static_cast<int64_t>(T.gs_smont[ti]) * (x - y), c));
      break;
    }
  }
}

template <class IO>
__device__ __forceinline__ uint64_t ld(const IO* p, size_t i, bool sgn) {
  const IO v = p[i];
  if (!sgn) return static_cast<uint64_t>(v);
  if constexpr (sizeof(IO) == 2) return static_cast<uint64_t>(static_cast<int64_t>(static_cast<int16_t>(v)));
  if constexpr (sizeof(IO) == 4) return static_cast<uint64_t>(static_cast<int64_t>(static_cast<int32_t>(v)));
  return static_cast<uint64_t>(v);
}

__device__ __forceinline__ uint64_t canon(uint64_t v, bool sgn, uint64_t p) {
  if (sgn) {
    const int64_t r = static_cast<int64_t>(v) % static_cast<int64_t>(p);
    return static_cast<uint64_t>(r < 0 ? r + static_cast<int64_t>(p) : r);
  }
  return v % p;
}

__device__ __forceinline__ uint64_t final_scale(int kind, uint64_t v, const GCtx& c) {
  if (kind == NTTK_IMPROVED) return mp64(c.n_inv_hat, v, c);  // transform.hpp:323-330
  if (kind == NTTK_SMONT) {
    const int64_t r = smont64(c.n_inv_smont * static_cast<int64_t>(v), c);
    return static_cast<uint64_t>(r < 0 ? r + static_cast<int64_t>(c.p) : r);
  }
  return mulmod64(v % c.p, c.n_inv, c.p);  // transform.hpp:331-335 (u128 there)
}

// whole transform of one polynomial per CTA, in shared memory
template <class IO>
__global__ void transform_smem_kernel(int kind, int dir, const IO* __restrict__ in,
                                      IO* __restrict__ out, size_t batch, GCtx c,
                                      DeviceTables T) {
  extern __shared__ uint64_t a[];
  const size_t poly = blockIdx.x;
  if (poly >= batch) return;
  const uint32_t N = c.N;
  const bool sgn = kind == NTTK_SMONT;
  for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
    uint64_t v = ld(in, poly * N + i, sgn);
    if (dir == 1) v = canon(v, sgn, c.p);  // transform.hpp:243
    a[i] = v;
  }
  __syncthreads();
  const bool per_index = c.tree == NTTK_CYCLIC && kind != NTTK_IMPROVED && kind != NTTK_SMONT;
  if (dir == 0) {  // run_split_layers, transform.hpp:77-96
    size_t cursor = 0;
    for (uint32_t s = 1; s <= c.layers; ++s) {
      const uint32_t len = N >> s, blocks = 1u << (s - 1);
      for (uint32_t k = threadIdx.x; k < N / 2; k += blockDim.x) {
        const uint32_t b = k / len, jj = k % len;
        const uint32_t i = b * 2 * len + jj;
        uint64_t X = a[i], Y = a[i + len];
        fwd_bf(kind, X, Y, cursor + (per_index ? jj : b), c, T);
        a[i] = X;
        a[i + len] = Y;
      }
      cursor += per_index ? len : blocks;
      __syncthreads();
    }
  } else {  // run_merge_layers, transform.hpp:99-116
    size_t cursor = 0;
    unsigned m = 0;
    for (uint32_t s = c.layers; s >= 1; --s) {
      ++m;
      const uint32_t len = N >> s, blocks = 1u << (s - 1);
      for (uint32_t k = threadIdx.x; k < N / 2; k += blockDim.x) {
        const uint32_t b = k / len, jj = k % len;
        const uint32_t i = b * 2 * len + jj;
        uint64_t X = a[i], Y = a[i + len];
        inv_bf(kind, X, Y, cursor + b, m, c, T);
        a[i] = X;
        a[i + len] = Y;
      }
      cursor += blocks;
      __syncthreads();
    }
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) a[i] = final_scale(kind, a[i], c);
    __syncthreads();
  }
  for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) out[poly * N + i] = static_cast<IO>(a[i]);
}

// large N: elementwise conversion into / out of a u64 work buffer, one launch per layer
template <class IO>
__global__ void load_u64_kernel(const IO* __restrict__ in, uint64_t* __restrict__ w, size_t n,
                                bool sgn, bool do_canon, uint64_t p) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    uint64_t v = ld(in, i, sgn);
    w[i] = do_canon ? canon(v, sgn, p) : v;
  }
}

template <class IO>
__global__ void store_u64_kernel(const uint64_t* __restrict__ w, IO* __restrict__ out, size_t n,
                                 int kind, bool scale, GCtx c) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    out[i] = static_cast<IO>(scale ? final_scale(kind, w[i], c) : w[i]);
}

__global__ void layer_kernel(int kind, int dir, uint64_t* __restrict__ a, size_t batch, uint32_t s,
                             size_t cursor, unsigned m, GCtx c, DeviceTables T) {
  const uint32_t N = c.N, len = N >> s;
  const size_t total = batch * (N / 2);
  const bool per_index = c.tree == NTTK_CYCLIC && kind != NTTK_IMPROVED && kind != NTTK_SMONT;
  for (size_t g = blockIdx.x * size_t(blockDim.x) + threadIdx.x; g < total;
       g += size_t(gridDim.x) * blockDim.x) {
    const size_t poly = g / (N / 2);
    const uint32_t k = static_cast<uint32_t>(g % (N / 2));
    const uint32_t b = k / len, jj = k % len;
    uint64_t* x = a + poly * N + b * 2 * len + jj;
    uint64_t X = x[0], Y = x[len];
    if (dir == 0) fwd_bf(kind, X, Y, cursor + (per_index ? jj : b), c, T);
    else inv_bf(kind, X, Y, cursor + b, m, c, T);
    x[0] = X;
    x[len] = Y;
  }
}

// ---------------------------------------------------------------------------
// pointwise / basemul: canonical outputs (transform.hpp:349-370; basemul extension)
template <class IO>
__global__ void pointwise_kernel(const IO* __restrict__ l, const IO* __restrict__ r,
                                 IO* __restrict__ out, size_t n, bool sgn, uint64_t p) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const uint64_t a = canon(ld(l, i, sgn), sgn, p), b = canon(ld(r, i, sgn), sgn, p);
    out[i] = static_cast<IO>(mulmod64(a, b, p));
  }
}

template <class IO>
__global__ void basemul_kernel(const IO* __restrict__ l, const IO* __restrict__ r,
                               IO* __restrict__ out, size_t pairs, uint32_t N, bool sgn,
                               uint64_t p, const uint64_t* __restrict__ gamma) {
  for (size_t g = blockIdx.x * size_t(blockDim.x) + threadIdx.x; g < pairs;
       g += size_t(gridDim.x) * blockDim.x) {
    const uint32_t k = static_cast<uint32_t>(g % (N / 2));
    const uint64_t a0 = canon(ld(l, 2 * g, sgn), sgn, p), a1 = canon(ld(l, 2 * g + 1, sgn), sgn, p);
    const uint64_t b0 = canon(ld(r, 2 * g, sgn), sgn, p), b1 = canon(ld(r, 2 * g + 1, sgn), sgn, p);
    const uint64_t gm = gamma[k];
    out[2 * g] = static_cast<IO>((mulmod64(a0, b0, p) + mulmod64(mulmod64(a1, b1, p), gm, p)) % p);
    out[2 * g + 1] = static_cast<IO>((mulmod64(a0, b1, p) + mulmod64(a1, b0, p)) % p);
  }
}

// flags[0] |= 1 when any coefficient is >= p (ntt_forward's canonical check)
template <class IO>
__global__ void check_canonical_kernel(const IO* __restrict__ in, size_t n, uint64_t p,
                                       unsigned* flag) {
  bool bad = false;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    bad |= static_cast<uint64_t>(in[i]) >= p;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

GCtx make_gctx(const HostParams& P) {
  GCtx c{};
  c.p = P.p;
  c.beta_mask = P.ctx.beta_mask;
  c.r2n_mask = P.ctx.r2n_mask;
  c.p_inv_beta = P.ctx.p_inv_beta;
  c.neg_p_inv_beta = P.ctx.neg_p_inv_beta;
  c.mu = P.ctx.mu;
  c.n_inv = P.n_inv;
  c.n_inv_hat = P.n_inv_hat;
  c.n_inv_smont = P.n_inv_smont;
  c.n_bits = P.n_bits;
  c.N = P.N;
  c.log2N = P.log2N;
  c.layers = P.layers;
  c.tree = P.tree;
  c.scott_off = P.scott_L ? uint64_t(P.N / P.scott_L) * P.p : 0;
  {
    const unsigned __int128 num = ((unsigned __int128)1 << (P.n_bits + 10)) + (P.p >> 1);
    c.barrett_v = static_cast<int64_t>(num / P.p);
  }
  return c;
}

int grid_for(size_t n, int threads) {
  size_t b = (n + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  return static_cast<int>(b ? b : 1);
}

template <class IO>
cudaError_t transform_io(const HostParams& P, const DeviceTables& T, int kind, int dir,
                         const void* in, void* out, size_t batch, cudaStream_t st) {
  const GCtx c = make_gctx(P);
  const IO* src = static_cast<const IO*>(in);
  IO* dst = static_cast<IO*>(out);
  if (P.N <= 4096) {
    const int threads = P.N / 2 < 256 ? static_cast<int>(P.N / 2 < 32 ? 32 : P.N / 2) : 256;
    const size_t smem = size_t(P.N) * 8;
    for (size_t done = 0; done < batch;) {  // grid.x limit
      const size_t chunk = batch - done < (size_t(1) << 30) ? batch - done : (size_t(1) << 30);
      transform_smem_kernel<IO><<<static_cast<unsigned>(chunk), threads, smem, st>>>(
          kind, dir, src + done * P.N, dst + done * P.N, chunk, c, T);
      done += chunk;
    }
    return cudaGetLastError();
  }
  const size_t n = batch * P.N;
  uint64_t* w = nullptr;
  cudaError_t e = cudaMallocAsync(&w, n * 8, st);
  if (e != cudaSuccess) return e;
  const bool sgn = kind == NTTK_SMONT;
  load_u64_kernel<IO><<<grid_for(n, 256), 256, 0, st>>>(src, w, n, sgn, dir == 1, P.p);
  const bool per_index = P.tree == NTTK_CYCLIC && kind != NTTK_IMPROVED && kind != NTTK_SMONT;
  size_t cursor = 0;
  if (dir == 0) {
    for (uint32_t s = 1; s <= P.layers; ++s) {
      layer_kernel<<<grid_for(batch * (P.N / 2), 256), 256, 0, st>>>(kind, 0, w, batch, s, cursor,
                                                                     0, c, T);
      cursor += per_index ? (P.N >> s) : (size_t(1) << (s - 1));
    }
  } else {
    unsigned m = 0;
    for (uint32_t s = P.layers; s >= 1; --s) {
      ++m;
      layer_kernel<<<grid_for(batch * (P.N / 2), 256), 256, 0, st>>>(kind, 1, w, batch, s, cursor,
                                                                     m, c, T);
      cursor += size_t(1) << (s - 1);
    }
  }
  store_u64_kernel<IO><<<grid_for(n, 256), 256, 0, st>>>(w, dst, n, kind, dir == 1, c);
  e = cudaGetLastError();
  cudaFreeAsync(w, st);
  return e;
}

}  // namespace

cudaError_t generic_transform(const HostParams& P, const DeviceTables& T, int kind, int dir,
                              const void* in, void* out, size_t batch, int elem_bytes,
                              cudaStream_t st) {
  if (batch == 0) return cudaSuccess;
  if (P.N <= 4096 && P.N * 8 > 48 * 1024) return cudaErrorInvalidValue;
  switch (elem_bytes) {
    case 2: return transform_io<uint16_t>(P, T, kind, dir, in, out, batch, st);
    case 4: return transform_io<uint32_t>(P, T, kind, dir, in, out, batch, st);
    case 8: return transform_io<uint64_t>(P, T, kind, dir, in, out, batch, st);
    default: return cudaErrorInvalidValue;
  }
}

namespace {
// storage-width conversions for the wide product composition (canonical words only)
template <class IO>
__global__ void widen_kernel(const IO* __restrict__ src, uint64_t* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    dst[i] = static_cast<uint64_t>(src[i]);
}
template <class IO>
__global__ void narrow_kernel(const uint64_t* __restrict__ src, IO* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    dst[i] = static_cast<IO>(src[i]);
}

}  // namespace

cudaError_t widen_to_u64(const void* src, int elem, uint64_t* dst, size_t n, cudaStream_t st) {
  if (!n) return cudaSuccess;
  if (elem == 2)
    widen_kernel<uint16_t><<<grid_for(n, 256), 256, 0, st>>>(static_cast<const uint16_t*>(src), dst, n);
  else if (elem == 4)
    widen_kernel<uint32_t><<<grid_for(n, 256), 256, 0, st>>>(static_cast<const uint32_t*>(src), dst, n);
  else
    return cudaMemcpyAsync(dst, src, n * 8, cudaMemcpyDeviceToDevice, st);
  return cudaGetLastError();
}

cudaError_t narrow_from_u64(const uint64_t* src, void* dst, int elem, size_t n, cudaStream_t st) {
  if (!n) return cudaSuccess;
  if (elem == 2)
    narrow_kernel<uint16_t><<<grid_for(n, 256), 256, 0, st>>>(src, static_cast<uint16_t*>(dst), n);
  else if (elem == 4)
    narrow_kernel<uint32_t><<<grid_for(n, 256), 256, 0, st>>>(src, static_cast<uint32_t*>(dst), n);
  else
    return cudaMemcpyAsync(dst, src, n * 8, cudaMemcpyDeviceToDevice, st);
  return cudaGetLastError();
}

// ntt_forward_observed / intt_inverse_observed (transform.hpp:77-116, 207-337): one
// polynomial, one launch per layer; after each layer the u64 state is read back and
// observe(layer, state) runs on the host (layers numbered as the reference's
// run_split_layers / run_merge_layers do).  d_io holds N u64 words (input, then output).
cudaError_t generic_transform_observed(const HostParams& P, const DeviceTables& T, int kind,
                                       int dir, uint64_t* d_io, uint64_t* h_state,
                                       const std::function<void(unsigned)>& observe,
                                       cudaStream_t st) {
  const GCtx c = make_gctx(P);
  const size_t n = P.N;
  uint64_t* w = nullptr;
  cudaError_t e = cudaMallocAsync(&w, n * 8, st);
  if (e != cudaSuccess) return e;
  const bool sgn = kind == NTTK_SMONT;
  load_u64_kernel<uint64_t><<<grid_for(n, 256), 256, 0, st>>>(d_io, w, n, sgn, dir == 1, P.p);
  const bool per_index = P.tree == NTTK_CYCLIC && kind != NTTK_IMPROVED && kind != NTTK_SMONT;
  auto after = [&](unsigned layer) -> cudaError_t {
    cudaError_t x = cudaMemcpyAsync(h_state, w, n * 8, cudaMemcpyDeviceToHost, st);
    if (x == cudaSuccess) x = cudaStreamSynchronize(st);
    if (x == cudaSuccess) observe(layer);
    return x;
  };
  size_t cursor = 0;
  if (dir == 0) {
    for (uint32_t s = 1; s <= P.layers && e == cudaSuccess; ++s) {
      layer_kernel<<<grid_for(P.N / 2, 256), 256, 0, st>>>(kind, 0, w, 1, s, cursor, 0, c, T);
      cursor += per_index ? (P.N >> s) : (size_t(1) << (s - 1));
      e = after(s);
    }
  } else {
    unsigned m = 0;
    for (uint32_t s = P.layers; s >= 1 && e == cudaSuccess; --s) {
      ++m;
      layer_kernel<<<grid_for(P.N / 2, 256), 256, 0, st>>>(kind, 1, w, 1, s, cursor, m, c, T);
      cursor += size_t(1) << (s - 1);
      e = after(m);
    }
  }
  if (e == cudaSuccess) {
    store_u64_kernel<uint64_t><<<grid_for(n, 256), 256, 0, st>>>(w, d_io, n, kind, dir == 1, c);
    e = cudaGetLastError();
  }
  cudaFreeAsync(w, st);
  return e;
}

cudaError_t generic_pointwise(const HostParams& P, int kind, const void* l, const void* r,
                              void* out, size_t batch, int elem_bytes, cudaStream_t st) {
  const size_t n = batch * P.N;
  if (!n) return cudaSuccess;
  const bool sgn = kind == NTTK_SMONT;
  switch (elem_bytes) {
    case 2:
      pointwise_kernel<<<grid_for(n, 256), 256, 0, st>>>(
          static_cast<const uint16_t*>(l), static_cast<const uint16_t*>(r),
          static_cast<uint16_t*>(out), n, sgn, P.p);
      break;
    case 4:
      pointwise_kernel<<<grid_for(n, 256), 256, 0, st>>>(
          static_cast<const uint32_t*>(l), static_cast<const uint32_t*>(r),
          static_cast<uint32_t*>(out), n, sgn, P.p);
      break;
    case 8:
      pointwise_kernel<<<grid_for(n, 256), 256, 0, st>>>(
          static_cast<const uint64_t*>(l), static_cast<const uint64_t*>(r),
          static_cast<uint64_t*>(out), n, sgn, P.p);
      break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t generic_basemul(const HostParams& P, const uint64_t* d_gamma, int kind, const void* l,
                            const void* r, void* out, size_t batch, int elem_bytes,
                            cudaStream_t st) {
  const size_t pairs = batch * P.N / 2;
  if (!pairs) return cudaSuccess;
  const bool sgn = kind == NTTK_SMONT;
  switch (elem_bytes) {
    case 2:
      basemul_kernel<<<grid_for(pairs, 256), 256, 0, st>>>(
          static_cast<const uint16_t*>(l), static_cast<const uint16_t*>(r),
          static_cast<uint16_t*>(out), pairs, P.N, sgn, P.p, d_gamma);
      break;
    case 4:
      basemul_kernel<<<grid_for(pairs, 256), 256, 0, st>>>(
          static_cast<const uint32_t*>(l), static_cast<const uint32_t*>(r),
          static_cast<uint32_t*>(out), pairs, P.N, sgn, P.p, d_gamma);
      break;
    case 8:
      basemul_kernel<<<grid_for(pairs, 256), 256, 0, st>>>(
          static_cast<const uint64_t*>(l), static_cast<const uint64_t*>(r),
          static_cast<uint64_t*>(out), pairs, P.N, sgn, P.p, d_gamma);
      break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t check_canonical(const void* in, size_t n, int elem_bytes, uint64_t p, unsigned* d_flag,
                            cudaStream_t st) {
  if (!n) return cudaSuccess;
  switch (elem_bytes) {
    case 2:
      check_canonical_kernel<<<grid_for(n, 256), 256, 0, st>>>(static_cast<const uint16_t*>(in),
                                                               n, p, d_flag);
      break;
    case 4:
      check_canonical_kernel<<<grid_for(n, 256), 256, 0, st>>>(static_cast<const uint32_t*>(in),
                                                               n, p, d_flag);
      break;
    case 8:
      check_canonical_kernel<<<grid_for(n, 256), 256, 0, st>>>(static_cast<const uint64_t*>(in),
                                                               n, p, d_flag);
      break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace nttk_b200
