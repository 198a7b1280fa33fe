"""Python mirror of the reference ``nttk`` interface over the B200 engine's C ABI.

The reference (/root/reference/proj/include/nttk) is a header-only C++20 library whose
hot path is ``ntt_forward`` / ``intt_inverse`` / ``pointwise_multiply`` /
``cyclic_convolution_via_ntt`` (transform.hpp:207-379) built on ``build_params``
(params.hpp:137-268).  This module keeps those names, argument meanings and error
behaviour (``ContractViolation`` carries the reference's contract_violation message),
and routes every call through ``libnttk_gpu.so`` (include/nttk_gpu.h) to the sm_100a
kernels.  There is no CPU fallback: without the built extension or a CUDA device the
compute calls raise.

Two layers:
  * reference-shaped host calls on Python lists / numpy arrays (checked, synchronous);
  * batched device calls on ``torch`` CUDA tensors (asynchronous on the current stream),
    which is what the benchmark and large workloads use.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnttk_gpu.so")


class ButterflyKind(enum.IntEnum):
    """butterfly.hpp:30 plus the signed-Montgomery extension kind."""

    ntl = 0
    harvey = 1
    scott = 2
    improved = 3
    smont = 4


class Ordering(enum.Enum):
    natural = 0
    bit_reversed = 1


class Tree(enum.IntEnum):
    cyclic = 0
    negacyclic = 1


class Redc(enum.IntEnum):
    mont = 0
    smont = 1
    plantard = 2
    modified_plantard = 3


class ContractViolation(ValueError):
    """nttk::contract_violation (int_util.hpp:17-21)."""


class PropertyViolation(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


def all_butterfly_kinds() -> list[ButterflyKind]:
    """params.hpp:192-195."""
    return [ButterflyKind.ntl, ButterflyKind.harvey, ButterflyKind.scott, ButterflyKind.improved]


def butterfly_kind_from_string(name: str) -> ButterflyKind:
    """butterfly.hpp:42-50."""
    try:
        return ButterflyKind[name]
    except KeyError:
        raise ContractViolation(
            f'unknown butterfly kind "{name}" (ntl, harvey, scott, improved)') from None


# ---------------------------------------------------------------------------
# library binding

class _Desc(C.Structure):
    _fields_ = [("p", C.c_uint64), ("N", C.c_uint32), ("n_bits", C.c_uint32),
                ("kinds_mask", C.c_uint32), ("tree", C.c_uint32), ("layers", C.c_uint32),
                ("root", C.c_uint64), ("flags", C.c_uint32)]


class ReductionContext(C.Structure):
    """reduction.hpp:44-78 (nttk_reduction_ctx); build with make_reduction_context()."""
    _fields_ = [("p", C.c_uint64), ("n_bits", C.c_uint32), ("alpha", C.c_uint32),
                ("ell", C.c_uint32), ("pad_", C.c_uint32), ("beta", C.c_uint64),
                ("beta_mask", C.c_uint64), ("r2n_mask", C.c_uint64), ("p_inv_beta", C.c_uint64),
                ("neg_p_inv_beta", C.c_uint64), ("mu", C.c_uint64), ("mu_centered", C.c_int64),
                ("beta_mod_p", C.c_uint64), ("r2n_mod_p", C.c_uint64)]

    def two_n(self) -> int:
        return 2 * self.n_bits

    def fits_plantard_bound(self) -> bool:
        return 5 * self.p * self.p < ((1 << (self.n_bits + 1)) - self.p) ** 2

    def fits_signed_plantard_bound(self) -> bool:
        return self.alpha + 1 < self.n_bits and self.p < (1 << (self.n_bits - self.alpha - 1))

    def fits_lazy_plantard_bound(self) -> bool:
        return self.ell + 2 < self.n_bits and self.p < (1 << (self.n_bits - self.ell - 2))

    def fits_signed_montgomery_bound(self) -> bool:
        return 2 * self.p < (1 << self.n_bits)


_OBSERVER = C.CFUNCTYPE(None, C.c_uint, C.POINTER(C.c_uint64), C.c_size_t, C.c_void_p)


class _Info(C.Structure):
    _fields_ = [("p", C.c_uint64), ("omega", C.c_uint64), ("omega_inv", C.c_uint64),
                ("n_inv", C.c_uint64), ("n_inv_hat", C.c_uint64), ("mu", C.c_uint64),
                ("N", C.c_uint32), ("log2N", C.c_uint32), ("n_bits", C.c_uint32),
                ("layers", C.c_uint32), ("tree", C.c_uint32), ("kinds_mask", C.c_uint32),
                ("scott_L", C.c_uint32), ("fast_path", C.c_uint32)]


EXPORTS = (
    "nttk_build_params", "nttk_preset", "nttk_params_destroy", "nttk_params_get_info",
    "nttk_params_fast_flags",
    "nttk_params_table", "nttk_ntt_forward", "nttk_intt_inverse", "nttk_pointwise_multiply",
    "nttk_basemul", "nttk_polymul", "nttk_ntt_forward_host", "nttk_intt_inverse_host",
    "nttk_roundtrip_host", "nttk_pointwise_multiply_host", "nttk_polymul_host",
    "nttk_modmul_sweep", "nttk_modmul_sweep_device", "nttk_make_reduction_context", "nttk_reduce", "nttk_reduce_host",
    "nttk_butterfly", "nttk_butterfly_host", "nttk_ntt_forward_observed",
    "nttk_intt_inverse_observed",
    "nttk_last_error", "nttk_launch_count", "nttk_device_available", "nttk_version",
    "nttk_plantard_correction_fires", "nttk_plan_create", "nttk_plan_launch", "nttk_plan_destroy",
)

_lib_handle = None


def lib() -> C.CDLL:
    """Load libnttk_gpu.so; fails loudly when the extension was not built."""
    global _lib_handle
    if _lib_handle is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} missing: the CUDA extension is not built (run `make lib` or "
                "__graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        vp, sz = C.c_void_p, C.c_size_t
        L.nttk_build_params.argtypes = [C.POINTER(_Desc), C.POINTER(vp)]
        L.nttk_preset.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.nttk_params_destroy.argtypes = [vp]
        L.nttk_params_get_info.argtypes = [vp, C.POINTER(_Info)]
        L.nttk_params_fast_flags.argtypes = [vp, C.c_int, C.c_int, C.POINTER(C.c_uint32)]
        L.nttk_params_table.restype = sz
        L.nttk_params_table.argtypes = [vp, C.c_char_p, vp, sz]
        for f in ("nttk_ntt_forward", "nttk_intt_inverse"):
            getattr(L, f).argtypes = [vp, C.c_int, vp, vp, sz, C.c_int, vp]
        for f in ("nttk_pointwise_multiply", "nttk_basemul", "nttk_polymul"):
            getattr(L, f).argtypes = [vp, C.c_int, vp, vp, vp, sz, C.c_int, vp]
        for f in ("nttk_ntt_forward_host", "nttk_intt_inverse_host"):
            getattr(L, f).argtypes = [vp, C.c_int, vp, vp, sz, C.c_int]
        L.nttk_roundtrip_host.argtypes = [vp, C.c_int, vp, vp, vp, sz, C.c_int]
        for f in ("nttk_pointwise_multiply_host", "nttk_polymul_host"):
            getattr(L, f).argtypes = [vp, C.c_int, vp, vp, vp, sz, C.c_int]
        L.nttk_modmul_sweep.argtypes = [C.c_int, C.c_uint64, C.c_uint32, C.c_uint32, vp, sz, vp,
                                        sz, vp, C.POINTER(C.c_uint64), vp]
        L.nttk_modmul_sweep_device.argtypes = [C.c_int, C.c_uint64, C.c_uint32, C.c_uint32, vp,
                                               sz, vp, sz, vp, vp, vp]
        L.nttk_make_reduction_context.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                                  C.POINTER(ReductionContext)]
        L.nttk_reduce.argtypes = [C.c_int, C.POINTER(ReductionContext), vp, vp, vp, sz, vp]
        L.nttk_reduce_host.argtypes = [C.c_int, C.POINTER(ReductionContext), vp, vp, vp, sz]
        for f in ("nttk_butterfly", "nttk_butterfly_host"):
            extra = [vp] if f == "nttk_butterfly" else []
            getattr(L, f).argtypes = ([C.c_int, C.POINTER(ReductionContext), C.c_uint32, C.c_uint32]
                                      + [vp] * 6 + [sz] + extra)
        for f in ("nttk_ntt_forward_observed", "nttk_intt_inverse_observed"):
            getattr(L, f).argtypes = [vp, C.c_int, vp, vp, _OBSERVER, vp]
        L.nttk_last_error.restype = C.c_char_p
        L.nttk_launch_count.restype = C.c_uint64
        L.nttk_plantard_correction_fires.restype = C.c_uint64
        L.nttk_version.restype = C.c_char_p
        L.nttk_plan_create.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp, sz, C.c_int, C.c_int,
                                       C.POINTER(vp)]
        L.nttk_plan_launch.argtypes = [vp, vp]
        L.nttk_plan_destroy.argtypes = [vp]
        L.nttk_plan_destroy.restype = None
        _lib_handle = L
    return _lib_handle


def _check(status: int) -> None:
    if status == 0:
        return
    msg = lib().nttk_last_error().decode()
    if status == 2:
        raise ContractViolation(msg)
    if status == 1:
        raise PropertyViolation(msg)
    raise CudaError(msg)


def device_available() -> bool:
    return bool(lib().nttk_device_available())


def plantard_correction_fires() -> int:
    """reduction.hpp:172-175: how often plantard_redc's r == p corner fired in this process
    (counted on the device by the reduce entry points and the synchronous modmul_sweep)."""
    return int(lib().nttk_plantard_correction_fires())


def launch_count() -> int:
    """Kernel launches issued by the engine in this process (bench gpu_launches)."""
    return int(lib().nttk_launch_count())


# ---------------------------------------------------------------------------
# parameters

class NttParams:
    """Handle over the engine's parameter bundle (params.hpp:107-128 NttParams)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        info = _Info()
        _check(lib().nttk_params_get_info(self._h, C.byref(info)))
        self.p = int(info.p)
        self.size = int(info.N)
        self.log2_size = int(info.log2N)
        self.n_bits = int(info.n_bits)
        self.omega = int(info.omega)
        self.omega_inv = int(info.omega_inv)
        self.n_inv = int(info.n_inv)
        self.n_inv_hat = int(info.n_inv_hat)
        self.mu = int(info.mu)
        self.layers = int(info.layers)
        self.tree = Tree(info.tree)
        self.scott_lazy_level = int(info.scott_L)
        self.kinds = [k for k in ButterflyKind if (info.kinds_mask >> k) & 1]
        self.fast_path = [k for k in ButterflyKind if (info.fast_path >> k) & 1]

    def __del__(self):
        try:
            if self._h:
                lib().nttk_params_destroy(self._h)
        except Exception:
            pass

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def has(self, kind) -> bool:
        return ButterflyKind(kind) in self.kinds

    def fast_flags(self, kind, direction: int) -> int:
        """Host-validated fast-kernel option bits of (kind, direction) -- see
        nttk_params_fast_flags in include/nttk_gpu.h (introspection, no device needed)."""
        f = C.c_uint32(0)
        _check(lib().nttk_params_fast_flags(self.handle, int(kind), int(direction), C.byref(f)))
        return f.value

    def table(self, name: str) -> np.ndarray:
        n = lib().nttk_params_table(self._h, name.encode(), None, 0)
        out = np.zeros(n, dtype=np.uint64)
        lib().nttk_params_table(self._h, name.encode(), out.ctypes.data, n)
        return out

    def __repr__(self):
        return (f"NttParams(p={self.p}, N={self.size}, n={self.n_bits}, tree={self.tree.name}, "
                f"layers={self.layers}, kinds={[k.name for k in self.kinds]})")


def build_params(p: int, N: int, n_bits: int, kinds: Iterable = None, *, tree=Tree.cyclic,
                 layers: int = 0, root: int = 0, exact_bound: bool = False) -> NttParams:
    """params.hpp:137-268; ``exact_bound`` admits `improved` under Prop. 4's exact bound."""
    kinds = all_butterfly_kinds() if kinds is None else list(kinds)
    mask = 0
    for k in kinds:
        mask |= 1 << int(k)
    d = _Desc(p, N, n_bits, mask, int(tree), layers, root, 1 if exact_bound else 0)
    h = C.c_void_p()
    _check(lib().nttk_build_params(C.byref(d), C.byref(h)))
    return NttParams(h.value)


def preset(name: str) -> NttParams:
    """params.hpp:303-306."""
    h = C.c_void_p()
    _check(lib().nttk_preset(name.encode(), C.byref(h)))
    return NttParams(h.value)


# ---------------------------------------------------------------------------
# reference-shaped host calls

@dataclass
class Spectrum:
    """transform.hpp:30-33."""

    values: list = field(default_factory=list)
    ordering: Ordering = Ordering.bit_reversed


_ELEM = {np.dtype(np.uint16): 2, np.dtype(np.int16): 2, np.dtype(np.uint32): 4,
         np.dtype(np.int32): 4, np.dtype(np.uint64): 8, np.dtype(np.int64): 8}


def _as_batch(x, N: int, signed: bool = False) -> np.ndarray:
    if isinstance(x, np.ndarray) and x.dtype in _ELEM:
        a = np.ascontiguousarray(x)
    else:
        a = np.ascontiguousarray(np.array(list(x) if not isinstance(x, np.ndarray) else x,
                                          dtype=np.int64 if signed else np.uint64))
    if a.size % N != 0 or a.size == 0:
        return None
    return a.reshape(-1, N)


def ntt_forward_batch(f: np.ndarray, P: NttParams, kind) -> np.ndarray:
    """Batched checked forward on host memory (transform.hpp:207-224 per polynomial)."""
    a = _as_batch(f, P.size)
    if a is None:
        raise ContractViolation("ntt_forward: wrong input length")
    out = np.empty_like(a)
    _check(lib().nttk_ntt_forward_host(P.handle, int(kind), a.ctypes.data, out.ctypes.data,
                                       a.shape[0], a.itemsize))
    return out


def intt_inverse_batch(s: np.ndarray, P: NttParams, kind) -> np.ndarray:
    """Batched inverse on host memory (transform.hpp:233-343 per polynomial)."""
    a = _as_batch(s, P.size, signed=ButterflyKind(kind) == ButterflyKind.smont)
    if a is None:
        raise ContractViolation("intt_inverse: wrong input length")
    out = np.empty_like(a)
    _check(lib().nttk_intt_inverse_host(P.handle, int(kind), a.ctypes.data, out.ctypes.data,
                                        a.shape[0], a.itemsize))
    return out


def ntt_forward(f: Sequence[int], P: NttParams, kind) -> Spectrum:
    """transform.hpp:220-224: natural-order canonical input, bit-reversed lazy spectrum."""
    if not P.has(kind):
        raise ContractViolation("ntt_forward: kind not built into these params")
    if len(f) != P.size:
        raise ContractViolation("ntt_forward: wrong input length")
    out = ntt_forward_batch(np.asarray(f, dtype=np.uint64), P, kind)
    vals = out.reshape(-1)
    if ButterflyKind(kind) == ButterflyKind.smont:
        vals = vals.view(np.int64)
    return Spectrum([int(v) for v in vals], Ordering.bit_reversed)


def ntt_forward_inplace(a: np.ndarray, P: NttParams, kind) -> None:
    """transform.hpp:228-231 (benchmark path): no validation beyond the engine's."""
    out = ntt_forward_batch(a, P, kind)
    a[...] = out.reshape(a.shape)


def intt_inverse(s: Spectrum, P: NttParams, kind) -> list:
    """transform.hpp:339-343."""
    if not P.has(kind):
        raise ContractViolation("intt_inverse: kind not built into these params")
    if len(s.values) != P.size:
        raise ContractViolation("intt_inverse: wrong input length")
    if s.ordering != Ordering.bit_reversed:
        raise ContractViolation("intt_inverse: spectrum must be in butterfly order")
    signed = ButterflyKind(kind) == ButterflyKind.smont or any(v < 0 for v in s.values)
    arr = np.array(s.values, dtype=np.int64 if signed else np.uint64)
    out = intt_inverse_batch(arr, P, kind)
    return [int(v) for v in out.reshape(-1)]


def pointwise_multiply(lhs: Spectrum, rhs: Spectrum, P: NttParams, kind) -> Spectrum:
    """transform.hpp:349-370 (canonical output)."""
    if len(lhs.values) != P.size or len(rhs.values) != P.size:
        raise ContractViolation("pointwise_multiply: wrong spectrum length")
    if lhs.ordering != rhs.ordering:
        raise ContractViolation("pointwise_multiply: mixed orderings")
    signed = ButterflyKind(kind) == ButterflyKind.smont
    dt = np.int64 if signed else np.uint64
    out = pointwise_multiply_batch(np.array(lhs.values, dtype=dt), np.array(rhs.values, dtype=dt),
                                   P, kind)
    return Spectrum([int(v) for v in out.reshape(-1)], lhs.ordering)


def pointwise_multiply_batch(lhs: np.ndarray, rhs: np.ndarray, P: NttParams, kind) -> np.ndarray:
    a = _as_batch(lhs, P.size)
    b = _as_batch(rhs, P.size)
    if a is None or b is None or a.shape != b.shape or a.dtype != b.dtype:
        raise ContractViolation("pointwise_multiply: wrong spectrum length")
    out = np.empty_like(a)
    _check(lib().nttk_pointwise_multiply_host(P.handle, int(kind), a.ctypes.data, b.ctypes.data,
                                              out.ctypes.data, a.shape[0], a.itemsize))
    return out


def polymul_batch(x: np.ndarray, y: np.ndarray, P: NttParams, kind) -> np.ndarray:
    """Batched product via NTT on host memory (cyclic: transform.hpp:372-379)."""
    a = _as_batch(x, P.size)
    b = _as_batch(y, P.size)
    if a is None or b is None or a.shape != b.shape or a.dtype != b.dtype:
        raise ContractViolation("polymul: size mismatch")
    out = np.empty_like(a)
    _check(lib().nttk_polymul_host(P.handle, int(kind), a.ctypes.data, b.ctypes.data,
                                   out.ctypes.data, a.shape[0], a.itemsize))
    return out


def cyclic_convolution_via_ntt(x: Sequence[int], y: Sequence[int], P: NttParams,
                               kind=ButterflyKind.improved) -> list:
    """transform.hpp:372-379."""
    if len(x) != P.size or len(y) != P.size:
        raise ContractViolation("ntt_forward: wrong input length")
    out = polymul_batch(np.asarray(x, dtype=np.uint64), np.asarray(y, dtype=np.uint64), P, kind)
    return [int(v) for v in out.reshape(-1)]


# ---------------------------------------------------------------------------
# batched device API on torch CUDA tensors

_TORCH_ELEM = None


def _torch_elem(t) -> int:
    global _TORCH_ELEM
    import torch

    if _TORCH_ELEM is None:
        _TORCH_ELEM = {torch.int16: 2, torch.uint16: 2, torch.int32: 4, torch.uint32: 4,
                       torch.int64: 8, torch.uint64: 8}
    if not t.is_cuda:
        raise ContractViolation("device API expects CUDA tensors")
    if not t.is_contiguous():
        raise ContractViolation("device API expects contiguous tensors")
    if t.dtype not in _TORCH_ELEM:
        raise ContractViolation(f"unsupported coefficient dtype {t.dtype}")
    return _TORCH_ELEM[t.dtype]


_RAW_STREAM = None


def _stream_ptr(stream, t=None) -> int:
    """cudaStream_t of `stream`, else torch's current stream on t's device (raw getter:
    building a torch.cuda.Stream object per call costs microseconds)."""
    global _RAW_STREAM
    if stream is not None:
        return stream.cuda_stream
    import torch

    if _RAW_STREAM is None:
        _RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", False)
    if _RAW_STREAM and t is not None:
        return _RAW_STREAM(t.device.index)
    return torch.cuda.current_stream().cuda_stream


def _batch_of(t, N: int) -> int:
    if t.numel() % N:
        raise ContractViolation("wrong input length")
    return t.numel() // N


def _match(ref, t, what: str):
    """A second operand or a caller-supplied output must be a CUDA tensor shaped like the
    first operand: same dtype, element count, device and contiguity (the C ABI only sees
    pointers and the first operand's batch)."""
    _torch_elem(t)
    if t.dtype != ref.dtype or t.numel() != ref.numel() or t.device != ref.device:
        raise ContractViolation(f"{what} must match the first operand (dtype {ref.dtype}, "
                                f"{ref.numel()} elements, {ref.device}); got {t.dtype}, "
                                f"{t.numel()} elements, {t.device}")
    return t


def _on_device(x, call):
    """Run `call` with x's device current: the C ABI resolves tables and launches on the
    current device."""
    import torch

    idx = x.device.index
    if idx == torch.cuda.current_device():
        return call()
    with torch.cuda.device(idx):
        return call()


def _out(x, out):
    import torch

    return torch.empty_like(x) if out is None else _match(x, out, "out")


def forward(P: NttParams, kind, x, out=None, stream=None):
    """Batched ntt_forward on device tensors (natural -> bit-reversed lazy spectrum)."""
    e = _torch_elem(x)
    out = _out(x, out)
    _on_device(x, lambda: _check(lib().nttk_ntt_forward(
        P.handle, int(kind), x.data_ptr(), out.data_ptr(), _batch_of(x, P.size), e,
        _stream_ptr(stream, x))))
    return out


def inverse(P: NttParams, kind, x, out=None, stream=None):
    """Batched intt_inverse on device tensors (canonical natural-order output)."""
    e = _torch_elem(x)
    out = _out(x, out)
    _on_device(x, lambda: _check(lib().nttk_intt_inverse(
        P.handle, int(kind), x.data_ptr(), out.data_ptr(), _batch_of(x, P.size), e,
        _stream_ptr(stream, x))))
    return out


class Plan:
    """A captured operation on fixed device tensors (nttk_plan_create, include/nttk_gpu.h):
    `repeat` back-to-back forward / inverse / polymul calls recorded into one CUDA graph;
    launch() replays it (small batches: one host call instead of `repeat`).  Creating a plan
    runs nothing; the tensors must stay alive while the plan is used."""

    FORWARD, INVERSE, POLYMUL = 0, 1, 2

    def __init__(self, P: NttParams, kind, op: int, a, out, b=None, repeat: int = 1):
        e = _torch_elem(a)
        _match(a, out, "out")
        if b is not None:
            _match(a, b, "b")
        self._keep = (P, a, b, out)  # the graph holds raw pointers
        h = C.c_void_p()
        _on_device(a, lambda: _check(lib().nttk_plan_create(
            P.handle, int(kind), int(op), a.data_ptr(), b.data_ptr() if b is not None else None,
            out.data_ptr(), _batch_of(a, P.size), e, int(repeat), C.byref(h))))
        self.handle = h.value
        self.device = a.device

    def launch(self, stream=None) -> None:
        import torch

        with torch.cuda.device(self.device):
            _check(lib().nttk_plan_launch(self.handle, _stream_ptr(stream, self._keep[1])))

    def __del__(self):
        if getattr(self, "handle", None) and _lib_handle is not None:
            _lib_handle.nttk_plan_destroy(self.handle)
            self.handle = None


def _binary(fn, P: NttParams, kind, a, b, out, stream):
    e = _torch_elem(a)
    _match(a, b, "b")
    out = _out(a, out)
    _on_device(a, lambda: _check(fn(P.handle, int(kind), a.data_ptr(), b.data_ptr(),
                                    out.data_ptr(), _batch_of(a, P.size), e,
                                    _stream_ptr(stream, a))))
    return out


def pointwise(P: NttParams, kind, a, b, out=None, stream=None):
    """Slotwise spectrum product (transform.hpp:349-370), canonical output."""
    return _binary(lib().nttk_pointwise_multiply, P, kind, a, b, out, stream)


def basemul(P: NttParams, kind, a, b, out=None, stream=None):
    """Degree-2 basemul of 7-layer negacyclic spectra (extension)."""
    return _binary(lib().nttk_basemul, P, kind, a, b, out, stream)


def polymul(P: NttParams, kind, a, b, out=None, stream=None):
    """Fused forward(a), forward(b), product, inverse (transform.hpp:372-379)."""
    return _binary(lib().nttk_polymul, P, kind, a, b, out, stream)


def roundtrip_host(P: NttParams, kind, h_in, h_spec, h_out) -> None:
    """forward + inverse over host memory (numpy or pinned torch CPU tensors)."""
    def ptr(t):
        return t.ctypes.data if isinstance(t, np.ndarray) else t.data_ptr()

    def n_elem(t):
        return t.itemsize if isinstance(t, np.ndarray) else t.element_size()

    n = h_in.size if isinstance(h_in, np.ndarray) else h_in.numel()
    _check(lib().nttk_roundtrip_host(P.handle, int(kind), ptr(h_in),
                                     ptr(h_spec) if h_spec is not None else None, ptr(h_out),
                                     n // P.size, n_elem(h_in)))


def modmul_sweep(variant, p: int, n_bits: int, ell: int, A, B, r=None, stream=None) -> int:
    """Run one reduction over the operand grid (A[i], B[j]) of int64 CUDA tensors.

    Results go to ``r`` (int64, len(A)*len(B), optional); returns the wrapping u64 sum.
    """
    _sweep_operands(A, B, r)
    s = C.c_uint64()
    _on_device(A, lambda: _check(lib().nttk_modmul_sweep(
        int(variant), p, n_bits, ell, A.data_ptr(), A.numel(), B.data_ptr(), B.numel(),
        r.data_ptr() if r is not None else None, C.byref(s), _stream_ptr(stream, A))))
    return int(s.value)


def _sweep_operands(A, B, r):
    import torch

    for t, what in ((A, "A"), (B, "B")):
        if t.dtype != torch.int64 or not t.is_cuda or not t.is_contiguous() or t.device != A.device:
            raise ContractViolation(f"modmul_sweep: {what} must be a contiguous int64 CUDA "
                                    f"tensor on {A.device}")
    if r is not None and (r.dtype != torch.int64 or r.numel() < A.numel() * B.numel()
                          or not r.is_contiguous() or r.device != A.device):
        raise ContractViolation("modmul_sweep: r must be a contiguous int64 CUDA tensor of "
                                "len(A) * len(B) elements on A's device")


def modmul_sweep_device(variant, p: int, n_bits: int, ell: int, A, B, checksum, r=None,
                        stream=None) -> None:
    """Device form of :func:`modmul_sweep`: adds the wrapping sum into ``checksum`` (a
    one-element int64 CUDA tensor the caller zeroes) without synchronising."""
    import torch
    if checksum.dtype != torch.int64 or checksum.numel() < 1 or checksum.device != A.device:
        raise ContractViolation("modmul_sweep: checksum must be an int64 CUDA tensor on A's device")
    _sweep_operands(A, B, r)
    _on_device(A, lambda: _check(lib().nttk_modmul_sweep_device(
        int(variant), p, n_bits, ell, A.data_ptr(), A.numel(), B.data_ptr(), B.numel(),
        r.data_ptr() if r is not None else None, checksum.data_ptr(), _stream_ptr(stream, A))))


# ---------------------------------------------------------------------------
# reduction.hpp: make_reduction_context + the word-level reductions, run on the GPU
# (reduce.cu).  Scalars in -> scalar out (reference signatures); numpy arrays in ->
# arrays out (one launch); `reduce` is the device-tensor form.

OP_MONT_REDC, OP_SIGNED_MONT_REDC, OP_PLANTARD_REDC, OP_MODIFIED_PLANTARD_MUL = 0, 1, 2, 3
OP_TO_PLANTARD_DOMAIN, OP_TO_MONTGOMERY_DOMAIN = 4, 5


def make_reduction_context(p: int, n_bits: int, alpha: int = 0, ell: int = 0) -> ReductionContext:
    """reduction.hpp:80-117 (same validation and messages)."""
    c = ReductionContext()
    _check(lib().nttk_make_reduction_context(p, n_bits, alpha, ell, C.byref(c)))
    return c


def _reduce_host(op, ctx, x, y=None):
    scalar = np.isscalar(x)
    xs = np.ascontiguousarray(np.atleast_1d(np.asarray(x)).astype(np.int64 if op == 1 else np.uint64)
                              .view(np.int64))
    ys = None
    if y is not None:
        ys = np.ascontiguousarray(np.atleast_1d(np.asarray(y)).astype(np.uint64).view(np.int64))
        if ys.size != xs.size:
            raise ContractViolation("reduce: operand lengths differ")
    out = np.empty_like(xs)
    _check(lib().nttk_reduce_host(op, C.byref(ctx), xs.ctypes.data,
                                  ys.ctypes.data if ys is not None else None, out.ctypes.data,
                                  xs.size))
    res = out if op == OP_SIGNED_MONT_REDC else out.view(np.uint64)
    return int(res[0]) if scalar else res


def mont_redc(T, ctx: ReductionContext):
    """reduction.hpp:125-135: T in [0, p^2) -> T 2^{-n} mod p."""
    return _reduce_host(OP_MONT_REDC, ctx, T)


def signed_mont_redc(A, ctx: ReductionContext):
    """reduction.hpp:141-165: A in (-p 2^{n-1}, p 2^{n-1}) -> A 2^{-n} mod p in (-p, p)."""
    return _reduce_host(OP_SIGNED_MONT_REDC, ctx, A)


def plantard_redc(W, T, ctx: ReductionContext):
    """reduction.hpp:178-191: W, T in [0, p] -> W T (-2^{-2n}) mod p."""
    return _reduce_host(OP_PLANTARD_REDC, ctx, W, T)


def modified_plantard_mul(W, T, ctx: ReductionContext):
    """reduction.hpp:264-273: W < p, T < 2^ell p -> W T (-2^{-2n}) mod p (Alg. 10)."""
    return _reduce_host(OP_MODIFIED_PLANTARD_MUL, ctx, W, T)


def to_plantard_domain(w, ctx: ReductionContext):
    """reduction.hpp:279-283."""
    return _reduce_host(OP_TO_PLANTARD_DOMAIN, ctx, w)


def to_montgomery_domain(w, ctx: ReductionContext):
    """reduction.hpp:287-291."""
    return _reduce_host(OP_TO_MONTGOMERY_DOMAIN, ctx, w)


def reduce(op: int, ctx: ReductionContext, x, y=None, out=None, stream=None):
    """Elementwise reduction on int64 CUDA tensors (synchronises `stream`: operand ranges
    are checked on the device like the reference's NTTK_REQUIRE)."""
    import torch

    if x.dtype != torch.int64 or not x.is_cuda or not x.is_contiguous():
        raise ContractViolation("reduce: x must be a contiguous int64 CUDA tensor")
    if y is not None:
        _match(x, y, "y")
    out = _out(x, out)
    _on_device(x, lambda: _check(lib().nttk_reduce(
        int(op), C.byref(ctx), x.data_ptr(), y.data_ptr() if y is not None else None,
        out.data_ptr(), x.numel(), _stream_ptr(stream, x))))
    return out


# ---------------------------------------------------------------------------
# butterfly.hpp checked entry points, run on the GPU (reduce.cu)

BF_NTL, BF_HARVEY, BF_SCOTT, BF_IMPROVED_CT, BF_IMPROVED_GS = 0, 1, 2, 3, 4


@dataclass
class ScottConfig:
    """butterfly.hpp:151-155 (the guard hook is not carried to the device)."""
    transform_size: int
    lazy_level: int


def make_scott_config(N: int, ctx: ReductionContext) -> ScottConfig:
    """butterfly.hpp:157-168: smallest power-of-two L with 4 N p < 2^n L."""
    if N <= 0 or N & (N - 1):
        raise ContractViolation("scott config: N must be a power of two")
    L = 1
    while L <= N:
        if 4 * N * ctx.p < ctx.beta * L:
            return ScottConfig(N, L)
        L *= 2
    raise ContractViolation(
        f"scott config: no lazy level satisfies 4*N*p/L < 2^n for p={ctx.p}")


def _butterfly_host(op, ctx, X, Y, W, Wq=None, aux0=0, aux1=0):
    scalar = np.isscalar(X)
    arrs = [np.ascontiguousarray(np.atleast_1d(np.asarray(v)).astype(np.uint64).view(np.int64))
            if v is not None else None for v in (X, Y, W, Wq)]
    n = arrs[0].size
    if any(a is not None and a.size != n for a in arrs):
        raise ContractViolation("butterfly: operand lengths differ")
    xo, yo = np.empty(n, np.int64), np.empty(n, np.int64)
    _check(lib().nttk_butterfly_host(op, C.byref(ctx), aux0, aux1,
                                     *[a.ctypes.data if a is not None else None for a in arrs],
                                     xo.ctypes.data, yo.ctypes.data, n))
    xo, yo = xo.view(np.uint64), yo.view(np.uint64)
    return (int(xo[0]), int(yo[0])) if scalar else (xo, yo)


def ntl_butterfly(X, Y, W, W_quot, ctx: ReductionContext):
    """butterfly.hpp:60-86 (Alg. 7)."""
    return _butterfly_host(BF_NTL, ctx, X, Y, W, W_quot)


def harvey_butterfly(X, Y, W_mont, ctx: ReductionContext):
    """butterfly.hpp:92-121 (Alg. 8)."""
    return _butterfly_host(BF_HARVEY, ctx, X, Y, W_mont)


harvey_butterfly_ref = harvey_butterfly  # butterfly.hpp:124-142: bit-identical twin


def scott_butterfly(X, Y, W_mont, ctx: ReductionContext, cfg: ScottConfig):
    """butterfly.hpp:172-212 (Alg. 9; no guard)."""
    return _butterfly_host(BF_SCOTT, ctx, X, Y, W_mont, None, cfg.transform_size, cfg.lazy_level)


def improved_ct_butterfly(X, Y, W_hat, ctx: ReductionContext):
    """butterfly.hpp:247-260 (Alg. 11)."""
    return _butterfly_host(BF_IMPROVED_CT, ctx, X, Y, W_hat)


def improved_gs_butterfly(X, Y, W_hat, ctx: ReductionContext, layer: int):
    """butterfly.hpp:263-279 (Alg. 12)."""
    return _butterfly_host(BF_IMPROVED_GS, ctx, X, Y, W_hat, None, layer)


# ---------------------------------------------------------------------------
# transform.hpp / params.hpp helpers (same names as the reference)

def spectrum_value_bound(P: NttParams, kind) -> int:
    """transform.hpp:61-70 (smont: bound on |value|)."""
    k = ButterflyKind(kind)
    return {ButterflyKind.ntl: P.p, ButterflyKind.harvey: 2 * P.p,
            ButterflyKind.scott: P.size * P.p, ButterflyKind.improved: (P.log2_size + 1) * P.p,
            ButterflyKind.smont: (P.log2_size + 2) * P.p}[k]


def canonicalize(v, p: int):
    """transform.hpp:38-40: every word mod p, on the device (returns a new array)."""
    a = np.ascontiguousarray(np.atleast_1d(np.asarray(v)).astype(np.uint64))
    c = ReductionContext()
    c.p, c.n_bits = p, 32  # the mod-p op reads only p
    out = np.empty_like(a)
    _check(lib().nttk_reduce_host(6, C.byref(c), a.ctypes.data, None, out.ctypes.data, a.size))
    return out


def bit_reverse_permutation(v) -> list:
    """transform.hpp:42-52 (index permutation only)."""
    n = len(v)
    if n == 0 or n & (n - 1):
        raise ContractViolation("bit_reverse_permutation: size must be a power of two")
    bits = n.bit_length() - 1
    out = [0] * n
    for i, x in enumerate(v):
        out[int(format(i, f"0{bits}b")[::-1], 2) if bits else 0] = x
    return out


def to_natural_order(s: Spectrum) -> list:
    """transform.hpp:54-58."""
    return list(s.values) if s.ordering == Ordering.natural else bit_reverse_permutation(s.values)


PRESET_TABLE = (("kyber256", 7681, 256, 32), ("kcl256", 7681, 256, 32),
                ("newhope512", 12289, 512, 32), ("falcon512", 12289, 512, 32),
                ("remblem512", 12289, 512, 32), ("newhope1024", 12289, 1024, 32),
                ("falcon1024", 12289, 1024, 32), ("hila5-1024", 12289, 1024, 32),
                ("toy13", 13, 4, 8))  # params.hpp:280-289


def preset_spec(name: str):
    """params.hpp:291-301 -> (name, p, size, n_bits)."""
    for spec in PRESET_TABLE:
        if spec[0] == name:
            return spec
    preset(name)  # raises the engine's "unknown preset ... (known: ...)" message
    raise ContractViolation(f"unknown preset '{name}'")


def find_primitive_root(p: int, N: int) -> int:
    """params.hpp:30-43: smallest w with w^N = 1 and w^{N/2} != 1 (host parameter search)."""
    if N <= 0 or N & (N - 1):
        raise ContractViolation("find_primitive_root: N must be a power of two")
    if (p - 1) % N:
        raise ContractViolation("find_primitive_root: N must divide p - 1")
    if N == 1:
        return 1
    for w in range(2, p):
        if pow(w, N, p) == 1 and pow(w, N // 2, p) != 1:
            return w
    raise ContractViolation("find_primitive_root: no root found")


def dif_forward_plain_twiddles(N: int, omega: int, p: int) -> list:
    """params.hpp:47-58."""
    out, ln = [], N // 2
    while ln >= 1:
        step = N // (2 * ln)
        out += [pow(omega, j * step, p) for j in range(ln)]
        ln //= 2
    return out


def ct_forward_plain_twiddles(N: int, omega: int, p: int) -> list:
    """params.hpp:60-72."""
    out, ln = [], N // 2
    while ln >= 1:
        blocks = N // (2 * ln)
        lvl = blocks.bit_length() - 1
        out += [pow(omega, ln * (int(format(b, f"0{lvl}b")[::-1], 2) if lvl else 0), p)
                for b in range(blocks)]
        ln //= 2
    return out


def gs_inverse_plain_twiddles(N: int, omega: int, p: int) -> list:
    """params.hpp:74-88."""
    out, ln = [], 1
    while ln < N:
        blocks = N // (2 * ln)
        lvl = blocks.bit_length() - 1
        for b in range(blocks):
            e = ln * (int(format(b, f"0{lvl}b")[::-1], 2) if lvl else 0) % N
            out.append(pow(omega, N - e if e else 0, p))
        ln *= 2
    return out


# ---------------------------------------------------------------------------
# observed transforms (transform.hpp:207-217, 233-337): observer(layer, state) per layer

def _observed(fn, P: NttParams, kind, words, observer):
    a = np.ascontiguousarray(np.array(words, dtype=np.uint64).reshape(-1))
    if a.size != P.size:
        raise ContractViolation(("ntt_forward" if fn.endswith("forward_observed") else "intt_inverse")
                                + ": wrong input length")
    out = np.empty_like(a)
    err = []

    def cb(layer, state, n, user):
        if err or observer is None:
            return
        try:
            observer(int(layer), [int(state[i]) for i in range(n)])
        except BaseException as e:  # re-raised after the call: never unwind through C
            err.append(e)

    cfn = _OBSERVER(cb)
    st = getattr(lib(), fn)(P.handle, int(kind), a.ctypes.data, out.ctypes.data, cfn, None)
    if err:
        raise err[0]
    _check(st)
    return [int(v) for v in out]


def ntt_forward_observed(f, P: NttParams, kind, observer) -> Spectrum:
    """transform.hpp:207-217."""
    return Spectrum(_observed("nttk_ntt_forward_observed", P, kind, f, observer), Ordering.bit_reversed)


def intt_inverse_observed(s: Spectrum, P: NttParams, kind, observer) -> list:
    """transform.hpp:233-337."""
    if s.ordering != Ordering.bit_reversed:
        raise ContractViolation("intt_inverse: spectrum must be in butterfly order")
    return _observed("nttk_intt_inverse_observed", P, kind, s.values, observer)
