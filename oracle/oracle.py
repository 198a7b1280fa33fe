"""ctypes bindings for the parity checker (TEST INFRASTRUCTURE ONLY).

``Oracle`` wraps ``oracle/liboracle.so`` -- the C restatement of the reference NTT path
(nttk_oracle.c).  ``Reference`` wraps ``oracle/_ref/libnttk_ref.so`` -- the unmodified
reference headers (/root/reference/proj/include/nttk) behind a C shim, built in this
container only.  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import
this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libnttk_ref.so")

NTL, HARVEY, SCOTT, IMPROVED, SMONT = range(5)
KIND_NAMES = {"ntl": NTL, "harvey": HARVEY, "scott": SCOTT, "improved": IMPROVED, "smont": SMONT}
CYCLIC, NEGA = 0, 1
SW_MONT, SW_SMONT, SW_PLANTARD, SW_MPLANTARD = range(4)

u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class Ctx(C.Structure):
    _fields_ = [
        ("p", C.c_uint32), ("n_bits", C.c_uint), ("alpha", C.c_uint), ("ell", C.c_uint),
        ("beta", C.c_uint64), ("beta_mask", C.c_uint64), ("r2n_mask", C.c_uint64),
        ("p_inv_beta", C.c_uint64), ("neg_p_inv_beta", C.c_uint64), ("mu", C.c_uint64),
        ("mu_centered", C.c_int64), ("beta_mod_p", C.c_uint64), ("r2n_mod_p", C.c_uint64),
    ]


class Params(C.Structure):
    _fields_ = [
        ("p", C.c_uint32), ("N", C.c_uint32), ("log2N", C.c_uint32), ("n_bits", C.c_uint32),
        ("tree", C.c_uint32), ("layers", C.c_uint32), ("kinds_mask", C.c_uint32),
        ("scott_L", C.c_uint32), ("omega", C.c_uint64), ("omega_inv", C.c_uint64),
        ("n_inv", C.c_uint64), ("n_inv_hat", C.c_uint64), ("n_inv_mont", C.c_uint64),
        ("n_inv_smont", C.c_int64), ("ctx", Ctx), ("fwd_len", C.c_size_t),
        ("inv_len", C.c_size_t),
        # table pointers follow; accessed through or_params_table
    ]


def build_oracle() -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        build_oracle()
    return C.CDLL(path)


class Oracle:
    _lib = None

    def __init__(self):
        if Oracle._lib is None:
            Oracle._lib = _load(ORACLE_SO)
            self._declare(Oracle._lib)
        self.lib = Oracle._lib

    @staticmethod
    def _declare(L):
        L.or_last_error.restype = C.c_char_p
        L.or_pow_mod.restype = C.c_uint64
        L.or_pow_mod.argtypes = [C.c_uint64] * 3
        L.or_bit_reverse.restype = C.c_uint64
        L.or_bit_reverse.argtypes = [C.c_uint64, C.c_uint]
        L.or_rng_fill.argtypes = [C.c_uint64, C.c_uint64, u64p, C.c_size_t]
        L.or_make_ctx.argtypes = [C.c_uint64, C.c_uint, C.c_uint, C.c_uint, C.POINTER(Ctx)]
        for f in ("or_ctx_fits_plantard", "or_ctx_fits_lazy_plantard",
                  "or_ctx_fits_signed_montgomery"):
            getattr(L, f).argtypes = [C.POINTER(Ctx)]
        L.or_mont_redc.argtypes = [C.c_uint64, C.POINTER(Ctx), C.POINTER(C.c_uint64)]
        L.or_signed_mont_redc.argtypes = [C.c_int64, C.POINTER(Ctx), C.POINTER(C.c_int64)]
        L.or_plantard_redc.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(Ctx),
                                       C.POINTER(C.c_uint64)]
        L.or_plantard_fires.restype = C.c_uint64
        L.or_modified_plantard_mul.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(Ctx),
                                               C.POINTER(C.c_uint64)]
        L.or_to_plantard_domain.argtypes = [C.c_uint64, C.POINTER(Ctx), C.POINTER(C.c_uint64)]
        L.or_to_montgomery_domain.argtypes = [C.c_uint64, C.POINTER(Ctx),
                                              C.POINTER(C.c_uint64)]
        L.or_signed_barrett.restype = C.c_int64
        L.or_signed_barrett.argtypes = [C.c_int64, C.POINTER(Ctx)]
        bf = [C.c_uint64, C.c_uint64]
        out2 = [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.or_ntl_core.argtypes = bf + [C.c_uint64, C.c_uint64, C.POINTER(Ctx)] + out2
        L.or_harvey_core.argtypes = bf + [C.c_uint64, C.POINTER(Ctx)] + out2
        L.or_harvey_ct_core.argtypes = bf + [C.c_uint64, C.POINTER(Ctx)] + out2
        L.or_scott_core.argtypes = bf + [C.c_uint64, C.c_uint64, C.POINTER(Ctx)] + out2
        L.or_improved_ct_core.argtypes = bf + [C.c_uint64, C.POINTER(Ctx)] + out2
        L.or_improved_gs_core.argtypes = bf + [C.c_uint64, C.c_uint64, C.POINTER(Ctx)] + out2
        L.or_scott_lazy_level.restype = C.c_uint32
        L.or_scott_lazy_level.argtypes = [C.c_uint32, C.POINTER(Ctx)]
        L.or_find_primitive_root.restype = C.c_uint64
        L.or_find_primitive_root.argtypes = [C.c_uint64, C.c_uint64]
        L.or_params_build.argtypes = [C.c_uint64, C.c_uint32, C.c_uint, C.c_uint32, C.c_uint32,
                                      C.c_uint32, C.c_uint64, C.c_int,
                                      C.POINTER(C.POINTER(Params))]
        L.or_params_free.argtypes = [C.POINTER(Params)]
        L.or_params_table.restype = C.c_size_t
        L.or_params_table.argtypes = [C.POINTER(Params), C.c_char_p, C.c_void_p, C.c_size_t]
        for f in ("or_forward", "or_inverse"):
            getattr(L, f).argtypes = [C.POINTER(Params), C.c_int, u64p, C.c_size_t]
        for f in ("or_pointwise", "or_basemul", "or_polymul"):
            getattr(L, f).argtypes = [C.POINTER(Params), C.c_int, u64p, u64p, u64p, C.c_size_t]
        L.or_naive_dft.argtypes = [u64p, C.c_size_t, C.c_uint64, C.c_uint64, u64p]
        L.or_schoolbook_cyclic.argtypes = [u64p, u64p, C.c_size_t, C.c_uint64, u64p]
        L.or_schoolbook_negacyclic.argtypes = [u64p, u64p, C.c_size_t, C.c_uint64, u64p]
        L.or_naive_nega_eval.argtypes = [C.POINTER(Params), u64p, u64p]
        L.or_sweep.argtypes = [C.c_int, C.POINTER(Ctx), i64p, C.c_size_t, i64p, C.c_size_t,
                               C.c_void_p, C.POINTER(C.c_uint64), C.c_int]
        L.or_fnv1a_u32.restype = C.c_uint64
        L.or_fnv1a_u32.argtypes = [u64p, C.c_size_t]

    # ---- helpers ----
    def _check(self, st: int):
        if st != 0:
            raise OracleError(st, self.lib.or_last_error().decode())

    def rng(self, seed: int, bound: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.uint64)
        self.lib.or_rng_fill(seed, bound, out, count)
        return out

    def ctx(self, p: int, n_bits: int, alpha: int = 0, ell: int = 0) -> Ctx:
        c = Ctx()
        self._check(self.lib.or_make_ctx(p, n_bits, alpha, ell, C.byref(c)))
        return c

    def mont_redc(self, T, c):
        o = C.c_uint64()
        self._check(self.lib.or_mont_redc(T, C.byref(c), C.byref(o)))
        return o.value

    def signed_mont_redc(self, A, c):
        o = C.c_int64()
        self._check(self.lib.or_signed_mont_redc(A, C.byref(c), C.byref(o)))
        return o.value

    def plantard_redc(self, W, T, c):
        o = C.c_uint64()
        self._check(self.lib.or_plantard_redc(W, T, C.byref(c), C.byref(o)))
        return o.value

    def modified_plantard_mul(self, W, T, c):
        o = C.c_uint64()
        self._check(self.lib.or_modified_plantard_mul(W, T, C.byref(c), C.byref(o)))
        return o.value

    def to_plantard_domain(self, w, c):
        o = C.c_uint64()
        self._check(self.lib.or_to_plantard_domain(w, C.byref(c), C.byref(o)))
        return o.value

    def to_montgomery_domain(self, w, c):
        o = C.c_uint64()
        self._check(self.lib.or_to_montgomery_domain(w, C.byref(c), C.byref(o)))
        return o.value

    def butterfly(self, name: str, X: int, Y: int, *args, c):
        x, y = C.c_uint64(), C.c_uint64()
        getattr(self.lib, f"or_{name}_core")(X, Y, *args, C.byref(c), C.byref(x), C.byref(y))
        return x.value, y.value

    def params(self, p, N, n_bits, kinds=(IMPROVED,), tree=CYCLIC, layers=0, root=0,
               exact=False) -> "OracleParams":
        mask = 0
        for k in kinds:
            mask |= 1 << k
        ptr = C.POINTER(Params)()
        self._check(self.lib.or_params_build(p, N, n_bits, mask, tree, layers, root,
                                             int(exact), C.byref(ptr)))
        return OracleParams(self, ptr)

    def naive_dft(self, f, omega, p):
        f = np.ascontiguousarray(f, dtype=np.uint64)
        out = np.empty_like(f)
        self.lib.or_naive_dft(f, f.size, omega, p, out)
        return out

    def schoolbook_cyclic(self, a, b, p):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        b = np.ascontiguousarray(b, dtype=np.uint64)
        out = np.empty_like(a)
        self.lib.or_schoolbook_cyclic(a, b, a.size, p, out)
        return out

    def schoolbook_negacyclic(self, a, b, p):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        b = np.ascontiguousarray(b, dtype=np.uint64)
        out = np.empty_like(a)
        self.lib.or_schoolbook_negacyclic(a, b, a.size, p, out)
        return out

    def sweep(self, variant, c, A, B, want_results=True, threads=1):
        A = np.ascontiguousarray(A, dtype=np.int64)
        B = np.ascontiguousarray(B, dtype=np.int64)
        r = np.empty(A.size * B.size, dtype=np.int64) if want_results else None
        s = C.c_uint64()
        self._check(self.lib.or_sweep(variant, C.byref(c), A, A.size, B, B.size,
                                      r.ctypes.data if r is not None else None, C.byref(s),
                                      threads))
        return r, s.value

    def fnv(self, v) -> int:
        v = np.ascontiguousarray(v, dtype=np.uint64)
        return self.lib.or_fnv1a_u32(v, v.size)


class OracleParams:
    def __init__(self, o: Oracle, ptr):
        self.o, self.ptr = o, ptr
        self.s = ptr.contents

    def __del__(self):
        try:
            self.o.lib.or_params_free(self.ptr)
        except Exception:
            pass

    def __getattr__(self, name):
        return getattr(self.s, name)

    def table(self, name: str) -> np.ndarray:
        n = self.o.lib.or_params_table(self.ptr, name.encode(), None, 0)
        out = np.zeros(n, dtype=np.uint64)
        self.o.lib.or_params_table(self.ptr, name.encode(), out.ctypes.data, n)
        return out

    def forward(self, kind, a):
        a = np.array(a, dtype=np.uint64).reshape(-1, self.N).copy()
        self.o._check(self.o.lib.or_forward(self.ptr, kind, a, a.shape[0]))
        return a

    def inverse(self, kind, a):
        a = np.array(a, dtype=np.uint64).reshape(-1, self.N).copy()
        self.o._check(self.o.lib.or_inverse(self.ptr, kind, a, a.shape[0]))
        return a

    def _binary(self, fn, kind, x, y):
        x = np.ascontiguousarray(np.array(x, dtype=np.uint64).reshape(-1, self.N))
        y = np.ascontiguousarray(np.array(y, dtype=np.uint64).reshape(-1, self.N))
        out = np.empty_like(x)
        self.o._check(getattr(self.o.lib, fn)(self.ptr, kind, x, y, out, x.shape[0]))
        return out

    def pointwise(self, kind, x, y):
        return self._binary("or_pointwise", kind, x, y)

    def basemul(self, kind, x, y):
        return self._binary("or_basemul", kind, x, y)

    def polymul(self, kind, x, y):
        return self._binary("or_polymul", kind, x, y)

    def naive_eval(self, f):
        f = np.ascontiguousarray(f, dtype=np.uint64)
        out = np.empty_like(f)
        self.o.lib.or_naive_nega_eval(self.ptr, f, out)
        return out


def reference_available() -> bool:
    return os.path.exists(REF_SO)


class Reference:
    """The unmodified reference (oracle/_ref/libnttk_ref.so)."""

    _lib = None

    def __init__(self):
        if Reference._lib is None:
            if not os.path.exists(REF_SO):
                build_oracle()
            L = C.CDLL(REF_SO)
            L.ref_last_error.restype = C.c_char_p
            L.ref_params_build.argtypes = [C.c_uint64, C.c_uint32, C.c_uint, C.c_uint32, C.c_int,
                                           C.POINTER(C.c_void_p)]
            L.ref_params_free.argtypes = [C.c_void_p]
            L.ref_params_scalars.argtypes = [C.c_void_p, u64p]
            L.ref_params_table.restype = C.c_size_t
            L.ref_params_table.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_size_t]
            for f in ("ref_forward", "ref_inverse"):
                getattr(L, f).argtypes = [C.c_void_p, C.c_int, u64p, C.c_size_t]
            for f in ("ref_pointwise", "ref_convolution"):
                getattr(L, f).argtypes = [C.c_void_p, C.c_int, u64p, u64p, u64p, C.c_size_t]
            L.ref_mont_redc.argtypes = [C.c_uint64, C.c_uint, C.c_uint64, C.POINTER(C.c_uint64)]
            L.ref_signed_mont_redc.argtypes = [C.c_uint64, C.c_uint, C.c_int64,
                                               C.POINTER(C.c_int64)]
            L.ref_plantard_redc.argtypes = [C.c_uint64, C.c_uint, C.c_uint64, C.c_uint64,
                                            C.POINTER(C.c_uint64)]
            L.ref_modified_plantard_mul.argtypes = [C.c_uint64, C.c_uint, C.c_uint, C.c_uint64,
                                                    C.c_uint64, C.POINTER(C.c_uint64)]
            L.ref_to_plantard_domain.argtypes = [C.c_uint64, C.c_uint, C.c_uint64,
                                                 C.POINTER(C.c_uint64)]
            L.ref_sweep.argtypes = [C.c_int, C.c_uint64, C.c_uint, C.c_uint, i64p, C.c_size_t,
                                    i64p, C.c_size_t, C.c_void_p, C.POINTER(C.c_uint64)]
            L.ref_plantard_fires.restype = C.c_uint64
            L.ref_rng_fill.argtypes = [C.c_uint64, C.c_uint64, u64p, C.c_size_t]
            L.ref_naive_dft.argtypes = [u64p, C.c_size_t, C.c_uint64, C.c_uint64, u64p]
            L.ref_time_batch.argtypes = [C.c_void_p, C.c_int, C.c_int, u64p, C.c_size_t, C.c_int,
                                         C.POINTER(C.c_uint64)]
            L.ref_run_all_suites.argtypes = [C.c_uint64, C.c_char_p, C.c_size_t,
                                             C.POINTER(C.c_uint64)]
            L.ref_observed.argtypes = [C.c_void_p, C.c_int, C.c_int, u64p, u64p, u64p]
            L.ref_tree_run.argtypes = [C.c_uint64, C.c_uint32, C.c_uint, C.c_int, C.c_uint32,
                                       C.c_int, C.c_int, u64p, C.c_void_p, C.c_size_t]
            L.ref_time_tree.argtypes = [C.c_uint64, C.c_uint32, C.c_uint, C.c_int, C.c_uint32,
                                        C.c_int, C.c_int, u64p, C.c_void_p, C.c_size_t, C.c_int,
                                        C.POINTER(C.c_uint64)]
            L.ref_time_convolution.argtypes = [C.c_void_p, C.c_int, u64p, u64p, u64p, C.c_size_t,
                                               C.c_int, C.POINTER(C.c_uint64)]
            if hasattr(L, "ref_run_bench"):
                L.ref_run_bench.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_int,
                                            C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
            Reference._lib = L
        self.lib = Reference._lib

    def _check(self, st):
        if st != 0:
            raise OracleError(st, self.lib.ref_last_error().decode())

    def run_all_suites(self, random_cases=100000):
        """verify.hpp run_all_suites of the unmodified reference -> ([(name, cases, failures)],
        total failures)."""
        buf = C.create_string_buffer(1 << 14)
        f = C.c_uint64()
        self._check(self.lib.ref_run_all_suites(random_cases, buf, len(buf), C.byref(f)))
        rows = [ln.rsplit(" ", 2) for ln in buf.value.decode().strip().splitlines()]
        return [(n, int(c), int(k)) for n, c, k in rows], f.value

    def run_bench(self, presets=("kyber256", "falcon512", "falcon1024"), iters=2000, seed=12345,
                  micro=False) -> dict:
        """The reference's own run_bench (bench.hpp:334-361) -> its BenchReport JSON
        (schema 1, bench.hpp:365-424), single-threaded as the reference is."""
        import json

        need = C.c_size_t(0)
        args = (",".join(presets).encode(), iters, seed, int(micro))
        cap = 1 << 20
        while True:  # each call re-runs the benchmark: size the buffer generously
            buf = C.create_string_buffer(cap)
            self._check(self.lib.ref_run_bench(*args, buf, cap, C.byref(need)))
            if need.value < cap:
                return json.loads(buf.value.decode())
            cap = 2 * need.value

    def params(self, p, N, n_bits, kinds=(IMPROVED,), exact=False) -> "RefParams":
        mask = 0
        for k in kinds:
            mask |= 1 << k
        h = C.c_void_p()
        self._check(self.lib.ref_params_build(p, N, n_bits, mask, int(exact), C.byref(h)))
        return RefParams(self, h, N)

    def rng(self, seed, bound, count):
        out = np.empty(count, dtype=np.uint64)
        self.lib.ref_rng_fill(seed, bound, out, count)
        return out

    def tree(self, p, N, n_bits, tree, layers, kind, direction, a, b=None):
        """Extension trees on the reference's unmodified cores (ref_shim.cpp
        ref_tree_run): direction 0 forward, 1 inverse, 2 polymul (fwd a, fwd b, basemul, inv).
        Signed (smont) words come back as two's complement uint64."""
        a = np.array(a, dtype=np.int64).astype(np.uint64).reshape(-1, N).copy()
        bp = None
        if b is not None:
            b = np.ascontiguousarray(np.array(b, dtype=np.int64).astype(np.uint64).reshape(-1, N))
            bp = b.ctypes.data
        self._check(self.lib.ref_tree_run(p, N, n_bits, tree, layers, kind, direction, a, bp,
                                          a.shape[0]))
        return a

    def time_tree(self, p, N, n_bits, tree, layers, kind, direction, a, b=None, threads=1):
        """Wall seconds of ref_tree_run over the batch `a` (modified in place) on `threads`
        host threads (the extension configs' CPU baseline)."""
        a = np.ascontiguousarray(a, dtype=np.uint64)
        bp = np.ascontiguousarray(b, dtype=np.uint64) if b is not None else None
        ns = C.c_uint64()
        self._check(self.lib.ref_time_tree(p, N, n_bits, tree, layers, kind, direction, a,
                                           bp.ctypes.data if bp is not None else None,
                                           a.size // N, threads, C.byref(ns)))
        return ns.value * 1e-9

    def sweep_checksum(self, variant, p, n, ell, A, B) -> int:
        """Wrapping u64 sum of the reference's checked reduction over the grid A x B,
        without materialising the results (ctypes drops the GIL: threads may split A)."""
        A = np.ascontiguousarray(A, dtype=np.int64)
        B = np.ascontiguousarray(B, dtype=np.int64)
        s = C.c_uint64()
        self._check(self.lib.ref_sweep(variant, p, n, ell, A, A.size, B, B.size, None, C.byref(s)))
        return s.value

    def sweep(self, variant, p, n, ell, A, B):
        A = np.ascontiguousarray(A, dtype=np.int64)
        B = np.ascontiguousarray(B, dtype=np.int64)
        r = np.empty(A.size * B.size, dtype=np.int64)
        s = C.c_uint64()
        self._check(self.lib.ref_sweep(variant, p, n, ell, A, A.size, B, B.size, r.ctypes.data,
                                       C.byref(s)))
        return r, s.value


class RefParams:
    def __init__(self, r: Reference, h, N):
        self.r, self.h, self.N = r, h, N

    def __del__(self):
        try:
            self.r.lib.ref_params_free(self.h)
        except Exception:
            pass

    def scalars(self):
        out = np.zeros(6, dtype=np.uint64)
        self.r.lib.ref_params_scalars(self.h, out)
        return dict(zip(("omega", "omega_inv", "n_inv", "n_inv_hat", "mu", "scott_L"),
                        (int(v) for v in out)))

    def table(self, name):
        n = self.r.lib.ref_params_table(self.h, name.encode(), None, 0)
        out = np.zeros(n, dtype=np.uint64)
        self.r.lib.ref_params_table(self.h, name.encode(), out.ctypes.data, n)
        return out

    def forward(self, kind, a):
        a = np.array(a, dtype=np.uint64).reshape(-1, self.N).copy()
        self.r._check(self.r.lib.ref_forward(self.h, kind, a, a.shape[0]))
        return a

    def inverse(self, kind, a):
        a = np.array(a, dtype=np.uint64).reshape(-1, self.N).copy()
        self.r._check(self.r.lib.ref_inverse(self.h, kind, a, a.shape[0]))
        return a

    def pointwise(self, kind, x, y):
        x = np.ascontiguousarray(np.array(x, dtype=np.uint64).reshape(-1, self.N))
        y = np.ascontiguousarray(np.array(y, dtype=np.uint64).reshape(-1, self.N))
        out = np.empty_like(x)
        self.r._check(self.r.lib.ref_pointwise(self.h, kind, x, y, out, x.shape[0]))
        return out

    def convolution(self, kind, x, y):
        x = np.ascontiguousarray(np.array(x, dtype=np.uint64).reshape(-1, self.N))
        y = np.ascontiguousarray(np.array(y, dtype=np.uint64).reshape(-1, self.N))
        out = np.empty_like(x)
        self.r._check(self.r.lib.ref_convolution(self.h, kind, x, y, out, x.shape[0]))
        return out

    def observed(self, kind, dir, a, layers):
        """The reference's *_observed on one polynomial -> (states[layers, N], output)."""
        a = np.ascontiguousarray(np.array(a, dtype=np.uint64).reshape(self.N))
        states = np.zeros((layers, self.N), dtype=np.uint64)
        out = np.empty(self.N, dtype=np.uint64)
        self.r._check(self.r.lib.ref_observed(self.h, kind, dir, a, states, out))
        return states, out

    def time_convolution(self, kind, x, y, threads=1):
        """Wall seconds of cyclic_convolution_via_ntt (transform.hpp:372-379) over a batch."""
        x = np.ascontiguousarray(x, dtype=np.uint64)
        y = np.ascontiguousarray(y, dtype=np.uint64)
        out = np.empty_like(x)
        ns = C.c_uint64()
        self.r._check(self.r.lib.ref_time_convolution(self.h, kind, x, y, out, x.size // self.N,
                                                      threads, C.byref(ns)))
        return ns.value * 1e-9

    def time_batch(self, kind, mode, a, threads):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        ns = C.c_uint64()
        self.r._check(self.r.lib.ref_time_batch(self.h, kind, mode, a, a.size // self.N,
                                                threads, C.byref(ns)))
        return ns.value * 1e-9
