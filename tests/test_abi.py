"""CPU checks of the C-ABI boundary and the host-side logic (no GPU needed).

* libnttk_gpu.so loads and exports every entry point include/nttk_gpu.h declares;
* the host parameter builder (B200 counterpart of build_params, params.hpp:137-268)
  produces the reference's tables bit for bit (checked against the pinned oracle) and
  the reference's fault messages;
* without a device every compute entry point fails loudly (no CPU fallback).
"""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle.oracle import CYCLIC, HARVEY, IMPROVED, NEGA, NTL, SCOTT, SMONT

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "nttk_gpu.h")).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(nttk_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_declared_symbol(engine):
    syms = header_symbols()
    assert len(syms) >= 19, syms
    lib = engine.lib()
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(engine.EXPORTS)


def test_no_gpu_fails_loudly(engine):
    if engine.device_available():
        pytest.skip("a device is present")
    P = engine.build_params(3329, 256, 16, [engine.ButterflyKind.improved], exact_bound=True)
    with pytest.raises(engine.CudaError, match="no CUDA device"):
        engine.ntt_forward_batch(np.zeros((2, 256), dtype=np.uint16), P, 3)
    with pytest.raises(engine.CudaError, match="no CUDA device"):  # reductions too
        engine.mont_redc(100, engine.make_reduction_context(17, 5))


@pytest.mark.parametrize("p,n,alpha,ell", [(13, 8, 0, 2), (17, 5, 0, 0), (3329, 16, 1, 2),
                                           (8380417, 32, 0, 7), (4294967291, 32, 3, 1)])
def test_reduction_context_matches_oracle(engine, oracle, p, n, alpha, ell):
    """make_reduction_context (reduction.hpp:80-117): host precompute == the oracle's."""
    c = engine.make_reduction_context(p, n, alpha, ell)
    o = oracle.ctx(p, n, alpha, ell)
    for f in ("p", "n_bits", "alpha", "ell", "beta", "beta_mask", "r2n_mask", "p_inv_beta",
              "neg_p_inv_beta", "mu", "mu_centered", "beta_mod_p", "r2n_mod_p"):
        assert getattr(c, f) == getattr(o, f), f


def test_reduction_context_messages(engine):
    for args, msg in (((13, 1), "word size n must be in [2, 32]"), ((12, 8), "odd and >= 3"),
                      ((301, 8), "p must be < 2^n"), ((13, 8, 8), "alpha must be < n"),
                      ((13, 8, 0, 8), "ell must be < n")):
        with pytest.raises(engine.ContractViolation, match=re.escape(msg)):
            engine.make_reduction_context(*args)


CONFIGS = [
    # (p, N, n, kinds, tree, layers, exact)
    (3329, 256, 16, (IMPROVED, HARVEY, SMONT), CYCLIC, 0, True),
    (3329, 256, 16, (IMPROVED, HARVEY, SMONT), NEGA, 7, True),
    (3329, 256, 32, (NTL, HARVEY, SCOTT, IMPROVED), CYCLIC, 0, False),
    (8380417, 256, 32, (NTL, HARVEY, SCOTT, IMPROVED, SMONT), CYCLIC, 0, True),
    (8380417, 256, 32, (IMPROVED, HARVEY, SMONT), NEGA, 8, True),
    (7681, 256, 32, (NTL, HARVEY, SCOTT, IMPROVED), CYCLIC, 0, False),
    (12289, 1024, 32, (NTL, HARVEY, SCOTT, IMPROVED), CYCLIC, 0, False),
    (13, 4, 8, (NTL, HARVEY, SCOTT, IMPROVED), CYCLIC, 0, False),
    (17, 8, 16, (IMPROVED, HARVEY, SMONT), NEGA, 2, True),
]
TABLES = ("dif_w", "dif_wq", "dif_mont", "ct_plain", "ct_plantard", "ct_mont", "ct_smont",
          "gs_plain", "gs_wq", "gs_mont", "gs_plantard", "gs_smont")


@pytest.mark.parametrize("cfg", CONFIGS)
def test_host_tables_match_oracle(engine, oracle, cfg):
    p, N, n, kinds, tree, layers, exact = cfg
    P = engine.build_params(p, N, n, kinds, tree=tree, layers=layers, exact_bound=exact)
    Q = oracle.params(p, N, n, kinds, tree=tree, layers=layers, exact=exact)
    assert (P.omega, P.omega_inv, P.n_inv) == (Q.omega, Q.omega_inv, Q.n_inv)
    if IMPROVED in kinds:
        assert P.n_inv_hat == Q.n_inv_hat
    for t in TABLES:
        a, b = P.table(t), Q.table(t)
        if len(a) == 0 and t.startswith("dif"):
            continue
        assert len(a) == len(b) and (a == b).all(), t


def test_fault_messages_match_reference(engine):
    C = engine.ContractViolation
    with pytest.raises(C, match="p must be prime"):
        engine.build_params(15, 4, 8)
    with pytest.raises(C, match="N must divide p - 1"):
        engine.build_params(13, 8, 8)
    with pytest.raises(C) as e:
        engine.build_params(15, 6, 40)
    assert all(s in str(e.value) for s in ("p must be prime", "power of two", "[2, 32]"))
    with pytest.raises(C, match=r"p < 2\^\{n-ell-2\}"):
        engine.build_params(7681, 256, 16)
    with pytest.raises(C, match="unknown preset"):
        engine.preset("nope")
    with pytest.raises(C, match="at least one butterfly kind"):
        engine.build_params(13, 4, 8, [])
    with pytest.raises(C, match="unknown butterfly kind"):
        engine.butterfly_kind_from_string("fancy")


def test_presets_and_fast_path_selection(engine):
    P = engine.preset("kyber256")
    assert (P.p, P.size, P.n_bits, P.omega) == (7681, 256, 32, 198)
    T = engine.preset("toy13")
    assert (T.omega, T.omega_inv, T.n_inv) == (5, 8, 10)
    K = engine.build_params(3329, 256, 16, [engine.ButterflyKind.improved], exact_bound=True)
    assert engine.ButterflyKind.improved in K.fast_path
    F = engine.preset("falcon512")  # N = 512: fastn_tma.cu for every kind
    assert sorted(F.fast_path) == sorted(engine.ButterflyKind)[:4]
    # partial trees at N = 512 and N = 2048 stay on the generic kernel
    G = engine.build_params(12289, 2048, 32, [engine.ButterflyKind.harvey])
    assert G.fast_path == []


def test_exact_bound_admits_kyber_n16_and_dilithium_n32(engine):
    with pytest.raises(engine.ContractViolation):
        engine.build_params(3329, 256, 16, [engine.ButterflyKind.improved])
    with pytest.raises(engine.ContractViolation):
        engine.build_params(8380417, 256, 32, [engine.ButterflyKind.improved])
    engine.build_params(3329, 256, 16, [engine.ButterflyKind.improved], exact_bound=True)
    engine.build_params(8380417, 256, 32, [engine.ButterflyKind.improved], exact_bound=True)


def test_params_helpers_match_engine_tables(engine):
    """params.hpp / transform.hpp helpers of the Python mirror (host parameter logic) against
    the engine's own tables and the reference's known values."""
    for name in ("kyber256", "falcon512", "toy13"):
        P = engine.preset(name)
        assert engine.find_primitive_root(P.p, P.size) == P.omega
        assert engine.ct_forward_plain_twiddles(P.size, P.omega, P.p) == list(P.table("ct_plain"))
        assert engine.gs_inverse_plain_twiddles(P.size, P.omega, P.p) == list(P.table("gs_plain"))
        assert engine.dif_forward_plain_twiddles(P.size, P.omega, P.p) == list(P.table("dif_w"))
        assert engine.preset_spec(name)[1:3] == (P.p, P.size)
    P = engine.preset("kyber256")
    assert engine.spectrum_value_bound(P, engine.ButterflyKind.scott) == 256 * 7681
    assert engine.to_natural_order(engine.Spectrum([0, 1, 2, 3])) == [0, 2, 1, 3]
    with pytest.raises(engine.ContractViolation, match="unknown preset"):
        engine.preset_spec("nope")


# ---------------------------------------------------------------------------
# host validation of the fast-kernel options (params.cpp fill_fast): the bounds that make the
# inverse shortcuts exact must be checked on the host, per parameter set
FWD_W1, CANON16, CANON32, FUSE16, LAZY, TW1, DEFER, PARTIAL = 16, 1, 2, 4, 8, 32, 64, 128


def test_fast_flags_kyber_dilithium(engine):
    K = engine.ButterflyKind
    Pk = engine.build_params(3329, 256, 16, [K.improved, K.harvey, K.ntl], exact_bound=True)
    fi = Pk.fast_flags(K.improved, 1)
    assert fi & (FUSE16 | LAZY | TW1 | DEFER) == FUSE16 | LAZY | TW1 | DEFER
    assert not fi & PARTIAL
    assert Pk.fast_flags(K.improved, 0) & FWD_W1
    assert Pk.fast_flags(K.harvey, 1) & TW1 and Pk.fast_flags(K.ntl, 1) & TW1
    Pd = engine.build_params(8380417, 256, 32, [K.improved], exact_bound=True)
    fd = Pd.fast_flags(K.improved, 1)
    # 2^9 p = 4 290 773 504 < 2^32: the doubled bounds of the partial canonicalisation fit
    assert fd & (CANON32 | LAZY | TW1 | PARTIAL) == CANON32 | LAZY | TW1 | PARTIAL
    assert not fd & (DEFER | FUSE16)


def test_fast_flags_refused_where_bounds_fail(engine):
    K = engine.ButterflyKind
    # 2^9 p >= 2^32: no partial canonicalisation (X + Y would overflow 32 bits), TW1 stays
    P = engine.build_params(8392193, 256, 32, [K.improved], exact_bound=True)
    f = P.fast_flags(K.improved, 1)
    assert f & TW1 and not f & PARTIAL
    # negacyclic / 7-layer trees: no twiddle-1 blocks, no DEFER (8 layers only)
    Pn = engine.build_params(3329, 256, 16, [K.improved], tree=engine.Tree.negacyclic, layers=7,
                             exact_bound=True)
    fn = Pn.fast_flags(K.improved, 1)
    assert not fn & (TW1 | DEFER)
    assert not Pn.fast_flags(K.improved, 0) & FWD_W1
    # N = 1024 full tree: TW1 on the phase-2 layers of fastn_tma.cu
    P10 = engine.build_params(12289, 1024, 32, [K.improved])
    assert P10.fast_flags(K.improved, 1) & TW1
    with pytest.raises(engine.ContractViolation):
        P10.fast_flags(K.harvey, 1)  # kind not built into these params


PM_LAZY = 256


def test_fast_flags_polymul_lazy_montgomery(engine):
    """params.cpp: the fused polymul's lazy twins (arith.cuh HarveyLazy16 / SmontLazy16, the
    improved kind's free F1 forwards) are admitted for Kyber n = 16 (config 2) and refused where their bounds or
    their n = 16 / CT-forward preconditions fail."""
    K = engine.ButterflyKind
    nega = engine.Tree.negacyclic
    Pk = engine.build_params(3329, 256, 16, [K.harvey, K.smont, K.improved], tree=nega, layers=7,
                             exact_bound=True)
    assert Pk.fast_flags(K.harvey, 1) & PM_LAZY and Pk.fast_flags(K.smont, 1) & PM_LAZY
    # improved: the free F1 forwards (tma_common.cuh fwd_body_f1_free)
    assert Pk.fast_flags(K.improved, 1) & PM_LAZY
    # cyclic harvey runs the DIF forward (no lazy twin); cyclic smont (CT) keeps it
    Pc = engine.build_params(3329, 256, 16, [K.harvey, K.smont], exact_bound=True)
    assert not Pc.fast_flags(K.harvey, 1) & PM_LAZY and Pc.fast_flags(K.smont, 1) & PM_LAZY
    # n = 32 (Dilithium): eager policies
    Pd = engine.build_params(8380417, 256, 32, [K.harvey, K.smont], tree=nega, layers=8,
                             exact_bound=True)
    assert not Pd.fast_flags(K.harvey, 1) & PM_LAZY and not Pd.fast_flags(K.smont, 1) & PM_LAZY
    # (1 + 2L) p >= 2^16: a forward operand could reach 2^16, refused
    Pb = engine.build_params(7681, 256, 16, [K.harvey, K.smont], tree=nega, layers=7,
                             exact_bound=True)
    assert not Pb.fast_flags(K.harvey, 1) & PM_LAZY and not Pb.fast_flags(K.smont, 1) & PM_LAZY


NARROW = 512


def test_fast_flags_narrow_image(engine):
    """params.cpp fill_narrow: an n = 32 improved parameter set whose forward operands stay
    inside the n = 16 Prop. 4 range runs on the n = 16 product (the paper's Table 2 presets);
    Dilithium (p > 2^15) and n = 16 sets do not."""
    K = engine.ButterflyKind
    for name in ("kyber256", "newhope512", "falcon1024"):
        P = engine.preset(name)
        assert P.fast_flags(K.improved, 0) & NARROW, name
        assert P.fast_flags(K.improved, 1) & NARROW, name  # inverse: bounded merge operands
        assert not P.fast_flags(K.harvey, 0) & NARROW
    Pd = engine.build_params(8380417, 256, 32, [K.improved], exact_bound=True)
    assert not Pd.fast_flags(K.improved, 0) & NARROW
    Pk = engine.build_params(3329, 256, 16, [K.improved], exact_bound=True)
    assert not Pk.fast_flags(K.improved, 0) & NARROW


CT_INV = 2048


def test_fast_flags_ct_inverse(engine):
    """params.cpp fill_ct_inverse: the Kyber tree (improved n = 16, cyclic N = 256) and the
    Dilithium tree (n = 32) admit the CT-form inverse (every product operand inside Prop. 4's
    range, every word below 2^32, under the host's interval propagation); negacyclic trees keep
    the GS inverse.  fill_ct_inverse_n: the narrow image at N = 512 / 1024 runs in CT form when
    kCtLimN p = 20 p lies inside the n = 16 range (the Table 2 modulus 12289), else the GS narrow
    body stays (p = 13313: 16 p fits, 20 p does not)."""
    K = engine.ButterflyKind
    Pk = engine.build_params(3329, 256, 16, [K.improved], exact_bound=True)
    assert Pk.fast_flags(K.improved, 1) & CT_INV
    assert not Pk.fast_flags(K.improved, 0) & CT_INV
    Pn = engine.build_params(3329, 256, 16, [K.improved], tree=engine.Tree.negacyclic, layers=7,
                             exact_bound=True)
    assert not Pn.fast_flags(K.improved, 1) & CT_INV
    Pd = engine.build_params(8380417, 256, 32, [K.improved], exact_bound=True)
    assert Pd.fast_flags(K.improved, 1) & CT_INV
    for N in (512, 1024):
        Pb = engine.build_params(12289, N, 32, [K.improved])
        assert Pb.fast_flags(K.improved, 1) & (CT_INV | NARROW) == CT_INV | NARROW
        assert not Pb.fast_flags(K.improved, 0) & CT_INV
    lim = lambda p: (1 << 16) * ((1 << 16) - p)  # noqa: E731
    p = 13313
    assert (p - 1) * (16 * p) < lim(p) <= (p - 1) * (20 * p - 1)
    Pc = engine.build_params(p, 512, 32, [K.improved])
    assert Pc.fast_flags(K.improved, 1) & (CT_INV | NARROW) == NARROW
    P7 = engine.build_params(7681, 256, 32, [K.improved])  # N = 256 narrow image: CT body on
    assert P7.fast_flags(K.improved, 1) & (CT_INV | NARROW) == CT_INV | NARROW  # canonicalised words
