"""GPU parity: the sm_100a engine through its C ABI vs the pinned CPU oracle.

Bit-exact comparisons (integer work) on seeded inputs drawn with the reference's own Rng
(int_util.hpp:90-138), at sizes the oracle finishes in seconds, plus size-independent
properties at BASELINE sizes (round trips, agreement with oracle on sampled polys).
Every test here needs a CUDA device; the engine has no CPU path.
"""
import numpy as np
import pytest
import torch

from oracle.oracle import CYCLIC, HARVEY, IMPROVED, NEGA, NTL, SCOTT, SMONT

import paper_2402_00675_b200.nttk as nttk
from paper_2402_00675_b200.nttk import ButterflyKind as K

pytestmark = pytest.mark.gpu

DT = {2: np.uint16, 4: np.uint32, 8: np.uint64}
SDT = {2: np.int16, 4: np.int32, 8: np.int64}
TDT = {2: torch.int16, 4: torch.int32, 8: torch.int64}


@pytest.fixture(scope="module", autouse=True)
def _device():
    assert torch.cuda.is_available(), "GPU parity tests need a CUDA device"
    assert nttk.device_available()
    torch.cuda.init()


def fnv(oracle, a):
    return "%016x" % oracle.fnv(np.asarray(a).astype(np.int64).astype(np.uint64).ravel())


def to_dev(a, elem, signed=False):
    arr = np.ascontiguousarray(np.asarray(a).astype(SDT[elem] if signed else DT[elem]))
    return torch.from_numpy(arr.view(SDT[elem])).cuda()


def from_dev(t, signed=False):
    a = t.cpu().numpy()
    return a.astype(np.int64) if signed else a.view({2: np.uint16, 4: np.uint32, 8: np.uint64}[a.itemsize]).astype(np.uint64)


def engine_params(p, N, n, kinds, tree=CYCLIC, layers=0, exact=False):
    return nttk.build_params(p, N, n, kinds, tree=tree, layers=layers, exact_bound=exact)


# ---------------------------------------------------------------------------
# golden vectors of the reference (tests/golden/golden.json)

def test_golden_forward_inverse_all_cases(oracle, golden):
    for c in golden["cases"]:
        p, N, n, kind = c["p"], c["N"], c["n_bits"], c["kind"]
        f = oracle.rng(c["seed"], p, c["polys"] * N).reshape(c["polys"], N)
        P = engine_params(p, N, n, [kind], exact=c["exact_bound"])
        assert P.omega == c["omega"]
        for elem in (8, 4, 2):
            try:
                x = to_dev(f, elem)
                y = nttk.forward(P, kind, x)
            except nttk.ContractViolation as e:
                assert "cannot hold" in str(e) and elem < 8
                continue
            fwd = from_dev(y)
            assert fnv(oracle, fwd) == c["fwd_fnv"], (c["label"], elem)
            inv = from_dev(nttk.inverse(P, kind, y))
            assert fnv(oracle, inv) == c["inv_fnv"], (c["label"], elem)
            assert (inv == f).all()
        # inverse of arbitrary in-range words (canonicalisation path, transform.hpp:243)
        g = oracle.rng(c["seed"] + 1, 1 << 15, c["polys"] * N).reshape(c["polys"], N)
        for elem in (8, 4, 2):
            if p > (1 << (8 * elem)):  # canonical output does not fit: refused
                with pytest.raises(nttk.ContractViolation, match="cannot hold canonical"):
                    nttk.inverse(P, kind, to_dev(g, elem))
                continue
            got = from_dev(nttk.inverse(P, kind, to_dev(g, elem)))
            assert fnv(oracle, got) == c["inv_g_fnv"], (c["label"], elem)


def test_golden_products(oracle, golden):
    for c in golden["products"]:
        p, N, n, kind = c["p"], c["N"], c["n_bits"], c["kind"]
        a = oracle.rng(c["seed"], p, 4 * N).reshape(4, N)
        b = oracle.rng(c["seed"] + 1, p, 4 * N).reshape(4, N)
        P = engine_params(p, N, n, [kind])
        fa = nttk.forward(P, kind, to_dev(a, 8))
        fb = nttk.forward(P, kind, to_dev(b, 8))
        assert fnv(oracle, from_dev(nttk.pointwise(P, kind, fa, fb))) == c["pointwise_fnv"]
        conv = from_dev(nttk.polymul(P, kind, to_dev(a, 8), to_dev(b, 8)))
        assert fnv(oracle, conv) == c["conv_fnv"]
        host = nttk.polymul_batch(a, b, P, kind)
        assert fnv(oracle, host) == c["conv_fnv"]


def test_golden_trees(oracle, golden):
    """Extension trees (Kyber 7-layer negacyclic, basemul polymul, Dilithium
    negacyclic, signed Montgomery) against reference-run words (tests/golden: the
    reference's unmodified cores on the a22 schedule), at every storage width that holds
    the kind's words: fast u16/u32 kernels, the fused polymul, the u64 generic kernel."""
    for c in golden["trees"]:
        p, N, n, kind, L, tree = c["p"], c["N"], c["n_bits"], c["kind"], c["layers"], c["tree"]
        sg = kind == SMONT
        P = engine_params(p, N, n, [kind], tree=tree, layers=L, exact=True)
        f = oracle.rng(c["seed"], p, c["polys"] * N).reshape(c["polys"], N)
        g = oracle.rng(c["seed"] + 1, 1 << 15, c["polys"] * N).reshape(c["polys"], N)
        if sg:
            g = g.astype(np.int64) - (1 << 14)
        h = oracle.rng(c["seed"] + 2, p, c["polys"] * N).reshape(c["polys"], N)
        widths = (2, 4, 8) if p < (1 << 15) else (4, 8)
        for elem in widths:
            y = nttk.forward(P, kind, to_dev(f, elem, sg))
            fwd = from_dev(y, sg)
            assert fnv(oracle, fwd) == c["fwd_fnv"], (c["label"], kind, elem)
            assert [int(v) for v in fwd[0]] == c["fwd_poly0"], (c["label"], kind, elem)
            assert (from_dev(nttk.inverse(P, kind, y)) == f).all(), (c["label"], kind, elem)
            inv_g = from_dev(nttk.inverse(P, kind, to_dev(g, elem, sg)))
            assert fnv(oracle, inv_g) == c["inv_g_fnv"], (c["label"], kind, elem)
            if "polymul_fnv" in c:
                pm = from_dev(nttk.polymul(P, kind, to_dev(f, elem), to_dev(h, elem)))
                assert fnv(oracle, pm) == c["polymul_fnv"], (c["label"], kind, elem)
                assert [int(v) for v in pm[0]] == c["polymul_poly0"], (c["label"], kind, elem)


def test_golden_reductions(golden):
    for c in golden["reductions"]:
        A = torch.tensor(c["A"], dtype=torch.int64, device="cuda")
        B = torch.tensor(c["B"], dtype=torch.int64, device="cuda")
        r = torch.empty(A.numel() * B.numel(), dtype=torch.int64, device="cuda")
        s = nttk.modmul_sweep(c["variant"], c["p"], c["n_bits"], c["ell"], A, B, r)
        assert "%016x" % s == c["checksum"], c
        assert r[:64].cpu().tolist() == c["r_first"], c


# ---------------------------------------------------------------------------
# BASELINE configs vs the oracle, bit-exact

KYBER, DILITHIUM = 3329, 8380417


@pytest.mark.parametrize("kind,n", [(IMPROVED, 16), (HARVEY, 16), (SMONT, 16), (IMPROVED, 32),
                                    (HARVEY, 32), (SMONT, 32)])
@pytest.mark.parametrize("tree,layers", [(CYCLIC, 8), (NEGA, 7)])
def test_kyber_transforms_vs_oracle(oracle, kind, n, tree, layers):
    P = engine_params(KYBER, 256, n, [kind], tree=tree, layers=layers, exact=True)
    Q = oracle.params(KYBER, 256, n, (kind,), tree=tree, layers=layers, exact=True)
    assert kind in P.fast_path
    B = 1027  # odd: exercises the half-warp tail
    f = oracle.rng(12345 + kind, KYBER, B * 256).reshape(B, 256)
    want = Q.forward(kind, f)
    sgn = kind == SMONT
    for elem in (2, 4, 8):
        y = nttk.forward(P, kind, to_dev(f, elem))
        got = from_dev(y, sgn)
        assert (got.astype(np.int64) == want.astype(np.int64)).all(), elem
        back = from_dev(nttk.inverse(P, kind, y))
        assert (back == f).all(), elem


@pytest.mark.parametrize("kind", [IMPROVED, HARVEY, SMONT])
@pytest.mark.parametrize("tree,layers", [(CYCLIC, 8), (NEGA, 8)])
def test_dilithium_transforms_vs_oracle(oracle, kind, tree, layers):
    P = engine_params(DILITHIUM, 256, 32, [kind], tree=tree, layers=layers, exact=True)
    Q = oracle.params(DILITHIUM, 256, 32, (kind,), tree=tree, layers=layers, exact=True)
    assert kind in P.fast_path
    B = 515
    f = oracle.rng(777 + kind, DILITHIUM, B * 256).reshape(B, 256)
    want = Q.forward(kind, f)
    sgn = kind == SMONT
    for elem in (4, 8):
        y = nttk.forward(P, kind, to_dev(f, elem))
        assert (from_dev(y, sgn).astype(np.int64) == want.astype(np.int64)).all(), elem
        assert (from_dev(nttk.inverse(P, kind, y)) == f).all(), elem


@pytest.mark.parametrize("p,n,kind", [(KYBER, 16, NTL), (KYBER, 32, NTL), (KYBER, 32, SCOTT),
                                      (DILITHIUM, 32, NTL), (DILITHIUM, 32, SCOTT),
                                      (7681, 32, SCOTT), (7681, 32, NTL)])
def test_dif_kinds_fast_path_vs_oracle(oracle, p, n, kind):
    """ntl (Alg. 7) and scott (Alg. 9) on the fast N=256 kernels (TMA for u16/u32, the
    register-prefetch kernel for u64): forward words, inverse of arbitrary in-bound
    spectra, round trips -- bit-exact with the oracle."""
    P = engine_params(p, 256, n, [kind])
    Q = oracle.params(p, 256, n, (kind,))
    assert kind in P.fast_path
    B = 291
    f = oracle.rng(4242 + kind + n, p, B * 256).reshape(B, 256)
    want = Q.forward(kind, f)
    bound = p if kind == NTL else 256 * p  # spectrum_value_bound (transform.hpp:61-70)
    elems = [e for e in (2, 4, 8) if bound <= (1 << (8 * e))]
    for elem in elems:
        y = nttk.forward(P, kind, to_dev(f, elem))
        assert (from_dev(y) == want).all(), elem
        assert (from_dev(nttk.inverse(P, kind, y)) == f).all(), elem
    rng = np.random.default_rng(kind * 100 + n)
    spec = rng.integers(0, bound, size=(B, 256), dtype=np.uint64)
    want_inv = Q.inverse(kind, spec)
    for elem in elems:
        assert (from_dev(nttk.inverse(P, kind, to_dev(spec, elem))) == want_inv).all(), elem


FASTN_CASES = [(32, NTL, CYCLIC), (32, HARVEY, CYCLIC), (32, SCOTT, CYCLIC), (32, IMPROVED, CYCLIC),
               (32, SMONT, CYCLIC), (16, NTL, CYCLIC), (16, HARVEY, CYCLIC),
               (32, IMPROVED, NEGA), (32, HARVEY, NEGA), (32, SMONT, NEGA), (16, HARVEY, NEGA)]


@pytest.mark.parametrize("N", [512, 1024])
@pytest.mark.parametrize("n,kind,tree", FASTN_CASES)
def test_fastn_transforms_vs_oracle(oracle, N, n, kind, tree):
    """N = 512 / 1024 fast kernels (fastn_tma.cu; the paper's Table 2 sizes, q = 12289):
    forward words, round trips and the inverse of arbitrary in-bound spectra, bit-exact."""
    p = 12289
    P = engine_params(p, N, n, [kind], tree=tree)
    Q = oracle.params(p, N, n, (kind,), tree=tree)
    assert kind in P.fast_path
    B = 37  # ragged: partial tiles, odd half-warp split at N = 512
    f = oracle.rng(900 + N + 10 * kind + n, p, B * N).reshape(B, N)
    want = Q.forward(kind, f)
    sgn = kind == SMONT
    L = N.bit_length() - 1
    bound = {NTL: p, HARVEY: 2 * p, SCOTT: N * p, IMPROVED: (L + 1) * p, SMONT: (L + 2) * p}[kind]
    lim = {2: 1 << 15, 4: 1 << 31, 8: 1 << 63} if sgn else {2: 1 << 16, 4: 1 << 32, 8: 1 << 64}
    elems = [e for e in (2, 4, 8) if bound <= lim[e]]
    for elem in elems:
        y = nttk.forward(P, kind, to_dev(f, elem, sgn))
        assert (from_dev(y, sgn).astype(np.int64) == want.astype(np.int64)).all(), elem
        assert (from_dev(nttk.inverse(P, kind, y)) == f).all(), elem
    if not sgn:
        rng = np.random.default_rng(N + kind + n)
        spec = rng.integers(0, bound, size=(B, N), dtype=np.uint64)
        want_inv = Q.inverse(kind, spec)
        for elem in elems:
            assert (from_dev(nttk.inverse(P, kind, to_dev(spec, elem))) == want_inv).all(), elem


@pytest.mark.parametrize("N", [512, 1024])
def test_fastn_inplace_and_misaligned(oracle, N):
    """In-place calls (d_in == d_out) on the fast N = 512/1024 kernels, and a buffer that
    is not 16-byte aligned (falls back to the generic kernel) -- same words either way."""
    p = 12289
    P = engine_params(p, N, 32, [IMPROVED])
    Q = oracle.params(p, N, 32, (IMPROVED,))
    B = 21
    f = oracle.rng(31 + N, p, B * N).reshape(B, N)
    want = Q.forward(IMPROVED, f)
    x = to_dev(f, 4)
    nttk.forward(P, IMPROVED, x, x)  # in place
    assert (from_dev(x) == want).all()
    nttk.inverse(P, IMPROVED, x, x)
    assert (from_dev(x) == f).all()
    # offset by one coefficient: 4-byte aligned only
    buf = torch.zeros(B * N + 1, dtype=torch.int32, device="cuda")
    view = buf[1:].view(B, N)
    view.copy_(to_dev(f, 4))
    out = torch.zeros_like(buf)[1:].view(B, N)
    nttk.forward(P, IMPROVED, view, out)
    assert (from_dev(out) == want).all()


def test_fastn_presets_all_kinds(oracle):
    """The reference presets at N = 512 / 1024 (params.hpp:280-289) on the fast kernels."""
    for name, p, N in (("newhope512", 12289, 512), ("falcon1024", 12289, 1024)):
        P = nttk.preset(name)
        kinds = (NTL, HARVEY, SCOTT, IMPROVED)
        Q = oracle.params(p, N, 32, kinds)
        f = oracle.rng(4, p, 19 * N).reshape(19, N)
        for k in kinds:
            assert k in P.fast_path, (name, k)
            got = from_dev(nttk.forward(P, k, to_dev(f, 4)))
            assert (got == Q.forward(k, f)).all(), (name, k)


def test_scott_n16_stays_on_generic_kernel(oracle):
    """scott at Kyber n=16 underflows uint64 in the reference; the engine
    keeps that configuration on the 64-bit generic kernel, which replicates it word for word."""
    P = engine_params(KYBER, 256, 16, [SCOTT])
    assert SCOTT not in P.fast_path
    Q = oracle.params(KYBER, 256, 16, (SCOTT,))
    f = oracle.rng(5, KYBER, 7 * 256).reshape(7, 256)
    assert (from_dev(nttk.forward(P, SCOTT, to_dev(f, 8))) == Q.forward(SCOTT, f)).all()


def test_dilithium_improved_matches_reference_exact_bound(oracle, golden):
    """config 3: modified Plantard (64-bit constant) vs 32-bit Montgomery round trip."""
    B = 4096
    f = oracle.rng(3, DILITHIUM, B * 256).reshape(B, 256)
    x = to_dev(f, 4)
    for kind in (IMPROVED, HARVEY):
        P = engine_params(DILITHIUM, 256, 32, [kind], exact=True)
        Q = oracle.params(DILITHIUM, 256, 32, (kind,), exact=True)
        y = nttk.forward(P, kind, x)
        sample = [0, 1, 2047, 4095]
        assert (from_dev(y)[sample] == Q.forward(kind, f[sample])).all()
        assert torch.equal(nttk.inverse(P, kind, y), x)


@pytest.mark.parametrize("kind,n,tree,layers", [(IMPROVED, 16, NEGA, 7), (HARVEY, 16, NEGA, 7),
                                                (SMONT, 16, NEGA, 7), (IMPROVED, 16, CYCLIC, 8),
                                                (HARVEY, 16, CYCLIC, 8), (SMONT, 16, CYCLIC, 8),
                                                (IMPROVED, 32, NEGA, 8), (SMONT, 32, NEGA, 8),
                                                (HARVEY, 32, CYCLIC, 8), (IMPROVED, 32, CYCLIC, 8)])
def test_polymul_vs_schoolbook(oracle, kind, n, tree, layers):
    p = KYBER if n == 16 else DILITHIUM
    P = engine_params(p, 256, n, [kind], tree=tree, layers=layers, exact=True)
    Q = oracle.params(p, 256, n, (kind,), tree=tree, layers=layers, exact=True)
    B = 33
    a = oracle.rng(10 + kind, p, B * 256).reshape(B, 256)
    b = oracle.rng(20 + kind, p, B * 256).reshape(B, 256)
    want = Q.polymul(kind, a, b)
    elem = 2 if p == KYBER else 4
    got = from_dev(nttk.polymul(P, kind, to_dev(a, elem), to_dev(b, elem)))  # fused kernel
    assert (got == want).all()
    got64 = from_dev(nttk.polymul(P, kind, to_dev(a, 8), to_dev(b, 8)))  # 4-kernel pipeline
    assert (got64 == want).all()
    # in-place (out aliases a)
    xa = to_dev(a, elem)
    nttk.polymul(P, kind, xa, to_dev(b, elem), out=xa)
    assert (from_dev(xa) == want).all()
    school = oracle.schoolbook_negacyclic if tree == NEGA else oracle.schoolbook_cyclic
    for i in (0, B - 1):
        assert (got[i] == school(a[i], b[i], p)).all()
    if tree == NEGA and layers == 7:
        fa = nttk.forward(P, kind, to_dev(a, elem))
        fb = nttk.forward(P, kind, to_dev(b, elem))
        bm = from_dev(nttk.basemul(P, kind, fa, fb))
        assert (bm == Q.basemul(kind, Q.forward(kind, a), Q.forward(kind, b))).all()


@pytest.mark.parametrize("kind,tree,layers", [(HARVEY, NEGA, 7), (SMONT, NEGA, 7), (SMONT, CYCLIC, 8)])
def test_polymul_lazy_montgomery_extremes(oracle, kind, tree, layers):
    """The fused polymul's lazy Montgomery twins (arith.cuh HarveyLazy16 / SmontLazy16, no
    intermediate normalisation) on the operands that drive every bound to its maximum:
    all p - 1, all zero, alternating extremes, one hot coefficient -- bit-exact with the
    oracle's eager reference loop."""
    p = KYBER
    P = engine_params(p, 256, 16, [kind], tree=tree, layers=layers, exact=True)
    assert P.fast_flags(kind, 1) & 256  # the lazy twin is the one that runs
    Q = oracle.params(p, 256, 16, (kind,), tree=tree, layers=layers, exact=True)
    rows = [np.full(256, p - 1), np.zeros(256, dtype=np.int64),
            np.where(np.arange(256) % 2 == 0, p - 1, 0), np.eye(256, dtype=np.int64)[0] * (p - 1),
            np.where(np.arange(256) < 128, p - 1, 0), np.arange(256) % p]
    a = np.stack(rows + [oracle.rng(71, p, 256)]).astype(np.int64)
    for b in (a, a[::-1].copy(), np.full_like(a, p - 1)):
        got = from_dev(nttk.polymul(P, kind, to_dev(a, 2), to_dev(b, 2)))
        assert (got == Q.polymul(kind, a, b)).all()


def test_all_reference_kinds_at_presets_via_host_api(oracle):
    """Every ButterflyKind at the reference presets (generic kernel for N != 256 and n=32)."""
    for name, p, N, n in (("kyber256", 7681, 256, 32), ("falcon512", 12289, 512, 32),
                          ("falcon1024", 12289, 1024, 32), ("toy13", 13, 4, 8)):
        P = nttk.preset(name)
        kinds = (NTL, HARVEY, SCOTT, IMPROVED)
        Q = oracle.params(p, N, n, kinds)
        f = oracle.rng(99, p, 5 * N).reshape(5, N)
        for k in kinds:
            got = nttk.ntt_forward_batch(f, P, k)
            assert (got == Q.forward(k, f)).all(), (name, k)
            for k2 in kinds:  # every kind pair inverts every other (transform_test.cpp:61-93)
                assert (nttk.intt_inverse_batch(got, P, k2) == f).all(), (name, k, k2)


def test_reference_shaped_single_poly_calls():
    """transform_test.cpp hand cases through the Python mirror of the reference API."""
    P = nttk.build_params(17, 4, 16)
    for k in nttk.all_butterfly_kinds():
        s = nttk.ntt_forward([1, 2, 3, 4], P, k)
        nat = [s.values[i] % 17 for i in (0, 2, 1, 3)]
        assert nat == [10, 7, 15, 6]
        assert nttk.intt_inverse(s, P, k) == [1, 2, 3, 4]
        assert nttk.cyclic_convolution_via_ntt([1, 2, 3, 4], [1, 0, 0, 1], P, k) == [3, 5, 7, 5]
    T = nttk.preset("toy13")
    for k in nttk.all_butterfly_kinds():
        s = nttk.ntt_forward([0, 1, 0, 0], T, k)
        assert [s.values[i] % 13 for i in (0, 2, 1, 3)] == [1, 5, 12, 8]
    lhs = nttk.Spectrum([1, 2, 3, 4])
    rhs = nttk.Spectrum([51, 40, 27, 14])
    out = nttk.pointwise_multiply(lhs, rhs, T, K.improved)
    assert out.values == [l * (r % 13) % 13 for l, r in zip(lhs.values, rhs.values)]
    assert nttk.pointwise_multiply(lhs, rhs, T, K.harvey).values == out.values
    # the left operand is reduced mod p before encoding (transform.hpp:362-365): only the
    # right one carries modified_plantard_mul's T < 2^ell p contract
    big = nttk.Spectrum([52, 1000, 2 ** 40 + 3, 2 ** 63 + 7])
    got = nttk.pointwise_multiply(big, rhs, T, K.improved)
    assert got.values == [(l % 13) * (r % 13) % 13 for l, r in zip(big.values, rhs.values)]


def test_device_api_operand_checks():
    """b / out must match the first operand (dtype, element count, device, contiguity)."""
    P = engine_params(KYBER, 256, 16, [IMPROVED], exact=True)
    a = torch.zeros((4, 256), dtype=torch.int16, device="cuda")
    for bad in (torch.zeros((3, 256), dtype=torch.int16, device="cuda"),
                torch.zeros((4, 256), dtype=torch.int32, device="cuda"),
                torch.zeros((4, 512), dtype=torch.int16, device="cuda")[:, ::2],
                torch.zeros((4, 256), dtype=torch.int16)):
        with pytest.raises(nttk.ContractViolation):
            nttk.polymul(P, K.improved, a, bad)
        with pytest.raises(nttk.ContractViolation):
            nttk.forward(P, K.improved, a, out=bad)
    A = torch.zeros(8, dtype=torch.int64, device="cuda")
    with pytest.raises(nttk.ContractViolation):
        nttk.modmul_sweep(0, 3329, 16, 2, A, A, torch.zeros(8, dtype=torch.int64, device="cuda"))


def test_contracts_match_reference_messages():
    T = nttk.preset("toy13")
    with pytest.raises(nttk.ContractViolation, match="wrong input length"):
        nttk.ntt_forward([1, 2], T, K.ntl)
    with pytest.raises(nttk.ContractViolation, match="coefficients must be canonical"):
        nttk.ntt_forward([13, 0, 0, 0], T, K.ntl)
    with pytest.raises(nttk.ContractViolation, match="butterfly order"):
        nttk.intt_inverse(nttk.Spectrum([1, 2, 3, 4], nttk.Ordering.natural), T, K.ntl)
    only = nttk.build_params(13, 4, 8, [K.ntl])
    with pytest.raises(nttk.ContractViolation, match="kind not built"):
        nttk.ntt_forward([1, 2, 3, 4], only, K.harvey)
    with pytest.raises(nttk.ContractViolation, match="mixed orderings"):
        nttk.pointwise_multiply(nttk.Spectrum([1, 2, 3, 4]),
                                nttk.Spectrum([1, 2, 3, 4], nttk.Ordering.natural), T, K.ntl)
    with pytest.raises(nttk.ContractViolation, match=r"T must be < 2\^ell \* p"):
        nttk.pointwise_multiply(nttk.Spectrum([1, 2, 3, 4]), nttk.Spectrum([52, 0, 0, 0]), T,
                                K.improved)


def test_edge_batches_and_extreme_values(oracle):
    P = engine_params(KYBER, 256, 16, [IMPROVED], exact=True)
    Q = oracle.params(KYBER, 256, 16, (IMPROVED,), exact=True)
    # empty batch is a no-op
    e = torch.empty(0, dtype=torch.int16, device="cuda")
    assert nttk.forward(P, IMPROVED, e).numel() == 0
    for B in (1, 2, 3, 31, 33):
        f = np.full((B, 256), KYBER - 1, dtype=np.uint64)
        f[0] = 0
        got = from_dev(nttk.forward(P, IMPROVED, to_dev(f, 2)))
        assert (got == Q.forward(IMPROVED, f)).all()
    # every u16 word through the inverse's canonicalisation
    w = np.arange(1 << 16, dtype=np.uint64).reshape(256, 256)
    got = from_dev(nttk.inverse(P, IMPROVED, to_dev(w, 2)))
    assert (got == Q.inverse(IMPROVED, w)).all()


@pytest.mark.slow
def test_large_batch_properties():
    """BASELINE config 4 sizes: round trip identity over 2^22 Kyber + 2^21 Dilithium."""
    g = torch.Generator(device="cuda").manual_seed(4)
    for p, n, elem, B in ((KYBER, 16, 2, 1 << 22), (DILITHIUM, 32, 4, 1 << 21)):
        P = engine_params(p, 256, n, [IMPROVED], exact=True)
        x = torch.randint(0, p, (B, 256), generator=g, device="cuda", dtype=torch.int64).to(TDT[elem])
        y = nttk.forward(P, IMPROVED, x)
        assert int(y.to(torch.int64).min()) >= 0 and int(y.to(torch.int64).max()) < 9 * p
        assert torch.equal(nttk.inverse(P, IMPROVED, y), x)
        # repeated runs are bit-identical (guards the TMA stage ring against races)
        z = torch.empty_like(y)
        for _ in range(4):
            nttk.forward(P, IMPROVED, x, z)
            assert torch.equal(z, y)
        # sampled polynomials against the oracle
        from oracle.oracle import Oracle
        Q = Oracle().params(p, 256, n, (IMPROVED,), exact=True)
        idx = [0, 15, 16, B // 2 + 7, B - 1]
        xs = x[idx].cpu().numpy().astype(np.int64) & ((1 << (8 * elem)) - 1)
        ys = y[idx].cpu().numpy().astype(np.int64) & ((1 << (8 * elem)) - 1)
        assert (Q.forward(IMPROVED, xs.astype(np.uint64)).astype(np.int64) == ys).all()
        del x, y, z
        torch.cuda.empty_cache()


def test_sweep_vs_oracle_grid(oracle):
    for p, n, ell in ((KYBER, 16, 2), (DILITHIUM, 32, 7)):
        ctx = oracle.ctx(p, n, 0, ell)
        rng = np.random.default_rng(5)
        for variant in range(4):
            na, nb = 96, 2100  # ragged: not a multiple of the 2048-column tile
            if variant == 1:
                A = rng.integers(0, p, na)
                B = rng.integers(-(1 << (n - 1)), 1 << (n - 1), nb)
            elif variant == 2:
                A = rng.integers(0, p + 1, na)
                B = rng.integers(0, p + 1, nb)
            elif variant == 3:
                A = rng.integers(0, p, na)
                B = rng.integers(0, p << ell, nb)
            else:
                A = rng.integers(0, p, na)
                B = rng.integers(0, p, nb)
            want, s = oracle.sweep(variant, ctx, A, B)
            dA = torch.tensor(A, dtype=torch.int64, device="cuda")
            dB = torch.tensor(B, dtype=torch.int64, device="cuda")
            r = torch.empty(na * nb, dtype=torch.int64, device="cuda")
            got = nttk.modmul_sweep(variant, p, n, ell, dA, dB, r)
            assert got == s and (r.cpu().numpy() == want).all(), (p, variant)
            assert nttk.modmul_sweep(variant, p, n, ell, dA, dB) == s


@pytest.mark.gpu
def test_sweep_device_form_ragged(oracle):
    """nttk_modmul_sweep_device: queued, accumulating; ragged rows/columns around the
    64-row x 4096-column tile, every word-size path (n = 16, 32 and the any-n form)."""
    rng = np.random.default_rng(11)
    for p, n, ell in ((KYBER, 16, 2), (DILITHIUM, 32, 7), (12289, 24, 3), (257, 12, 1)):
        ctx = oracle.ctx(p, n, 0, ell)
        for variant in range(4):
            if variant == 2 and not 5 * p * p < ((1 << (n + 1)) - p) ** 2:
                continue  # plantard_redc context bound
            for na, nb in ((1, 1), (65, 4097), (130, 4095), (3, 8193)):
                A = rng.integers(0, p, na)
                B = rng.integers(0, p, nb)
                want, s = oracle.sweep(variant, ctx, A, B)
                dA = torch.tensor(A, dtype=torch.int64, device="cuda")
                dB = torch.tensor(B, dtype=torch.int64, device="cuda")
                cs = torch.zeros(1, dtype=torch.int64, device="cuda")
                r = torch.empty(na * nb, dtype=torch.int64, device="cuda")
                nttk.modmul_sweep_device(variant, p, n, ell, dA, dB, cs, r)
                nttk.modmul_sweep_device(variant, p, n, ell, dA, dB, cs)
                assert (int(cs.item()) & (2**64 - 1)) == (2 * s) & (2**64 - 1), (p, variant, na, nb)
                assert (r.cpu().numpy() == want).all(), (p, variant, na, nb)


def test_launch_counter_moves():
    before = nttk.launch_count()
    P = engine_params(KYBER, 256, 16, [IMPROVED], exact=True)
    x = torch.zeros(64, 256, dtype=torch.int16, device="cuda")
    nttk.forward(P, IMPROVED, x)
    assert nttk.launch_count() == before + 1


@pytest.mark.parametrize("name", ["toy13", "kyber256", "falcon512"])
def test_observed_transforms_match_reference_layer_by_layer(name):
    """ntt_forward_observed / intt_inverse_observed: every intermediate layer state equals the
    unmodified reference's (transform.hpp:77-116 observer calls), every kind."""
    from oracle.oracle import Oracle, Reference, reference_available

    if not reference_available():
        pytest.skip("oracle/_ref not built")
    P = nttk.preset(name)
    R = Reference().params(P.p, P.size, P.n_bits, (NTL, HARVEY, SCOTT, IMPROVED))
    L = P.size.bit_length() - 1
    f = Oracle().rng(17, P.p, P.size)
    for k in (NTL, HARVEY, SCOTT, IMPROVED):
        got = []
        spec = nttk.ntt_forward_observed(f, P, k, lambda layer, st: got.append((layer, st)))
        want_states, want_out = R.observed(k, 0, f, L)
        assert [g[0] for g in got] == list(range(1, L + 1))
        for (layer, st), w in zip(got, want_states):
            assert st == [int(x) for x in w], (name, k, layer)
        assert spec.values == [int(x) for x in want_out]
        got_i = []
        back = nttk.intt_inverse_observed(spec, P, k, lambda layer, st: got_i.append(st))
        want_states, want_out = R.observed(k, 1, spec.values, L)
        assert got_i == [[int(x) for x in w] for w in want_states], (name, k)
        assert back == [int(x) for x in f]


@pytest.mark.parametrize("p,N,n,tree,layers", [(40961, 4096, 32, CYCLIC, 0), (65537, 8192, 32, CYCLIC, 0),
                                               (65537, 16384, 32, CYCLIC, 0),
                                               (40961, 4096, 32, NEGA, 10)])
def test_generic_large_n_vs_oracle(oracle, p, N, n, tree, layers):
    """The generic kernel at large N: one CTA per polynomial up to N = 4096, one launch per
    layer beyond (generic.cu) -- every admitted kind, forward words and round trips."""
    kinds = (NTL, HARVEY, SCOTT, IMPROVED) if tree == CYCLIC else (HARVEY, IMPROVED, SMONT)
    admitted = []
    for k in kinds:
        try:
            engine_params(p, N, n, [k], tree=tree, layers=layers, exact=True)
            admitted.append(k)
        except nttk.ContractViolation:
            pass
    assert admitted
    B = 3
    f = oracle.rng(N + p, p, B * N).reshape(B, N)
    for k in admitted:
        P = engine_params(p, N, n, [k], tree=tree, layers=layers, exact=True)
        Q = oracle.params(p, N, n, (k,), tree=tree, layers=layers, exact=True)
        assert k not in P.fast_path
        sgn = k == SMONT
        y = nttk.forward(P, k, to_dev(f, 8, sgn))
        assert (from_dev(y, sgn).astype(np.int64) == Q.forward(k, f).astype(np.int64)).all(), k
        assert (from_dev(nttk.inverse(P, k, y)) == f).all(), k


def test_randomized_dispatch_sweep(oracle):
    """Seeded random (kind, N, tree, storage width, batch, buffer offset) cases across every
    dispatch path (TMA N=256 / N=512/1024 kernels, the register-prefetch u64 kernel, the
    generic kernel for misaligned buffers): forward vs oracle, round trip."""
    rng = np.random.default_rng(2402)
    cases = 0
    while cases < 40:
        N = int(rng.choice([256, 512, 1024]))
        p = {256: int(rng.choice([3329, 7681, 8380417])), 512: 12289, 1024: 12289}[N]
        n = 16 if (p == 3329 and rng.random() < 0.5) else 32
        tree = CYCLIC if (N > 256 or rng.random() < 0.6) else NEGA
        kinds = [IMPROVED, HARVEY, SMONT] + ([NTL, SCOTT] if tree == CYCLIC else [])
        k = int(rng.choice(kinds))
        layers = 0 if tree == CYCLIC else (7 if p == 3329 else 8)
        try:
            P = engine_params(p, N, n, [k], tree=tree, layers=layers, exact=True)
            Q = oracle.params(p, N, n, (k,), tree=tree, layers=layers, exact=True)
        except (nttk.ContractViolation, Exception):
            continue
        sgn = k == SMONT
        L = N.bit_length() - 1 if not layers else layers
        bound = {NTL: p, HARVEY: 2 * p, SCOTT: N * p, IMPROVED: (L + 1) * p, SMONT: (L + 2) * p}[k]
        lim = {2: 1 << 15, 4: 1 << 31, 8: 1 << 63} if sgn else {2: 1 << 16, 4: 1 << 32, 8: 1 << 64}
        elems = [e for e in (2, 4, 8) if bound <= lim[e]]
        if not elems:
            continue
        elem = int(rng.choice(elems))
        B = int(rng.integers(1, 70))
        off = int(rng.choice([0, 0, 1, 8]))  # 1: not 16-byte aligned -> fallback path
        f = oracle.rng(int(rng.integers(1 << 30)), p, B * N).reshape(B, N)
        dt = (SDT if sgn else DT)[elem]
        tdt = TDT[elem]
        buf = torch.zeros(B * N + off, dtype=tdt, device="cuda")
        x = buf[off:].view(B, N)
        x.copy_(torch.from_numpy(np.ascontiguousarray(f.astype(dt)).view(SDT[elem])).cuda())
        y = nttk.forward(P, k, x)
        want = Q.forward(k, f)
        assert (from_dev(y, sgn).astype(np.int64) == want.astype(np.int64)).all(), (p, N, n, tree, k, elem, B, off)
        assert (from_dev(nttk.inverse(P, k, y)) == f).all(), (p, N, n, tree, k, elem, B, off)
        cases += 1


def test_randomized_products_and_host_calls(oracle):
    """Seeded random cases for the product paths (fused polymul when aligned, the four-kernel
    composition otherwise, pointwise / basemul) and the host entry points, vs the oracle."""
    rng = np.random.default_rng(675)
    done = 0
    while done < 30:
        N = int(rng.choice([256, 256, 512, 1024]))
        p = {256: int(rng.choice([3329, 8380417])), 512: 12289, 1024: 12289}[N]
        n = 16 if (p == 3329 and rng.random() < 0.6) else 32
        tree = NEGA if (N == 256 and rng.random() < 0.5) else CYCLIC
        layers = (7 if p == 3329 else 8) if tree == NEGA else 0
        k = int(rng.choice([IMPROVED, HARVEY, SMONT] + ([NTL, SCOTT] if tree == CYCLIC else [])))
        try:
            P = engine_params(p, N, n, [k], tree=tree, layers=layers, exact=True)
            Q = oracle.params(p, N, n, (k,), tree=tree, layers=layers, exact=True)
        except Exception:
            continue
        B = int(rng.integers(1, 40))
        a = oracle.rng(int(rng.integers(1 << 30)), p, B * N).reshape(B, N)
        b = oracle.rng(int(rng.integers(1 << 30)), p, B * N).reshape(B, N)
        elem = 2 if p < (1 << 16) and rng.random() < 0.5 else (4 if rng.random() < 0.7 else 8)
        off = int(rng.choice([0, 0, 1]))
        tdt = TDT[elem]

        def dev(v):
            buf = torch.zeros(B * N + off, dtype=tdt, device="cuda")
            x = buf[off:].view(B, N)
            x.copy_(torch.from_numpy(np.ascontiguousarray(v.astype(DT[elem])).view(SDT[elem])).cuda())
            return x
        got = from_dev(nttk.polymul(P, k, dev(a), dev(b)))
        assert (got == Q.polymul(k, a, b)).all(), (p, N, n, tree, k, elem, B, off)
        # host forward at a width that holds the kind's spectrum (narrower ones are refused)
        L = N.bit_length() - 1 if not layers else layers
        bound = {NTL: p, HARVEY: 2 * p, SCOTT: N * p, IMPROVED: (L + 1) * p, SMONT: (L + 2) * p}[k]
        # (scott at n = 16 wraps in the reference: only 64-bit words hold it, and the engine
        # refuses the narrower ones -- SURVEY §0 item 6)
        host = None
        for hel in (e for e in (2, 4, 8) if bound <= (1 << (8 * e - (1 if k == SMONT else 0)))):
            try:
                host = nttk.ntt_forward_batch(a.astype({2: np.uint16, 4: np.uint32, 8: np.uint64}[hel]), P, k)
                break
            except nttk.ContractViolation as e:
                assert "cannot hold" in str(e) and k == SCOTT and n == 16, e
        host = np.asarray(host).astype({2: np.int16, 4: np.int32, 8: np.int64}[hel]).astype(np.int64) \
            if k == SMONT else np.asarray(host).astype(np.int64)
        assert (host == Q.forward(k, a).astype(np.int64)).all(), (p, N, k, hel)
        done += 1


def test_scott_n16_refuses_narrow_storage(oracle):
    """scott at Kyber n = 16 wraps uint64 in the reference; only 64-bit
    storage holds those words, so the engine refuses 16/32-bit storage instead of
    truncating -- and its 64-bit results (and polymul at any width) match the oracle."""
    P = engine_params(KYBER, 256, 16, [SCOTT])
    Q = oracle.params(KYBER, 256, 16, (SCOTT,))
    f = oracle.rng(8, KYBER, 5 * 256).reshape(5, 256)
    g = oracle.rng(9, KYBER, 5 * 256).reshape(5, 256)
    for elem in (2, 4):
        with pytest.raises(nttk.ContractViolation, match="cannot hold the scott spectrum bound"):
            nttk.forward(P, SCOTT, to_dev(f, elem))
        assert (from_dev(nttk.polymul(P, SCOTT, to_dev(f, elem), to_dev(g, elem))) ==
                Q.polymul(SCOTT, f, g)).all(), elem
    assert (from_dev(nttk.forward(P, SCOTT, to_dev(f, 8))) == Q.forward(SCOTT, f)).all()


def test_randomized_pointwise_basemul_and_aliasing(oracle):
    """pointwise / basemul on real forward spectra (lazy words) at random sizes and widths,
    and polymul with its output aliasing either operand."""
    rng = np.random.default_rng(2024)
    for case in range(16):
        p, n = (KYBER, 16) if case % 2 else (DILITHIUM, 32)
        tree = NEGA if case % 4 < 2 else CYCLIC
        layers = (7 if p == KYBER else 8) if tree == NEGA else 0
        k = int(rng.choice([IMPROVED, HARVEY, SMONT]))
        P = engine_params(p, 256, n, [k], tree=tree, layers=layers, exact=True)
        Q = oracle.params(p, 256, n, (k,), tree=tree, layers=layers, exact=True)
        B = int(rng.integers(1, 50))
        a = oracle.rng(100 + case, p, B * 256).reshape(B, 256)
        b = oracle.rng(200 + case, p, B * 256).reshape(B, 256)
        sgn = k == SMONT
        elem = 4 if p == DILITHIUM else int(rng.choice([2, 4]))
        fa, fb = nttk.forward(P, k, to_dev(a, elem)), nttk.forward(P, k, to_dev(b, elem))
        Fa, Fb = Q.forward(k, a), Q.forward(k, b)
        if tree == NEGA and layers == 7:
            assert (from_dev(nttk.basemul(P, k, fa, fb)) == Q.basemul(k, Fa, Fb)).all(), case
        else:
            assert (from_dev(nttk.pointwise(P, k, fa, fb)) == Q.pointwise(k, Fa, Fb)).all(), case
        want = Q.polymul(k, a, b)
        xa, xb = to_dev(a, elem), to_dev(b, elem)
        nttk.polymul(P, k, xa, xb, out=xb)  # out aliases b
        assert (from_dev(xb) == want).all(), case
        xa, xb = to_dev(a, elem), to_dev(b, elem)
        nttk.polymul(P, k, xa, xb, out=xa)  # out aliases a
        assert (from_dev(xa) == want).all(), case


def _extreme_words(p, bits, B, seed, N=256):
    """Inverse inputs that drive the merge bounds: all-max words, max/zero patterns that
    maximise T = X + off - Y, and random draws from boundary values (words need not be
    canonical: the inverse canonicalises, transform.hpp:243)."""
    top = (1 << bits) - 1
    rs = np.random.RandomState(seed)
    pts = np.array([0, 1, p - 1, p, 2 * p - 1, 9 * p - 1, top - p, top - 1, top], dtype=np.uint64)
    pts = pts[pts <= top]
    w = pts[rs.randint(0, len(pts), size=(B, N))]
    w[0] = top
    w[1] = 0
    w[2, ::2], w[2, 1::2] = top, 0
    w[3, :N // 2], w[3, N // 2:] = top, 0
    idx = np.arange(N)
    L = N.bit_length() - 1
    for k in range(L):  # X max / Y zero at every merge span 2^k
        w[4 + k] = np.where((idx >> k) & 1, 0, top)
    return w


@pytest.mark.parametrize("p,n,elem,tree,layers", [(KYBER, 16, 2, CYCLIC, 8),
                                                   (KYBER, 16, 2, NEGA, 7), (DILITHIUM, 32, 4, CYCLIC, 8),
                                                   (DILITHIUM, 32, 4, NEGA, 8), (7681, 32, 4, CYCLIC, 8),
                                                   (12289, 32, 4, CYCLIC, 8)])
@pytest.mark.parametrize("kind", [IMPROVED, HARVEY, NTL])
def test_inverse_extreme_words(oracle, p, n, elem, tree, layers, kind):
    """Worst-case words through the fast inverse (TW1 multiply-free block-0 merges for the
    improved / harvey / ntl kinds, the u16 DEFER path without input canonicalisation, the
    u32 partial canonicalisation) vs the oracle, bit-exact."""
    if kind == NTL and tree == NEGA:
        pytest.skip("ntl is a DIF kind: cyclic tree only")
    P = engine_params(p, 256, n, [kind], tree=tree, layers=layers, exact=True)
    Q = oracle.params(p, 256, n, (kind,), tree=tree, layers=layers, exact=True)
    assert kind in P.fast_path
    w = _extreme_words(p, 8 * elem, 515, 7 + p + layers)
    got = from_dev(nttk.inverse(P, kind, to_dev(w, elem)))
    assert (got == Q.inverse(kind, w)).all()
    # and the round trip of their forward images
    f = np.asarray(Q.inverse(kind, w))
    y = nttk.forward(P, kind, to_dev(f, elem))
    assert (from_dev(nttk.inverse(P, kind, y)) == f).all()


@pytest.mark.parametrize("N", [512, 1024])
@pytest.mark.parametrize("n,elem", [(32, 4), (32, 8)])
def test_fastn_inverse_extreme_words(oracle, N, n, elem):
    """Worst-case words through the N = 512 / 1024 inverse (TW1 multiply-free block-0
    merges of the phase-2 layers) vs the oracle, bit-exact."""
    p = 12289
    P = engine_params(p, N, n, [IMPROVED])
    Q = oracle.params(p, N, n, (IMPROVED,))
    assert IMPROVED in P.fast_path
    w = _extreme_words(p, 8 * elem if elem < 8 else 40, 131, 3 + N + n, N)
    got = from_dev(nttk.inverse(P, IMPROVED, to_dev(w, elem)))
    assert (got == Q.inverse(IMPROVED, w)).all()


def test_sweep_full_grid_vs_reference_checksums():
    """BASELINE config 5 at its stated size: every 2^15 x 2^15 = 2^30-pair grid of
    tests/golden/sweep_inputs.py (boundary values first) on the GPU reproduces the checksum
    of the reference's checked reductions over the same grid (tests/golden/sweep_2p30.json)."""
    import json
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from sweep_inputs import grid

    with open(os.path.join(os.path.dirname(__file__), "golden", "sweep_2p30.json")) as fh:
        rows = json.load(fh)["rows"]
    for row in rows:
        A, B = grid(row["q"], row["n_bits"], row["ell"], row["variant"])
        s = nttk.modmul_sweep(row["variant"], row["q"], row["n_bits"], row["ell"],
                              torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
        assert "%016x" % s == row["checksum"], row


@pytest.mark.parametrize("p,n,tree,layers", [(KYBER, 16, NEGA, 7), (KYBER, 16, CYCLIC, 8),
                                             (DILITHIUM, 32, NEGA, 8), (DILITHIUM, 32, CYCLIC, 8),
                                             (12289, 32, CYCLIC, 9)])
@pytest.mark.parametrize("kind", [IMPROVED, HARVEY, SMONT])
def test_standalone_products_vs_oracle(oracle, p, n, tree, layers, kind):
    """Standalone pointwise / basemul (product.cu: 32-bit per-kind reductions, 128-bit I/O)
    on lazy forward spectra and on arbitrary storage words vs the oracle, every storage
    width that holds the words; a misaligned view exercises the generic fallback."""
    N = 1 << layers if tree == CYCLIC else 256
    P = engine_params(p, N, n, [kind], tree=tree, layers=layers, exact=True)
    Q = oracle.params(p, N, n, (kind,), tree=tree, layers=layers, exact=True)
    sg = kind == SMONT
    B = 37
    a = oracle.rng(300 + kind, p, B * N).reshape(B, N)
    b = oracle.rng(400 + kind, p, B * N).reshape(B, N)
    fa, fb = Q.forward(kind, a), Q.forward(kind, b)
    prod = Q.basemul if (N >> layers) == 2 else Q.pointwise
    want = prod(kind, fa, fb)
    fits16 = max(np.abs(fa.astype(np.int64)).max(), np.abs(fb.astype(np.int64)).max()) < (1 << 15)
    for elem in ((2, 4) if fits16 else (4,)):
        xa, xb = to_dev(fa, elem, sg), to_dev(fb, elem, sg)
        fn = nttk.basemul if (N >> layers) == 2 else nttk.pointwise
        assert (from_dev(fn(P, kind, xa, xb)) == want).all(), (elem, "spectra")
        # arbitrary storage words: canonicalised first
        wa = oracle.rng(500 + kind, 1 << (8 * elem - 1), B * N).reshape(B, N)
        wb = oracle.rng(600 + kind, 1 << (8 * elem - 1), B * N).reshape(B, N)
        if sg:
            wa = wa.astype(np.int64) - (1 << (8 * elem - 2))
            wb = wb.astype(np.int64) - (1 << (8 * elem - 2))
        ca = np.array([[int(v) % p for v in row] for row in wa], dtype=np.uint64)
        cb = np.array([[int(v) % p for v in row] for row in wb], dtype=np.uint64)
        got = from_dev(fn(P, kind, to_dev(wa, elem, sg), to_dev(wb, elem, sg)))
        assert (got == prod(kind, ca, cb)).all(), (elem, "words")
        # misaligned (not 16-byte aligned) buffers: the generic kernel, same result
        buf_a = torch.zeros(B * N + 1, dtype=TDT[elem], device="cuda")
        buf_b = torch.zeros(B * N + 1, dtype=TDT[elem], device="cuda")
        buf_a[1:] = xa.view(-1)
        buf_b[1:] = xb.view(-1)
        got = from_dev(fn(P, kind, buf_a[1:], buf_b[1:]))
        assert (got.reshape(B, N) == want).all(), (elem, "misaligned")


def test_plantard_correction_fires_counter():
    """plantard_correction_fires (reduction.hpp:172-191): within the admitted operand range
    the r == p corner never fires (the reference's own observation, reduction_test.cpp and
    Appendix: exhaustive toy radices) -- the counter stays put over a full grid; operands
    outside the range (the sweep does not check per pair) reach the corner, and the device
    count equals a numpy count of h_hi == 2^16 - 1."""
    q, n = 3329, 16
    before = nttk.plantard_correction_fires()
    A = torch.arange(0, q + 1, dtype=torch.int64, device="cuda")
    nttk.modmul_sweep(2, q, n, 0, A, A)
    assert nttk.plantard_correction_fires() == before
    # the corner needs W T = 2^32 - k p (k < 2^16): large 16-bit operands
    W = np.arange(65024, 65536, dtype=np.int64)
    T = np.arange(0, 1 << 16, dtype=np.int64)
    mu = pow(q, -1, 1 << 32)
    wt = (W[:, None] * T[None, :]).astype(np.uint64)  # < 2^32
    h = (wt * np.uint64(mu)) & np.uint64(0xFFFFFFFF)  # uint64 products wrap mod 2^64
    want = int(((h >> 16) == 0xFFFF).sum())
    assert want > 0
    nttk.modmul_sweep(2, q, n, 0, torch.from_numpy(W).cuda(), torch.from_numpy(T).cuda())
    assert nttk.plantard_correction_fires() - before == want


def test_captured_plans_match_eager_calls(oracle):
    """nttk_plan_create / nttk_plan_launch (include/nttk_gpu.h): a captured forward, inverse
    and fused polymul (config 1 / config 2 shapes, small batch) give the eager calls' words;
    creating a plan runs nothing; repeat > 1 replays the operation in place."""
    Pn = engine_params(KYBER, 256, 16, [IMPROVED, HARVEY], tree=NEGA, layers=7, exact=True)
    Q = oracle.params(KYBER, 256, 16, (IMPROVED, HARVEY), tree=NEGA, layers=7, exact=True)
    B = 4096
    f = oracle.rng(81, KYBER, B * 256).reshape(B, 256)
    g = oracle.rng(82, KYBER, B * 256).reshape(B, 256)
    x, y = to_dev(f, 2), to_dev(g, 2)
    out = torch.zeros_like(x)
    plan = nttk.Plan(Pn, IMPROVED, nttk.Plan.FORWARD, x, out)
    torch.cuda.synchronize()
    assert not out.any()  # nothing ran at creation
    plan.launch()
    torch.cuda.synchronize()
    assert (from_dev(out) == Q.forward(IMPROVED, f)).all()
    inv = torch.empty_like(x)
    nttk.Plan(Pn, IMPROVED, nttk.Plan.INVERSE, out, inv).launch()
    torch.cuda.synchronize()
    assert torch.equal(inv, x)
    for k in (IMPROVED, HARVEY):
        pm = torch.empty_like(x)
        nttk.Plan(Pn, k, nttk.Plan.POLYMUL, x, pm, b=y).launch()
        torch.cuda.synchronize()
        assert (from_dev(pm) == Q.polymul(k, f, g)).all()
    # repeat: 3 in-place forwards of the N = 1024 preset (fastn kernel, narrow image)
    P = nttk.preset("newhope1024")
    Qn = oracle.params(12289, 1024, 32, (IMPROVED,))
    h = oracle.rng(83, 12289, 8 * 1024).reshape(8, 1024)
    z = to_dev(h, 4)
    nttk.Plan(P, IMPROVED, nttk.Plan.INVERSE, z, z, repeat=3).launch()
    torch.cuda.synchronize()
    want = h
    for _ in range(3):
        want = Qn.inverse(IMPROVED, want)
    assert (from_dev(z) == want).all()
    with pytest.raises(nttk.ContractViolation):
        nttk.Plan(Pn, SCOTT, nttk.Plan.FORWARD, x, out)  # kind not built into Pn


@pytest.mark.parametrize("name", ["kyber256", "newhope512", "newhope1024"])
def test_narrow_image_extremes(oracle, name):
    """The paper's Table 2 presets run on the narrow image (n = 16 product on the n = 32 set;
    F1/F3 forward, bound-exponent inverse with paper-form products): extreme canonical inputs
    through the forward and extreme storage words through the inverse, bit-exact with the
    oracle's n = 32 reference loop."""
    P = nttk.preset(name)
    assert P.fast_flags(IMPROVED, 0) & 512 and P.fast_flags(IMPROVED, 1) & 512
    p, N = P.p, P.size
    Q = oracle.params(p, N, 32, (IMPROVED,))
    rows = [np.full(N, p - 1), np.zeros(N, dtype=np.int64), np.where(np.arange(N) % 2 == 0, p - 1, 0),
            np.where(np.arange(N) < N // 2, p - 1, 0), np.arange(N) % p, oracle.rng(91, p, N)]
    f = np.stack(rows).astype(np.int64)
    assert (from_dev(nttk.forward(P, IMPROVED, to_dev(f, 4))) == Q.forward(IMPROVED, f)).all()
    w = _extreme_words(p, 32, 67, 5 + N, N)
    assert (from_dev(nttk.inverse(P, IMPROVED, to_dev(w, 4))) == Q.inverse(IMPROVED, w)).all()


@pytest.mark.parametrize("N", [512, 1024])
def test_ct_narrow_inverse_and_its_fallback(oracle, N):
    """N = 512 / 1024 improved inverses: the Table 2 modulus 12289 runs the CT-form narrow inverse
    (fastn_tma.cu inv_body_n_ct, flags bit 11); p = 13313 fits the narrow image but not
    kCtLimN p, so it keeps the GS narrow body.  Extreme and random storage words, ragged batches, bit-exact with the oracle's n = 32 reference inverse
    (transform.hpp:233-343)."""
    for p, ct in ((12289, True), (13313, False)):
        P = nttk.build_params(p, N, 32, [IMPROVED])
        fl = P.fast_flags(IMPROVED, 1)
        assert bool(fl & 2048) == ct and fl & 512
        Q = oracle.params(p, N, 32, (IMPROVED,))
        for batch in (15, 33, 67):
            w = _extreme_words(p, 32, batch, 7 + N + batch, N)
            assert (from_dev(nttk.inverse(P, IMPROVED, to_dev(w, 4))) == Q.inverse(IMPROVED, w)).all()
            assert (from_dev(nttk.inverse(P, IMPROVED, to_dev(w[:1], 4))) == Q.inverse(IMPROVED, w[:1])).all()
        f = oracle.rng(17, p, 70 * N).reshape(70, N).astype(np.int64)
        s = nttk.forward(P, IMPROVED, to_dev(f, 4))
        assert (from_dev(s) == Q.forward(IMPROVED, f)).all()
        assert (from_dev(nttk.inverse(P, IMPROVED, s)) == f).all()


def test_ct_inverse_canonical_input_images(oracle):
    """N = 256 CT-form inverse on canonicalised (unpacked) words (HostParams::fast_ctinv_c): the
    Kyber n = 16 set in u32 storage and the narrow image of the kyber256 preset (q = 7681,
    n = 32).  Extreme, raw 32-bit and random words, ragged batches, bit-exact with the oracle."""
    for p, n, exact in ((3329, 16, True), (7681, 32, False)):
        P = nttk.build_params(p, 256, n, [IMPROVED], exact_bound=exact)
        assert P.fast_flags(IMPROVED, 1) & 2048
        Q = oracle.params(p, 256, n, (IMPROVED,), exact=exact)
        for batch in (13, 35, 130):
            w = _extreme_words(p, 32, batch, 11 + batch + p)
            assert (from_dev(nttk.inverse(P, IMPROVED, to_dev(w, 4))) == Q.inverse(IMPROVED, w)).all()
        f = oracle.rng(23, p, 77 * 256).reshape(77, 256).astype(np.int64)
        s = nttk.forward(P, IMPROVED, to_dev(f, 4))
        assert (from_dev(s) == Q.forward(IMPROVED, f)).all()
        assert (from_dev(nttk.inverse(P, IMPROVED, s)) == f).all()


def test_pdl_dependent_chains(oracle):
    """The TMA kernels are launched with programmatic dependent launch allowed
    (launch_cache.hpp launch_pdl): a small launch becomes resident while the previous one still
    runs and must not read its input before that grid has completed.  Chains of dependent small
    launches -- in place, each reading what the previous wrote, on idle SMs so the next grid
    starts early -- end in the oracle's words."""
    p = 3329
    P = engine_params(p, 256, 16, [IMPROVED], exact=True)
    Q = oracle.params(p, 256, 16, (IMPROVED,), exact=True)
    for batch in (1, 37, 300):
        f = oracle.rng(41 + batch, p, batch * 256).reshape(batch, 256).astype(np.int64)
        buf = to_dev(f, 2)
        for _ in range(25):
            nttk.forward(P, IMPROVED, buf, buf)
            nttk.inverse(P, IMPROVED, buf, buf)
        assert (from_dev(buf) == f).all()
        nttk.forward(P, IMPROVED, buf, buf)
        assert (from_dev(buf) == Q.forward(IMPROVED, f)).all()
    # Dilithium u32 (tensor-map producer) and the N = 1024 kernel in the same kind of chain
    for pp, N, n, exact in ((8380417, 256, 32, True), (12289, 1024, 32, False)):
        Pd = engine_params(pp, N, n, [IMPROVED], exact=exact)
        f = oracle.rng(5, pp, 19 * N).reshape(19, N).astype(np.int64)
        buf = to_dev(f, 4)
        for _ in range(15):
            nttk.forward(Pd, IMPROVED, buf, buf)
            nttk.inverse(Pd, IMPROVED, buf, buf)
        assert (from_dev(buf) == f).all()
    # inside a captured plan the launches are back to back on the device, so the next grid really
    # starts while the previous one runs (the kernels signal launch_dependents as they start):
    # the in-place inverse of arbitrary words, 16 times per replay, against the oracle's iterate
    for pp, n, elem in ((3329, 16, 2), (8380417, 32, 4)):
        Pi = engine_params(pp, 256, n, [IMPROVED], exact=True)
        Qi = oracle.params(pp, 256, n, (IMPROVED,), exact=True)
        w = _extreme_words(pp, 8 * elem, 37, 77 + elem)
        buf = to_dev(w, elem)
        plan = nttk.Plan(Pi, IMPROVED, nttk.Plan.INVERSE, buf, buf, repeat=16)
        plan.launch()
        want = w
        for _ in range(16):
            want = np.asarray(Qi.inverse(IMPROVED, want)).astype(np.uint64)
        assert (from_dev(buf) == want).all()
        del plan
    # fused polymul chain: c <- c * b, ten times (negacyclic Kyber tree, basemul)
    Pn = engine_params(p, 256, 16, [IMPROVED], tree=NEGA, layers=7, exact=True)
    Qn = oracle.params(p, 256, 16, (IMPROVED,), tree=NEGA, layers=7, exact=True)
    a = oracle.rng(7, p, 21 * 256).reshape(21, 256).astype(np.int64)
    b = oracle.rng(8, p, 21 * 256).reshape(21, 256).astype(np.int64)
    c, db, want = to_dev(a, 2), to_dev(b, 2), a
    for _ in range(10):
        nttk.polymul(Pn, IMPROVED, c, db, c)
        want = np.asarray(Qn.polymul(IMPROVED, want, b)).astype(np.int64)
    assert (from_dev(c) == want).all()
