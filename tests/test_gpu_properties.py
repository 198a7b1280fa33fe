"""Device-side property suites: the reference's verify.hpp patterns
run on the B200 engine, with the pinned oracle as the checker.

* reductions (verify_montgomery / _signed_montgomery / _plantard / _modified_plantard,
  verify.hpp:65-213): exhaustive operand grids on the toy radices and 10^6 seeded random
  pairs on each production context (verify.hpp:114-122, 201-211), bit-exact;
* transforms (verify_transform, verify.hpp:375-483): every butterfly kind's forward
  spectrum equals the naive DFT (cyclic) or the naive evaluation at the tree's roots
  (negacyclic) modulo p, in butterfly order, and every kind's inverse inverts every
  other kind's forward -- on toy sizes (generic kernel) and on the production sizes
  N = 256 / 512 / 1024 (fast kernels).
"""
import numpy as np
import pytest
import torch

from oracle.oracle import CYCLIC, HARVEY, IMPROVED, NEGA, NTL, SCOTT, SMONT, OracleError

import paper_2402_00675_b200.nttk as nttk

pytestmark = pytest.mark.gpu

MONT, SMONT_R, PLANTARD, MPLANTARD = 0, 1, 2, 3


@pytest.fixture(scope="module", autouse=True)
def _device():
    assert torch.cuda.is_available() and nttk.device_available()


def operand_ranges(variant, p, n, ell):
    """Valid operand domains per reduction (reduction.hpp)."""
    if variant == MONT:
        return (0, p), (0, p)
    if variant == SMONT_R:
        return (0, p), (-(1 << (n - 1)), 1 << (n - 1))
    if variant == PLANTARD:
        return (0, p + 1), (0, p + 1)
    return (0, p), (0, p << ell)


def run_sweep(oracle, variant, p, n, ell, A, B):
    ctx = oracle.ctx(p, n, 0, ell)
    want, s = oracle.sweep(variant, ctx, A, B)
    dA = torch.tensor(A, dtype=torch.int64, device="cuda")
    dB = torch.tensor(B, dtype=torch.int64, device="cuda")
    r = torch.empty(A.size * B.size, dtype=torch.int64, device="cuda")
    got = nttk.modmul_sweep(variant, p, n, ell, dA, dB, r)
    return want, s, r.cpu().numpy(), got


TOY = [(13, 8, 2), (17, 6, 1), (17, 8, 2), (31, 8, 1), (97, 12, 2)]


@pytest.mark.parametrize("p,n,ell", TOY)
@pytest.mark.parametrize("variant", [MONT, SMONT_R, PLANTARD, MPLANTARD])
def test_reductions_exhaustive_toy(oracle, p, n, ell, variant):
    """Every operand pair of the variant's domain on a toy radix."""
    (a0, a1), (b0, b1) = operand_ranges(variant, p, n, ell)
    A = np.arange(a0, a1, dtype=np.int64)
    B = np.arange(b0, b1, dtype=np.int64)
    try:
        want, s, got, gs = run_sweep(oracle, variant, p, n, ell, A, B)
    except (OracleError, nttk.ContractViolation) as e:
        pytest.skip(f"context not admitted: {e}")
    assert gs == s and (got == want).all()


@pytest.mark.parametrize("variant", [MONT, SMONT_R, PLANTARD, MPLANTARD])
def test_reductions_exhaustive_kyber_n16(oracle, variant):
    """Every operand pair of the variant's domain at Kyber's q = 3329, n = 16 (the
    specialised 32-bit sweep bodies), in row blocks of <= 2^24 pairs."""
    p, n, ell = 3329, 16, 2
    (a0, a1), (b0, b1) = operand_ranges(variant, p, n, ell)
    B = np.arange(b0, b1, dtype=np.int64)
    rows = max(1, (1 << 24) // B.size)
    for r0 in range(a0, a1, rows):
        A = np.arange(r0, min(a1, r0 + rows), dtype=np.int64)
        want, s, got, gs = run_sweep(oracle, variant, p, n, ell, A, B)
        assert gs == s and (got == want).all(), (variant, r0)


def boundary_operands(lo, hi, p, ell, signed):
    """SURVEY §8(d) config 5 boundary set: {0, 1, q-1, q, 2^k q - 1, 2^k q (k <= ell + 1),
    range max - 1, range max - 2}, plus the negative mirrors for the signed operand;
    clipped to [lo, hi)."""
    v = {0, 1, p - 1, p, hi - 1, hi - 2}
    for k in range(ell + 2):
        v |= {(p << k) - 1, p << k}
    if signed:
        v |= {-x for x in list(v)} | {lo, lo + 1}
    return np.array(sorted(x for x in v if lo <= x < hi), dtype=np.int64)


@pytest.mark.parametrize("p,n,ell", [(3329, 16, 2), (8380417, 32, 7)])
@pytest.mark.parametrize("variant", [MONT, SMONT_R, PLANTARD, MPLANTARD])
def test_reductions_boundary_grid(oracle, p, n, ell, variant):
    """Boundary x boundary, boundary x random and random x boundary grids (config 5's
    boundary values) through the sweep kernel, bit-exact against the reference."""
    rng = np.random.default_rng(777 + 7 * variant + n)
    (a0, a1), (b0, b1) = operand_ranges(variant, p, n, ell)
    Ab = boundary_operands(a0, a1, p, ell, False)
    Bb = boundary_operands(b0, b1, p, ell, variant == SMONT_R)
    Ar = rng.integers(a0, a1, 4099, dtype=np.int64)
    Br = rng.integers(b0, b1, 4099, dtype=np.int64)
    for A, B in ((Ab, Bb), (Ab, Br), (Ar, Bb)):
        want, s, got, gs = run_sweep(oracle, variant, p, n, ell, A, B)
        assert gs == s and (got == want).all(), (variant, A.size, B.size)


@pytest.mark.parametrize("p,n,ell", [(3329, 16, 2), (8380417, 32, 7)])
@pytest.mark.parametrize("variant", [MONT, SMONT_R, PLANTARD, MPLANTARD])
def test_reductions_random_production(oracle, p, n, ell, variant):
    """10^6 seeded random pairs (1000 x 1000 grid) plus the domain boundaries."""
    rng = np.random.default_rng(12345 + 31 * variant + n)
    (a0, a1), (b0, b1) = operand_ranges(variant, p, n, ell)
    A = rng.integers(a0, a1, 1000, dtype=np.int64)
    B = rng.integers(b0, b1, 1000, dtype=np.int64)
    A[:3] = [a0, a0 + 1, a1 - 1]
    B[:3] = [b0, b0 + 1, b1 - 1]
    want, s, got, gs = run_sweep(oracle, variant, p, n, ell, A, B)
    assert gs == s and (got == want).all()


def bitrev(i, bits):
    return int(format(i, f"0{bits}b")[::-1], 2) if bits else 0


TRANSFORMS = [  # (p, N, n, tree, exact)
    (17, 8, 16, CYCLIC, False), (97, 16, 16, CYCLIC, False), (7681, 64, 32, CYCLIC, False),
    (3329, 256, 16, CYCLIC, True), (8380417, 256, 32, CYCLIC, True), (12289, 512, 32, CYCLIC, False),
    (12289, 1024, 32, CYCLIC, False), (97, 16, 16, NEGA, False), (7681, 256, 32, NEGA, False),
    (12289, 1024, 32, NEGA, False),
]


def kinds_for(tree, p, N, n):
    ks = [HARVEY, IMPROVED, SMONT] if tree == NEGA else [NTL, HARVEY, SCOTT, IMPROVED, SMONT]
    out = []
    for k in ks:
        try:
            nttk.build_params(p, N, n, [k], tree=tree, exact_bound=True)
            out.append(k)
        except nttk.ContractViolation:
            pass
    return out


@pytest.mark.parametrize("p,N,n,tree,exact", TRANSFORMS)
def test_transform_properties(oracle, p, N, n, tree, exact):
    kinds = kinds_for(tree, p, N, n)
    assert kinds, "no kind admitted"
    B = 9
    f = oracle.rng(4000 + N + n, p, B * N).reshape(B, N)
    bits = N.bit_length() - 1
    spectra = {}
    for k in kinds:
        P = nttk.build_params(p, N, n, [k], tree=tree, exact_bound=True)
        x = torch.from_numpy(f.astype(np.int64)).cuda()
        y = nttk.forward(P, k, x).cpu().numpy().astype(np.int64) % p
        if tree == CYCLIC:
            for b in range(B):
                dft = oracle.naive_dft(f[b], P.omega, p).astype(np.int64)
                assert (y[b] == dft[[bitrev(i, bits) for i in range(N)]]).all(), (k, b)
        else:
            Q = oracle.params(p, N, n, (k,), tree=tree, exact=True)
            for b in range(B):  # naive_eval takes one polynomial
                assert (y[b] == Q.naive_eval(f[b]).astype(np.int64)).all(), (k, b)
        spectra[k] = (P, nttk.forward(P, k, x))
    for k, (P, y) in spectra.items():  # every inverse undoes every forward (same residues)
        for k2, (P2, _) in spectra.items():
            if (k == SMONT) != (k2 == SMONT):
                continue  # signed spectra are two's complement words: only smont reads them
            back = nttk.inverse(P2, k2, y)
            assert (back.cpu().numpy() == f).all(), (k, k2)


# ---------------------------------------------------------------------------
# reduction.hpp signatures on the GPU (nttk_reduce): the reference's known answers,
# exhaustive toy ranges and random production operands vs the oracle, contract messages

def test_reductions_known_answers():
    c = nttk.make_reduction_context(13, 8, 0, 2)
    assert c.mu == 20165
    assert nttk.mont_redc(100, nttk.make_reduction_context(17, 5)) == 1
    s = nttk.make_reduction_context(17, 6)
    assert nttk.signed_mont_redc(100, s) == 9 and nttk.signed_mont_redc(-100, s) == -9
    assert nttk.plantard_redc(5, 12, nttk.make_reduction_context(13, 8)) == 6
    assert nttk.modified_plantard_mul(5, 20, c) == 10 and nttk.modified_plantard_mul(1, 1, c) == 4
    assert nttk.to_plantard_domain(7, c) == 5


@pytest.mark.parametrize("p,n,alpha,ell", [(13, 8, 0, 2), (17, 6, 0, 1), (31, 8, 1, 1)])
def test_elementwise_reductions_exhaustive_toy(oracle, p, n, alpha, ell):
    c = nttk.make_reduction_context(p, n, alpha, ell)
    o = oracle.ctx(p, n, alpha, ell)
    T = np.arange(p * p, dtype=np.uint64)
    assert (nttk.mont_redc(T, c) == [oracle.mont_redc(int(t), o) for t in T]).all()
    if c.fits_signed_montgomery_bound():
        lim = p << (n - 1)
        A = np.arange(-lim + 1, lim, dtype=np.int64)
        assert (nttk.signed_mont_redc(A, c) == [oracle.signed_mont_redc(int(a), o) for a in A]).all()
    W, Tt = np.meshgrid(np.arange(p + 1, dtype=np.uint64), np.arange(p + 1, dtype=np.uint64))
    W, Tt = W.ravel(), Tt.ravel()
    if c.fits_plantard_bound():
        assert (nttk.plantard_redc(W, Tt, c) ==
                [oracle.plantard_redc(int(a), int(b), o) for a, b in zip(W, Tt)]).all()
    if c.fits_lazy_plantard_bound():
        W2, T2 = np.meshgrid(np.arange(p, dtype=np.uint64), np.arange(p << ell, dtype=np.uint64))
        W2, T2 = W2.ravel(), T2.ravel()
        assert (nttk.modified_plantard_mul(W2, T2, c) ==
                [oracle.modified_plantard_mul(int(a), int(b), o) for a, b in zip(W2, T2)]).all()
    w = np.arange(p, dtype=np.uint64)
    assert (nttk.to_plantard_domain(w, c) == [oracle.to_plantard_domain(int(v), o) for v in w]).all()
    assert (nttk.to_montgomery_domain(w, c) == [oracle.to_montgomery_domain(int(v), o) for v in w]).all()


@pytest.mark.parametrize("p,n,ell", [(3329, 16, 2), (8380417, 32, 7)])
def test_elementwise_reductions_random_production(oracle, p, n, ell):
    """10^5 random operands per op through the device-tensor API vs the oracle."""
    rng = np.random.default_rng(p + n)
    c = nttk.make_reduction_context(p, n, 0, ell)
    o = oracle.ctx(p, n, 0, ell)
    m = 100000
    cases = [(nttk.OP_MONT_REDC, rng.integers(0, p * p, m, dtype=np.uint64), None,
              lambda a, b: oracle.mont_redc(a, o)),
             (nttk.OP_SIGNED_MONT_REDC, rng.integers(-(p << (n - 1)) + 1, p << (n - 1), m,
                                                     dtype=np.int64), None,
              lambda a, b: oracle.signed_mont_redc(a, o)),
             (nttk.OP_MODIFIED_PLANTARD_MUL, rng.integers(0, p, m, dtype=np.uint64),
              rng.integers(0, p << ell, m, dtype=np.uint64),
              lambda a, b: oracle.modified_plantard_mul(a, b, o))]
    if c.fits_plantard_bound():
        cases.append((nttk.OP_PLANTARD_REDC, rng.integers(0, p + 1, m, dtype=np.uint64),
                      rng.integers(0, p + 1, m, dtype=np.uint64),
                      lambda a, b: oracle.plantard_redc(a, b, o)))
    for op, x, y, ref in cases:
        dx = torch.from_numpy(x.view(np.int64)).cuda()
        dy = torch.from_numpy(y.view(np.int64)).cuda() if y is not None else None
        got = nttk.reduce(op, c, dx, dy).cpu().numpy()
        idx = rng.integers(0, m, 2000)
        want = [ref(int(x[i]), int(y[i]) if y is not None else 0) for i in idx]
        got_i = got[idx] if op == nttk.OP_SIGNED_MONT_REDC else got[idx].view(np.uint64)
        assert (got_i.astype(np.int64) == np.array(want, dtype=np.int64)).all(), op


def test_reduction_contract_messages():
    c = nttk.make_reduction_context(13, 8, 0, 2)
    m = nttk.make_reduction_context(17, 5)
    for call, msg in ((lambda: nttk.mont_redc(17 * 17, m), "mont_redc: T must be < p^2"),
                      (lambda: nttk.modified_plantard_mul(13, 0, c), "W must be < p"),
                      (lambda: nttk.modified_plantard_mul(0, 52, c), "T must be < 2^ell * p"),
                      (lambda: nttk.plantard_redc(14, 0, nttk.make_reduction_context(13, 8)),
                       "inputs exceed p"),
                      (lambda: nttk.to_plantard_domain(13, c), "w must be < p"),
                      (lambda: nttk.signed_mont_redc(1, nttk.make_reduction_context(31, 5)),
                       "requires 2p < 2^n"),
                      (lambda: nttk.modified_plantard_mul(1, 1, nttk.make_reduction_context(17, 8, 0, 2)),
                       "requires p < 2^{n-ell-2}")):
        with pytest.raises(nttk.ContractViolation, match=__import__("re").escape(msg)):
            call()


# ---------------------------------------------------------------------------
# butterfly.hpp checked entry points on the GPU (nttk_butterfly)

def test_butterfly_hand_examples_on_gpu():  # butterfly_test.cpp:31-197
    c8 = nttk.make_reduction_context(13, 8)
    assert nttk.ntl_butterfly(5, 9, 3, 59, c8) == (1, 1)
    assert nttk.harvey_butterfly(100, 4000, 4583, nttk.make_reduction_context(7681, 16)) == (4100, 3662)
    assert nttk.scott_butterfly(5, 9, 3, c8, nttk.make_scott_config(4, c8)) == (14, 3)
    c = nttk.make_reduction_context(13, 8, 0, 2)
    assert nttk.improved_ct_butterfly(3, 20, 5, c) == (13, 6)
    assert nttk.improved_gs_butterfly(5, 9, 5, c, 1) == (14, 11)


@pytest.mark.parametrize("p,n,ell", [(3329, 16, 2), (3329, 32, 7), (8380417, 32, 7), (7681, 32, 4)])
def test_butterflies_random_vs_oracle(oracle, p, n, ell):
    """Every checked butterfly on 20000 random in-range operands vs the oracle cores."""
    rng = np.random.default_rng(p * n + ell)
    c = nttk.make_reduction_context(p, n, 0, ell)
    o = oracle.ctx(p, n, 0, ell)
    m = 20000
    idx = rng.integers(0, m, 400)
    W = rng.integers(1, p, m, dtype=np.uint64)
    if 2 * p < (1 << n):  # ntl
        X, Y = rng.integers(0, p, m, dtype=np.uint64), rng.integers(0, p, m, dtype=np.uint64)
        Wq = np.array([(int(w) << n) // p for w in W], dtype=np.uint64)
        xo, yo = nttk.ntl_butterfly(X, Y, W, Wq, c)
        for i in idx:
            assert (xo[i], yo[i]) == oracle.butterfly("ntl", int(X[i]), int(Y[i]), int(W[i]), int(Wq[i]), c=o)
    if 4 * p < (1 << n):  # harvey
        X, Y = rng.integers(0, 2 * p, m, dtype=np.uint64), rng.integers(0, 2 * p, m, dtype=np.uint64)
        xo, yo = nttk.harvey_butterfly(X, Y, W, c)
        for i in idx:
            assert (xo[i], yo[i]) == oracle.butterfly("harvey", int(X[i]), int(Y[i]), int(W[i]), c=o)
    try:
        cfg = nttk.make_scott_config(256, c)
    except nttk.ContractViolation:
        cfg = None
    if cfg is not None:  # scott
        off = (cfg.transform_size // cfg.lazy_level) * p
        X, Y = rng.integers(0, off, m, dtype=np.uint64), rng.integers(0, off, m, dtype=np.uint64)
        xo, yo = nttk.scott_butterfly(X, Y, W, c, cfg)
        for i in idx:
            assert (xo[i], yo[i]) == oracle.butterfly("scott", int(X[i]), int(Y[i]), int(W[i]), off, c=o)
    if c.fits_lazy_plantard_bound():  # improved CT / GS
        Wh = rng.integers(0, p, m, dtype=np.uint64)
        b = (p << ell) // 2
        X, Y = rng.integers(0, b, m, dtype=np.uint64), rng.integers(0, b, m, dtype=np.uint64)
        xo, yo = nttk.improved_ct_butterfly(X, Y, Wh, c)
        for i in idx:
            assert (xo[i], yo[i]) == oracle.butterfly("improved_ct", int(X[i]), int(Y[i]), int(Wh[i]), c=o)
        for layer in range(1, ell + 1):
            b = p << (layer - 1)
            X, Y = rng.integers(0, b, m, dtype=np.uint64), rng.integers(0, b, m, dtype=np.uint64)
            xo, yo = nttk.improved_gs_butterfly(X, Y, Wh, c, layer)
            for i in idx[:50]:
                assert (xo[i], yo[i]) == oracle.butterfly("improved_gs", int(X[i]), int(Y[i]), b,
                                                          int(Wh[i]), c=o), layer


def test_butterfly_contract_messages():
    c8 = nttk.make_reduction_context(13, 8)
    c = nttk.make_reduction_context(13, 8, 0, 2)
    h = nttk.make_reduction_context(7681, 16)
    for call, msg in ((lambda: nttk.ntl_butterfly(5, 9, 3, 58, c8), "ntl_butterfly: stale W_quot"),
                      (lambda: nttk.ntl_butterfly(13, 9, 3, 59, c8), "inputs must be canonical"),
                      (lambda: nttk.harvey_butterfly(1, 1, 0, h), "harvey_butterfly: W out of (0, p)"),
                      (lambda: nttk.harvey_butterfly(2 * 7681, 1, 3, h), "inputs must be < 2p"),
                      (lambda: nttk.scott_butterfly(52, 0, 3, c8, nttk.make_scott_config(4, c8)),
                       "inputs must be < (N/L)*p"),
                      (lambda: nttk.improved_ct_butterfly(26, 0, 5, c), "inputs must be < 2^ell * p / 2"),
                      (lambda: nttk.improved_gs_butterfly(5, 9, 5, c, 3), "layer out of [1, ell]"),
                      (lambda: nttk.improved_gs_butterfly(13, 9, 5, c, 1), "inputs must be < 2^{layer-1} * p"),
                      (lambda: nttk.make_scott_config(6, c8), "N must be a power of two")):
        with pytest.raises(nttk.ContractViolation, match=__import__("re").escape(msg)):
            call()


def test_canonicalize_on_device():
    """transform.hpp:38-40 through the device mod-p op."""
    v = np.array([0, 7680, 7681, 7682, 2**63 + 5, 2**64 - 1], dtype=np.uint64)
    got = nttk.canonicalize(v, 7681)
    assert got.tolist() == [int(x) % 7681 for x in v.tolist()]


def test_randomized_reduction_contexts(oracle):
    """Random (p, n, alpha, ell), valid or not: context validation accepts/refuses exactly as
    the oracle does, and every admitted op agrees with it on random in-range operands."""
    rng = np.random.default_rng(90)
    for _ in range(60):
        n = int(rng.integers(2, 33))
        p = int(rng.integers(2, min(1 << n, 1 << 31) + 3))
        alpha, ell = int(rng.integers(0, n + 1)), int(rng.integers(0, n + 1))
        try:
            o = oracle.ctx(p, n, alpha, ell)
        except OracleError:
            with pytest.raises(nttk.ContractViolation, match="reduction context"):
                nttk.make_reduction_context(p, n, alpha, ell)
            continue
        c = nttk.make_reduction_context(p, n, alpha, ell)
        m = 2000
        ops = [("mont", lambda: (rng.integers(0, p * p, m, dtype=np.uint64),), nttk.mont_redc,
                oracle.mont_redc, True)]
        if c.fits_signed_montgomery_bound():
            lim = p << (n - 1) >> 1
            ops.append(("smont", lambda: (rng.integers(-lim + 1, lim, m, dtype=np.int64),),
                        nttk.signed_mont_redc, oracle.signed_mont_redc, True))
        if c.fits_plantard_bound():
            ops.append(("plantard", lambda: (rng.integers(0, p + 1, m, dtype=np.uint64),
                                             rng.integers(0, p + 1, m, dtype=np.uint64)),
                        nttk.plantard_redc, oracle.plantard_redc, True))
        if c.fits_lazy_plantard_bound():
            ops.append(("mplantard", lambda: (rng.integers(0, p, m, dtype=np.uint64),
                                              rng.integers(0, p << ell, m, dtype=np.uint64)),
                        nttk.modified_plantard_mul, oracle.modified_plantard_mul, True))
        for name, gen, fn, ref, _ in ops:
            args = gen()
            got = fn(*args, c)
            for i in range(0, m, 97):
                want = ref(*[int(a[i]) for a in args], o)
                assert int(got[i]) == want, (name, p, n, alpha, ell)
