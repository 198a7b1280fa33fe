"""Pins the CPU oracle (oracle/nttk_oracle.c) before it is trusted as the checker.

(a) known-answer values from the reference's own GoogleTest suites
    (proj/tests/reduction_test.cpp, butterfly_test.cpp, params_test.cpp,
    transform_test.cpp, oracle_test.cpp);
(b) golden vectors produced by the unmodified reference (tests/golden/golden.json,
    tests/golden/make_golden.py via oracle/_ref);
(c) when oracle/_ref is present, live cross-checks against the reference itself.
"""
import numpy as np
import pytest

from oracle.oracle import (CYCLIC, HARVEY, IMPROVED, NEGA, NTL, SCOTT, SMONT, OracleError,
                           Reference, reference_available)


# ---- (a) reference known answers ------------------------------------------------

def test_ctx_frozen_toy_constants(oracle):  # reduction_test.cpp:11-25
    c = oracle.ctx(13, 8, 0, 2)
    assert (c.beta, c.beta_mask, c.r2n_mask, c.mu, c.mu_centered) == (256, 255, 65535, 20165, 20165)
    assert (c.p_inv_beta * 13) & 255 == 1 and (c.neg_p_inv_beta * 13 + 1) & 255 == 0
    assert oracle.ctx(17, 5).p_inv_beta == 17


def test_ctx_rejects_bad_parameters(oracle):  # reduction_test.cpp:27-35
    for args in ((12, 8), (1, 8), (13, 1), (13, 33), (17, 4), (13, 8, 8), (13, 8, 0, 8)):
        with pytest.raises(OracleError):
            oracle.ctx(*args)


def test_bound_predicates(oracle):  # reduction_test.cpp:37-46
    L = oracle.lib
    from ctypes import byref
    assert L.or_ctx_fits_plantard(byref(oracle.ctx(13, 8)))
    assert not L.or_ctx_fits_plantard(byref(oracle.ctx(13, 4)))
    assert L.or_ctx_fits_lazy_plantard(byref(oracle.ctx(13, 8, 0, 2)))
    assert not L.or_ctx_fits_lazy_plantard(byref(oracle.ctx(17, 8, 0, 2)))
    assert L.or_ctx_fits_signed_montgomery(byref(oracle.ctx(13, 5)))
    assert not L.or_ctx_fits_signed_montgomery(byref(oracle.ctx(31, 5)))


def test_mont_redc_kat_and_exhaustive(oracle):  # reduction_test.cpp:48-68
    c = oracle.ctx(17, 5)
    assert oracle.mont_redc(100, c) == 1
    inv32 = pow(32, -1, 17)
    for T in range(17 * 17):
        assert oracle.mont_redc(T, c) == T * inv32 % 17
    for k in range(17):
        assert oracle.mont_redc(17 * k, c) == 0
    with pytest.raises(OracleError):
        oracle.mont_redc(17 * 17, c)


def test_signed_mont_redc_kat_and_range(oracle):  # reduction_test.cpp:70-86
    c = oracle.ctx(17, 6)
    assert oracle.signed_mont_redc(100, c) == 9
    assert oracle.signed_mont_redc(-100, c) == -9
    limit = 17 << 5
    inv64 = pow(64, -1, 17)
    for A in range(-limit + 1, limit):
        r = oracle.signed_mont_redc(A, c)
        assert -17 < r < 17 and (r - A * inv64) % 17 == 0
    for A in (limit, -limit):
        with pytest.raises(OracleError):
            oracle.signed_mont_redc(A, c)


def test_plantard_redc_kat_and_exhaustive(oracle):  # reduction_test.cpp:88-106
    c = oracle.ctx(13, 8)
    assert oracle.plantard_redc(5, 12, c) == 6
    before = oracle.lib.or_plantard_fires()
    neg = (-pow(65536, -1, 13)) % 13
    for W in range(14):
        for T in range(14):
            assert oracle.plantard_redc(W, T, c) == W * T * neg % 13
    assert oracle.lib.or_plantard_fires() == before
    with pytest.raises(OracleError):
        oracle.plantard_redc(14, 0, c)


def test_modified_plantard_kat_exhaustive_and_exact_quotient(oracle):  # reduction_test.cpp:153-175
    c = oracle.ctx(13, 8, 0, 2)
    assert oracle.modified_plantard_mul(5, 20, c) == 10
    assert oracle.modified_plantard_mul(1, 1, c) == 4
    neg = (-pow(65536, -1, 13)) % 13
    for W in range(13):
        for T in range(13 * 4):
            r = oracle.modified_plantard_mul(W, T, c)
            assert r == W * T * neg % 13
            h = (W * T * c.mu) & c.r2n_mask
            num = h * 13 - W * T
            assert num % 65536 == 0 and num // 65536 == r
    with pytest.raises(OracleError):
        oracle.modified_plantard_mul(13, 0, c)
    with pytest.raises(OracleError):
        oracle.modified_plantard_mul(0, 52, c)


def test_domain_conversions(oracle):  # reduction_test.cpp:177-190
    c = oracle.ctx(13, 8, 0, 2)
    assert oracle.to_plantard_domain(7, c) == 5
    for w in range(13):
        assert oracle.to_montgomery_domain(w, c) == w * 256 % 13
        assert oracle.to_plantard_domain(w, c) == (13 - w * (65536 % 13) % 13) % 13
        assert oracle.modified_plantard_mul(oracle.to_plantard_domain(w, c), 1, c) == w


def test_butterfly_hand_examples(oracle):  # butterfly_test.cpp:31-197
    assert oracle.butterfly("ntl", 5, 9, 3, 59, c=oracle.ctx(13, 8)) == (1, 1)
    assert oracle.butterfly("harvey", 100, 4000, 4583, c=oracle.ctx(7681, 16)) == (4100, 3662)
    assert oracle.butterfly("scott", 5, 9, 3, 52, c=oracle.ctx(13, 8)) == (14, 3)
    assert oracle.butterfly("improved_ct", 3, 20, 5, c=oracle.ctx(13, 8, 0, 2)) == (13, 6)
    assert oracle.butterfly("improved_gs", 5, 9, 13, 5, c=oracle.ctx(13, 8, 0, 2)) == (14, 11)


def test_scott_lazy_level(oracle):  # butterfly_test.cpp:96-109
    from ctypes import byref
    c = oracle.ctx(13, 8)
    assert oracle.lib.or_scott_lazy_level(4, byref(c)) == 1
    assert oracle.lib.or_scott_lazy_level(256, byref(c)) == 64


def test_primitive_roots(oracle):  # params_test.cpp:10-28
    for (p, N), w in {(17, 4): 4, (13, 4): 5, (7681, 256): 198, (12289, 512): 3,
                      (12289, 1024): 49, (13, 1): 1}.items():
        assert oracle.lib.or_find_primitive_root(p, N) == w


def test_toy13_bundle_and_tables(oracle):  # params_test.cpp:56-69,112-149
    P = oracle.params(13, 4, 8, (NTL, HARVEY, SCOTT, IMPROVED))
    assert (P.omega, P.omega_inv, P.n_inv, P.scott_L) == (5, 8, 10, 1)
    c = oracle.ctx(13, 8, 0, 2)
    assert P.n_inv_hat == oracle.to_plantard_domain(10, c)
    assert list(P.table("dif_w")) == [1, 5, 1]
    assert list(P.table("gs_plain")) == [1, 8, 1]
    P2 = oracle.params(7681, 256, 32, (NTL, HARVEY, SCOTT, IMPROVED))
    assert P2.omega == 198 and len(P2.table("ct_plantard")) == 255 and P2.scott_L == 1


def test_build_params_fault_messages(oracle):  # params_test.cpp:71-110
    with pytest.raises(OracleError, match="p must be prime"):
        oracle.params(15, 4, 8)
    with pytest.raises(OracleError, match="N must divide p - 1"):
        oracle.params(13, 8, 8)
    with pytest.raises(OracleError) as e:
        oracle.params(15, 6, 40)
    assert "p must be prime" in str(e.value) and "power of two" in str(e.value) and "[2, 32]" in str(e.value)
    with pytest.raises(OracleError, match=r"p < 2\^\{n-ell-2\}") as e:
        oracle.params(7681, 256, 16, (IMPROVED,))
    assert "7681" in str(e.value)


def test_dft_hand_case_all_kinds(oracle):  # transform_test.cpp:39-48, oracle_test.cpp:47-52
    kinds = (NTL, HARVEY, SCOTT, IMPROVED)
    P = oracle.params(17, 4, 16, kinds)
    f = np.array([1, 2, 3, 4], dtype=np.uint64)
    assert list(oracle.naive_dft(f, 4, 17)) == [10, 7, 15, 6]
    for k in kinds:
        s = P.forward(k, f)[0]
        nat = [int(s[int(oracle.lib.or_bit_reverse(i, 2))]) % 17 for i in range(4)]
        assert nat == [10, 7, 15, 6]
        assert list(P.inverse(k, s)[0]) == [1, 2, 3, 4]


def test_convolution_hand_case(oracle):  # transform_test.cpp:373-383
    assert list(oracle.schoolbook_cyclic([1, 2, 3, 4], [1, 0, 0, 1], 17)) == [3, 5, 7, 5]
    P = oracle.params(17, 4, 16, (NTL, HARVEY, SCOTT, IMPROVED))
    for k in (NTL, HARVEY, SCOTT, IMPROVED):
        assert list(P.polymul(k, [1, 2, 3, 4], [1, 0, 0, 1])[0]) == [3, 5, 7, 5]


def test_rng_stream(oracle):
    # xoshiro256** values are what make the golden inputs reproducible
    a = oracle.rng(12345, 3329, 8)
    assert all(int(x) < 3329 for x in a)
    if reference_available():
        assert (Reference().rng(12345, 3329, 4096) == oracle.rng(12345, 3329, 4096)).all()


# ---- (b) golden vectors from the reference ------------------------------------------

def test_golden_transforms(oracle, golden):
    for c in golden["cases"]:
        p, N, n, kind = c["p"], c["N"], c["n_bits"], c["kind"]
        f = oracle.rng(c["seed"], p, c["polys"] * N)
        P = oracle.params(p, N, n, (kind,), exact=c["exact_bound"])
        assert P.omega == c["omega"], c["label"]
        fwd = P.forward(kind, f)
        assert "%016x" % oracle.fnv(fwd) == c["fwd_fnv"], c["label"]
        assert [int(v) for v in fwd[0][:16]] == c["fwd_first"], c["label"]
        inv = P.inverse(kind, fwd)
        assert "%016x" % oracle.fnv(inv) == c["inv_fnv"], c["label"]
        g = oracle.rng(c["seed"] + 1, 1 << 15, c["polys"] * N)
        assert "%016x" % oracle.fnv(P.inverse(kind, g)) == c["inv_g_fnv"], c["label"]


def test_golden_products(oracle, golden):
    for c in golden["products"]:
        p, N, n, kind = c["p"], c["N"], c["n_bits"], c["kind"]
        a = oracle.rng(c["seed"], p, 4 * N)
        b = oracle.rng(c["seed"] + 1, p, 4 * N)
        P = oracle.params(p, N, n, (kind,))
        pw = P.pointwise(kind, P.forward(kind, a), P.forward(kind, b))
        assert "%016x" % oracle.fnv(pw) == c["pointwise_fnv"]
        assert "%016x" % oracle.fnv(P.polymul(kind, a, b)) == c["conv_fnv"]


def test_golden_reductions(oracle, golden):
    for c in golden["reductions"]:
        ctx = oracle.ctx(c["p"], c["n_bits"], 0, c["ell"])
        r, s = oracle.sweep(c["variant"], ctx, np.array(c["A"]), np.array(c["B"]))
        assert "%016x" % s == c["checksum"]
        assert [int(x) for x in r[:64]] == c["r_first"]
    assert golden["plantard_fires"] == 0


def test_golden_trees(oracle, golden):
    """Extension trees pinned to reference-run words: the golden rows come from
    the reference's unmodified cores driven on the negacyclic / 7-layer schedules
    (oracle/ref_shim.cpp ref_tree_run); the C restatement must reproduce every word."""
    assert len(golden["trees"]) >= 11
    for c in golden["trees"]:
        p, N, n, kind, L, tree = c["p"], c["N"], c["n_bits"], c["kind"], c["layers"], c["tree"]
        P = oracle.params(p, N, n, (kind,), tree=tree, layers=L, exact=True)
        f = oracle.rng(c["seed"], p, c["polys"] * N).reshape(c["polys"], N)
        fwd = P.forward(kind, f)
        assert "%016x" % oracle.fnv(fwd) == c["fwd_fnv"], c["label"]
        got0 = fwd[0].astype(np.int64) if kind == SMONT else fwd[0]
        assert [int(v) for v in got0] == c["fwd_poly0"], c["label"]
        g = oracle.rng(c["seed"] + 1, 1 << 15, c["polys"] * N).reshape(c["polys"], N)
        if kind == SMONT:
            g = (g.astype(np.int64) - (1 << 14)).astype(np.uint64)
        assert "%016x" % oracle.fnv(P.inverse(kind, g)) == c["inv_g_fnv"], c["label"]
        if "polymul_fnv" in c:
            h = oracle.rng(c["seed"] + 2, p, c["polys"] * N).reshape(c["polys"], N)
            pm = P.polymul(kind, f, h)
            assert "%016x" % oracle.fnv(pm) == c["polymul_fnv"], c["label"]
            assert (pm[0] == oracle.schoolbook_negacyclic(f[0], h[0], p)).all()


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("p,N,n,L", [(3329, 256, 16, 7), (3329, 256, 32, 7), (8380417, 256, 32, 8),
                                     (12289, 1024, 32, 9), (17, 8, 16, 2)])
def test_live_trees_against_reference_cores(oracle, p, N, n, L):
    """Live cross-check of the restated extension trees against the reference's own cores
    on fresh seeds (forward words, inverse of arbitrary words, polymul)."""
    ref = Reference()
    for kind in (IMPROVED, HARVEY, SMONT):
        P = oracle.params(p, N, n, (kind,), tree=NEGA, layers=L, exact=True)
        f = oracle.rng(9000 + kind, p, 4 * N).reshape(4, N)
        fwd = P.forward(kind, f)
        assert (fwd == ref.tree(p, N, n, NEGA, L, kind, 0, f)).all(), (p, kind)
        g = oracle.rng(9100 + kind, min(1 << 15, 8 * p), 4 * N).reshape(4, N)
        assert (P.inverse(kind, g) == ref.tree(p, N, n, NEGA, L, kind, 1, g)).all(), (p, kind)
        if (N >> L) == 2:
            h = oracle.rng(9200 + kind, p, 4 * N).reshape(4, N)
            assert (P.polymul(kind, f, h) == ref.tree(p, N, n, NEGA, L, kind, 2, f, h)).all()


# ---- extension rows: also checked against naive evaluation ---------------------------

@pytest.mark.parametrize("p,N,n,L,root", [(3329, 256, 16, 7, 0), (8380417, 256, 32, 8, 0),
                                          (3329, 256, 32, 7, 0), (17, 8, 16, 2, 0)])
def test_negacyclic_trees_against_naive(oracle, p, N, n, L, root):
    kinds = (IMPROVED, HARVEY, SMONT)
    P = oracle.params(p, N, n, kinds, tree=NEGA, layers=L, root=root, exact=True)
    for seed in range(3):
        a = oracle.rng(100 + seed, p, N)
        b = oracle.rng(200 + seed, p, N)
        ev = P.naive_eval(a)
        want = oracle.schoolbook_negacyclic(a, b, p)
        for k in kinds:
            fa = P.forward(k, a)
            assert ((fa.astype(np.int64) % p).astype(np.uint64).ravel() == ev).all()
            assert (P.inverse(k, fa).ravel() == a).all()
            assert (P.polymul(k, a, b).ravel() == want).all()


def test_dilithium_root_is_the_standard_one(oracle):
    assert oracle.lib.or_find_primitive_root(8380417, 512) == 1753
    assert oracle.lib.or_find_primitive_root(3329, 256) == 17


# ---- (c) live cross-check with the reference when oracle/_ref is built -------------

@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_live_against_reference(oracle):
    ref = Reference()
    for p, N, n, kinds in ((7681, 256, 32, (NTL, HARVEY, SCOTT, IMPROVED)),
                           (12289, 1024, 32, (NTL, HARVEY, SCOTT, IMPROVED)),
                           (8380417, 256, 32, (NTL, HARVEY, SCOTT)),
                           (3329, 256, 16, (NTL, HARVEY))):
        f = oracle.rng(4242, p, 3 * N)
        P = oracle.params(p, N, n, kinds)
        R = ref.params(p, N, n, kinds)
        for k in kinds:
            a, b = P.forward(k, f), R.forward(k, f)
            assert (a == b).all()
            assert (P.inverse(k, a) == R.inverse(k, b)).all()


def test_reference_self_verification_suites():
    """The unmodified reference's own property suites (verify.hpp run_all_suites) pass
    when built here: the checker behind the golden vectors verifies itself first."""
    from oracle.oracle import Reference, reference_available

    if not reference_available():
        pytest.skip("oracle/_ref not built (no /root/reference on this host)")
    rows, failures = Reference().run_all_suites(100000)
    names = {n for n, _, _ in rows}
    assert {"montgomery", "signed-montgomery", "plantard", "modified-plantard", "butterflies",
            "transform"} <= names
    assert failures == 0, rows
    assert all(c > 0 for _, c, _ in rows)


def test_sweep_full_grid_checksums_match_reference(oracle):
    """BASELINE config 5 at its stated size: the restated reductions over every 2^30-pair
    grid of tests/golden/sweep_inputs.py reproduce the reference's checksums
    (tests/golden/sweep_2p30.json, generated by the reference's checked reductions)."""
    import json
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from sweep_inputs import grid

    with open(os.path.join(os.path.dirname(__file__), "golden", "sweep_2p30.json")) as fh:
        rows = json.load(fh)["rows"]
    assert len(rows) == 8
    threads = max(1, len(os.sched_getaffinity(0)))
    for row in rows:
        A, B = grid(row["q"], row["n_bits"], row["ell"], row["variant"])
        assert A.size * B.size == row["pairs"] == 1 << 30
        ctx = oracle.ctx(row["q"], row["n_bits"], 0, row["ell"])
        _, s = oracle.sweep(row["variant"], ctx, A, B, want_results=False, threads=threads)
        assert "%016x" % s == row["checksum"], row


def _f1_schedule_model(a, ct, p, S, w1_layer2=True):
    """Integer model of the F1 forwards (tma_common.cuh fwd_body_f1 at N = 256 with the layer-2
    W1 block, fastn_tma.cu fwd_body_n_f1 at N = 512 / 1024 without it): surplus S p injected
    by layer 1 (twiddle 1), paper-form Y' = X - r on layers 2..L-1, the last layer subtracts
    sigma p; asserts every F1 X input keeps a surplus >= 1 and every product operand lies
    inside Prop. 4's n = 16 range."""
    a = [int(v) for v in a]
    N = len(a)
    L = N.bit_length() - 1
    lim = (1 << 16) * ((1 << 16) - p)
    for s in range(1, L + 1):
        span = N >> s
        for i in range(N):
            if i & span:
                continue
            x, y, blk = a[i], a[i + span], i >> (L + 1 - s)
            if s == 1:
                a[i], a[i + span] = x + y + S * p, x + (S + 1) * p - y
                continue
            if w1_layer2 and s == 2 and blk == 0:
                c = y - S * p
                c = c - p if c >= p else c
                a[i], a[i + span] = x + c, x + p - c
                continue
            w = int(ct[(1 << (s - 1)) - 1 + blk])
            assert w * y < lim
            r = w * y % p
            if s < L:
                assert x - r >= 0
                a[i], a[i + span] = x + r, x - r
            else:
                b = lambda k: (i >> k) & 1  # noqa: E731
                spent = sum(b(k) for k in range(1, L - 1))
                if w1_layer2:  # the layer-2 W1 block (bit L-1 = 0) spends nothing
                    spent -= b(L - 2) * (1 - b(L - 1))
                sig = S - spent
                a[i], a[i + span] = x + r - sig * p, x + p - r - sig * p
    return a


def _f1_nega7_model(a, ct, p):
    """Integer model of tma_common.cuh fwd_body_f1_nega7 (Kyber, 7-layer negacyclic tree, N = 256):
    layer 1 multiplies and injects the surplus S = 5, layers 2..6 run Y' = X - r, layer 7 removes
    sigma = S - popcount(i6..i2); asserts every F-layer X input keeps a surplus >= 1 (no
    underflow) and every product operand lies inside Prop. 4's n = 16 range."""
    a = [int(v) for v in a]
    N, L, S = 256, 7, 5
    lim = (1 << 16) * ((1 << 16) - p)
    for s in range(1, L + 1):
        span = N >> s
        for i in range(N):
            if i & span:
                continue
            x, y, blk = a[i], a[i + span], i >> (9 - s)
            w = int(ct[(1 << (s - 1)) - 1 + blk])
            assert w * y < lim
            r = w * y % p
            if s == 1:
                a[i], a[i + span] = x + r + S * p, x + (S + 1) * p - r
            elif s < L:
                assert x - r >= 0
                a[i], a[i + span] = x + r, x - r
            else:
                sig = S - sum((i >> k) & 1 for k in range(2, 7))
                assert sig >= 0
                a[i], a[i + span] = x + r - sig * p, x + p - r - sig * p
    return a


def test_f1_forward_schedule_nega7(oracle):
    """The F1 forward of the 7-layer negacyclic Kyber tree (fwd_body_f1_nega7) reproduces the
    words of the reference's cores driven on that schedule (row a22: the oracle's tree forward is
    pinned to reference-run words), on extreme and random canonical inputs."""
    p = 3329
    Q = oracle.params(p, 256, 16, (IMPROVED,), tree=NEGA, layers=7, exact=True)
    ct = Q.table("ct_plain")
    rs = np.random.RandomState(21)
    rows = [np.full(256, p - 1), np.zeros(256, dtype=np.int64), np.where(np.arange(256) % 2 == 0, p - 1, 0),
            np.where(np.arange(256) < 128, p - 1, 0), np.where(np.arange(256) < 128, 0, p - 1),
            rs.randint(0, p, 256), rs.randint(0, p, 256)]
    want = Q.forward(IMPROVED, np.stack(rows).astype(np.uint64))
    for k, row in enumerate(rows):
        assert _f1_nega7_model(row, ct, p) == [int(v) for v in want[k]]


@pytest.mark.parametrize("p", [3329, 7681])
def test_f1_forward_schedule_matches_reference_loop(oracle, p):
    """The surplus bookkeeping of the F1 forward (kF1Surplus = 6) reproduces the reference's
    lazy forward words (butterfly.hpp:224-230 driven by transform.hpp:77-96) on extreme and
    random inputs -- the CPU proof of the schedule the GPU kernel runs."""
    Q = oracle.params(p, 256, 16 if p == 3329 else 32, (IMPROVED,), exact=p == 3329)
    ct = Q.table("ct_plain")
    rows = [np.full(256, p - 1), np.zeros(256, dtype=np.int64), oracle.rng(5, p, 256),
            oracle.rng(6, p, 256), np.where(np.arange(256) % 3 == 0, p - 1, 0)]
    want = Q.forward(IMPROVED, np.stack(rows))
    for k, row in enumerate(rows):
        assert _f1_schedule_model(row, ct, p, 6) == [int(v) for v in want[k]]


@pytest.mark.parametrize("N", [512, 1024])
def test_f1_forward_schedule_n512_1024(oracle, N):
    """The N = 512 / 1024 F1 forward (fastn_tma.cu fwd_body_n_f1, surplus L - 2) reproduces the
    reference's lazy forward words at the paper's Table 2 modulus."""
    p = 12289
    Q = oracle.params(p, N, 32, (IMPROVED,))
    ct = Q.table("ct_plain")
    L = N.bit_length() - 1
    rows = [np.full(N, p - 1), oracle.rng(7, p, N), np.where(np.arange(N) % 2 == 0, p - 1, 0)]
    want = Q.forward(IMPROVED, np.stack(rows))
    for k, row in enumerate(rows):
        assert _f1_schedule_model(row, ct, p, L - 2, w1_layer2=False) == [int(v) for v in want[k]]


def _ct_inverse_model(F, p, omega, in_hi=65535):
    """Integer model of tma_common.cuh inv_body_ct (Kyber N = 256): radix-2 DIT on the
    bit-reversed spectrum with omega^{-1}, raw words in, the multiply-free jb = 0 butterflies of
    len 1..8 adding per-layer offsets chosen as params.cpp fill_ct_inverse chooses them (interval
    propagation, worst case merged at the transpose), F3 products elsewhere, N^{-1} folded into
    the last layer.  Asserts the bounds the host validates."""
    N = 256
    lim = (1 << 16) * ((1 << 16) - p)
    neg = in_hi != 65535  # the canonical-input image may subtract multiples of p as well
    rup = lambda x: (-((-x) // p) * p if neg else 0) if x <= 0 else (x + p - 1) // p * p  # noqa: E731
    oi = pow(omega, p - 2, p)
    ninv = pow(N, p - 2, p)
    lo, hi = [0] * 16, [in_hi] * 16
    consts = []
    for li, fl in enumerate((6 * p, 5 * p, 4 * p, 3 * p)):
        ln = 1 << li
        free = [r for r in range(16) if not r & ln and r & (ln - 1) == 0]
        c1 = max(rup(fl - lo[r] - lo[r + ln]) for r in free)
        c2 = max(rup(fl - lo[r] + hi[r + ln]) for r in free)
        consts.append((c1, c2))
        nlo, nhi = lo[:], hi[:]
        for r in range(16):
            if r & ln:
                continue
            if r & (ln - 1) == 0:
                nlo[r], nhi[r] = lo[r] + lo[r + ln] + c1, hi[r] + hi[r + ln] + c1
                nlo[r + ln], nhi[r + ln] = lo[r] - hi[r + ln] + c2, hi[r] - lo[r + ln] + c2
            else:
                nlo[r], nhi[r] = lo[r], hi[r] + p - 1
                nlo[r + ln], nhi[r + ln] = lo[r] - p + 1, hi[r]
        lo, hi = nlo, nhi
    if in_hi == p - 1:  # the unpacked variant canonicalises its input words first
        F = [int(x) % p for x in F]
    v = [[int(F[16 * j + r]) for r in range(16)] for j in range(16)]
    for a in v:  # contiguous phase: position 16 j + r
        for li in range(4):
            ln = 1 << li
            c1, c2 = consts[li]
            for r in range(16):
                if r & ln:
                    continue
                jb = r & (ln - 1)
                u, x = a[r], a[r + ln]
                if jb == 0:
                    a[r], a[r + ln] = u + x + c1, u - x + c2
                else:
                    assert x * (p - 1) < lim
                    rr = x * pow(oi, (128 // ln) * jb, p) % p
                    assert u - rr >= 0
                    a[r], a[r + ln] = u + rr, u - rr
    pos = {16 * j + r: v[j][r] for j in range(16) for r in range(16)}
    out = [0] * N
    for j in range(16):  # strided phase: position j + 16 r
        a = [pos[j + 16 * r] for r in range(16)]
        for h in (1, 2, 4):
            for r in range(16):
                if r & h:
                    continue
                u, x = a[r], a[r + h]
                assert x * (p - 1) < lim
                rr = x * pow(oi, (8 // h) * (j + 16 * (r % h)), p) % p
                assert u - rr >= 0
                a[r], a[r + h] = u + rr, u - rr
        for r in range(8):
            assert a[r] * (p - 1) < lim and a[r + 8] * (p - 1) < lim
            A = a[r] * ninv % p
            B = a[r + 8] * (ninv * pow(oi, j + 16 * r, p) % p) % p
            out[j + 16 * r], out[j + 16 * (r + 8)] = (A + B) % p, (A - B) % p
    return out


def _ct_inverse_model32(F, p, omega):
    """Integer model of tma_common.cuh inv_body_ct32 (Dilithium, n = 32): inputs partially reduced
    to [0, 2p) by the shift reduction, umulhi-form CT butterflies (X + r, X + p - r) on the DIT
    schedule of _ct_inverse_model, the multiply-free jb = 0 butterflies adding the multiple of p
    that params.cpp fill_ct_inverse32 picks (>= their Y input), N^{-1} folded.  Asserts that
    every word stays below 2^32 and non-negative."""
    N = 256
    s = p.bit_length()  # 2^s >= p: v - (v >> s) p lies in [0, 2p) for every 32-bit v
    oi, ninv = pow(omega, p - 2, p), pow(N, p - 2, p)
    rup = lambda x: (x + p - 1) // p * p  # noqa: E731
    hi = [2 * p - 1] * 16
    consts = []
    for li in range(4):
        ln = 1 << li
        c2 = max(rup(hi[r + ln]) for r in range(16) if not r & ln and r & (ln - 1) == 0)
        consts.append(c2)
        nhi = hi[:]
        for r in range(16):
            if r & ln:
                continue
            if r & (ln - 1) == 0:
                nhi[r], nhi[r + ln] = hi[r] + hi[r + ln], hi[r] + c2
            else:
                nhi[r], nhi[r + ln] = hi[r] + p - 1, hi[r] + p
        hi = nhi
    assert max(hi) + 3 * p < 1 << 32
    red = [int(x) - (int(x) >> s) * p for x in F]
    assert all(0 <= x < 2 * p for x in red)
    v = [[red[16 * j + r] for r in range(16)] for j in range(16)]
    for a in v:
        for li in range(4):
            ln = 1 << li
            for r in range(16):
                if r & ln:
                    continue
                jb = r & (ln - 1)
                u, x = a[r], a[r + ln]
                if jb == 0:
                    assert consts[li] >= x
                    a[r], a[r + ln] = u + x, u + consts[li] - x
                else:
                    rr = x * pow(oi, (128 // ln) * jb, p) % p
                    a[r], a[r + ln] = u + rr, u + p - rr
                assert 0 <= a[r] < 1 << 32 and 0 <= a[r + ln] < 1 << 32
    pos = {16 * j + r: v[j][r] for j in range(16) for r in range(16)}
    out = [0] * N
    for j in range(16):
        a = [pos[j + 16 * r] for r in range(16)]
        for h in (1, 2, 4):
            for r in range(16):
                if r & h:
                    continue
                rr = a[r + h] * pow(oi, (8 // h) * (j + 16 * (r % h)), p) % p
                a[r], a[r + h] = a[r] + rr, a[r] + p - rr
                assert a[r] < 1 << 32 and a[r + h] < 1 << 32
        for r in range(8):
            A = a[r] * ninv % p
            B = a[r + 8] * (ninv * pow(oi, j + 16 * r, p) % p) % p
            out[j + 16 * r], out[j + 16 * (r + 8)] = (A + B) % p, (A - B) % p
    return out


def test_ct_inverse_schedule32_matches_reference(oracle):
    """The CT-form Dilithium inverse (tma_common.cuh inv_body_ct32) gives the reference's
    canonical inverse (transform.hpp:233-343) on arbitrary 32-bit words."""
    p = 8380417
    Q = oracle.params(p, 256, 32, (IMPROVED,), exact=True)
    rs = np.random.RandomState(9)
    rows = [np.full(256, (1 << 32) - 1), np.zeros(256, dtype=np.int64),
            np.where(np.arange(256) % 2 == 0, (1 << 32) - 1, 0), rs.randint(0, 1 << 32, 256),
            rs.randint(0, p, 256)]
    want = Q.inverse(IMPROVED, np.stack(rows).astype(np.uint64))
    for k, row in enumerate(rows):
        assert _ct_inverse_model32(row, p, Q.omega) == [int(v) for v in want[k]]


def _ct_inverse_model_n(F, p, omega, N):
    """Integer model of fastn_tma.cu inv_body_n_ct (N = 512 / 1024, narrow image): canonical
    input, compile-time interval schedule in units of p (floors rq, offsets m p, canon1 when a
    multiply-free input is wider than kT p), F-form products, N^{-1} folded.  Asserts every bound
    the schedule promises with the actual values, and Prop. 4's n = 16 range below kCtLimN p."""
    G, FS = N // 32, (4 if N == 1024 else 3)
    H0 = 1 if N == 1024 else 2
    kT, LIM = (1, 2, 4, 1, 2), 20
    lim = (1 << 16) * ((1 << 16) - p)
    assert (p - 1) * (LIM * p - 1) < lim
    oi, ninv = pow(omega, p - 2, p), pow(N, p - 2, p)
    rq = [[0] * 32 for _ in range(6)]
    rq[5] = [FS] * 32
    for li in range(4, -1, -1):
        ln = 1 << li
        for k in range(32):
            if k & ln or k & (ln - 1) == 0:
                continue
            rq[li][k] = max(rq[li + 1][k], rq[li + 1][k + ln] + 1)
    ncanon = 0
    pos = {}
    for j in range(N // 32):  # contiguous phase: position 32 j + k
        v = [int(F[32 * j + k]) % p for k in range(32)]
        lo, hi = [0] * 32, [1] * 32
        for li in range(5):
            ln = 1 << li
            for k in range(32):
                if k & ln:
                    continue
                m, jb = k + ln, k & (ln - 1)
                if jb == 0:
                    for r in (k, m):
                        if hi[r] - lo[r] > kT[li]:
                            assert v[r] < LIM * p
                            v[r], lo[r], hi[r] = v[r] % p, 0, 1
                            ncanon += j == 0
                    c1 = max(0, rq[li + 1][k] - (lo[k] + lo[m]))
                    c2 = max(0, rq[li + 1][m] - (lo[k] - hi[m]))
                    assert c1 < 12 and c2 < 12
                    u, w = v[k], v[m]
                    v[k], v[m] = u + w + c1 * p, u - w + c2 * p
                    lo[k], hi[k], lo[m], hi[m] = (lo[k] + lo[m] + c1, hi[k] + hi[m] + c1,
                                                  lo[k] - hi[m] + c2, hi[k] - lo[m] + c2)
                else:
                    assert v[m] < LIM * p and lo[k] >= rq[li][k] >= 1
                    rr = v[m] * pow(oi, (N // (2 * ln)) * jb, p) % p
                    v[k], v[m] = v[k] + rr, v[k] - rr
                    lo[m], hi[m], hi[k] = lo[k] - 1, hi[k], hi[k] + 1
                for r in (k, m):
                    assert lo[r] * p <= v[r] < hi[r] * p and lo[r] >= rq[li + 1][r]
        assert min(lo) >= FS and max(hi) + FS <= LIM
        for k in range(32):
            pos[32 * j + k] = v[k]
    assert ncanon == 4
    out = [0] * N
    for j in range(G):  # strided phase: position j + G k
        a = [pos[j + G * k] for k in range(32)]
        h = H0
        while h <= 8:
            for k in range(32):
                if k & h:
                    continue
                assert a[k + h] * (p - 1) < lim
                rr = a[k + h] * pow(oi, (16 // h) * (j + G * (k % h)), p) % p
                assert a[k] - rr >= 0
                a[k], a[k + h] = a[k] + rr, a[k] - rr
            h *= 2
        for k in range(16):
            assert a[k] < LIM * p and a[k + 16] < LIM * p
            A = a[k] * ninv % p
            B = a[k + 16] * (ninv * pow(oi, j + G * k, p) % p) % p
            out[j + G * k], out[j + G * (k + 16)] = (A + B) % p, (A - B) % p
    return out


@pytest.mark.parametrize("N", [512, 1024])
def test_ct_inverse_schedule_n_matches_reference(oracle, N):
    """The CT-form narrow inverse at N = 512 / 1024 (fastn_tma.cu inv_body_n_ct) gives the
    reference's canonical inverse (transform.hpp:233-343) for the Table 2 modulus: extreme,
    alternating and random canonical spectra (the kernel canonicalises raw words first)."""
    p = 12289
    Q = oracle.params(p, N, 32, (IMPROVED,))
    rs = np.random.RandomState(11)
    rows = [np.full(N, p - 1), np.zeros(N, dtype=np.int64), np.where(np.arange(N) % 2 == 0, p - 1, 0),
            np.where(np.arange(N) % 2 == 1, p - 1, 0), rs.randint(0, p, N), rs.randint(0, 1 << 32, N)]
    want = Q.inverse(IMPROVED, np.stack(rows).astype(np.uint64))
    for k, row in enumerate(rows):
        assert _ct_inverse_model_n(row, p, Q.omega, N) == [int(v) for v in want[k]]


def test_ct_inverse_schedule_matches_reference(oracle):
    """The CT-form Kyber inverse (tma_common.cuh inv_body_ct) gives the reference's canonical
    inverse (transform.hpp:233-343) on raw u16 words: all-max, all-zero, alternating, random."""
    p = 3329
    Q = oracle.params(p, 256, 16, (IMPROVED,), exact=True)
    rs = np.random.RandomState(5)
    rows = [np.full(256, 65535), np.zeros(256, dtype=np.int64),
            np.where(np.arange(256) % 2 == 0, 65535, 0), rs.randint(0, 65536, 256),
            rs.randint(0, p, 256)]
    want = Q.inverse(IMPROVED, np.stack(rows).astype(np.uint64))
    for k, row in enumerate(rows):
        assert _ct_inverse_model(row, p, Q.omega) == [int(v) for v in want[k]]
