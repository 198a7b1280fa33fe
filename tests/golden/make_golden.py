"""Generate golden vectors by running the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The reference is the header-only nttk library compiled by oracle/Makefile; this script
only calls it through oracle/_ref/libnttk_ref.so.  Output: tests/golden/golden.json.
Inputs come from the reference's own Rng (int_util.hpp:90-138), seed 12345 unless
stated, drawn poly-major like bench.hpp:201-205.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import HARVEY, IMPROVED, NTL, SCOTT, Reference, Oracle  # noqa: E402

ref = Reference()
orc = Oracle()  # only for the FNV helper (pure hashing)


def fnv(a):
    return "%016x" % orc.fnv(np.asarray(a, dtype=np.uint64).ravel())


out = {"generator": "tests/golden/make_golden.py via oracle/_ref/libnttk_ref.so", "cases": []}

# SURVEY Appendix A + reference presets, every kind the reference builds there
CASES = [
    # (label, p, N, n, kind, exact, polys, seed)
    ("kyber_q3329_n32_improved", 3329, 256, 32, IMPROVED, False, 16, 12345),
    ("kyber_q3329_n16_harvey", 3329, 256, 16, HARVEY, False, 16, 12345),
    ("kyber_q3329_n16_ntl", 3329, 256, 16, NTL, False, 16, 12345),
    ("kyber_q3329_n32_scott", 3329, 256, 32, SCOTT, False, 16, 12345),
    ("kyber_q3329_n32_harvey", 3329, 256, 32, HARVEY, False, 16, 12345),
    ("dilithium_q8380417_n32_harvey", 8380417, 256, 32, HARVEY, False, 16, 12345),
    ("dilithium_q8380417_n32_ntl", 8380417, 256, 32, NTL, False, 16, 12345),
    ("dilithium_q8380417_n32_scott", 8380417, 256, 32, SCOTT, False, 16, 12345),
    ("dilithium_q8380417_n32_improved_exact", 8380417, 256, 32, IMPROVED, True, 16, 12345),
    ("kyber_q3329_n16_improved_exact", 3329, 256, 16, IMPROVED, True, 16, 12345),
]
for kind in (NTL, HARVEY, SCOTT, IMPROVED):
    CASES.append((f"kyber256_preset_k{kind}", 7681, 256, 32, kind, False, 4, 99))
    CASES.append((f"falcon512_preset_k{kind}", 12289, 512, 32, kind, False, 2, 21))
    CASES.append((f"falcon1024_preset_k{kind}", 12289, 1024, 32, kind, False, 2, 404))
    CASES.append((f"toy13_preset_k{kind}", 13, 4, 8, kind, False, 8, 7))
    CASES.append((f"p17_N4_n16_k{kind}", 17, 4, 16, kind, False, 8, 5))

for label, p, N, n, kind, exact, polys, seed in CASES:
    f = ref.rng(seed, p, polys * N).reshape(polys, N)
    P = ref.params(p, N, n, (kind,), exact=exact)
    fwd = P.forward(kind, f)
    inv = P.inverse(kind, fwd)
    assert (inv == f).all(), label
    # inverse of an arbitrary (non-spectrum) in-range word: canonicalisation path
    g = ref.rng(seed + 1, 1 << 15, polys * N).reshape(polys, N)
    inv_g = P.inverse(kind, g)
    out["cases"].append({
        "label": label, "p": p, "N": N, "n_bits": n, "kind": kind, "exact_bound": exact,
        "polys": polys, "seed": seed, "omega": P.scalars()["omega"],
        "fwd_fnv": fnv(fwd), "inv_fnv": fnv(inv), "inv_g_fnv": fnv(inv_g),
        "fwd_first": [int(v) for v in fwd[0][:16]],
        "fwd_poly0": [int(v) for v in fwd[0]] if N <= 256 else None,
        "inv_g_poly0": [int(v) for v in inv_g[0]] if N <= 256 else None,
    })

# pointwise (transform.hpp:349-370) and convolution (transform.hpp:372-379)
prod = []
for p, N, n, kinds, seed in ((7681, 256, 32, (NTL, HARVEY, SCOTT, IMPROVED), 31337),
                             (3329, 256, 16, (NTL, HARVEY), 31338),
                             (13, 4, 8, (NTL, HARVEY, SCOTT, IMPROVED), 31339)):
    a = ref.rng(seed, p, 4 * N).reshape(4, N)
    b = ref.rng(seed + 1, p, 4 * N).reshape(4, N)
    for kind in kinds:
        P = ref.params(p, N, n, (kind,))
        fa, fb = P.forward(kind, a), P.forward(kind, b)
        pw = P.pointwise(kind, fa, fb)
        cv = P.convolution(kind, a, b)
        prod.append({"p": p, "N": N, "n_bits": n, "kind": kind, "seed": seed,
                     "pointwise_fnv": fnv(pw), "conv_fnv": fnv(cv),
                     "conv_first": [int(v) for v in cv[0][:16]]})
out["products"] = prod

# extension trees: the reference's unmodified cores driven on the
# negacyclic / 7-layer schedules (oracle/ref_shim.cpp ref_tree_run) -- the Kyber 7-layer
# forward, degree-2 basemul polymul, the Dilithium 8-layer negacyclic tree and the
# signed-Montgomery transform, at the storage words the GPU keeps (u16 Kyber, u32 Dilithium)
from oracle.oracle import CYCLIC, NEGA, SMONT  # noqa: E402

trees = []
TREES = [
    # (label, p, N, n, tree, layers, polys, seed)
    ("kyber_nega7_n16", 3329, 256, 16, NEGA, 7, 16, 4242),
    ("kyber_nega7_n32", 3329, 256, 32, NEGA, 7, 8, 4243),
    ("dilithium_nega8_n32", 8380417, 256, 32, NEGA, 8, 16, 4244),
    ("kyber_cyclic8_n16", 3329, 256, 16, CYCLIC, 8, 8, 4245),
    ("dilithium_cyclic8_n32", 8380417, 256, 32, CYCLIC, 8, 8, 4246),
]
for label, p, N, n, tree, L, polys, seed in TREES:
    f = ref.rng(seed, p, polys * N).reshape(polys, N)
    g = ref.rng(seed + 1, 1 << 15, polys * N).reshape(polys, N)  # arbitrary inverse input
    h = ref.rng(seed + 2, p, polys * N).reshape(polys, N)
    for kind in ((IMPROVED, HARVEY, SMONT) if tree == NEGA else (SMONT,)):
        fwd = ref.tree(p, N, n, tree, L, kind, 0, f)
        inv = ref.tree(p, N, n, tree, L, kind, 1, fwd)
        assert (inv == f).all(), (label, kind)
        gi = g.astype(np.int64) - (1 << 14) if kind == SMONT else g  # signed words for smont
        inv_g = ref.tree(p, N, n, tree, L, kind, 1, gi)
        row = {"label": label, "p": p, "N": N, "n_bits": n, "tree": tree, "layers": L,
               "kind": kind, "polys": polys, "seed": seed,
               "fwd_fnv": fnv(fwd), "inv_g_fnv": fnv(inv_g),
               "fwd_poly0": [int(np.int64(v)) if kind == SMONT else int(v) for v in fwd[0]],
               "inv_g_poly0": [int(v) for v in inv_g[0]]}
        if (N >> L) == 2:
            pm = ref.tree(p, N, n, tree, L, kind, 2, f, h)
            row["polymul_fnv"] = fnv(pm)
            row["polymul_poly0"] = [int(v) for v in pm[0]]
        trees.append(row)
out["trees"] = trees

# reductions over operand grids incl. boundary values (reduction.hpp:125-273)
def grid(p, n, variant, ell):
    rng_a = ref.rng(777 + variant, 1 << 62, 64)
    rng_b = ref.rng(888 + variant, 1 << 62, 64)
    if variant == 0:      # mont: a, b in [0, p)
        A = rng_a % p; B = rng_b % p
        edge = [0, 1, p - 1]
        A[:3] = edge; B[:3] = edge
    elif variant == 1:    # signed mont: a in [0, p), b in [-2^{n-1}, 2^{n-1})
        A = (rng_a % p).astype(np.int64)
        B = (rng_b % (1 << n)).astype(np.int64) - (1 << (n - 1))
        A[:3] = [0, 1, p - 1]; B[:4] = [-(1 << (n - 1)), (1 << (n - 1)) - 1, 0, -1]
    elif variant == 2:    # plantard: W, T in [0, p]
        A = rng_a % (p + 1); B = rng_b % (p + 1)
        A[:3] = [0, 1, p]; B[:3] = [0, 1, p]
    else:                 # modified plantard: W in [0, p), T in [0, 2^ell p)
        A = rng_a % p; B = rng_b % (p << ell)
        A[:3] = [0, 1, p - 1]; B[:4] = [0, 1, (p << ell) - 1, p]
    return np.asarray(A, dtype=np.int64), np.asarray(B, dtype=np.int64)


red = []
for p, n, ell in ((3329, 16, 2), (8380417, 32, 7)):
    for variant in range(4):
        A, B = grid(p, n, variant, ell)
        r, s = ref.sweep(variant, p, n, ell, A, B)
        red.append({"p": p, "n_bits": n, "ell": ell, "variant": variant,
                    "A": [int(x) for x in A], "B": [int(x) for x in B],
                    "checksum": "%016x" % s, "r_first": [int(x) for x in r[:64]]})
out["reductions"] = red
out["plantard_fires"] = int(ref.lib.ref_plantard_fires())

path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
with open(path, "w") as fh:
    json.dump(out, fh, indent=0)
print("wrote", path, len(out["cases"]), "cases")
