"""Seeded operand grids of BASELINE config 5 (the reduction sweep), shared by the golden
generator (make_sweep_golden.py), the GPU test and bench.py.

2^15 row operands x 2^15 column operands = 2^30 pairs per (q, reduction), drawn with
numpy's PCG64 (stable across machines) from the variant's valid input range (SURVEY
§8(d) config 5, reduction.hpp:125-273), with the boundary values placed first:
  mont_redc              a, b in [0, q)                     (T = a b < q^2)
  signed_mont_redc       a in [0, q), b in [-2^{n-1}, 2^{n-1})  (A = a b inside
                         (-q 2^{n-1}, q 2^{n-1}), reduction.hpp:145-147)
  plantard_redc          W, T in [0, q]                     (reduction.hpp:182)
  modified_plantard_mul  W in [0, q), T in [0, 2^ell q)     (ell = 2 at n = 16, 7 at n = 32)
"""
import numpy as np

CONFIGS = ((3329, 16, 2), (8380417, 32, 7))
NAMES = ("mont_redc", "signed_mont_redc", "plantard_redc", "modified_plantard_mul")
LOG2 = 15


def grid(q: int, n: int, ell: int, variant: int, log2: int = LOG2):
    """(A, B) int64 arrays of 2^log2 operands each for one (q, reduction)."""
    rng = np.random.default_rng(5000 + 10 * variant + (1 if q > (1 << 16) else 0))
    m = 1 << log2
    if variant == 0:
        A, B = rng.integers(0, q, m), rng.integers(0, q, m)
        ea, eb = [0, 1, q - 1, q // 2], [0, 1, q - 1, q // 2 + 1]
    elif variant == 1:
        h = 1 << (n - 1)
        A, B = rng.integers(0, q, m), rng.integers(-h, h, m)
        ea, eb = [0, 1, q - 1, q // 2], [-h, h - 1, 0, -1, 1, -q, q, -(q - 1) * 2]
    elif variant == 2:
        A, B = rng.integers(0, q + 1, m), rng.integers(0, q + 1, m)
        ea, eb = [0, 1, q, q - 1], [0, 1, q, q - 1]
    else:
        top = q << ell
        A, B = rng.integers(0, q, m), rng.integers(0, top, m)
        ea = [0, 1, q - 1, q // 2]
        eb = [0, 1, top - 1, q, q - 1] + [(q << k) - 1 for k in range(1, ell)] + [q << k for k in range(1, ell)]
    A = np.asarray(A, dtype=np.int64)
    B = np.asarray(B, dtype=np.int64)
    A[:len(ea)] = ea
    B[:len(eb)] = eb
    return A, B
