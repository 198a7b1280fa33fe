"""Checksums of BASELINE config 5 at its full size, computed by the UNMODIFIED reference.

For every (q, reduction) the reference's checked entry points (reduction.hpp:125-273,
through oracle/ref_shim.cpp ref_sweep) run over the whole 2^15 x 2^15 = 2^30 operand grid
of tests/golden/sweep_inputs.py; the wrapping u64 sum of the results is the checksum the
GPU sweep must reproduce (tests/test_gpu_parity.py, bench.py config 5).  Run here:
    python tests/golden/make_sweep_golden.py      (about a minute on 8 host threads)
Output: tests/golden/sweep_2p30.json.
"""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
from oracle.oracle import Reference  # noqa: E402
from sweep_inputs import CONFIGS, LOG2, NAMES, grid  # noqa: E402


def main():
    ref = Reference()
    threads = max(1, len(os.sched_getaffinity(0)))
    rows = []
    t0 = time.time()
    for q, n, ell in CONFIGS:
        for v in range(4):
            A, B = grid(q, n, ell, v)
            chunks = np.array_split(A, threads * 4)
            with ThreadPoolExecutor(threads) as ex:
                sums = list(ex.map(lambda a: ref.sweep_checksum(v, q, n, ell, a, B), chunks))
            s = sum(sums) % (1 << 64)
            rows.append({"q": q, "n_bits": n, "ell": ell, "variant": v, "name": NAMES[v],
                         "pairs": int(A.size) * int(B.size), "checksum": "%016x" % s})
            print(q, NAMES[v], "%016x" % s, f"{time.time() - t0:.1f}s", flush=True)
    out = {"generator": "tests/golden/make_sweep_golden.py via oracle/_ref/libnttk_ref.so "
                        "(the reference's checked reductions)",
           "inputs": "tests/golden/sweep_inputs.py grid(), 2^%d x 2^%d" % (LOG2, LOG2),
           "rows": rows}
    with open(os.path.join(HERE, "sweep_2p30.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
