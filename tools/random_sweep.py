#!/usr/bin/env python3
"""Extended seeded random parity sweep (one-off validation beside tests/test_gpu_parity.py):
random (kind, N, tree, n, storage width, batch) cases; forward of canonical inputs and inverse
of ARBITRARY storage words against the CPU oracle, plus the round trip.
usage: python tools/random_sweep.py [cases] [seed]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import CYCLIC, HARVEY, IMPROVED, NEGA, NTL, SCOTT, SMONT, Oracle  # noqa: E402
import paper_2402_00675_b200.nttk as nttk  # noqa: E402

cases_wanted = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 20261021)
o = Oracle()
DT = {2: np.uint16, 4: np.uint32, 8: np.uint64}
SDT = {2: np.int16, 4: np.int32, 8: np.int64}
cache, done, by_path = {}, 0, {}
while done < cases_wanted:
    N = int(rng.choice([256, 256, 512, 1024]))
    p = {256: int(rng.choice([3329, 7681, 8380417])), 512: int(rng.choice([12289, 13313])), 1024: 12289}[N]
    n = 16 if (p == 3329 and rng.random() < 0.6) else 32
    tree = CYCLIC if (N > 256 or rng.random() < 0.6) else NEGA
    k = int(rng.choice([IMPROVED, IMPROVED, IMPROVED, HARVEY, SMONT] + ([NTL, SCOTT] if tree == CYCLIC else [])))
    layers = 0 if tree == CYCLIC else (7 if p == 3329 else 8)
    key = (p, N, n, tree, k, layers)
    if key not in cache:
        try:
            cache[key] = (nttk.build_params(p, N, n, [k], tree=tree, layers=layers, exact_bound=True),
                          o.params(p, N, n, (k,), tree=tree, layers=layers, exact=True))
        except Exception:
            cache[key] = None
    if cache[key] is None:
        continue
    P, Q = cache[key]
    sgn = k == SMONT
    L = N.bit_length() - 1 if not layers else layers
    bound = {NTL: p, HARVEY: 2 * p, SCOTT: N * p, IMPROVED: (L + 1) * p, SMONT: (L + 2) * p}[k]
    lim = {2: 1 << 15, 4: 1 << 31, 8: 1 << 63} if sgn else {2: 1 << 16, 4: 1 << 32, 8: 1 << 64}
    elems = [e for e in (2, 4) if bound <= lim[e]]
    if not elems:
        continue
    elem = int(rng.choice(elems))
    B = int(rng.integers(1, 200))
    f = o.rng(int(rng.integers(1 << 30)), p, B * N).reshape(B, N)
    x = torch.from_numpy(np.ascontiguousarray(f.astype((SDT if sgn else DT)[elem])).view(SDT[elem])).cuda()
    try:
        y = nttk.forward(P, k, x)
    except nttk.ContractViolation as e:  # a width the engine refuses for this kind's spectrum
        if "cannot hold" in str(e):
            continue
        raise
    got = y.cpu().numpy()
    got = got.astype(np.int64) if sgn else got.view(DT[elem]).astype(np.int64)
    assert (got == Q.forward(k, f).astype(np.int64)).all(), ("forward", key, elem, B)
    z = nttk.inverse(P, k, y).cpu().numpy().view(DT[elem]).astype(np.uint64)
    assert (z == f).all(), ("round trip", key, elem, B)
    if not sgn:  # arbitrary storage words through the inverse
        w = rng.integers(0, 1 << (8 * elem), size=(B, N), dtype=np.uint64)
        t = torch.from_numpy(w.astype(DT[elem]).view(SDT[elem])).cuda()
        zi = nttk.inverse(P, k, t).cpu().numpy().view(DT[elem]).astype(np.uint64)
        assert (zi == Q.inverse(k, w)).all(), ("inverse of arbitrary words", key, elem, B)
    tag = f"N={N} p={p} n={n} {'cyc' if tree == CYCLIC else 'nega'} kind={k} u{8 * elem}"
    by_path[tag] = by_path.get(tag, 0) + 1
    done += 1
print(f"{done} random cases, 0 mismatches; {len(by_path)} distinct (N, p, n, tree, kind, width) paths")
for tag in sorted(by_path):
    print(f"  {by_path[tag]:3d} x {tag}")
