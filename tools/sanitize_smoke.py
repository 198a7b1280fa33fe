"""Small-batch run of every kernel family for compute-sanitizer (memcheck / racecheck).

Exercises the TMA forward/inverse kernels (u16/u32, both trees, improved/harvey/smont),
the fused polymul, the v1 kernels (u64 storage), the generic kernel, pointwise/basemul and
the reduction sweep, checking each result against the CPU oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_2402_00675_b200.nttk as nttk  # noqa: E402
from oracle.oracle import CYCLIC, HARVEY, IMPROVED, NEGA, SMONT, Oracle  # noqa: E402

o = Oracle()
bad = 0
B = 37
for p, n, elem in ((3329, 16, 2), (8380417, 32, 4), (3329, 16, 8)):
    for tree, L in ((CYCLIC, 8), (NEGA, 7 if p == 3329 else 8)):
        for kind in (IMPROVED, HARVEY, SMONT):
            P = nttk.build_params(p, 256, n, [kind], tree=tree, layers=L, exact_bound=True)
            Q = o.params(p, 256, n, (kind,), tree=tree, layers=L, exact=True)
            f = o.rng(5 + kind, p, B * 256).reshape(B, 256)
            g = o.rng(6 + kind, p, B * 256).reshape(B, 256)
            dt = {2: torch.int16, 4: torch.int32, 8: torch.int64}[elem]
            x = torch.from_numpy(f.astype(np.int64)).to(dt).cuda()
            y = torch.from_numpy(g.astype(np.int64)).to(dt).cuda()
            s = nttk.forward(P, kind, x)
            mask = (1 << (8 * elem)) - 1 if elem < 8 else -1
            want = Q.forward(kind, f).astype(np.int64)
            got = s.cpu().numpy().astype(np.int64)
            if kind == SMONT:
                ok = (got == want).all()
            else:
                ok = ((got & mask) == (want & mask)).all()
            ok &= torch.equal(nttk.inverse(P, kind, s), x)
            c = nttk.polymul(P, kind, x, y)
            ok &= (c.cpu().numpy().astype(np.int64) & (mask if elem < 8 else -1) ==
                   Q.polymul(kind, f, g).astype(np.int64)).all()
            if not ok:
                bad += 1
                print("MISMATCH", p, n, elem, tree, L, kind)
# generic kernel: falcon512 preset, all reference kinds
P = nttk.preset("falcon512")
Q = o.params(12289, 512, 32, (0, 1, 2, 3))
f = o.rng(9, 12289, 3 * 512).reshape(3, 512)
for k in range(4):
    s = nttk.ntt_forward_batch(f, P, k)
    if not ((s == Q.forward(k, f)).all() and (nttk.intt_inverse_batch(s, P, k) == f).all()):
        bad += 1
        print("MISMATCH generic", k)
# sweep
A = torch.tensor([0, 1, 3328, 17, 999], dtype=torch.int64, device="cuda")
Bv = torch.arange(0, 4 * 3329, 7, dtype=torch.int64, device="cuda")
for v in (0, 3):
    r = torch.empty(A.numel() * Bv.numel(), dtype=torch.int64, device="cuda")
    bb = Bv if v == 3 else Bv % 3329
    nttk.modmul_sweep(v, 3329, 16, 2, A, bb, r)
    want, _ = o.sweep(v, o.ctx(3329, 16, 0, 2), A.cpu().numpy(), bb.cpu().numpy())
    if not (r.cpu().numpy() == want).all():
        bad += 1
        print("MISMATCH sweep", v)
torch.cuda.synchronize()
print("sanitize smoke:", "OK" if bad == 0 else f"{bad} mismatches")
sys.exit(1 if bad else 0)
