import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2402_00675_b200.nttk as nttk
from oracle.oracle import Oracle, IMPROVED
o = Oracle()
for p, n, dt, B in ((8380417, 32, torch.int32, 1 << 21), (8380417, 32, torch.int32, 1 << 16), (3329, 16, torch.int16, 1 << 22)):
    P = nttk.build_params(p, 256, n, [3], exact_bound=True)
    Q = o.params(p, 256, n, (IMPROVED,), exact=True)
    g = torch.Generator(device="cuda").manual_seed(4)
    x = torch.randint(0, p, (B, 256), generator=g, device="cuda", dtype=torch.int64).to(dt)
    for trial in range(3):
        y = nttk.forward(P, 3, x)
        z = nttk.inverse(P, 3, y)
        bad = (z != x).any(dim=1).nonzero().flatten()
        print(p, B, 'trial', trial, 'bad rows', bad.numel(), bad[:10].tolist())
        if bad.numel():
            i = int(bad[0])
            xi = x[i].cpu().numpy().astype(np.int64) & 0xffffffff
            yi = y[i].cpu().numpy().astype(np.int64) & 0xffffffff
            fw = Q.forward(IMPROVED, xi.astype(np.uint64))[0]
            print('  fwd ok?', (fw.astype(np.int64) == yi).all(), ' inv of good fwd:', (Q.inverse(IMPROVED, fw)[0].astype(np.int64)==xi).all())
            zi = z[i].cpu().numpy().astype(np.int64) & 0xffffffff
            print('  z vs x mism positions', np.nonzero(zi != xi)[0][:20])
