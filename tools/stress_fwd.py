"""Stress: compare the engine's forward output over many repetitions against a saved
v1 (register-prefetch kernel) result.  Usage: NTTK_KERNEL=v1 python tools/stress_fwd.py save
then python tools/stress_fwd.py check."""
import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2402_00675_b200.nttk as nttk
mode = sys.argv[1]
cases = [(8380417, 32, torch.int32, 1 << 21), (3329, 16, torch.int16, 1 << 22)]
for p, n, dt, B in cases:
    P = nttk.build_params(p, 256, n, [3], exact_bound=True)
    g = torch.Generator(device="cuda").manual_seed(4)
    x = torch.randint(0, p, (B, 256), generator=g, device="cuda", dtype=torch.int64).to(dt)
    path = f"/tmp/fwd_{p}.pt"
    if mode == "save":
        torch.save(nttk.forward(P, 3, x).cpu(), path)
        continue
    ref = torch.load(path).cuda()
    y = torch.empty_like(x)
    nbad = 0
    for t in range(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
        y.fill_(0)
        nttk.forward(P, 3, x, y)
        bad = (y != ref).nonzero()
        if bad.numel():
            nbad += 1
            rows = bad[:, 0].unique()
            print(p, "trial", t, "bad elems", bad.shape[0], "rows", rows[:8].tolist(),
                  "cols", bad[:32, 1].tolist())
    print(p, "trials with mismatches:", nbad)
