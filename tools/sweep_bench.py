"""Time every reduction-sweep variant (BASELINE config 5) with CUDA events."""
import os, sys, time
import torch
sys.path.insert(0, os.getcwd())
import paper_2402_00675_b200.nttk as nttk
g = torch.Generator(device="cuda").manual_seed(1)
for q, n, ell in ((3329, 16, 2), (8380417, 32, 7)):
    for v in range(4):
        hi = q + 1 if v == 2 else (q << ell if v == 3 else q)
        A = torch.randint(0, q + (1 if v == 2 else 0), (1 << 15,), generator=g, device="cuda", dtype=torch.int64)
        if v == 1:
            B = torch.randint(-(1 << (n - 1)), 1 << (n - 1), (1 << 15,), generator=g, device="cuda", dtype=torch.int64)
        else:
            B = torch.randint(0, hi, (1 << 15,), generator=g, device="cuda", dtype=torch.int64)
        nttk.modmul_sweep(v, q, n, ell, A, B)
        ts = []
        for _ in range(30):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            nttk.modmul_sweep(v, q, n, ell, A, B)
            ts.append(time.perf_counter() - t0)
        print(q, v, "min %.3f ms  -> %.3f T mults/s" % (min(ts) * 1e3, (1 << 30) / min(ts) / 1e12))
