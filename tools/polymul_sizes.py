import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2402_00675_b200.nttk as nttk
K = nttk.ButterflyKind
P = nttk.build_params(3329, 256, 16, [K.improved], tree=nttk.Tree.negacyclic, layers=7, exact_bound=True)
for lg in (14, 15, 16, 17, 18, 20):
    B = 1 << lg
    xa = torch.randint(0, 3329, (B, 256), device="cuda", dtype=torch.int32).to(torch.int16)
    xb = torch.randint(0, 3329, (B, 256), device="cuda", dtype=torch.int32).to(torch.int16)
    xc = torch.empty_like(xa)
    for _ in range(5): nttk.polymul(P, K.improved, xa, xb, xc)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record()
    for _ in range(reps): nttk.polymul(P, K.improved, xa, xb, xc)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"B=2^{lg}: {ms*1e3:.1f} us  {B/ms/1e6:.3f} G products/s")
