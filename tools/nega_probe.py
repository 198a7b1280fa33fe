#!/usr/bin/env python3
"""Time the Kyber 7-layer negacyclic transforms (row a22) at a large batch, next to the cyclic
8-layer ones.  usage: python tools/nega_probe.py [log2 batch] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_00675_b200.nttk as nttk  # noqa: E402

K = nttk.ButterflyKind
B = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 22)
reps = int(sys.argv[2] if len(sys.argv) > 2 else 20)
x = torch.randint(0, 3329, (B, 256), device="cuda", dtype=torch.int32).to(torch.int16)
y, z = torch.empty_like(x), torch.empty_like(x)
for name, P in (("nega7", nttk.build_params(3329, 256, 16, [K.improved], tree=nttk.Tree.negacyclic, layers=7, exact_bound=True)),
                ("cyclic8", nttk.build_params(3329, 256, 16, [K.improved], exact_bound=True))):
    for _ in range(3):
        nttk.forward(P, K.improved, x, y)
        nttk.inverse(P, K.improved, y, z)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    for _ in range(reps):
        nttk.forward(P, K.improved, x, y)
    e[1].record()
    for _ in range(reps):
        nttk.inverse(P, K.improved, y, z)
    e[2].record()
    torch.cuda.synchronize()
    assert torch.equal(z, x)
    print(f"{name} B={B}: fwd {e[0].elapsed_time(e[1]) / reps:.4f} ms, inv {e[1].elapsed_time(e[2]) / reps:.4f} ms "
          f"(flags fwd {P.fast_flags(K.improved, 0):#x} inv {P.fast_flags(K.improved, 1):#x})")
