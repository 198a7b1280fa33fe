#!/usr/bin/env python3
"""Time (or drive under ncu) the N = 512 / 1024 fast kernels on one preset and kind.

usage: python tools/fastn_probe.py [preset] [kind] [log2 batch] [reps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_00675_b200.nttk as nttk  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "newhope1024"
kind = nttk.ButterflyKind[sys.argv[2] if len(sys.argv) > 2 else "improved"]
B = 1 << int(sys.argv[3] if len(sys.argv) > 3 else 16)
reps = int(sys.argv[4] if len(sys.argv) > 4 else 10)
P = nttk.preset(name)
x = torch.randint(0, P.p, (B, P.size), device="cuda", dtype=torch.int32)
s, o = torch.empty_like(x), torch.empty_like(x)
for _ in range(2):
    nttk.forward(P, kind, x, s)
    nttk.inverse(P, kind, s, o)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record()
for _ in range(reps):
    nttk.forward(P, kind, x, s)
e[1].record()
for _ in range(reps):
    nttk.inverse(P, kind, s, o)
e[2].record()
torch.cuda.synchronize()
assert torch.equal(o, x)
f, i = e[0].elapsed_time(e[1]) / reps, e[1].elapsed_time(e[2]) / reps
print(f"{name} {kind.name} B={B}: fwd {f * 1e6 / B:.3f} ns/poly, inv {i * 1e6 / B:.3f} ns/poly")
