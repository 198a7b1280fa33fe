#!/usr/bin/env python3
"""Time the N = 256 forward alone (no correctness check: usable with A/B kernel variants).
usage: python tools/fwd_probe.py [kyber|dilithium] [log2 batch] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_00675_b200.nttk as nttk  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "dilithium"
B = 1 << int(sys.argv[2] if len(sys.argv) > 2 else 21)
reps = int(sys.argv[3] if len(sys.argv) > 3 else 10)
q, n, dt = (3329, 16, torch.int16) if which == "kyber" else (8380417, 32, torch.int32)
P = nttk.build_params(q, 256, n, [nttk.ButterflyKind.improved], exact_bound=True)
x = torch.randint(0, q, (B, 256), device="cuda", dtype=torch.int32).to(dt)
y = torch.empty_like(x)
for _ in range(3):
    nttk.forward(P, nttk.ButterflyKind.improved, x, y)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    nttk.forward(P, nttk.ButterflyKind.improved, x, y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
gbs = 2 * x.numel() * x.element_size() / (ms / 1e3) / 1e9
print(f"{which} fwd B={B}: {ms:.4f} ms, {gbs:.0f} GB/s (alg.)")
