#!/usr/bin/env python3
"""Time the N = 256 inverse alone on arbitrary storage words (round trip checked once).
usage: python tools/inv_probe.py [kyber|dilithium] [log2 batch] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_00675_b200.nttk as nttk  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "kyber"
B = 1 << int(sys.argv[2] if len(sys.argv) > 2 else 22)
reps = int(sys.argv[3] if len(sys.argv) > 3 else 20)
q, n, dt = (3329, 16, torch.int16) if which == "kyber" else (8380417, 32, torch.int32)
K = nttk.ButterflyKind
P = nttk.build_params(q, 256, n, [K.improved], exact_bound=True)
x = torch.randint(0, q, (B, 256), device="cuda", dtype=torch.int32).to(dt)
y = nttk.forward(P, K.improved, x)
z = torch.empty_like(x)
for _ in range(3):
    nttk.inverse(P, K.improved, y, z)
assert torch.equal(z, x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    nttk.inverse(P, K.improved, y, z)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"{which} inv B={B}: {ms:.4f} ms, {2 * x.numel() * x.element_size() / (ms / 1e3) / 1e9:.0f} GB/s (alg.)")
