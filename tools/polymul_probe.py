#!/usr/bin/env python3
"""BASELINE config 2 (Kyber 7-layer negacyclic polymul, 65536 pairs) per reduction kind,
fused kernel, CUDA events; usable with A/B variants of libnttk_gpu.so (no parity check).
usage: python tools/polymul_probe.py [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_00675_b200.nttk as nttk  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
K = nttk.ButterflyKind
B = 65536
g = torch.Generator(device="cuda").manual_seed(2)
xa = torch.randint(0, 3329, (B, 256), generator=g, device="cuda", dtype=torch.int32).to(torch.int16)
xb = torch.randint(0, 3329, (B, 256), generator=g, device="cuda", dtype=torch.int32).to(torch.int16)
xc = torch.empty_like(xa)
out = []
for name, kind in (("improved", K.improved), ("harvey", K.harvey), ("smont", K.smont)):
    P = nttk.build_params(3329, 256, 16, [kind], tree=nttk.Tree.negacyclic, layers=7, exact_bound=True)
    for _ in range(5):
        nttk.polymul(P, kind, xa, xb, xc)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        nttk.polymul(P, kind, xa, xb, xc)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out.append(f"{name} {ms * 1e3:.1f} us ({B / ms / 1e6:.3f} G products/s)")
# Dilithium (u32, n = 32, 8-layer negacyclic, slotwise product)
xa = torch.randint(0, 8380417, (B, 256), generator=g, device="cuda", dtype=torch.int32)
xb = torch.randint(0, 8380417, (B, 256), generator=g, device="cuda", dtype=torch.int32)
xc = torch.empty_like(xa)
for name, kind in (("dil_improved", K.improved), ("dil_harvey", K.harvey), ("dil_smont", K.smont)):
    P = nttk.build_params(8380417, 256, 32, [kind], tree=nttk.Tree.negacyclic, layers=8, exact_bound=True)
    for _ in range(5):
        nttk.polymul(P, kind, xa, xb, xc)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        nttk.polymul(P, kind, xa, xb, xc)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out.append(f"{name} {ms * 1e3:.1f} us")
print(" | ".join(out))
