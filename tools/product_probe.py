"""Standalone pointwise / basemul kernels (product.cu) at config-2 / config-4 sizes:
device time per call and GB/s of algorithmic traffic (3 x storage bytes per slot)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2402_00675_b200.nttk as nttk  # noqa: E402

K = nttk.ButterflyKind
NEG, CYC = nttk.Tree.negacyclic, nttk.Tree.cyclic
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6462.7


def t_ms(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


g = torch.Generator(device="cuda").manual_seed(1)
for label, q, n, tree, L, dt, B in (("kyber nega7 basemul u16", 3329, 16, NEG, 7, torch.int16, 1 << 16),
                                    ("kyber nega7 basemul u16 big", 3329, 16, NEG, 7, torch.int16, 1 << 20),
                                    ("kyber cyclic pointwise u16 big", 3329, 16, CYC, 8, torch.int16, 1 << 20),
                                    ("dilithium cyclic pointwise u32 big", 8380417, 32, CYC, 8, torch.int32, 1 << 20)):
    for kind in (K.improved, K.harvey, K.smont):
        P = nttk.build_params(q, 256, n, [kind], tree=tree, layers=L, exact_bound=True)
        xa = torch.randint(0, q, (B, 256), generator=g, device="cuda", dtype=torch.int32).to(dt)
        xb = torch.randint(0, q, (B, 256), generator=g, device="cuda", dtype=torch.int32).to(dt)
        fa, fb = nttk.forward(P, kind, xa), nttk.forward(P, kind, xb)
        out = torch.empty_like(fa)
        fn = nttk.basemul if L == 7 else nttk.pointwise
        ms = t_ms(lambda: fn(P, kind, fa, fb, out))
        gbs = 3 * fa.numel() * fa.element_size() / (ms / 1e3) / 1e9
        print(f"{label:36s} {kind.name:9s} {ms * 1e3:8.1f} us  {gbs:7.1f} GB/s  {gbs / peak:.2f} of HBM")
