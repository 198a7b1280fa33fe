#!/usr/bin/env python3
"""BASELINE config 3 shape: Dilithium (q = 8380417, n = 32, u32) round trip of B polys per
kind, forward and inverse timed separately (CUDA events, HBM-resident).
usage: python tools/c3_probe.py [log2 batch ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_00675_b200.nttk as nttk  # noqa: E402

K = nttk.ButterflyKind
for lb in [int(a) for a in sys.argv[1:]] or [16]:
    B = 1 << lb
    x = torch.randint(0, 8380417, (B, 256), device="cuda", dtype=torch.int32)
    s, o = torch.empty_like(x), torch.empty_like(x)
    out = []
    for kind in (K.improved, K.harvey, K.scott):
        P = nttk.build_params(8380417, 256, 32, [kind], exact_bound=True)
        for _ in range(3):
            nttk.forward(P, kind, x, s)
            nttk.inverse(P, kind, s, o)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        for _ in range(20):
            nttk.forward(P, kind, x, s)
        e[1].record()
        for _ in range(20):
            nttk.inverse(P, kind, s, o)
        e[2].record()
        torch.cuda.synchronize()
        assert torch.equal(o, x)
        out.append(f"{kind.name} fwd {e[0].elapsed_time(e[1]) / 20 * 1e3:.1f} inv {e[1].elapsed_time(e[2]) / 20 * 1e3:.1f} us")
    print(f"B=2^{lb}: " + " | ".join(out))
