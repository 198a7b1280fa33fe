#!/usr/bin/env python3
"""Per-kind forward / inverse at 2^20 polys (Kyber u16 n = 16, Dilithium u32 n = 32), CUDA events."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_00675_b200.nttk as nttk  # noqa: E402

K = nttk.ButterflyKind
B = 1 << 20
for q, n, dt, kinds in ((3329, 16, torch.int16, (K.improved, K.harvey, K.ntl, K.smont)),
                        (8380417, 32, torch.int32, (K.improved, K.harvey, K.ntl, K.scott, K.smont))):
    x = torch.randint(0, q, (B, 256), device="cuda", dtype=torch.int32).to(dt)
    s, o = torch.empty_like(x), torch.empty_like(x)
    out = []
    for kind in kinds:
        P = nttk.build_params(q, 256, n, [kind], exact_bound=True)
        for _ in range(3):
            nttk.forward(P, kind, x, s)
            nttk.inverse(P, kind, s, o)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        for _ in range(10):
            nttk.forward(P, kind, x, s)
        e[1].record()
        for _ in range(10):
            nttk.inverse(P, kind, s, o)
        e[2].record()
        torch.cuda.synchronize()
        assert torch.equal(o, x)
        out.append(f"{kind.name} {e[0].elapsed_time(e[1]) / 10:.3f}/{e[1].elapsed_time(e[2]) / 10:.3f}")
    print(f"q={q}: " + " | ".join(out))
