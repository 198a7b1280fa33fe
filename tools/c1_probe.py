#!/usr/bin/env python3
"""BASELINE config 1 latency: 4096 Kyber polys, 7-layer negacyclic forward, one call, CUDA-graph
replay (device time per call without host launch overhead) and eager, plus a batch sweep."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_00675_b200.nttk as nttk  # noqa: E402

K = nttk.ButterflyKind
P1 = nttk.build_params(3329, 256, 16, [K.improved], tree=nttk.Tree.negacyclic, layers=7, exact_bound=True)
out = []
BS = [int(b) for b in sys.argv[1].split(',')] if len(sys.argv) > 1 else [1024, 4096, 16384, 65536]
for B in BS:
    x = torch.randint(0, 3329, (B, 256), device="cuda", dtype=torch.int32).to(torch.int16)
    y = torch.empty_like(x)
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        nttk.forward(P1, K.improved, x, y)
    torch.cuda.current_stream().wait_stream(cs)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(50):
            nttk.forward(P1, K.improved, x, y)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    fi = nttk.build_params(3329, 256, 16, [K.improved], exact_bound=True)
    t = e0.elapsed_time(e1) / 1000 * 1e3
    # the same batch through the cyclic 8-layer inverse (u16, DEFER path), eager
    z = torch.empty_like(x)
    for _ in range(3):
        nttk.inverse(fi, K.improved, x, z)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        nttk.inverse(fi, K.improved, x, z)
    e1.record()
    torch.cuda.synchronize()
    out.append(f"B={B}: fwd7 {t:.2f} us, inv8 {e0.elapsed_time(e1) / 20 * 1e3:.2f} us")
print(" | ".join(out))
