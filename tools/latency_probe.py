#!/usr/bin/env python3
"""Per-call latency of the reference-shaped host calls (one polynomial per call) and of the
device calls, through the Python mirror and the C ABI."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_00675_b200.nttk as nttk  # noqa: E402

K = nttk.ButterflyKind
P = nttk.preset("kyber256")
f = np.random.default_rng(1).integers(0, P.p, 256, dtype=np.uint64)
for B in (1, 16, 256, 4096):
    x = np.tile(f, (B, 1))
    nttk.ntt_forward_batch(x, P, K.improved)
    t0 = time.perf_counter()
    n = 200 if B < 4096 else 50
    for _ in range(n):
        nttk.ntt_forward_batch(x, P, K.improved)
    dt = (time.perf_counter() - t0) / n
    print(f"host call, {B:5d} polys: {dt * 1e6:8.1f} us/call, {dt * 1e6 / B:8.3f} us/poly")
xd = torch.from_numpy(np.tile(f, (16, 1)).astype(np.int32)).cuda()
yd = torch.empty_like(xd)
for _ in range(10):
    nttk.forward(P, K.improved, xd, yd)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(1000):
    nttk.forward(P, K.improved, xd, yd)
torch.cuda.synchronize()
print(f"device call (16 polys, async, Python): {(time.perf_counter() - t0) * 1e3:.1f} us/call")
