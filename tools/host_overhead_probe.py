#!/usr/bin/env python3
"""Host-side cost per device call (config 1 shape: 4096 Kyber polys, 7-layer negacyclic
forward): the Python mirror vs direct C-ABI calls with cached pointers vs a no-op ABI call.
The GPU work (~4 us) is shorter than the host path, so the issue rate is the host cost."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_00675_b200.nttk as nttk  # noqa: E402

K = nttk.ButterflyKind
P1 = nttk.build_params(3329, 256, 16, [K.improved], tree=nttk.Tree.negacyclic, layers=7,
                       exact_bound=True)
x = torch.randint(0, 3329, (4096, 256), device="cuda", dtype=torch.int32).to(torch.int16)
y = torch.empty_like(x)
L = nttk.lib()
h, xp, yp = P1.handle, x.data_ptr(), y.data_ptr()
sp = torch.cuda.current_stream().cuda_stream


def rate(fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return (t1 - t0) / n * 1e6, (t2 - t0) / n * 1e6


for name, fn in (("python mirror nttk.forward", lambda: nttk.forward(P1, K.improved, x, y)),
                 ("direct ctypes nttk_ntt_forward", lambda: L.nttk_ntt_forward(h, 3, xp, yp, 4096, 2, sp)),
                 ("ctypes no-op (nttk_version)", lambda: L.nttk_version())):
    a, b = rate(fn)
    print(f"{name:34s}: issue {a:7.2f} us/call, issue+drain {b:7.2f} us/call")
