#!/usr/bin/env python3
"""Where do the 4-6 % between a kernel timed alone and inside the config-4 step go?  Times each
of the four kernels (a) looped alone, (b) inside the step in several orders, with CUDA events
around every launch.  usage: python tools/step_probe.py [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_00675_b200.nttk as nttk  # noqa: E402

K = nttk.ButterflyKind.improved
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
Pk = nttk.build_params(3329, 256, 16, [K], exact_bound=True)
Pd = nttk.build_params(8380417, 256, 32, [K], exact_bound=True)
xk = torch.randint(0, 3329, (1 << 22, 256), device="cuda", dtype=torch.int32).to(torch.int16)
xd = torch.randint(0, 8380417, (1 << 21, 256), device="cuda", dtype=torch.int32)
sk, ok, sd, od = (torch.empty_like(t) for t in (xk, xk, xd, xd))
ops = {"kf": lambda: nttk.forward(Pk, K, xk, sk), "ki": lambda: nttk.inverse(Pk, K, sk, ok),
       "df": lambda: nttk.forward(Pd, K, xd, sd), "di": lambda: nttk.inverse(Pd, K, sd, od)}
for f in ops.values():
    f()
torch.cuda.synchronize()


def timed(order):
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(order) + 1)] for _ in range(reps)]
    for r in range(reps):
        ev[r][0].record()
        for i, name in enumerate(order):
            ops[name]()
            ev[r][i + 1].record()
    torch.cuda.synchronize()
    per = {}
    for i, name in enumerate(order):
        per.setdefault(name, []).append(sum(ev[r][i].elapsed_time(ev[r][i + 1]) for r in range(2, reps)) / (reps - 2))
    tot = sum(ev[r][0].elapsed_time(ev[r][-1]) for r in range(2, reps)) / (reps - 2)
    return " ".join(f"{k}=" + "/".join(f"{v:.4f}" for v in vs) for k, vs in per.items()) + f" | total {tot:.4f}"


for order in (["kf"], ["ki"], ["df"], ["di"], ["kf", "ki", "df", "di"], ["kf", "kf", "ki", "ki"],
              ["df", "kf", "di", "ki"], ["kf", "df", "ki", "di"], ["df", "di", "kf", "ki"]):
    print(",".join(order), "->", timed(order))
