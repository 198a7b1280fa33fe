"""Stress: compare the engine's forward (or inverse) output over many repetitions against a
saved result of the v1 (register-prefetch) kernels, at BASELINE config-4 sizes.  Guards the
TMA stage rings (mbarrier phases, proxy-fenced stage release) against races.

Usage: NTTK_KERNEL=v1 python tools/stress_fwd.py save [fwd|inv]
       python tools/stress_fwd.py check [trials] [fwd|inv]
The inverse is fed arbitrary storage words (seeded), so it also covers the DEFER / partial
canonicalisation paths."""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2402_00675_b200.nttk as nttk  # noqa: E402

mode = sys.argv[1]
args = sys.argv[2:]
direction = "inv" if "inv" in args else "fwd"
nums = [a for a in args if a.isdigit()]
trials = int(nums[0]) if nums else 20
cases = [(8380417, 32, torch.int32, 1 << 21), (3329, 16, torch.int16, 1 << 22)]
for p, n, dt, B in cases:
    P = nttk.build_params(p, 256, n, [3], exact_bound=True)
    g = torch.Generator(device="cuda").manual_seed(4)
    if direction == "fwd":
        x = torch.randint(0, p, (B, 256), generator=g, device="cuda", dtype=torch.int64).to(dt)
    else:
        bits = 16 if dt == torch.int16 else 32
        x = torch.randint(0, 1 << bits, (B, 256), generator=g, device="cuda", dtype=torch.int64)
        x = (x - (1 << (bits - 1))).to(dt)
    run = nttk.forward if direction == "fwd" else nttk.inverse
    path = f"/tmp/{direction}_{p}.pt"
    if mode == "save":
        torch.save(run(P, 3, x).cpu(), path)
        continue
    ref = torch.load(path).cuda()
    y = torch.empty_like(x)
    nbad = 0
    for t in range(trials):
        y.fill_(0)
        run(P, 3, x, y)
        bad = (y != ref).nonzero()
        if bad.numel():
            nbad += 1
            rows = bad[:, 0].unique()
            print(p, "trial", t, "bad elems", bad.shape[0], "rows", rows[:8].tolist(),
                  "cols", bad[:32, 1].tolist())
    print(direction, p, "trials with mismatches:", nbad)
