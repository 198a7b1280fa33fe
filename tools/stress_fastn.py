"""Stress the N = 512 / 1024 TMA kernels (fastn_tma.cu: F1 forward, narrow inverse, two-box
inverse stages with 16 consumers): repeat forward and inverse over a batch much larger than
the stage rings and require every trial to reproduce trial 0 word for word and the round trip
to return the input.  A stage-ring race (mbarrier phase, proxy-fenced release) would show up as
a trial-to-trial difference.
Usage: python tools/stress_fastn.py [trials]"""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2402_00675_b200.nttk as nttk  # noqa: E402

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 20
K = nttk.ButterflyKind
for name in ("newhope512", "newhope1024", "kyber256"):
    P = nttk.preset(name)
    B = (1 << 27) // P.size
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randint(0, P.p, (B, P.size), generator=g, device="cuda", dtype=torch.int32)
    for kind in (K.improved, K.harvey):
        s0 = nttk.forward(P, kind, x)
        w = torch.randint(0, 1 << 31, (B, P.size), generator=g, device="cuda", dtype=torch.int32)
        i0 = nttk.inverse(P, kind, w)  # arbitrary words through the inverse
        bad = 0
        s, o, i = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
        for _ in range(trials):
            nttk.forward(P, kind, x, s)
            nttk.inverse(P, kind, s, o)
            nttk.inverse(P, kind, w, i)
            bad += int(not (torch.equal(s, s0) and torch.equal(o, x) and torch.equal(i, i0)))
        print(f"{name} {kind.name} B={B}: trials with mismatches: {bad} / {trials}", flush=True)
