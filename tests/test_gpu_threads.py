"""Concurrent host threads through the C ABI (ctypes drops the GIL): first-call launch
caches, per-thread error state and per-stream launches must hold up.  Runs in a fresh
process so the per-kernel caches are populated concurrently."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, threading
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
import paper_2402_00675_b200.nttk as nttk
K = nttk.ButterflyKind
jobs = [(3329, 256, 16, K.improved, torch.int16, True), (8380417, 256, 32, K.improved, torch.int32, True),
        (3329, 256, 16, K.harvey, torch.int16, True), (12289, 1024, 32, K.improved, torch.int32, False),
        (12289, 512, 32, K.ntl, torch.int32, False), (8380417, 256, 32, K.scott, torch.int32, False),
        (3329, 256, 16, K.smont, torch.int16, True), (7681, 256, 32, K.ntl, torch.int16, False)]
inputs, want = [], []
for j, (p, N, n, k, dt, ex) in enumerate(jobs):
    g = torch.Generator(device="cuda").manual_seed(j)
    inputs.append(torch.randint(0, p, (1031, N), generator=g, device="cuda", dtype=torch.int32).to(dt))
errors, results = [], [None] * len(jobs)
barrier = threading.Barrier(len(jobs))
def work(j):
    try:
        p, N, n, k, dt, ex = jobs[j]
        P = nttk.build_params(p, N, n, [k], exact_bound=ex)
        s = torch.cuda.Stream()
        barrier.wait()
        with torch.cuda.stream(s):
            for _ in range(20):
                y = nttk.forward(P, k, inputs[j], stream=s)
                z = nttk.inverse(P, k, y, stream=s)
        s.synchronize()
        results[j] = (y.cpu(), z.cpu())
        try:  # per-thread error state: this thread's message, not another's
            nttk.build_params(15, N, n, [k])
        except nttk.ContractViolation as e:
            assert "p must be prime" in str(e), str(e)
    except Exception as e:
        errors.append(repr(e))
ts = [threading.Thread(target=work, args=(j,)) for j in range(len(jobs))]
[t.start() for t in ts]; [t.join() for t in ts]
assert not errors, errors
for j, (p, N, n, k, dt, ex) in enumerate(jobs):  # single-threaded replay must agree
    P = nttk.build_params(p, N, n, [k], exact_bound=ex)
    y = nttk.forward(P, k, inputs[j])
    assert torch.equal(y.cpu(), results[j][0]), j
    assert torch.equal(results[j][1], inputs[j].cpu()), j
print("threads ok")
'''


def test_concurrent_threads_fresh_process(tmp_path):
    script = tmp_path / "threads.py"
    script.write_text(SCRIPT)
    r = subprocess.run([sys.executable, str(script), ROOT], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "threads ok" in r.stdout, r.stdout + r.stderr


AB_SCRIPT = r'''
import sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
from oracle.oracle import Oracle, IMPROVED, HARVEY, SMONT, NEGA
import paper_2402_00675_b200.nttk as nttk
o = Oracle()
K = nttk.ButterflyKind
# Kyber forward (F1 off: umulhi form everywhere)
P = nttk.build_params(3329, 256, 16, [K.improved], exact_bound=True)
Q = o.params(3329, 256, 16, (IMPROVED,), exact=True)
f = o.rng(31, 3329, 257 * 256).reshape(257, 256)
y = nttk.forward(P, K.improved, torch.from_numpy(f.astype(np.int16)).cuda())
assert (y.cpu().numpy().astype(np.int64) & 0xffff == Q.forward(IMPROVED, f)).all()
# the 7-layer negacyclic Kyber forward (F1 off: umulhi form)
P7 = nttk.build_params(3329, 256, 16, [K.improved], tree=nttk.Tree.negacyclic, layers=7, exact_bound=True)
Q7 = o.params(3329, 256, 16, (IMPROVED,), tree=NEGA, layers=7, exact=True)
y7 = nttk.forward(P7, K.improved, torch.from_numpy(f.astype(np.int16)).cuda())
assert (y7.cpu().numpy().astype(np.int64) & 0xffff == Q7.forward(IMPROVED, f)).all()
# Kyber u16 inverse on arbitrary words (CT off: the GS lazy-merge body)
w = np.random.RandomState(3).randint(0, 1 << 16, size=(129, 256)).astype(np.uint16)
z = nttk.inverse(P, K.improved, torch.from_numpy(w.view(np.int16)).cuda())
assert (z.cpu().numpy().astype(np.int64) == Q.inverse(IMPROVED, w.astype(np.uint64))).all()
# Dilithium u32 inverse on arbitrary words (CT off: the GS lazy merge with partial canonicalisation)
Pd = nttk.build_params(8380417, 256, 32, [K.improved], exact_bound=True)
Qd = o.params(8380417, 256, 32, (IMPROVED,), exact=True)
wd = np.random.RandomState(4).randint(0, 1 << 32, size=(65, 256), dtype=np.uint64)
zd = nttk.inverse(Pd, K.improved, torch.from_numpy(wd.astype(np.uint32).view(np.int32)).cuda())
assert (zd.cpu().numpy().view(np.uint32).astype(np.int64) == Qd.inverse(IMPROVED, wd)).all()
# Table 2 presets, inverse on arbitrary words (CT off: the GS narrow bodies)
for name in ("kyber256", "newhope512", "newhope1024"):
    Pn = nttk.preset(name)
    Qn = o.params(Pn.p, Pn.size, 32, (IMPROVED,))
    wn = np.random.RandomState(5).randint(0, 1 << 32, size=(35, Pn.size), dtype=np.uint64)
    zn = nttk.inverse(Pn, K.improved, torch.from_numpy(wn.astype(np.uint32).view(np.int32)).cuda())
    assert (zn.cpu().numpy().view(np.uint32).astype(np.int64) == Qn.inverse(IMPROVED, wn)).all(), name
# fused polymul with the eager policies of every kind
for kind, k in ((K.improved, IMPROVED), (K.harvey, HARVEY), (K.smont, SMONT)):
    P = nttk.build_params(3329, 256, 16, [kind], tree=nttk.Tree.negacyclic, layers=7, exact_bound=True)
    Q = o.params(3329, 256, 16, (k,), tree=NEGA, layers=7, exact=True)
    a = o.rng(32, 3329, 65 * 256).reshape(65, 256)
    b = o.rng(33, 3329, 65 * 256).reshape(65, 256)
    c = nttk.polymul(P, kind, torch.from_numpy(a.astype(np.int16)).cuda(),
                     torch.from_numpy(b.astype(np.int16)).cuda())
    assert (c.cpu().numpy().astype(np.int64) == Q.polymul(k, a, b)).all(), kind
print("ok")
'''


def test_ab_switches_keep_parity(tmp_path):
    """The runtime A/B switches (NTTK_FWD_F1=0: umulhi-form Kyber forward; NTTK_INV_CT=0: the
    GS lazy-merge Kyber / Dilithium inverses and the GS narrow inverse at N = 512 / 1024; NTTK_POLYMUL_EAGER=1: the standalone policies inside the fused
    polymul) select other exact arithmetic; in a fresh process their words must equal the
    oracle's too."""
    script = tmp_path / "ab.py"
    script.write_text(AB_SCRIPT)
    env = dict(os.environ, NTTK_FWD_F1="0", NTTK_POLYMUL_EAGER="1", NTTK_INV_CT="0")
    r = subprocess.run([sys.executable, str(script), ROOT], capture_output=True, text=True,
                       timeout=600, env=env)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
