#!/usr/bin/env python3
"""Benchmark of the B200 NTT engine (driver contract: one JSON line on rank 0).

Workload (BASELINE.json config 4, the large-batch throughput config), per step:
  * 2^22 Kyber polynomials  (q = 3329,    N = 256, cyclic 8 layers, int16),
  * 2^21 Dilithium polys    (q = 8380417, N = 256, cyclic 8 layers, int32),
  each run forward then inverse with the paper's modified-Plantard ("improved")
  butterfly: n = 16 (32-bit Plantard constant) for Kyber, n = 32 (64-bit) for Dilithium.
Inputs are seeded uniform [0, q) synthetic data (no dataset is involved: the reference
benchmarks seeded random polynomials too, bench.hpp:198-230).  The working set
(4 GiB in + 4 GiB spectra at N = 1) is far above the 126 MB L2, so no flush is needed.

Multi-GPU: one process per GPU.  `--gpus N` run without torchrun re-launches
itself through torch.distributed.run (127.0.0.1); under torchrun WORLD_SIZE must equal
--gpus.  --scaling strong (default, config 4 "sharded evenly"): every rank draws the same
seeded global batch and paper_2402_00675_b200.shard.Sharder.run hands it its contiguous
shard -- no collective on the compute path; --scaling weak: each rank transforms the full
per-GPU sizes.  The step time is the max over ranks.  --gather: the result shards are
all-gathered with Sharder.gather (NCCL, timed separately) and rank 0 checks sampled
polynomials against the CPU oracle.

--impl reference times the reference's own CPU path (oracle/_ref: ntt_forward_inplace
+ intt_inverse, transform.hpp:228-231,339-343) on the host cores, same metric/config.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

KYBER_Q, DIL_Q = 3329, 8380417
METRIC = "NTT polys/sec (fwd+inv round trip, modified-Plantard butterfly)"
UNIT = "polys/s"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the fixed config-4 batch is sharded over the ranks; "
                         "weak: every rank transforms the full per-GPU batch")
    ap.add_argument("--kyber-log2", type=int, default=22)
    ap.add_argument("--dil-log2", type=int, default=21)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--gather", action="store_true",
                    help="all-gather the result shards (NCCL, timed separately) and check "
                         "sampled polynomials against the CPU oracle on rank 0")
    ap.add_argument("--no-extras", action="store_true", help="skip BASELINE configs 1/2/3/5")
    ap.add_argument("--plan-only", action="store_true",
                    help="print the per-rank shard plan (launcher / sharder check; no GPU work)")
    ap.add_argument("--bench-report", metavar="DIR",
                    help="write the reference BenchReport schema (bench.hpp:365-424) for the GPU "
                         "and for the reference's own run_bench, then exit")
    return ap.parse_args(argv)


def shard_plan(a, rank: int, world: int):
    """Per-rank (Kyber, Dilithium) polynomial ranges of one step."""
    from paper_2402_00675_b200.shard import Sharder

    nk, nd = 1 << a.kyber_log2, 1 << a.dil_log2
    if a.scaling == "weak":
        return {"kyber": (0, nk), "dilithium": (0, nd), "kyber_total": nk * world,
                "dilithium_total": nd * world}
    sh = Sharder(rank, world)
    return {"kyber": sh.local(nk), "dilithium": sh.local(nd), "kyber_total": nk,
            "dilithium_total": nd}


def workload_config(a, world, shards=None):
    nk, nd = 1 << a.kyber_log2, 1 << a.dil_log2
    per = "per GPU " if a.scaling == "weak" else "in total, sharded over the GPUs: "
    cfg = {
        "workload": (f"config4: {per}2^{a.kyber_log2} Kyber (q=3329,N=256,cyclic 8 layers,"
                     f"improved n=16,int16) + 2^{a.dil_log2} Dilithium (q=8380417,N=256,cyclic"
                     " 8 layers,improved n=32,int32); step = forward + inverse of both"),
        "kyber_polys_total": nk * (world if a.scaling == "weak" else 1),
        "dilithium_polys_total": nd * (world if a.scaling == "weak" else 1),
        "parallelism": f"dp{world} (batch sharding, no collective on the compute path)",
        "l2": "working set >= 8 GiB / GPU at N = 1 (>> 126 MB L2): no flush needed",
        "storage": "int16 (Kyber) / int32 (Dilithium) words; arithmetic on 32-bit registers",
    }
    if shards is not None:
        cfg["shards"] = shards
    return cfg


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform

    return platform.processor() or "unknown"


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(argv, n):
    """`bench.py --gpus N` without torchrun: one process per GPU through torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           os.path.abspath(__file__)] + list(argv)
    return subprocess.call(cmd)


# ---------------------------------------------------------------------------
# clocks sampled DURING the timed region (B200_PROFILING.md clocks line)

class ClockSampler:
    """SM clock + throttle reasons via NVML every 10 ms (nvidia-smi as a fallback)."""

    REASONS = {  # nvmlClocksEventReason* bits
        "hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
        "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.dev)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(sm), float(mx), int(rs)))
                self._stop.wait(0.01)
            return
        except Exception:
            pass
        fields = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={fields}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                s = [x.strip() for x in out.stdout.strip().split(",")]
                self.samples.append((float(s[0]), float(s[1]), int(s[2], 16)))
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        time.sleep(0.05)
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [s[0] for s in self.samples]
        reasons = sorted({name for s in self.samples for name, bit in self.REASONS.items()
                          if s[2] & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples)}


NCU_KERNELS = {"kyber_fwd": "fwd256_tma_kernel<ImprovedN16", "kyber_inv": "inv256_tma_kernel<ImprovedN16",
               "dil_fwd": "fwd256_tma_kernel<ImprovedN32", "dil_inv": "inv256_tma_kernel<ImprovedN32"}
# the SASS-census instantiations of the bench kernels (MODE 82 / 67 = the CT-form Kyber /
# Dilithium inverses; F1 + W1 forwards -- the last matching census row wins)
CENSUS_KERNELS = {"kyber_fwd": "fwd256_tma_kernelINS_11ImprovedN16ILb0EEEtLi8ELb0ELb1E",
                  "kyber_inv": "inv256_tma_kernelINS_11ImprovedN16ILb0EEEtLi8ELi82E",
                  "dil_fwd": "fwd256_tma_kernelINS_11ImprovedN32EjLi8ELb0ELb1E",
                  "dil_inv": "inv256_tma_kernelINS_11ImprovedN32EjLi8ELi67E",
                  # config 2 (fused polymul, 7-layer negacyclic, u16): the kernels that run
                  "pm_modified_plantard": "polymul256_tma_kernelINS_11ImprovedN16ILb0EEEtLi7ELb0ELb1ELb0ELb1E",
                  "pm_montgomery_R2^16": "polymul256_tma_kernelINS_12HarveyLazy16EtLi7E",
                  "pm_signed_montgomery": "polymul256_tma_kernelINS_11SmontLazy16EtLi7E"}


def latest_profile(pattern: str):
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", pattern)))
    return files[-1] if files else None


def ncu_traffic(kernel: str, nk: int, nd: int):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu --set full
    capture of the N = 1 bench configuration (profiles/r*_ncu_full.json), else None."""
    if (nk, nd) != (1 << 22, 1 << 21):
        return None
    path = latest_profile("r*_ncu_full.json")
    if not path:
        return None
    with open(path) as fh:
        caps = json.load(fh)["kernels"]
    for k in caps:
        if NCU_KERNELS[kernel] in k["kernel"].replace("nttk_b200::", "").replace("unnamed>::", ""):
            return k["dram_bytes"]
    return None


def kernel_source_sha():
    """sha256 over the sources the library is compiled from (csrc/, include/, Makefile):
    the SASS of a rebuild from the same sources with the same nvcc is the same."""
    import glob
    import hashlib

    h = hashlib.sha256()
    files = sorted(glob.glob(os.path.join(ROOT, "paper_2402_00675_b200", "csrc", "*")))
    files += [os.path.join(ROOT, "include", "nttk_gpu.h"), os.path.join(ROOT, "Makefile")]
    for f in files:
        with open(f, "rb") as fh:
            h.update(os.path.basename(f).encode() + b"\0" + fh.read())
    return h.hexdigest()


def sass_census():
    """Executed fmaheavy cycles per polynomial of the bench kernels from the committed SASS
    census (tools/sass_census.py --json), flagged stale when the kernel sources changed
    since (the census records their sha256; a rebuild of the same sources is the same SASS)."""
    path = latest_profile("r*_sass_census.json")
    if not path:
        return None, None
    with open(path) as fh:
        d = json.load(fh)
    try:
        stale = kernel_source_sha() != d.get("src_sha256")
    except OSError:
        stale = True
    out = {}
    for key, pat in CENSUS_KERNELS.items():
        for r in d["rows"]:
            if pat in r["kernel"]:
                out[key] = r["fmaheavy_cycles_per_iter"] / r["polys_per_iter"]
    return out, {"file": os.path.relpath(path, ROOT), "stale": stale}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# CPU legs (reference code; test-infrastructure libraries under oracle/)

def cpu_reference_rate(n_kyber: int, n_dil: int, threads: int):
    """Reference round trip (forward_inplace + intt_inverse) on host threads.

    Returns (polys/s, kind, seconds).  Uses oracle/_ref (the unmodified reference) when
    it was built; otherwise the C restatement (oracle/liboracle.so)."""
    from oracle.oracle import IMPROVED, Oracle, Reference, reference_available

    o = Oracle()
    kyb = o.rng(12345, KYBER_Q, n_kyber * 256)
    dil = o.rng(54321, DIL_Q, n_dil * 256)
    if reference_available():
        ref = Reference()
        # the reference admits `improved` for Kyber at n = 32 (bit-identical outputs to the
        # engine's n = 16) and for Dilithium via exact-bound params
        pk = ref.params(KYBER_Q, 256, 32, (IMPROVED,))
        pd = ref.params(DIL_Q, 256, 32, (IMPROVED,), exact=True)
        t = pk.time_batch(IMPROVED, 1, kyb, threads) + pd.time_batch(IMPROVED, 1, dil, threads)
        return (n_kyber + n_dil) / t, "reference", t
    # fallback: the oracle port, threaded over polynomials
    from concurrent.futures import ThreadPoolExecutor

    qk = o.params(KYBER_Q, 256, 32, (IMPROVED,))
    qd = o.params(DIL_Q, 256, 32, (IMPROVED,), exact=True)

    def work(args):
        P, arr = args
        P.inverse(IMPROVED, P.forward(IMPROVED, arr))

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        jobs = [(qk, c) for c in np.array_split(kyb.reshape(-1, 256), threads)]
        jobs += [(qd, c) for c in np.array_split(dil.reshape(-1, 256), threads)]
        list(ex.map(work, jobs))
    t = time.perf_counter() - t0
    return (n_kyber + n_dil) / t, "port", t


def run_reference_arm(a, rank, world):
    if rank != 0:
        return 0
    threads = host_threads()
    per_step_k = max(2, threads * 2048)   # bounded sample per step, 2:1 Kyber:Dilithium
    per_step_d = max(1, threads * 1024)
    for _ in range(a.warmup):
        cpu_reference_rate(per_step_k // 8, per_step_d // 8, threads)
    total_t, total_polys, kind = 0.0, 0, "reference"
    for _ in range(a.steps):
        r, kind, t = cpu_reference_rate(per_step_k, per_step_d, threads)
        total_t += t
        total_polys += per_step_k + per_step_d
    value = total_polys / total_t
    sample = (f"each step: {per_step_k} Kyber + {per_step_d} Dilithium polys, fwd+inv, "
              f"{threads} host threads ({cpu_model()})")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * total_t / a.steps,
        "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (reference Rng, uniform [0,q))",
        "config": workload_config(a, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "cpu": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# engine arm

def _time_ms(torch, fn, iters, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def _cpu_rate(fn, units, min_s=0.3):
    """units/s of fn() repeated until at least min_s of wall time."""
    t, reps = 0.0, 0
    while t < min_s:
        t += fn()
        reps += 1
    return units * reps / t, t, reps


def table2_cpu_reference(q, N):
    """The reference's own path at a Table 2 preset on ONE host thread (the reference is
    single-threaded), per kind: ntt_forward_inplace and intt_inverse, each timed directly
    (transform.hpp:228-231, 339-343) over >= 1 s / >= 2 s of repeated batches
    (oracle/_ref, the unmodified reference headers); None if not built."""
    from oracle.oracle import HARVEY, IMPROVED, NTL, SCOTT, Oracle, Reference, reference_available

    if not reference_available():
        return None
    ref = Reference()
    kinds = {"ntl": NTL, "harvey": HARVEY, "scott": SCOTT, "improved": IMPROVED}
    rp = ref.params(q, N, 32, tuple(kinds.values()))
    n = 256 if N <= 512 else 128
    a = Oracle().rng(77, q, n * N)
    out = {}
    for kname, k in kinds.items():
        fwd, tf, rf = _cpu_rate(lambda: rp.time_batch(k, 0, a.copy(), 1), n, 1.0)
        spec = rp.forward(k, a.reshape(n, N)).ravel()
        inv, ti, ri = _cpu_rate(lambda: rp.time_batch(k, 2, spec.copy(), 1), n, 2.0)
        out[kname] = {"cpu_ref_fwd_ns_per_poly": 1e9 / fwd, "cpu_ref_inv_ns_per_poly": 1e9 / inv,
                      "cpu_ref_sample": f"{n} polys x {rf} (fwd, {tf:.1f} s) / x {ri} (inv, "
                                        f"{ti:.1f} s), 1 thread"}
    return out


def extras_cpu_baselines():
    """The reference's CPU path beside every BASELINE config (1 thread and all host threads):
    config 1/2 negacyclic trees through the reference's own cores (oracle/_ref ref_tree_run,
    restated loop), config 2's reference-pinned twin cyclic_convolution_via_ntt
    (transform.hpp:372-379), config 3 the Dilithium round trip (ntt_forward_inplace +
    intt_inverse), config 5 the checked reductions (reduction.hpp:125-273)."""
    from oracle.oracle import HARVEY, IMPROVED, NEGA, SMONT, Oracle, Reference, reference_available

    if not reference_available():
        return None
    ref, o = Reference(), Oracle()
    thr = host_threads()
    out = {"cpu": cpu_model(), "threads": thr}

    def both(fn, units):  # (1 thread, all threads) units/s
        r1, t1, _ = _cpu_rate(lambda: fn(1), units, 0.3)
        rn, tn, _ = _cpu_rate(lambda: fn(thr), units, 0.3)
        return {"one_thread": r1, "all_threads": rn}

    B = 8192
    f = o.rng(101, KYBER_Q, B * 256)
    g = o.rng(102, KYBER_Q, B * 256)
    out["config1_kyber7_fwd"] = dict(unit="polys/s", kind="reference cores (ref_tree_run)",
                                     **both(lambda t: ref.time_tree(KYBER_Q, 256, 16, NEGA, 7, IMPROVED, 0,
                                                                    f.copy(), threads=t), B))
    c2 = {"unit": "products/s", "kind": "reference cores (ref_tree_run: 2 fwd + basemul + inv)"}
    for name, k in (("modified_plantard", IMPROVED), ("montgomery_R2^16", HARVEY),
                    ("signed_montgomery", SMONT)):
        c2[name] = both(lambda t, k=k: ref.time_tree(KYBER_Q, 256, 16, NEGA, 7, k, 2, f[:2048 * 256].copy(),
                                                     g[:2048 * 256], threads=t), 2048)
    RP = ref.params(KYBER_Q, 256, 32, (IMPROVED, HARVEY))
    c2["cyclic_convolution_via_ntt_improved_n32"] = both(
        lambda t: RP.time_convolution(IMPROVED, f[:2048 * 256], g[:2048 * 256], t), 2048)
    out["config2_kyber_polymul"] = c2
    dil = o.rng(103, DIL_Q, B * 256)
    c3 = {"unit": "polys/s", "kind": "reference (ntt_forward_inplace + intt_inverse)"}
    for name, k, exact in (("modified_plantard_n32", IMPROVED, True), ("montgomery_n32", HARVEY, False)):
        R3 = ref.params(DIL_Q, 256, 32, (k,), exact=exact)
        c3[name] = both(lambda t, R3=R3, k=k: R3.time_batch(k, 1, dil.copy(), t), B)
    out["config3_dilithium_roundtrip"] = c3
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from sweep_inputs import CONFIGS, NAMES, grid

    c5 = {"unit": "mults/s", "kind": "reference checked reductions (ref_sweep)",
          "sample": "2^10 rows x 2^15 columns of each config-5 grid"}
    for q, n, ell in CONFIGS:
        for v in range(4):
            A, Bv = grid(q, n, ell, v)
            A = A[:1024]

            def sweep(t, A=A, Bv=Bv, v=v, q=q, n=n, ell=ell):
                from concurrent.futures import ThreadPoolExecutor

                t0 = time.perf_counter()
                with ThreadPoolExecutor(t) as ex:
                    list(ex.map(lambda a: ref.sweep_checksum(v, q, n, ell, a, Bv),
                                np.array_split(A, t)))
                return time.perf_counter() - t0
            c5[f"q{q}_{NAMES[v]}"] = both(sweep, A.size * Bv.size)
    out["config5_sweep"] = c5
    return out

def run_extras(dev):
    """The other BASELINE.json configs, device-resident, CUDA events (secondary fields)."""
    import torch

    import paper_2402_00675_b200.nttk as nttk

    K = nttk.ButterflyKind
    NEG = nttk.Tree.negacyclic
    g = torch.Generator(device=dev).manual_seed(99)
    ex = {}
    # config 1: Kyber-style forward, 4096 polys, 7 layers (degree-2 leaves), improved n=16
    P1 = nttk.build_params(KYBER_Q, 256, 16, [K.improved], tree=NEG, layers=7, exact_bound=True)
    x = torch.randint(0, KYBER_Q, (4096, 256), generator=g, device=dev, dtype=torch.int32).to(torch.int16)
    y = torch.empty_like(x)
    ms = _time_ms(torch, lambda: nttk.forward(P1, K.improved, x, y), 200, 10)
    # the same call through a captured plan (nttk_plan_create: 50 forwards in one CUDA graph):
    # device time per call without the host's per-call work
    gms = None
    try:
        plan = nttk.Plan(P1, K.improved, nttk.Plan.FORWARD, x, y, repeat=50)
        gms = _time_ms(torch, plan.launch, 20, 3) / 50
        del plan
    except Exception as e:  # report, do not fail the bench line
        gms = f"plan capture failed: {e}"
    ex["config1_kyber7_fwd_4096"] = {
        "us_per_call": ms * 1e3, "polys_per_s": 4096 / (ms / 1e3),
        "graph_us_per_call": gms * 1e3 if isinstance(gms, float) else gms,
        "graph_polys_per_s": 4096 / (gms / 1e3) if isinstance(gms, float) else None}
    # config 2: Kyber-style polymul (7-layer fwd x2, basemul, inverse), 65536 pairs, per variant
    B = 65536
    xa = torch.randint(0, KYBER_Q, (B, 256), generator=g, device=dev, dtype=torch.int32).to(torch.int16)
    xb = torch.randint(0, KYBER_Q, (B, 256), generator=g, device=dev, dtype=torch.int32).to(torch.int16)
    xc = torch.empty_like(xa)
    c2 = {}
    census, _ = sass_census()
    n_smsp = 4 * torch.cuda.get_device_properties(dev).multi_processor_count
    clk_hz = 1.965e9  # the pool's SM clock under load (bench clocks record)
    for name, kind in (("modified_plantard", K.improved), ("montgomery_R2^16", K.harvey),
                       ("signed_montgomery", K.smont)):
        P2 = nttk.build_params(KYBER_Q, 256, 16, [kind], tree=NEG, layers=7, exact_bound=True)
        ms = _time_ms(torch, lambda: nttk.polymul(P2, kind, xa, xb, xc), 20)
        c2[name] = {"ms": ms, "products_per_s": B / (ms / 1e3)}
        # executed-instruction roof: fmaheavy cycles per product of the kernel's SASS loop
        cyc = (census or {}).get("pm_" + name)
        if cyc:
            roof = n_smsp * clk_hz / cyc
            c2[name].update({"imad_executed_roof_products_per_s": roof,
                             "frac_of_imad_executed_roof": B / (ms / 1e3) / roof,
                             "fmaheavy_cycles_per_product": cyc})
    # the standalone basemul kernel (product.cu) on the same 65536 pairs of forward spectra:
    # HBM-bound, 3 x 512 B per polynomial pair (two spectra in, one product out)
    peak, _ = measured_peaks()
    for name, kind in (("modified_plantard", K.improved), ("montgomery_R2^16", K.harvey),
                       ("signed_montgomery", K.smont)):
        P2 = nttk.build_params(KYBER_Q, 256, 16, [kind], tree=NEG, layers=7, exact_bound=True)
        fa, fb = nttk.forward(P2, kind, xa), nttk.forward(P2, kind, xb)
        ms = _time_ms(torch, lambda: nttk.basemul(P2, kind, fa, fb, xc), 20)
        gbs = 3 * B * 512 / (ms / 1e3) / 1e9
        c2[name]["standalone_basemul"] = {"ms": ms, "GBps": gbs, "frac_of_hbm": gbs / peak}
    ex["config2_kyber_polymul_65536_fused"] = c2
    # config 3: Dilithium round trip, 65536 polys, modified Plantard n=32 vs 32-bit Montgomery
    xd = torch.randint(0, DIL_Q, (B, 256), generator=g, device=dev, dtype=torch.int32)
    sd, od = torch.empty_like(xd), torch.empty_like(xd)
    c3 = {}
    # the paper's comparison set (Alg. 7-12): every butterfly kind at n = 32, each on its
    # own fast kernel
    for name, kind in (("modified_plantard_n32", K.improved), ("montgomery_n32", K.harvey),
                       ("scott_montgomery_n32", K.scott), ("ntl_shoup_n32", K.ntl),
                       ("signed_montgomery_n32", K.smont)):
        P3 = nttk.build_params(DIL_Q, 256, 32, [kind], exact_bound=True)
        assert kind in P3.fast_path, name

        def rt():
            nttk.forward(P3, kind, xd, sd)
            nttk.inverse(P3, kind, sd, od)

        ms = _time_ms(torch, rt, 20)
        assert torch.equal(od, xd)
        c3[name] = {"ms": ms, "polys_per_s": B / (ms / 1e3)}
    ex["config3_dilithium_roundtrip_65536"] = c3
    # every butterfly kind at an HBM-resident batch (2^20 polys, 512 MiB / 1 GiB in + out):
    # forward and inverse per kind, the GPU analogue of the paper's Table 2 comparison
    kt = {}
    for label, q, n, dt, kinds in (
            ("kyber_u16_n16", KYBER_Q, 16, torch.int16, (K.improved, K.harvey, K.ntl, K.smont)),
            ("dilithium_u32_n32", DIL_Q, 32, torch.int32,
             (K.improved, K.harvey, K.scott, K.ntl, K.smont))):
        Bk = 1 << 20
        xk = torch.randint(0, q, (Bk, 256), generator=g, device=dev, dtype=torch.int32).to(dt)
        sk, ok = torch.empty_like(xk), torch.empty_like(xk)
        row = {}
        for kind in kinds:
            Pk = nttk.build_params(q, 256, n, [kind], exact_bound=True)
            assert kind in Pk.fast_path, (label, kind)
            fms = _time_ms(torch, lambda: nttk.forward(Pk, kind, xk, sk), 10)
            ims = _time_ms(torch, lambda: nttk.inverse(Pk, kind, sk, ok), 10)
            assert torch.equal(ok, xk), (label, kind)
            row[kind.name] = {"fwd_ms": fms, "inv_ms": ims,
                              "fwd_polys_per_s": Bk / (fms / 1e3), "inv_polys_per_s": Bk / (ims / 1e3)}
        kt[label] = row
        del xk, sk, ok
    ex["kinds_2^20"] = kt
    # the paper's Table 2 parameter sets (params.hpp:273-306 presets, n = 32, u32 storage):
    # every kind, forward and inverse, a steady-state batch of 2^27 coefficients (512 MiB in
    # + 512 MiB out: 2^19 / 2^18 / 2^17 polys), with each kernel's HBM roof per polynomial
    peak, _ = measured_peaks()
    t2 = {"batch": "2^27 coefficients (u32) per call", "hbm_peak_GBps": peak}
    for name in ("kyber256", "newhope512", "newhope1024"):
        Pp = nttk.preset(name)
        Np, qp = Pp.size, Pp.p
        Bp = (1 << 27) // Np
        xp = torch.randint(0, qp, (Bp, Np), generator=g, device=dev, dtype=torch.int32)
        sp, op = torch.empty_like(xp), torch.empty_like(xp)
        row = {}
        for kind in (K.ntl, K.harvey, K.scott, K.improved):
            fms = _time_ms(torch, lambda: nttk.forward(Pp, kind, xp, sp), 10)
            ims = _time_ms(torch, lambda: nttk.inverse(Pp, kind, sp, op), 10)
            assert torch.equal(op, xp), (name, kind)
            roof = 2 * Np * 4 / (peak * 1e9) * 1e9  # ns per polynomial at the HBM peak
            row[kind.name] = {"fwd_ns_per_poly": fms * 1e6 / Bp, "inv_ns_per_poly": ims * 1e6 / Bp,
                              "hbm_roof_ns_per_poly": roof,
                              "fwd_frac_of_hbm": roof / (fms * 1e6 / Bp),
                              "inv_frac_of_hbm": roof / (ims * 1e6 / Bp),
                              "fast_path": kind in Pp.fast_path,
                              "n16_product": bool(kind == K.improved and Pp.fast_flags(kind, 0) & 512),
                              "ct_form_inverse": bool(kind == K.improved and Pp.fast_flags(kind, 1) & 2048)}
        cpu = table2_cpu_reference(qp, Np)
        if cpu:
            for kname, v in cpu.items():
                row[kname].update(v)
        t2[name] = row
        del xp, sp, op
    ex["table2_presets"] = t2
    # config 5: reduction sweep, 2^30 operand pairs (2^15 x 2^15 grid) per (q, variant) from
    # tests/golden/sweep_inputs.py; every checksum must equal the unmodified reference's over
    # the same full grid (tests/golden/sweep_2p30.json) or the bench line fails.  "mults" are
    # grid pairs: the row operand's premultiplication (a mu, a k, a p^-1) is done once per
    # row, so each pair costs the reduction's remaining multiplies (IMAD 1/64, IMAD.HI and
    # IMAD.WIDE 1/32 SM-cycles per lane-op, measured)
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from sweep_inputs import CONFIGS, NAMES, grid

    with open(os.path.join(ROOT, "tests", "golden", "sweep_2p30.json")) as fh:
        ref_sums = {(r["q"], r["variant"]): r["checksum"] for r in json.load(fh)["rows"]}
    cost = {(16, 0): 3 / 64, (16, 1): 3 / 64, (16, 2): 2 / 64, (16, 3): 2 / 64,
            (32, 0): 5 / 64, (32, 1): 5 / 64, (32, 2): 5 / 64, (32, 3): 5 / 64}
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    c5 = {"grid": "2^15 rows x 2^15 columns per (q, reduction), tests/golden/sweep_inputs.py",
          "validated": "checksum == the reference's checked reductions over the full grid "
                       "(tests/golden/sweep_2p30.json)"}
    for q, n, ell in CONFIGS:
        for v in range(4):
            Ah, Bh = grid(q, n, ell, v)
            A, Bv = torch.from_numpy(Ah).to(dev), torch.from_numpy(Bh).to(dev)
            got = "%016x" % nttk.modmul_sweep(v, q, n, ell, A, Bv)  # synchronous form
            if got != ref_sums[(q, v)]:
                raise RuntimeError(f"config5 sweep checksum {got} != reference {ref_sums[(q, v)]} "
                                   f"(variant {NAMES[v]}, q {q})")
            want = int(got, 16)
            cs = torch.zeros(1, dtype=torch.int64, device=dev)
            for _ in range(3):  # warm-up (module load, occupancy query, clocks)
                nttk.modmul_sweep_device(v, q, n, ell, A, Bv, cs)
            reps = 20
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            cs.zero_()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):  # device form: queued back to back, one checksum word
                nttk.modmul_sweep_device(v, q, n, ell, A, Bv, cs)
            e1.record()
            torch.cuda.synchronize()
            sec = e0.elapsed_time(e1) / 1e3 / reps
            if (int(cs.item()) & (2**64 - 1)) != (want * reps) & (2**64 - 1):
                raise RuntimeError(f"config5 timed sweep checksum mismatch (variant {v}, q {q})")
            rate = (1 << 30) / sec
            roof = n_sm * 1965e6 / cost[(n, v)]
            c5[f"q{q}_{NAMES[v]}"] = {"grid_pairs_per_s": rate, "imad_roof_pairs_per_s": roof,
                                      "frac": rate / roof, "checksum": got}
    ex["config5_sweep_2^30"] = c5
    return ex


def run_e2e(a, torch, dist, nttk, Pk, Pd, IMP, xk, xd, world, dev, polys_per_step):
    """The same step end to end through the C ABI host entry point (nttk_roundtrip_host:
    pinned host buffers, H2D + kernels + D2H inside the timed region), each rank on its own
    shard.  The pinned allocation is agreed on by all ranks first, so a rank that cannot pin
    fails the e2e leg everywhere instead of leaving the others in a collective."""
    err, okf = None, torch.ones(1, device=dev)
    try:
        hk = torch.empty(tuple(xk.shape), dtype=torch.int16, pin_memory=True)
        hd = torch.empty(tuple(xd.shape), dtype=torch.int32, pin_memory=True)
        ohk, ohd = torch.empty_like(hk, pin_memory=True), torch.empty_like(hd, pin_memory=True)
    except Exception as ex:
        err = f"{type(ex).__name__}: {ex}"
        okf.zero_()
    if world > 1:
        dist.all_reduce(okf, op=dist.ReduceOp.MIN)
    if okf.item() == 0:
        raise RuntimeError(err or "pinned host allocation failed on another rank")
    hk.copy_(xk)
    hd.copy_(xd)
    nttk.roundtrip_host(Pk, IMP, hk, None, ohk)
    nttk.roundtrip_host(Pd, IMP, hd, None, ohd)
    if world > 1:
        dist.barrier()
    te = time.perf_counter()
    for _ in range(a.e2e_steps):
        nttk.roundtrip_host(Pk, IMP, hk, None, ohk)
        nttk.roundtrip_host(Pd, IMP, hd, None, ohd)
    dt = torch.tensor([time.perf_counter() - te], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    assert torch.equal(ohk, hk) and torch.equal(ohd, hd), "e2e round trip mismatch"
    nbytes = torch.tensor([hk.numel() * 2 + hd.numel() * 4], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(nbytes)
    return {"value": polys_per_step * a.e2e_steps / float(dt.item()), "unit": UNIT,
            "h2d_bytes_per_step": int(nbytes.item()), "d2h_bytes_per_step": int(nbytes.item()),
            "path": "nttk_roundtrip_host (C ABI, pinned host buffers, 3-stream pipeline); "
                    "wall clock, max over ranks"}


def gather_check(a, torch, dist, sh, sk, sd, nk_total, nd_total, seed_k, seed_d, dev):
    """All-gather the forward-spectrum shards (Sharder.gather: NCCL), timed with CUDA
    events; rank 0 checks sampled polynomials of the gathered batch against the CPU oracle
    (the checker, outside every timed region)."""
    from oracle.oracle import IMPROVED, Oracle

    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gk = sh.gather(sk, nk_total)
    gd = sh.gather(sd, nd_total)
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    out = {"gather_ms": float(ms.item()),
           "bytes": int(gk.numel() * 2 + gd.numel() * 4), "collective": "Sharder.gather "
           "(torch.distributed all_gather, NCCL)"}
    if sh.rank == 0:
        o = Oracle()
        rs = np.random.RandomState(0)
        ok = True
        for P, g, q, n, seed, total in (
                (o.params(KYBER_Q, 256, 16, (IMPROVED,), exact=True), gk, KYBER_Q, 16, seed_k, nk_total),
                (o.params(DIL_Q, 256, 32, (IMPROVED,), exact=True), gd, DIL_Q, 32, seed_d, nd_total)):
            idx = np.sort(rs.choice(total, 16, replace=False))
            x = global_batch(torch, seed, q, total, torch.int16 if q == KYBER_Q else torch.int32, dev)
            f = x[torch.from_numpy(idx).to(dev)].cpu().numpy().astype(np.int64).astype(np.uint64)
            want = P.forward(IMPROVED, f).astype(np.int64)
            mask = 0xFFFF if q == KYBER_Q else 0xFFFFFFFF
            got = g[torch.from_numpy(idx).to(dev)].cpu().numpy().astype(np.int64) & mask
            ok &= bool((got == want).all())
            del x
        out["sampled_polys_vs_oracle"] = "16 Kyber + 16 Dilithium, bit-exact" if ok else "MISMATCH"
        if not ok:
            raise RuntimeError("gathered spectra differ from the oracle")
    return out


def global_batch(torch, seed, q, total, dtype, dev):
    """The seeded global input batch every rank draws identically (strong scaling)."""
    g = torch.Generator(device=dev).manual_seed(seed)
    return torch.randint(0, q, (total, 256), generator=g, device=dev, dtype=torch.int32).to(dtype)


def run_engine_arm(a, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2402_00675_b200.nttk as nttk
    from paper_2402_00675_b200.shard import Sharder

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    Pk = nttk.build_params(KYBER_Q, 256, 16, [nttk.ButterflyKind.improved], exact_bound=True)
    Pd = nttk.build_params(DIL_Q, 256, 32, [nttk.ButterflyKind.improved], exact_bound=True)
    IMP = nttk.ButterflyKind.improved
    assert IMP in Pk.fast_path and IMP in Pd.fast_path

    plan = shard_plan(a, rank, world)
    nk_total, nd_total = plan["kyber_total"], plan["dilithium_total"]
    seed_k, seed_d = 1234, 4321
    sh = Sharder(rank, world) if a.scaling == "strong" else Sharder(0, 1)
    if a.scaling == "strong":  # one global seeded batch, this rank's contiguous shard
        xk_all = global_batch(torch, seed_k, KYBER_Q, nk_total, torch.int16, dev)
        xd_all = global_batch(torch, seed_d, DIL_Q, nd_total, torch.int32, dev)
        xk = sh.run(lambda part: part, xk_all)
        xd = sh.run(lambda part: part, xd_all)
    else:  # weak: every rank its own full per-GPU batch
        xk = global_batch(torch, seed_k + rank, KYBER_Q, 1 << a.kyber_log2, torch.int16, dev)
        xd = global_batch(torch, seed_d + rank, DIL_Q, 1 << a.dil_log2, torch.int32, dev)
    nk, nd = xk.shape[0], xd.shape[0]
    sk, sd = torch.empty_like(xk), torch.empty_like(xd)
    ok, od = torch.empty_like(xk), torch.empty_like(xd)
    stream = torch.cuda.current_stream(dev)

    names = ["kyber_fwd", "kyber_inv", "dil_fwd", "dil_inv"]
    calls = [lambda: nttk.forward(Pk, IMP, xk, sk), lambda: nttk.inverse(Pk, IMP, sk, ok),
             lambda: nttk.forward(Pd, IMP, xd, sd), lambda: nttk.inverse(Pd, IMP, sd, od)]
    # algorithmic HBM bytes per launch: read + write of the coefficient arrays
    alg_bytes = [nk * 256 * 2 * 2, nk * 256 * 2 * 2, nd * 256 * 4 * 2, nd * 256 * 4 * 2]

    def step(evs=None):
        for i, c in enumerate(calls):
            if evs is not None:
                evs[i][0].record(stream)
            c()
            if evs is not None:
                evs[i][1].record(stream)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    # correctness guard on the measured data: round trip must be the identity
    assert torch.equal(ok, xk) and torch.equal(od, xd), "round trip mismatch"

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in calls]
           for _ in range(a.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = nttk.launch_count()
    with ClockSampler(local_rank) as clk:
        t0.record(stream)
        for k in range(a.steps):
            step(evs[k])
        t1.record(stream)
        torch.cuda.synchronize()
    launches = nttk.launch_count() - launches0
    if world > 1:
        dist.barrier()
    elapsed_ms = t0.elapsed_time(t1)
    per_kernel = [np.mean([evs[k][i][0].elapsed_time(evs[k][i][1]) for k in range(a.steps)])
                  for i in range(len(calls))]
    tm = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    max_ms = float(tm.item())
    polys_per_step = nk_total + nd_total
    value = polys_per_step * a.steps / (max_ms / 1e3)
    shards = None
    if world > 1:
        sizes = torch.tensor([nk, nd], dtype=torch.int64, device=dev)
        allz = [torch.empty_like(sizes) for _ in range(world)]
        dist.all_gather(allz, sizes)
        shards = [{"rank": r, "kyber_polys": int(z[0]), "dilithium_polys": int(z[1])}
                  for r, z in enumerate(allz)]

    # roofline of the dominant kernel: HBM (algorithmic bytes in + out) against the measured
    # copy bandwidth, beside the IMAD issue roof under two cost models:
    # algorithmic = the reference algorithm's modmuls per polynomial (N/2 log N forward,
    # + N inverse) x the fmaheavy cost of one modmul (measured IMAD 1/64, IMAD.HI 1/32
    # SM-cycles per lane-op, profiles/r2_imad_microbench.txt); executed = the fmaheavy cycles
    # of the kernel's own SASS loop (profiles/r*_sass_census.json)
    dom = int(np.argmax(per_kernel))
    peak, peak_src = measured_peaks()
    achieved = alg_bytes[dom] / (per_kernel[dom] / 1e3) / 1e9
    sm_hz = 1965e6 if not clk.samples else 1e6 * float(np.median([s[0] for s in clk.samples]))
    n_sm = torch.cuda.get_device_properties(local_rank).multi_processor_count
    cyc = [3 / 64, 3 / 64, 5 / 64, 5 / 64]
    modmuls = [1024, 1024 + 256, 1024, 1024 + 256]
    polys = [nk, nk, nd, nd]
    alg_ms = [p_ * m * c / (n_sm * sm_hz) * 1e3 for p_, m, c in zip(polys, modmuls, cyc)]
    census, census_src = sass_census()
    exe_ms = None
    if census and all(k in census for k in names):
        # SMSP-cycles per polynomial spread over 4 sub-partitions per SM
        exe_ms = [p_ * census[k] / (4 * n_sm * sm_hz) * 1e3 for p_, k in zip(polys, names)]
    hbm_ms = [b / (peak * 1e9) * 1e3 for b in alg_bytes]
    traffic = ncu_traffic(names[dom], nk, nd)

    def bind(imad_ms):
        return ["imad" if i > h else "hbm" for i, h in zip(imad_ms, hbm_ms)]

    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "kernel": names[dom],
                "peak_source": peak_src,
                "per_kernel_ms": dict(zip(names, [round(x, 4) for x in per_kernel])),
                "per_kernel_GBps": dict(zip(names, [round(b / (t / 1e3) / 1e9, 1)
                                                    for b, t in zip(alg_bytes, per_kernel)])),
                "per_kernel_frac_of_hbm": dict(zip(names, [round(h / t, 3)
                                                           for h, t in zip(hbm_ms, per_kernel)])),
                "step_frac_of_hbm": sum(hbm_ms) / sum(per_kernel),
                "imad_algorithmic": {
                    "definition": "reference modmuls per poly (fwd 1024, inv 1280) x fmaheavy "
                                  "cost per modmul (n=16 IMAD+IMAD.HI = 3/64, n=32 IMAD+2 IMAD.HI "
                                  "= 5/64 SM-cycles per lane-op) at the sampled SM clock",
                    "roof_ms": dict(zip(names, [round(x, 4) for x in alg_ms])),
                    "frac": dict(zip(names, [round(r / t, 3) for r, t in zip(alg_ms, per_kernel)])),
                    "binding_roof": dict(zip(names, bind(alg_ms)))}}
    if exe_ms is not None:
        roofline["imad_executed"] = {
            "definition": "fmaheavy cycles of the kernel's SASS loop (2 x IMAD + 4 x IMAD.HI/WIDE "
                          "per warp-iteration of 2 polys) at the sampled SM clock",
            "source": census_src,
            "roof_ms": dict(zip(names, [round(x, 4) for x in exe_ms])),
            "frac": dict(zip(names, [round(r / t, 3) for r, t in zip(exe_ms, per_kernel)])),
            "binding_roof": dict(zip(names, bind(exe_ms)))}
    fwd_rate = polys_per_step / (max(per_kernel[0] + per_kernel[2], 1e-9) / 1e3)

    # end-to-end through the C ABI host entry point (pinned host buffers, copies timed)
    e2e = None
    if not a.no_e2e:
        try:
            e2e = run_e2e(a, torch, dist, nttk, Pk, Pd, IMP, xk, xd, world, dev, polys_per_step)
        except Exception as ex:  # e.g. pinned host memory exhausted with many ranks per host
            e2e = {"value": None, "unit": UNIT, "error": f"{type(ex).__name__}: {ex}"[:300]}
    gathered = None
    if a.gather and world > 1:  # NCCL only to gather results when asked, outside timing
        if a.scaling != "strong":
            raise SystemExit("--gather needs --scaling strong (one global batch)")
        gathered = gather_check(a, torch, dist, sh, sk, sd, nk_total, nd_total, seed_k, seed_d, dev)

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        threads = host_threads()
        smp_k, smp_d = threads * 4096, threads * 2048
        tot_t, reps, kind = 0.0, 0, "reference"
        while tot_t < 2.0 and reps < 50:  # ~2 s wall x all host threads of CPU work
            _, kind, t = cpu_reference_rate(smp_k, smp_d, threads)
            tot_t += t
            reps += 1
        rate = reps * (smp_k + smp_d) / tot_t
        # the reference is single-threaded: one core, same workload mix
        _, _, t1 = cpu_reference_rate(16384, 8192, 1)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": kind, "cpu": cpu_model(),
               "sample": (f"{reps} x ({smp_k} Kyber + {smp_d} Dilithium) polys fwd+inv, "
                          f"{tot_t:.1f} s wall on {threads} threads"),
               "value_1_core": 24576 / t1,
               "sample_1_core": f"16384 Kyber + 8192 Dilithium polys fwd+inv, 1 thread, {t1:.2f} s"}

    extras = None
    if rank == 0 and world == 1 and not a.no_extras:  # single-GPU configs: N = 1 runs only
        extras = run_extras(dev)
        if not a.no_cpu_baseline:
            extras["cpu_reference_per_config"] = extras_cpu_baselines()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": max_ms / a.steps, "higher_is_better": True,
            "scaling": a.scaling, "vs_baseline": None, "dtype": "u32",
            "data": "synthetic uniform [0,q) (torch.randint, seeded)",
            "config": workload_config(a, world, shards),
            "fwd_only_polys_per_s": fwd_rate,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clk.summary(),
        }
        if extras is not None:
            line["extras"] = extras
        if gathered is not None:
            line["gather"] = gathered
        print(json.dumps(line), flush=True)
    return 0


KIND_ORDER = ("ntl", "harvey", "scott", "improved")  # all_butterfly_kinds()


def pairwise_gains(results):
    """bench.hpp:146-175: later-over-earlier kind pairs per preset, (base - kind)/base %."""
    out = []
    for preset in dict.fromkeys(r["preset"] for r in results):
        mean = {r["kind"]: r["mean_us"] for r in results if r["preset"] == preset}
        for b in range(len(KIND_ORDER)):
            for k in range(b + 1, len(KIND_ORDER)):
                kb, kk = KIND_ORDER[b], KIND_ORDER[k]
                if kb in mean and kk in mean:
                    out.append({"preset": preset, "kind": kk, "baseline": kb,
                                "gain_percent": (mean[kb] - mean[kk]) / mean[kb] * 100.0})
    return out


def bench_report(outdir, presets=("kyber256", "falcon512", "falcon1024"), seed=12345):
    """GPU rows in the reference's BenchReport schema 1 (transform mode: per-polynomial
    forward time), next to the reference's own run_bench on one host thread."""
    import platform

    import torch

    import paper_2402_00675_b200.nttk as nttk

    K = nttk.ButterflyKind
    B, R = 1 << 16, 10
    g = torch.Generator(device="cuda").manual_seed(seed)
    results = []
    for name in presets:
        P = nttk.preset(name)
        x = torch.randint(0, P.p, (B, P.size), generator=g, device="cuda", dtype=torch.int32)
        y = torch.empty_like(x)
        for kname in KIND_ORDER:
            kind = K[kname]
            for _ in range(3):
                nttk.forward(P, kind, x, y)
            samples = []
            for _ in range(R):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                nttk.forward(P, kind, x, y)
                e1.record()
                torch.cuda.synchronize()
                samples.append(e0.elapsed_time(e1) * 1e3 / B)  # us per polynomial
            m = float(np.mean(samples))
            results.append({"preset": name, "kind": kname, "iters": B * R, "mean_us": m,
                            "std_us": float(np.std(samples, ddof=1))})
    try:
        nv = subprocess.run(["nvcc", "--version"], capture_output=True, text=True).stdout.strip()
        nv = nv.splitlines()[-1]
    except Exception:
        nv = "nvcc"
    gpu = {"schema": 1, "mode": "transform", "iters": B * R, "seed": seed,
           "machine": {"os": f"{platform.system()} {platform.release()} {platform.machine()}",
                       "cpu": f"{torch.cuda.get_device_name(0)} (sm_100a), batched 2^16 polys/launch",
                       "compiler": nv,
                       "flags": "-O3 -gencode arch=compute_100a,code=sm_100a"},
           "results": results, "gains": pairwise_gains(results)}
    os.makedirs(outdir, exist_ok=True)
    with open(os.path.join(outdir, "gpu_bench_report.json"), "w") as fh:
        json.dump(gpu, fh, indent=1)
    cpu = None
    from oracle.oracle import Reference, reference_available

    if reference_available():
        cpu = Reference().run_bench(presets, iters=2000, seed=seed)
        with open(os.path.join(outdir, "cpu_reference_bench_report.json"), "w") as fh:
            json.dump(cpu, fh, indent=1)
    lines = ["| preset | kind | GPU us/poly | CPU reference us/poly (1 thread) | ratio |",
             "|---|---|---|---|---|"]
    cmap = {(r["preset"], r["kind"]): r["mean_us"] for r in (cpu or {}).get("results", [])}
    for r in results:
        c = cmap.get((r["preset"], r["kind"]))
        lines.append(f"| {r['preset']} | {r['kind']} | {r['mean_us']:.5f} | "
                     f"{'' if c is None else f'{c:.3f}'} | {'' if c is None else f'{c / r['mean_us']:.0f}x'} |")
    with open(os.path.join(outdir, "bench_report.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))
    return 0


def plan_only(a, rank, world):
    """Launcher / sharder check without GPU work: every rank computes its shard plan, the
    plans are all-gathered (gloo), rank 0 prints one JSON line."""
    import torch.distributed as dist

    plan = shard_plan(a, rank, world)
    rows = [None] * world
    if world > 1:
        dist.all_gather_object(rows, plan)
    else:
        rows = [plan]
    if rank == 0:
        print(json.dumps({"n_gpus": world, "scaling": a.scaling,
                          "shards": [{"rank": r, "kyber": list(p["kyber"]),
                                      "dilithium": list(p["dilithium"])}
                                     for r, p in enumerate(rows)],
                          "kyber_total": plan["kyber_total"],
                          "dilithium_total": plan["dilithium_total"]}), flush=True)
    return 0


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    a = parse(argv)
    if a.bench_report:
        return bench_report(a.bench_report)
    if "WORLD_SIZE" not in os.environ and a.gpus > 1:
        return relaunch(argv, a.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        print(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if a.impl == "reference":
        if world > 1 and rank != 0:
            return 0
        return run_reference_arm(a, rank, world)
    if a.plan_only:
        import torch.distributed as dist

        if world > 1:
            dist.init_process_group("gloo")
        try:
            return plan_only(a, rank, world)
        finally:
            if world > 1:
                dist.destroy_process_group()
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return run_engine_arm(a, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
