"""bench.py's multi-GPU launcher and sharding on CPU (gloo, world size 2): `--gpus 2`
without torchrun re-launches itself as 2 ranks, each computes its Sharder shard of the fixed
config-4 batch (strong scaling) and rank 0 prints the plan.  No GPU work (--plan-only)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, env=None):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=240, env=env)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    return out.returncode, lines


def test_gpus2_strong_shards_the_fixed_batch():
    rc, lines = _run("--gpus", "2", "--plan-only", "--kyber-log2", "10", "--dil-log2", "9")
    assert rc == 0 and len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    k = [tuple(s["kyber"]) for s in d["shards"]]
    dl = [tuple(s["dilithium"]) for s in d["shards"]]
    assert k == [(0, 512), (512, 1024)] and dl == [(0, 256), (256, 512)]
    assert d["kyber_total"] == 1024 and d["dilithium_total"] == 512


def test_gpus2_weak_keeps_per_rank_batches():
    rc, lines = _run("--gpus", "2", "--plan-only", "--scaling", "weak", "--kyber-log2", "10",
                     "--dil-log2", "9")
    d = json.loads(lines[0])
    assert rc == 0 and d["scaling"] == "weak"
    assert all(tuple(s["kyber"]) == (0, 1024) for s in d["shards"])
    assert d["kyber_total"] == 2048


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    rc, _ = _run("--gpus", "2", "--plan-only", env=env)
    assert rc == 2
