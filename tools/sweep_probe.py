"""Config-5 reduction-sweep probe: the bench's 2^30-pair sweep for every (q, variant),
device-timed over queued launches, printed as one line per case (frac of the IMAD roof)."""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_00675_b200.nttk as nttk  # noqa: E402

COST = {(16, 0): 3 / 64, (16, 1): 3 / 64, (16, 2): 2 / 64, (16, 3): 2 / 64,
        (32, 0): 5 / 64, (32, 1): 5 / 64, (32, 2): 5 / 64, (32, 3): 5 / 64}
NAMES = ["mont_redc", "signed_mont_redc", "plantard_redc", "modified_plantard_mul"]


def main():
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    for q, n, ell in ((3329, 16, 2), (8380417, 32, 7)):
        for v in range(4):
            if len(sys.argv) > 1 and sys.argv[1] not in f"q{q}_{NAMES[v]}":
                continue
            hi_b = {1: None, 2: q + 1, 3: q << ell}.get(v, q)
            A = torch.randint(0, q + (v == 2), (1 << 15,), generator=g, device=dev, dtype=torch.int64)
            if v == 1:
                B = torch.randint(-(1 << (n - 1)), 1 << (n - 1), (1 << 15,), generator=g, device=dev,
                                  dtype=torch.int64)
            else:
                B = torch.randint(0, hi_b, (1 << 15,), generator=g, device=dev, dtype=torch.int64)
            want = nttk.modmul_sweep(v, q, n, ell, A, B)
            cs = torch.zeros(1, dtype=torch.int64, device=dev)
            for _ in range(3):
                nttk.modmul_sweep_device(v, q, n, ell, A, B, cs)
            reps = 20
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            cs.zero_()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):
                nttk.modmul_sweep_device(v, q, n, ell, A, B, cs)
            e1.record()
            torch.cuda.synchronize()
            sec = e0.elapsed_time(e1) / 1e3 / reps
            ok = (int(cs.item()) & (2**64 - 1)) == (want * reps) & (2**64 - 1)
            rate = (1 << 30) / sec
            roof = n_sm * 1965e6 / COST[(n, v)]
            print(f"q{q} {NAMES[v]:24s} {sec * 1e6:8.1f} us  {rate:.3e} mults/s  frac {rate / roof:.3f}"
                  f"  checksum {'ok' if ok else 'MISMATCH'}", flush=True)


if __name__ == "__main__":
    main()
