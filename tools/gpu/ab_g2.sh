# A/B of the paper-form (G2) Kyber inverse (NTTK_INV_G2=0 runs the umulhi lazy-merge form)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-g2}
mkdir -p $O
./tools/bff_mb.bin > $O/bff.txt 2>&1; grep -E "^G|^F3|^F1 paper|^F0 umulhi" $O/bff.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
tail -2 $O/gputest.log
cat > /tmp/inv_probe.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_2402_00675_b200.nttk as nttk
K = nttk.ButterflyKind
P = nttk.build_params(3329, 256, 16, [K.improved], exact_bound=True)
x = torch.randint(0, 3329, (1 << 22, 256), device="cuda", dtype=torch.int32).to(torch.int16)
y = nttk.forward(P, K.improved, x); z = torch.empty_like(x)
for _ in range(3): nttk.inverse(P, K.improved, y, z)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): nttk.inverse(P, K.improved, y, z)
e1.record(); torch.cuda.synchronize()
assert torch.equal(z, x)
print(f"kyber inv 2^22: {e0.elapsed_time(e1) / 20:.4f} ms")
PY
for rep in 1 2; do for x in 0 1; do echo -n "G2=$x "; NTTK_INV_G2=$x python /tmp/inv_probe.py; done; done 2>&1 | tee $O/ab.txt
python tools/fwd_probe.py kyber 22 20 | tee -a $O/ab.txt
