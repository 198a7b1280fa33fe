cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-ct32}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
tail -3 $O/gputest.log
for rep in 1 2 3; do for x in 0 1; do echo "CT=$x $(NTTK_INV_CT=$x python tools/inv_probe.py dilithium 21 20) | $(NTTK_INV_CT=$x python tools/inv_probe.py kyber 22 20)"; done; done 2>&1 | tee $O/ab.txt
