# F1/F3 forward of the 7-layer negacyclic Kyber tree vs the umulhi form (NTTK_FWD_F1=0): parity, then timing
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-f1n7}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
tail -2 $O/gputest.log
for rep in 1 2 3; do for x in 0 1; do echo "F1=$x $(NTTK_FWD_F1=$x python tools/nega_probe.py 22 20 | head -1)"; done; done 2>&1 | tee $O/ab.txt
NTTK_FWD_F1=1 python tools/c1_probe.py 4096,65536 | tee -a $O/ab.txt
NTTK_FWD_F1=0 python tools/c1_probe.py 4096,65536 | tee -a $O/ab.txt
