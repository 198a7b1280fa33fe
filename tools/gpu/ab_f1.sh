# A/B of the F1 forward (NTTK_FWD_F1=0 keeps the umulhi form): parity first, then timing
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-f1}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
tail -2 $O/gputest.log
NTTK_FWD_F1=0 timeout 900 python -m pytest tests -m gpu -x -q -k "forward or golden or smoke or config or extreme" > $O/gputest_f0.log 2>&1; echo "pytest(F1 off) rc=$?" >> $O/gputest_f0.log
tail -2 $O/gputest_f0.log
for rep in 1 2 3; do
  for x in 0 1; do echo -n "F1=$x "; NTTK_FWD_F1=$x python tools/fwd_probe.py kyber 22 20; done
done 2>&1 | tee $O/ab.txt
NTTK_FWD_F1=1 python tools/fastn_probe.py kyber256 improved 20 10 | tee -a $O/ab.txt
NTTK_FWD_F1=0 python tools/fastn_probe.py kyber256 improved 20 10 | tee -a $O/ab.txt
