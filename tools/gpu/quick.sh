# quick check: parity suite + forward/inverse/polymul/fastn timings
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-q}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
tail -2 $O/gputest.log
{ python tools/fwd_probe.py kyber 22 20; python tools/fwd_probe.py kyber 22 20
  for pr in kyber256 newhope512 newhope1024; do timeout 120 python tools/fastn_probe.py $pr improved 17 10; done
  timeout 300 python tools/polymul_probe.py 50; } 2>&1 | tee $O/times.txt
