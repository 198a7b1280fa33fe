# GPU check: parity suite, smoke, A/B probes of the changed kernels (outputs under gpurun_out/$1)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-chk}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
tail -3 $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
tail -1 $O/smoke.log
for x in 0 1; do NTTK_POLYMUL_EAGER=$x timeout 300 python tools/polymul_probe.py 50 > $O/polymul_eager$x.txt 2>&1; done
for pr in kyber256 newhope512 newhope1024; do
  for k in improved harvey; do timeout 120 python tools/fastn_probe.py $pr $k 17 10 >> $O/fastn.txt 2>&1; done
done
cat $O/polymul_eager*.txt $O/fastn.txt
