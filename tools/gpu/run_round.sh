# parity suite + smoke + polymul A/B + full bench line (outputs under gpurun_out/$1)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-rr}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
tail -2 $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
tail -1 $O/smoke.log
for x in 0 1; do NTTK_POLYMUL_EAGER=$x timeout 300 python tools/polymul_probe.py 50 > $O/polymul_eager$x.txt 2>&1; done
cat $O/polymul_eager*.txt
timeout 600 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
tail -1 $O/bench.log
