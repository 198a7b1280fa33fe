cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-cf}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
tail -2 $O/gputest.log
for pr in kyber256 newhope512 newhope1024; do timeout 120 python tools/fastn_probe.py $pr improved 17 10; done 2>&1 | tee $O/fastn.txt
python tools/fwd_probe.py kyber 22 20 | tee -a $O/fastn.txt
