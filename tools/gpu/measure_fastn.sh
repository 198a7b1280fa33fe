# after the CT-form narrow inverse (N = 512 / 1024): full parity, stress, bench line, reference
# arm, ncu captures of the fastn inverses -- outputs under gpurun_out/$1
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-measure_fastn}
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
tail -2 $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python tools/stress_fastn.py 20 > $O/stress_fastn.txt 2>&1; tail -2 $O/stress_fastn.txt
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/bench_ref.log
cap() {  # name, kernel regex, count, skip, command...
  n=$1; k=$2; c=$3; sk=$4; shift 4
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $sk -c $c -o /tmp/$n -f "$@" > $O/$n.log 2>&1
  ncu -i /tmp/$n.ncu-rep --page raw --csv > $O/$n.raw.csv 2>/dev/null
}
cap fastn512 "fwdn_tma|invn_tma" 2 4 python tools/fastn_probe.py newhope512 improved 17 1
cap fastn1024 "fwdn_tma|invn_tma" 2 4 python tools/fastn_probe.py newhope1024 improved 17 1
ls $O
