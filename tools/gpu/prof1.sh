# ncu captures of the N=512/1024 and Kyber N=256 kernels; summaries only travel back
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/p1
O=gpurun_out/p1
python tools/fastn_probe.py newhope512 improved 17 10 > $O/fastn_times.txt 2>&1
python tools/fastn_probe.py newhope1024 improved 16 10 >> $O/fastn_times.txt 2>&1
python tools/fastn_probe.py kyber256 improved 17 10 >> $O/fastn_times.txt 2>&1
cap() {  # name, kernel regex, command...
  n=$1; k=$2; shift 2
  timeout 900 ncu --set full --clock-control none -k regex:"$k" -c 2 -o /tmp/$n -f "$@" > $O/$n.log 2>&1
  ncu -i /tmp/$n.ncu-rep --page raw --csv > $O/$n.raw.csv 2>/dev/null
  ncu -i /tmp/$n.ncu-rep --page details --csv > $O/$n.details.csv 2>/dev/null
}
cap fastn512 "fwdn_tma|invn_tma" python tools/fastn_probe.py newhope512 improved 17 1
cap fastn1024 "fwdn_tma|invn_tma" python tools/fastn_probe.py newhope1024 improved 16 1
cap kyber "fwd256_tma|inv256_tma" python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline --no-e2e
tail -5 $O/*.log
du -sh $O
