# round-2 evidence: ncu launch list of the bench command, ncu --set full of the bench kernels,
# the fused polymul and the N = 512/1024 kernels (raw pages exported on the box), SASS-free
# microbenchmarks (transpose A/B) -- outputs under gpurun_out/$1
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-prof2}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/xpose_mb.bin tools/xpose_microbench.cu && /tmp/xpose_mb.bin > $O/xpose_mb.txt 2>&1
# launch list of the bench command (cold-cache, serialised; share of the step matters)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline --no-e2e > $O/launches_run.log 2>&1
cap() {  # name, kernel regex, count, command...
  n=$1; k=$2; c=$3; shift 3
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$k" -c $c -o /tmp/$n -f "$@" > $O/$n.log 2>&1
  ncu -i /tmp/$n.ncu-rep --page raw --csv > $O/$n.raw.csv 2>/dev/null
  ncu -i /tmp/$n.ncu-rep --page details --csv > $O/$n.details.csv 2>/dev/null
  ncu -i /tmp/$n.ncu-rep --page source --csv --print-source sass > $O/$n.source.csv 2>/dev/null
  ls -la /tmp/$n.ncu-rep >> $O/$n.log
}
cap bench "fwd256_tma|inv256_tma" 4 python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline --no-e2e
cap polymul "polymul256" 3 python tools/polymul_probe.py 1
cap fastn "fwdn_tma|invn_tma" 4 python tools/fastn_probe.py newhope1024 improved 17 1
du -sh $O; ls $O
