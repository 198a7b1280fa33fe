# round-2 closing measurement after the CT-form inverses: parity, smoke, bench line, reference
# arm, ncu launch list and one full capture of the four config-4 kernels -- outputs under gpurun_out/$1
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-measure}
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
tail -2 $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/bench_ref.log
tail -1 $O/bench.log | cut -c1-600; tail -2 $O/bench_ref.log | cut -c1-400
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/ncu_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fwd256_tma|inv256_tma" -s 12 -c 4 -o /tmp/c4 -f \
  python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
ncu -i /tmp/c4.ncu-rep --page raw --csv > $O/ncu_full.raw.csv 2>/dev/null
ncu -i /tmp/c4.ncu-rep --page details --csv > $O/ncu_full.details.csv 2>/dev/null
ls -la $O
