cp paper_2402_00675_b200/libnttk_gpu.so /tmp/base.so
for r in 1 2; do
for v in base s3 s4; do
  if [ $v = base ]; then cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so; else cp variants/$v.so paper_2402_00675_b200/libnttk_gpu.so; fi
  echo -n "$v "; python bench.py --no-extras --no-cpu-baseline --no-e2e --steps 20 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,4), d['roofline']['per_kernel_ms'])"
done
done
cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so
