cp paper_2402_00675_b200/libnttk_gpu.so /tmp/swz3.so
for rep in 1 2; do for v in swz0 swz1 swz2 swz3; do
  if [ $v = swz3 ]; then cp /tmp/swz3.so paper_2402_00675_b200/libnttk_gpu.so; else cp variants/$v.so paper_2402_00675_b200/libnttk_gpu.so; fi
  timeout 300 python bench.py --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$v', round(d['value']/1e9,4), d['roofline']['per_kernel_ms'])"
done; done
