# 256-bit vs 128-bit stores of the u16 forward output (variants/no256.so: tools/build_variant.sh with a temporary -D switch, removed afterwards)
cd $GRAFT_REPO_ROOT
cp paper_2402_00675_b200/libnttk_gpu.so /tmp/base.so
for rep in 1 2 3; do
  for v in base variants/no256; do
    if [ $v = base ]; then cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so; else cp $v.so paper_2402_00675_b200/libnttk_gpu.so; fi
    echo "$v: $(python tools/fwd_probe.py kyber 22 20) | $(python tools/nega_probe.py 22 20 2>/dev/null | head -1)"
  done
done
cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so
timeout 600 python -m pytest tests -m gpu -x -q -k "forward or golden or misaligned or offset or random or smoke" 2>&1 | tail -2
for v in base variants/no256; do
  if [ $v = base ]; then cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so; else cp $v.so paper_2402_00675_b200/libnttk_gpu.so; fi
  python bench.py --steps 100 --warmup 30 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v step', d['ms_per_step'], d['roofline']['per_kernel_ms'], d['clocks']['sm_mhz'])"
done
cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so
