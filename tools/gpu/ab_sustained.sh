# F1 (IADD3) vs F3 (IMAD) forms of Y' = 2X - X' under SUSTAINED load (the bench step, power-capped).
# The variants were built with tools/build_variant.sh from temporary -D switches in tma_common.cuh
# (removed after the measurement: F3 stayed); the base rows and tools/step_probe.py re-run as is.
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-sus}
mkdir -p $O
cp paper_2402_00675_b200/libnttk_gpu.so /tmp/base.so
for rep in 1 2; do
  for v in base variants/f1fwd variants/f1ct variants/f1both; do
    if [ $v = base ]; then cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so; else cp $v.so paper_2402_00675_b200/libnttk_gpu.so; fi
    python bench.py --steps 100 --warmup 30 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v', d['ms_per_step'], d['roofline']['per_kernel_ms'], d['clocks'])"
  done
done 2>&1 | tee $O/ab.txt
cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so
python tools/step_probe.py 20 | tee $O/step_probe.txt
