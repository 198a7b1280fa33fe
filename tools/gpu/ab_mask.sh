# A/B of the F1 layer mask (variants/f1m*.so built by tools/build_variant.sh)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-mask}
mkdir -p $O
cp paper_2402_00675_b200/libnttk_gpu.so /tmp/base.so
for rep in 1 2; do
  for v in base variants/f1m3c variants/f1m5c variants/f1mcc variants/f1m1c variants/f1mf0 variants/f1me0; do
    if [ $v = base ]; then cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so; else cp $v.so paper_2402_00675_b200/libnttk_gpu.so; fi
    echo -n "$v: "; python tools/fwd_probe.py kyber 22 20
  done
done 2>&1 | tee $O/ab.txt
cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so
