cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-ctm}
mkdir -p $O
cp paper_2402_00675_b200/libnttk_gpu.so /tmp/base.so
for rep in 1 2; do
  for v in base variants/ct00 variants/ct07 variants/ct38 variants/ct15 variants/ct2a variants/ct3c; do
    if [ $v = base ]; then cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so; else cp $v.so paper_2402_00675_b200/libnttk_gpu.so; fi
    echo "$v: $(python tools/inv_probe.py kyber 22 20)"
  done
done 2>&1 | tee $O/ab.txt
cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so
