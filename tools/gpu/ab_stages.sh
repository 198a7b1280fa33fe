# A/B of the u16 stage counts (variants/st*.so from tools/build_variant.sh)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-stages}
mkdir -p $O
cp paper_2402_00675_b200/libnttk_gpu.so /tmp/base.so
for rep in 1 2; do
  for v in base variants/stf5 variants/stf6 variants/stf8 variants/sti3 variants/sti4; do
    if [ $v = base ]; then cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so; else cp $v.so paper_2402_00675_b200/libnttk_gpu.so; fi
    echo "$v: $(python tools/fwd_probe.py kyber 22 20) | $(python tools/inv_probe.py kyber 22 20)"
  done
done 2>&1 | tee $O/ab.txt
cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so
