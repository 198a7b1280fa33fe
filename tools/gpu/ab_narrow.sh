cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-nf}
mkdir -p $O
cp paper_2402_00675_b200/libnttk_gpu.so /tmp/base.so
for rep in 1 2; do
  for v in base variants/nf1 variants/nf2 variants/nf1n variants/nf2n; do
    if [ $v = base ]; then cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so; else cp $v.so paper_2402_00675_b200/libnttk_gpu.so; fi
    echo "$v: $(python tools/fastn_probe.py kyber256 improved 17 10) | $(python tools/fastn_probe.py newhope512 improved 17 10) | $(python tools/fastn_probe.py newhope1024 improved 17 10)"
  done
done 2>&1 | tee $O/ab.txt
cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so
