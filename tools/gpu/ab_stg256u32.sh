# 256-bit direct stores of the u32 forward outputs (N = 256 Dilithium, N = 512 / 1024) vs the coalesced stores
# through the transpose tile (variants/no256u32.so: temporary -D switch, removed afterwards)
cd $GRAFT_REPO_ROOT
cp paper_2402_00675_b200/libnttk_gpu.so /tmp/base.so
for rep in 1 2 3; do
  for v in base variants/no256u32; do
    if [ $v = base ]; then cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so; else cp $v.so paper_2402_00675_b200/libnttk_gpu.so; fi
    echo "$v: $(python tools/fwd_probe.py dilithium 21 20) | $(python tools/fastn_probe.py newhope512 improved 18 20) | $(python tools/fastn_probe.py newhope1024 improved 17 20) | $(python tools/fastn_probe.py newhope1024 harvey 17 20)"
  done
done
cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
