# CT-form narrow inverse at N = 512 / 1024: parity of the fastn / narrow tests, then the A/B
# against the GS narrow body (NTTK_INV_CT=0) and the F-form masks (variants/ctnCS.so, built with
# tools/build_variant.sh from temporary -D switches of ct_f3_contiguous; the switches were removed
# once the per-N choice was made, so only the GS / CT rows can be re-run as is)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-ctn}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "fastn or narrow or preset or table2 or smoke" > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
tail -3 $O/gputest.log
cp paper_2402_00675_b200/libnttk_gpu.so /tmp/base.so
for rep in 1 2; do
  for p in newhope512 newhope1024; do
    echo "GS  $(NTTK_INV_CT=0 python tools/fastn_probe.py $p improved 17 20)"
    for v in base variants/ctn00 variants/ctn10 variants/ctn11; do
      if [ $v = base ]; then cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so; else cp $v.so paper_2402_00675_b200/libnttk_gpu.so; fi
      echo "$v $(python tools/fastn_probe.py $p improved 17 20)"
    done
    cp /tmp/base.so paper_2402_00675_b200/libnttk_gpu.so
  done
done 2>&1 | tee $O/ab.txt
