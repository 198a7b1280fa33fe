#!/usr/bin/env bash
# A/B variants of the TMA kernels: recompile fast256_tma.cu with extra -D flags and link
# it against the already built objects into variants/<name>.so (travels with gpurun).
#   tools/build_variant.sh alt0 -DNTTK_ALT_MASK=0
#   SRC=sweep tools/build_variant.sh r256 -DNTTK_SWEEP_ROWS=256   (another csrc/<SRC>.cu)
# On the box:  cp variants/alt0.so paper_2402_00675_b200/libnttk_gpu.so && python bench.py ...
set -euo pipefail
name=$1
shift
src=${SRC:-fast256_tma}
cd "$(dirname "$0")/.."
make -s lib
mkdir -p variants build/variants
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc -O3 -lineinfo -std=c++17 $ARCH -Xcompiler -fPIC --expt-relaxed-constexpr "$@" \
  -c paper_2402_00675_b200/csrc/$src.cu -o build/variants/$name.o
objs=$(ls build/obj/*.o | grep -v "/$src.o")
nvcc $ARCH -shared -o variants/$name.so build/variants/$name.o $objs -cudart static \
  -Xlinker -z,defs -lpthread -ldl -lrt
echo "variants/$name.so"
