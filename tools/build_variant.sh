#!/usr/bin/env bash
# A/B variants of the TMA kernels: recompile fast256_tma.cu with extra -D flags and link
# it against the already built objects into variants/<name>.so (travels with gpurun).
#   tools/build_variant.sh alt0 -DNTTK_ALT_MASK=0
# On the box:  cp variants/alt0.so paper_2402_00675_b200/libnttk_gpu.so && python bench.py ...
set -euo pipefail
name=$1
shift
cd "$(dirname "$0")/.."
make -s lib
mkdir -p variants build/variants
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc -O3 -lineinfo -std=c++17 $ARCH -Xcompiler -fPIC --expt-relaxed-constexpr "$@" \
  -c paper_2402_00675_b200/csrc/fast256_tma.cu -o build/variants/$name.o
objs=$(ls build/obj/*.o | grep -v fast256_tma.o)
nvcc $ARCH -shared -o variants/$name.so build/variants/$name.o $objs -cudart static \
  -Xlinker -z,defs -lpthread -ldl -lrt
echo "variants/$name.so"
