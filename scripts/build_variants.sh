#!/bin/bash
# Builds kernel variants of libgosma.so into scripts/variants/ for A/B timing:
#   [SRC=objective_kernel] scripts/build_variants.sh NAME "-DFLAG=..." [NAME "-D..."]...
# (SRC: the csrc/*.cu translation unit the flags apply to; default bounds_kernel)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_1812_01232_b200/csrc
SRC=${SRC:-bounds_kernel}
mkdir -p $ROOT/scripts/variants
make -s -C $C
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC -I$ROOT/include -I$C -Xptxas -v --expt-relaxed-constexpr $flags \
    -c -o /tmp/bk_$name.o $C/$SRC.cu 2> $ROOT/scripts/variants/$name.ptxas.log
  objs=$(ls $C/build/*.o | grep -v $SRC.o)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared \
    -o $ROOT/scripts/variants/libgosma_$name.so /tmp/bk_$name.o $objs -lpthread
  echo "$name: $(grep -E 'Used' $ROOT/scripts/variants/$name.ptxas.log | head -3 | tr '\n' ' ')"
done
