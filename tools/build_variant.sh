#!/bin/bash
# A/B builds: relink lib/libifgf_b200.so with CUDA sources recompiled under extra flags.
#   tools/build_variant.sh <name> "<cuda/a.cu cuda/b.cu ...>" "<nvcc flags>"  -> lib/variants/<name>.so
# (select with IFGF_B200_LIB=paper_2112_06316_b200/lib/variants/<name>.so)
set -e
NAME=$1; SRCS=$2; FLAGS=$3
cd "$(dirname "$0")/../paper_2112_06316_b200/csrc"
make -s -j8 >/dev/null
OBJ=../build/obj; VD=../build/variants/$NAME; rm -rf $VD; mkdir -p $VD ../lib/variants
OBJS=$(find $OBJ -name '*.o')
: > $VD/ptxas.log
for SRC in $SRCS; do
  B=$(basename $SRC .cu)
  EXTRA=""
  case $SRC in cuda/beta_kernel.cu|cuda/coneplan_kernels.cu|cuda/proximity_kernels.cu) EXTRA=--fmad=false;; esac
  /usr/local/cuda/bin/nvcc -std=c++20 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
    -Xcompiler -fopenmp -ccbin /usr/bin/g++ --expt-relaxed-constexpr -Xptxas -v $EXTRA $FLAGS -c $SRC \
    -o $VD/$B.o 2>> $VD/ptxas.log
  OBJS=$(echo "$OBJS" | grep -v "/cuda/$B.o$")
done
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -ccbin /usr/bin/g++ \
  -o ../lib/variants/$NAME.so $OBJS $VD/*.o -lgomp -lnccl
grep -B1 Used $VD/ptxas.log | grep -o "[0-9]* bytes spill stores\|Used [0-9]* registers" | paste - - | sort | uniq -c
