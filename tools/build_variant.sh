#!/bin/bash
# build_variant.sh <csrc_dir> <out.so> [nvcc -D flags...]: experimental library builds (not product)
set -e
SRC=$1; OUT=$2; shift 2
OBJ=$(mktemp -d)
for f in capi.cu fill.cu fused.cu keyctr.cu scaled.cu keygen.cpp; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 "$@" -c $SRC/$f -o $OBJ/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT $OBJ/*.o
rm -rf $OBJ
