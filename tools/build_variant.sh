#!/bin/bash
# build_variant.sh NAME "-DFLAGS..." : builds tune/libxft_NAME.so (tuning only)
set -e
cd "$(dirname "$0")/../paper_0912_1379_b200/csrc"
OUT=../../tune/libxft_$1.so
B=../../tune/build_$1
mkdir -p $B
A="-gencode arch=compute_100a,code=sm_100a"
OBJS=""
for f in *.cu; do
  nvcc -O3 -std=c++17 -lineinfo $A -Xcompiler -fPIC --expt-relaxed-constexpr $2 -c $f -o $B/${f%.cu}.o &
  OBJS="$OBJS $B/${f%.cu}.o"
done
wait
nvcc $A -shared -o $OUT $OBJS -lcudart
