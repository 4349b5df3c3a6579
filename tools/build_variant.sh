#!/bin/bash
# build_variant.sh NAME "-DFLAGS..." : builds tune/libxft_NAME.so (tuning only)
set -e
cd "$(dirname "$0")/../paper_0912_1379_b200/csrc"
OUT=../../tune/libxft_$1.so
B=../../tune/build_$1
mkdir -p $B
A="-gencode arch=compute_100a,code=sm_100a"
nvcc -O3 -std=c++17 -lineinfo $A -Xcompiler -fPIC --expt-relaxed-constexpr $2 -c xft_capi.cu -o $B/capi.o
nvcc -O3 -std=c++17 -lineinfo $A -Xcompiler -fPIC --expt-relaxed-constexpr $2 -c xft_tables.cu -o $B/tables.o
nvcc $A -shared -o $OUT $B/capi.o $B/tables.o -lcudart
