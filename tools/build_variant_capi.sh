#!/bin/bash
# build_variant_capi.sh NAME "-DFLAGS..." : tune/libxft_NAME.so = the default objects (csrc/build, `make` first)
# with xft_capi.cu alone rebuilt under the flags (row-kernel tuning only)
set -e
cd "$(dirname "$0")/../paper_0912_1379_b200/csrc"
mkdir -p ../../tune
A="-gencode arch=compute_100a,code=sm_100a"
nvcc -O3 -std=c++17 -lineinfo $A -Xcompiler -fPIC --expt-relaxed-constexpr -diag-suppress 177 $2 -c xft_capi.cu -o ../../tune/capi_$1.o
OBJS=$(ls build/*.o | grep -v xft_capi.o)
nvcc $A -shared -o ../../tune/libxft_$1.so $OBJS ../../tune/capi_$1.o -lcudart -ldl
rm -f ../../tune/capi_$1.o
