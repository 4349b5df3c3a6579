#!/bin/bash
# build_variant_blue.sh NAME "-DFLAGS..." : tune/libxft_NAME.so = the default objects (csrc/build, `make` first)
# with xft_bluestein.cu alone rebuilt under the flags (chirp-z / Mehler kernel tuning only)
set -e
cd "$(dirname "$0")/../paper_0912_1379_b200/csrc"
mkdir -p ../../tune
A="-gencode arch=compute_100a,code=sm_100a"
nvcc -O3 -std=c++17 -lineinfo $A -Xcompiler -fPIC --expt-relaxed-constexpr -diag-suppress 177 $2 -c xft_bluestein.cu -o ../../tune/blue_$1.o
OBJS=$(ls build/*.o | grep -v xft_bluestein.o)
nvcc $A -shared -o ../../tune/libxft_$1.so $OBJS ../../tune/blue_$1.o -lcudart -ldl
rm -f ../../tune/blue_$1.o
