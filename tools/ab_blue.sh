#!/bin/bash
# Mehler apply A/B: hoff = no staging/prefetch, st0 = shared-memory staging only, pf1/pf2/pf3 = L2 prefetches only
mkdir -p gpurun_out/ab6
for round in 1 2; do
  for v in hoff st0 pf1 pf2 pf3; do
    export XFT_LIB=tune/libxft_$v.so
    timeout 300 python tools/time_cfg3.py >> gpurun_out/ab6/cfg3.txt 2>> gpurun_out/ab6/err.txt
  done
done
cat gpurun_out/ab6/cfg3.txt; tail -5 gpurun_out/ab6/err.txt
