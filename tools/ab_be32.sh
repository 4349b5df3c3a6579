#!/bin/bash
mkdir -p gpurun_out/ab14
for round in 1 2; do
  for v in default be32; do
    if [ $v = default ]; then unset XFT_LIB; else export XFT_LIB=tune/libxft_$v.so; fi
    timeout 300 python tools/time_cfg3.py >> gpurun_out/ab14/cfg3.txt 2>> gpurun_out/ab14/err.txt
  done
done
cat gpurun_out/ab14/cfg3.txt; tail -5 gpurun_out/ab14/err.txt
