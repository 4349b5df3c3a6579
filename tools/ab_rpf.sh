#!/bin/bash
mkdir -p gpurun_out/ab11
for round in 1 2; do
  for v in default rpf1 rpf2 rpf4; do
    if [ $v = default ]; then unset XFT_LIB; else export XFT_LIB=tune/libxft_$v.so; fi
    timeout 200 python tools/time_colring.py >> gpurun_out/ab11/colring.txt 2>> gpurun_out/ab11/err.txt
  done
done
cat gpurun_out/ab11/colring.txt; tail -5 gpurun_out/ab11/err.txt
