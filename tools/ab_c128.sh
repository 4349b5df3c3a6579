#!/bin/bash
mkdir -p gpurun_out/ab10
for round in 1 2; do
  for v in default early sp2 sp2e; do
    if [ $v = default ]; then unset XFT_LIB; else export XFT_LIB=tune/libxft_$v.so; fi
    timeout 200 python tools/tune_time.py --tag $v >> gpurun_out/ab10/cfg2.txt 2>> gpurun_out/ab10/err.txt
  done
done
cat gpurun_out/ab10/cfg2.txt; tail -5 gpurun_out/ab10/err.txt
