#!/bin/bash
mkdir -p gpurun_out/ab7
for round in 1 2; do
  for v in default e16; do
    if [ $v = default ]; then unset XFT_LIB; else export XFT_LIB=tune/libxft_$v.so; fi
    timeout 200 python tools/time_rows16k.py >> gpurun_out/ab7/rows.txt 2>> gpurun_out/ab7/err.txt
  done
done
cat gpurun_out/ab7/rows.txt; tail -5 gpurun_out/ab7/err.txt
