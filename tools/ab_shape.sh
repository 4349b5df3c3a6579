#!/bin/bash
mkdir -p gpurun_out/ab8
for round in 1 2; do
  for v in default m3s2 m2s3 m3s1; do
    if [ $v = default ]; then unset XFT_LIB; else export XFT_LIB=tune/libxft_$v.so; fi
    timeout 200 python tools/tune_time.py --tag $v >> gpurun_out/ab8/cfg2.txt 2>> gpurun_out/ab8/err.txt
  done
done
for v in default m3s2 m2s3 m3s1; do
  if [ $v = default ]; then unset XFT_LIB; else export XFT_LIB=tune/libxft_$v.so; fi
  timeout 200 python tools/time_rows.py --n 8192 --rows 8192 --dtype c64 >> gpurun_out/ab8/rows.txt 2>> gpurun_out/ab8/err.txt
  timeout 200 python tools/time_rows.py --n 2048 --rows 32768 --dtype c64 >> gpurun_out/ab8/rows.txt 2>> gpurun_out/ab8/err.txt
done
cat gpurun_out/ab8/cfg2.txt gpurun_out/ab8/rows.txt; tail -5 gpurun_out/ab8/err.txt
