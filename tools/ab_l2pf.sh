#!/bin/bash
# A/B of the row kernels' L2 prefetch depth: in-tree build (depth 1 where enabled) vs depth 2, 3 and off
mkdir -p gpurun_out/ab4
for round in 1 2; do
  for v in default d2a d3 off; do
    if [ $v = default ]; then unset XFT_LIB; else export XFT_LIB=tune/libxft_$v.so; fi
    timeout 200 python tools/tune_time.py --tag $v >> gpurun_out/ab4/cfg2.txt 2>> gpurun_out/ab4/err.txt
    timeout 200 python tools/tune_time.py --config cfg4 --tag $v >> gpurun_out/ab4/cfg4.txt 2>> gpurun_out/ab4/err.txt
    timeout 200 python tools/time_rows16k.py >> gpurun_out/ab4/rows.txt 2>> gpurun_out/ab4/err.txt
  done
done
for v in default d2a d3 off; do
  if [ $v = default ]; then unset XFT_LIB; else export XFT_LIB=tune/libxft_$v.so; fi
  timeout 200 python tools/time_rows.py --n 8192 --rows 4096 --dtype c128 >> gpurun_out/ab4/rows.txt 2>> gpurun_out/ab4/err.txt
  timeout 200 python tools/time_rows.py --n 2048 --rows 16384 --dtype c128 >> gpurun_out/ab4/rows.txt 2>> gpurun_out/ab4/err.txt
  timeout 200 python tools/time_rows.py --n 2048 --rows 32768 --dtype c64 >> gpurun_out/ab4/rows.txt 2>> gpurun_out/ab4/err.txt
  timeout 200 python tools/time_rows.py --n 256 --rows 262144 --dtype c64 >> gpurun_out/ab4/rows.txt 2>> gpurun_out/ab4/err.txt
done
cat gpurun_out/ab4/cfg2.txt gpurun_out/ab4/cfg4.txt gpurun_out/ab4/rows.txt; tail -5 gpurun_out/ab4/err.txt
