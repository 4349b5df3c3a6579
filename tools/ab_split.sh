#!/bin/bash
# A/B: split next-row prefetch at 2/4 CTAs per SM (c64) and the L2 bulk prefetch, vs the in-tree build
mkdir -p gpurun_out/ab3
for round in 1 2; do
  for v in default sp4 l2pf sp4l; do
    if [ $v = default ]; then unset XFT_LIB; else export XFT_LIB=tune/libxft_$v.so; fi
    timeout 200 python tools/tune_time.py --tag $v >> gpurun_out/ab3/cfg2.txt 2>> gpurun_out/ab3/err.txt
  done
done
for v in default sp4 l2pf sp4l; do
  if [ $v = default ]; then unset XFT_LIB; else export XFT_LIB=tune/libxft_$v.so; fi
  timeout 200 python tools/time_rows.py --n 8192 --rows 8192 --dtype c64 >> gpurun_out/ab3/rows.txt 2>> gpurun_out/ab3/err.txt
  timeout 200 python tools/tune_time.py --config cfg4 --tag $v >> gpurun_out/ab3/cfg4.txt 2>> gpurun_out/ab3/err.txt
  timeout 200 python tools/time_rows16k.py >> gpurun_out/ab3/rows.txt 2>> gpurun_out/ab3/err.txt
done
cat gpurun_out/ab3/cfg2.txt gpurun_out/ab3/rows.txt gpurun_out/ab3/cfg4.txt; tail -5 gpurun_out/ab3/err.txt
