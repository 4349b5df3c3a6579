#!/bin/bash
# A/B: the row's last rendezvous replaced by "the last-arriving warp hands the stage back" (XFT_XTAIL=1: issue after
# the last pass as before, 2: c128 too issues right away) vs the in-tree build
mkdir -p gpurun_out/ab13
for round in 1 2; do
  for v in default xt1 xt2; do
    if [ $v = default ]; then unset XFT_LIB; else export XFT_LIB=tune/libxft_$v.so; fi
    timeout 200 python tools/tune_time.py --tag $v >> gpurun_out/ab13/cfg2.txt 2>> gpurun_out/ab13/err.txt
    timeout 200 python tools/tune_time.py --config cfg4 --tag $v >> gpurun_out/ab13/cfg2.txt 2>> gpurun_out/ab13/err.txt
    timeout 200 python tools/time_rows.py --n 8192 --rows 4096 --dtype c128 >> gpurun_out/ab13/cfg2.txt 2>> gpurun_out/ab13/err.txt
    timeout 200 python tools/time_rows.py --n 8192 --rows 8192 --dtype c64 >> gpurun_out/ab13/cfg2.txt 2>> gpurun_out/ab13/err.txt
    timeout 200 python tools/time_rows16k.py >> gpurun_out/ab13/cfg2.txt 2>> gpurun_out/ab13/err.txt
  done
done
cat gpurun_out/ab13/cfg2.txt; tail -5 gpurun_out/ab13/err.txt
