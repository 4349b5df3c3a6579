#!/bin/bash
# full GPU suite on the in-tree build, then A/B of the prefetch placement (tune/libxft_pfe.so)
mkdir -p gpurun_out/s8
python -m pytest tests -m gpu -x -q > gpurun_out/s8/gputest.log 2>&1; tail -3 gpurun_out/s8/gputest.log
for round in 1 2; do
  for v in default pfe; do
    if [ $v = default ]; then unset XFT_LIB; else export XFT_LIB=tune/libxft_$v.so; fi
    timeout 200 python tools/tune_time.py --tag $v >> gpurun_out/s8/cfg2.txt 2>> gpurun_out/s8/err.txt
    timeout 200 python tools/tune_time.py --config cfg4 --tag $v >> gpurun_out/s8/cfg4.txt 2>> gpurun_out/s8/err.txt
    timeout 200 python tools/time_rows16k.py >> gpurun_out/s8/rows.txt 2>> gpurun_out/s8/err.txt
  done
done
cat gpurun_out/s8/cfg2.txt gpurun_out/s8/cfg4.txt gpurun_out/s8/rows.txt; tail -5 gpurun_out/s8/err.txt
