#!/bin/bash
# Mehler plan wave balancing (in-tree) vs off (tune/libxft_nowave.so), then the Mehler / chirp-z / concurrency tests
mkdir -p gpurun_out/ab9
for round in 1 2; do
  for v in default nowave; do
    if [ $v = default ]; then unset XFT_LIB; else export XFT_LIB=tune/libxft_$v.so; fi
    timeout 300 python tools/time_cfg3.py >> gpurun_out/ab9/cfg3.txt 2>> gpurun_out/ab9/err.txt
  done
done
unset XFT_LIB
cat gpurun_out/ab9/cfg3.txt; tail -5 gpurun_out/ab9/err.txt
timeout 1200 python -m pytest tests/test_gpu_chirpz.py tests/test_gpu_concurrency.py tests/test_gpu_cli_dense.py -m gpu -x -q > gpurun_out/ab9/test.log 2>&1; tail -5 gpurun_out/ab9/test.log
