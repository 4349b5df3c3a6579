#!/bin/bash
# ncu captures of the final round-2 kernels (run under gpurun; one ncu use per call).
# Each program first runs without ncu (the recipe's rule), then one --set full capture.
set -e
O=gpurun_out/prof2
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
python tools/prof_cfg.py cfg2c128 3 > $O/plain_c128.log 2>&1 && \
  $NCU -k regex:xft_pipe_kernel -s 2 -c 1 -o $O/c128 python tools/prof_cfg.py cfg2c128 3 > $O/ncu_c128.log 2>&1
python tools/prof_cfg.py cfg2c64 3 > $O/plain_c64.log 2>&1 && \
  $NCU -k regex:xft_pipe_kernel -s 2 -c 1 -o $O/c64 python tools/prof_cfg.py cfg2c64 3 > $O/ncu_c64.log 2>&1
python tools/prof_cfg.py cfg3 2 > $O/plain_cfg3.log 2>&1 && \
  $NCU -k regex:xft_blue_kernel -s 2 -c 3 -o $O/cfg3 python tools/prof_cfg.py cfg3 2 > $O/ncu_cfg3.log 2>&1
python tools/prof_2d.py 1 > $O/plain_2d.log 2>&1 && \
  $NCU -k regex:xft_pipe_kernel -s 1 -c 1 -o $O/rows16k python tools/prof_2d.py 1 > $O/ncu_rows16k.log 2>&1
# launch lists (per-launch device time and DRAM bytes) of the bench workloads
for c in cfg2 cfg3 cfg5; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $O/launches_$c.csv python tools/prof_cfg.py $c 2 > $O/ncu_launch_$c.log 2>&1 || true
done
