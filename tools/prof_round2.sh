#!/bin/bash
# ncu captures of the final round-2 kernels (run under gpurun; one ncu use per call).
# Each program first runs without ncu (the recipe's rule), then one --set full capture;
# the reports are summarised on the box (text only comes back: gpurun_out <= 64 MiB).
O=gpurun_out/prof2
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
summ() {  # report, kernel substring, tag
  python tools/ncu_summary.py $1.ncu-rep > $O/summary_$3.txt 2>&1
  python tools/ncu_stalls.py $1.ncu-rep $2 30 > $O/stalls_$3.txt 2>&1
  python tools/ncu_lines.py $1.ncu-rep $2 > $O/lines_$3.txt 2>&1
  python tools/ncu_opmix.py $1.ncu-rep $2 > $O/opmix_$3.txt 2>&1
  rm -f $1.ncu-rep
}
T=/tmp/prof2
mkdir -p $T
python tools/prof_cfg.py cfg2c128 3 > $O/plain_c128.log 2>&1 && \
  $NCU -k regex:xft_pipe_kernel -s 2 -c 1 -o $T/c128 python tools/prof_cfg.py cfg2c128 3 > $O/ncu_c128.log 2>&1 && \
  summ $T/c128 xft_pipe_kernel c128
python tools/prof_cfg.py cfg2c64 3 > $O/plain_c64.log 2>&1 && \
  $NCU -k regex:xft_pipe_kernel -s 2 -c 1 -o $T/c64 python tools/prof_cfg.py cfg2c64 3 > $O/ncu_c64.log 2>&1 && \
  summ $T/c64 xft_pipe_kernel c64
python tools/prof_cfg.py cfg3 2 > $O/plain_cfg3.log 2>&1 && \
  $NCU -k regex:xft_blue_kernel -s 2 -c 2 -o $T/cfg3 python tools/prof_cfg.py cfg3 2 > $O/ncu_cfg3.log 2>&1 && \
  summ $T/cfg3 xft_blue_kernel cfg3_blue
python tools/prof_2d.py 1 > $O/plain_2d.log 2>&1 && \
  $NCU -k regex:xft_pipe_kernel -s 1 -c 1 -o $T/rows16k python tools/prof_2d.py 1 > $O/ncu_rows16k.log 2>&1 && \
  summ $T/rows16k xft_pipe_kernel rows16k
# launch lists (per-launch device time and DRAM bytes) of the bench workloads
for c in cfg2 cfg3 cfg5; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $O/launches_$c.csv python tools/prof_cfg.py $c 2 > $O/ncu_launch_$c.log 2>&1 || true
done
ls -la $O
