#!/bin/bash
# Round-2 final captures (after the split-barrier / L2-prefetch row kernels): --set full of the c128 config-2 row
# kernel and of the n = 16384 c64 row pass, launch lists of config 2, config 5 and of the bench command.
# Each program first runs without ncu (the recipe's rule); summaries only come back (gpurun_out <= 64 MiB).
O=gpurun_out/prof3
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
summ() {  # report, kernel substring, tag
  python tools/ncu_summary.py $1.ncu-rep > $O/ncu_full_$3.txt 2>&1
  python tools/ncu_stalls.py $1.ncu-rep $2 30 > $O/stalls_$3.txt 2>&1
  python tools/ncu_lines.py $1.ncu-rep $2 > $O/lines_$3.txt 2>&1
  rm -f $1.ncu-rep
}
T=/tmp/prof3
mkdir -p $T
python tools/prof_cfg.py cfg2c128 3 > $O/plain_c128.log 2>&1 && \
  $NCU -k regex:xft_pipe_kernel -s 2 -c 1 -o $T/c128 python tools/prof_cfg.py cfg2c128 3 > $O/ncu_c128.log 2>&1 && \
  summ $T/c128 xft_pipe_kernel c128_final
python tools/prof_2d.py 1 > $O/plain_2d.log 2>&1 && \
  $NCU -k regex:xft_pipe_kernel -s 1 -c 1 -o $T/rows16k python tools/prof_2d.py 1 > $O/ncu_rows16k.log 2>&1 && \
  summ $T/rows16k xft_pipe_kernel rows16k_final
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
for c in cfg2 cfg5; do
  python tools/prof_cfg.py $c 2 > $O/plain_$c.log 2>&1 && \
    ncu $M --log-file $O/launches_${c}_final.csv python tools/prof_cfg.py $c 2 > $O/ncu_launch_$c.log 2>&1
  python tools/launch_summary.py $O/launches_${c}_final.csv > $O/launches_${c}_final.txt 2>&1
done
python bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu > $O/plain_bench.log 2>&1 && \
  ncu $M -c 800 --log-file $O/launches_bench_final.csv python bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu > $O/ncu_bench.log 2>&1
python tools/launch_summary.py $O/launches_bench_final.csv > $O/launches_bench_final.txt 2>&1
ls -la $O
# the driver's command, last (no profiler)
python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; tail -c 600 $O/bench.err
