#!/bin/bash
# Round-2 (K7) captures: one --set full capture of the column kernel, the cfg5 launch list and the bench launch list.
O=gpurun_out/prof2b
mkdir -p $O
bash tools/prof_colring.sh > $O/prof_colring.log 2>&1
cp gpurun_out/prof_ring/summary.txt $O/ncu_full_colring.txt
cp gpurun_out/prof_ring/stalls.txt $O/stalls_colring.txt
cp gpurun_out/prof_ring/lines.txt $O/lines_colring.txt
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
python tools/prof_cfg.py cfg5 2 > $O/plain_cfg5.log 2>&1 && \
  ncu $M --log-file $O/launches_cfg5.csv python tools/prof_cfg.py cfg5 2 > $O/ncu_cfg5.log 2>&1
python tools/launch_summary.py $O/launches_cfg5.csv > $O/launches_cfg5.txt 2>&1
python bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu > $O/plain_bench.log 2>&1 && \
  ncu $M -c 800 --log-file $O/launches_bench.csv python bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu > $O/ncu_bench.log 2>&1
python tools/launch_summary.py $O/launches_bench.csv > $O/launches_bench.txt 2>&1
ls -la $O
