#!/bin/bash
# ncu --set full capture of one K7 (xft_colring_kernel) launch on the 16384^2 c64 field; summaries only come back.
O=gpurun_out/prof_ring
mkdir -p $O
T=/tmp/prof_ring
mkdir -p $T
python tools/prof_2d.py 1 > $O/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:xft_colring_kernel -s 1 -c 1 -o $T/ring python tools/prof_2d.py 1 > $O/ncu.log 2>&1
python tools/ncu_summary.py $T/ring.ncu-rep > $O/summary.txt 2>&1
python tools/ncu_stalls.py $T/ring.ncu-rep xft_colring_kernel 30 > $O/stalls.txt 2>&1
python tools/ncu_lines.py $T/ring.ncu-rep xft_colring_kernel > $O/lines.txt 2>&1
python tools/ncu_opmix.py $T/ring.ncu-rep 40 > $O/opmix.txt 2>&1
ncu -i $T/ring.ncu-rep --page details > $O/details.txt 2>&1
rm -f $T/ring.ncu-rep
ls -la $O
