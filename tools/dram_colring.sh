#!/bin/bash
# DRAM bytes + duration of the K7 launches of one 2-D transform: bash tools/dram_colring.sh [XFT_LIB path]
export XFT_LIB=$1
python tools/time_colring.py 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:xft_colring -c 2 python tools/time_colring.py > /tmp/ncu_dram.txt 2>&1
grep -E "dram__bytes|gpu__time" /tmp/ncu_dram.txt | tail -3
