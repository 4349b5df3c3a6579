#!/bin/bash
# A/B of the split-barrier column ring kernel (tune/libxft_rxb.so, -DXFT_RING_XBAR=1) against the in-tree build
# (row kernels: split barriers for the one-CTA-per-SM c64 kernel); the sha lines must match
mkdir -p gpurun_out/ab2
for round in 1 2; do
  for v in default rxb; do
    if [ $v = default ]; then unset XFT_LIB; else export XFT_LIB=tune/libxft_$v.so; fi
    timeout 200 python tools/time_colring.py >> gpurun_out/ab2/colring.txt 2>> gpurun_out/ab2/err.txt
  done
done
unset XFT_LIB
timeout 200 python tools/time_rows16k.py >> gpurun_out/ab2/rows16k.txt 2>> gpurun_out/ab2/err.txt
timeout 200 python tools/tune_time.py >> gpurun_out/ab2/cfg2.txt 2>> gpurun_out/ab2/err.txt
for v in default rxb; do
  if [ $v = default ]; then unset XFT_LIB; else export XFT_LIB=tune/libxft_$v.so; fi
  timeout 300 python tools/time_2d_shapes.py >> gpurun_out/ab2/shapes.txt 2>> gpurun_out/ab2/err.txt
done
cat gpurun_out/ab2/*.txt | grep -v "^$" | tail -40
