#!/bin/bash
# Generic A/B driver for variant libraries (tools/build_variant*.sh -> tune/libxft_NAME.so):
#   bash tools/ab.sh TAG "NAME1 NAME2 ..." "command 1" ["command 2" ...]
# runs every command with the in-tree library ("default") and with each variant (XFT_LIB, read by
# tools/_variant.py), two rounds, under a per-command timeout, into gpurun_out/ab_TAG/out.txt.
# The timing tools print an output fingerprint (sha): scheduling-only variants must reproduce the default's.
# Example (the round-2 row-kernel experiments):
#   bash tools/build_variant_capi.sh l2pf "-DXFT_L2PF=1"
#   gpurun -- 'bash tools/ab.sh l2pf "l2pf" "python tools/tune_time.py" "python tools/time_rows16k.py"'
TAG=$1; VARIANTS=$2; shift 2
O=gpurun_out/ab_$TAG
mkdir -p $O
for round in 1 2; do
  for v in default $VARIANTS; do
    if [ $v = default ]; then unset XFT_LIB; else export XFT_LIB=tune/libxft_$v.so; fi
    for cmd in "$@"; do
      echo "# $v: $cmd" >> $O/out.txt
      timeout 300 $cmd >> $O/out.txt 2>> $O/err.txt
    done
  done
done
cat $O/out.txt; tail -5 $O/err.txt
