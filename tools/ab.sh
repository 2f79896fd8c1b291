#!/bin/bash
# A/B timing of library variants on the GPU box:
#   bash tools/ab.sh "base clip" [configs] [views]
mkdir -p gpurun_out
cfgs=${2:-"c3 c4 c5"}; views=${3:-128}
for rep in 1 2; do
for v in $1; do
  lib=build/variants/libcvpb200_$v.so
  for cfg in $cfgs; do
    n=512; [ $cfg = c5 ] && n=1024; [ $cfg = c2 ] && n=256
    CVPB_LIB=$lib timeout 300 python tools/prof_cvp.py --config $cfg --n $n --views $views --reps 2 2>&1 | tail -1 | sed "s/^/$v /"
  done
done
done
