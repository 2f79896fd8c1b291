#!/bin/bash
# Time (and parity-test) kernel variants on the GPU box:
#   bash tools/variants.sh "base bk64" [--tests] [--configs "c3 c4 c5"]
mkdir -p gpurun_out
cfgs="c3 c4 c5"; [ "$3" = "--configs" ] && cfgs=$4
for v in $1; do
  lib=build/variants/libcvpb200_$v.so
  for cfg in $cfgs; do
    n=512; [ $cfg = c5 ] && n=1024
    CVPB_LIB=$lib timeout 300 python tools/prof_cvp.py --config $cfg --n $n --views 64 --reps 2 2>&1 | tail -1 | sed "s/^/$v /"
  done
  if [ "$2" = "--tests" ]; then
    CVPB_LIB=$lib timeout 300 python -m pytest -x -q tests/test_cvp_gpu.py tests/test_cvp_edge_gpu.py 2>&1 | tail -2 | sed "s/^/$v tests: /"
  fi
done
