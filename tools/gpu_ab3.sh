#!/bin/bash
# A/B/C of a multi-valued environment knob on the C2 bench (one GPU):
#   gpurun -- 'bash tools/gpu_ab3.sh VAR tag v0 v1 v2'   each value three times, interleaved
VAR=${1:-HPS_CHECK_L2}
TAG=${2:-ab3}
shift 2
VALS=${@:-0 1 2}
mkdir -p gpurun_out
A="--steps 50 --warmup 5 --e2e-steps 0 --no-cpu-baseline --soak-seconds 0"
: > gpurun_out/rc_$TAG.txt
for i in 1 2 3; do
  for v in $VALS; do
    env $VAR=$v timeout 300 python bench.py $A > gpurun_out/${TAG}_${v}_$i.log 2>&1
  done
done
for f in gpurun_out/${TAG}_*.log; do
  echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"update": [0-9.]*' $f) $(grep -o '"check": [0-9.]*' $f)"
done >> gpurun_out/rc_$TAG.txt
