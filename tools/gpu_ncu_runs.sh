#!/bin/bash
# ncu --set full of update_runs (C3, one eager step) with source correlation
mkdir -p gpurun_out
TAG=${1:-runs}; KREGEX=${2:-update_runs}
ARGS="--config c3 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --soak-seconds 0 --batches 2 --no-graph"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -c 1 \
  -o gpurun_out/prof_${TAG} python bench.py $ARGS > gpurun_out/ncu_${TAG}.log 2>&1
echo ncu=$? > gpurun_out/rc_${TAG}.txt
