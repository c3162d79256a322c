#!/bin/bash
# A/B of environment settings on the C2 bench (one GPU), interleaved, twice each:
#   gpurun -- 'bash tools/gpu_ab2.sh TAG "ENV_A" "ENV_B" ["ENV_C"]'   (ENV_x e.g. "X=1" or "HPS_L2_FETCH_BYTES=32")
TAG=$1; shift
mkdir -p gpurun_out
A="--steps 50 --warmup 5 --e2e-steps 0 --no-cpu-baseline --soak-seconds 0"
: > gpurun_out/rc_$TAG.txt
for i in 1 2; do
  k=0
  for E in "$@"; do
    k=$((k+1))
    env $E timeout 300 python bench.py $A > gpurun_out/${TAG}_${k}_$i.log 2>&1
    echo "$E run$i $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/${TAG}_${k}_$i.log) $(grep -o '"kernels_ms": {[^}]*}' gpurun_out/${TAG}_${k}_$i.log)" >> gpurun_out/rc_$TAG.txt
  done
done
