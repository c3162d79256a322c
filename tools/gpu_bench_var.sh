#!/bin/bash
# bench variants on one box: default, then with env overrides given as args
mkdir -p gpurun_out
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/var_default.log 2>&1
for v in "$@"; do
  env $v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/var_${v//[^A-Za-z0-9]/_}.log 2>&1
done
