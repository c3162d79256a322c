#!/bin/bash
mkdir -p gpurun_out
HPS_LIB=tools/exp/libhps_prof.so timeout 600 python bench.py --config c3 --batches 1 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --soak-seconds 0 --no-graph > gpurun_out/hotprof.log 2>&1
echo rc=$? >> gpurun_out/hotprof.log
