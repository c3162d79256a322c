#!/bin/bash
mkdir -p gpurun_out
A="--config c3 --batches 1 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --soak-seconds 0 --no-graph"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"update_hot" -s 1 -c 1 -o gpurun_out/prof_c3 python bench.py $A > gpurun_out/ncu_c3_full.log 2>&1
echo rc=$? > gpurun_out/rc_c3ncu.txt
