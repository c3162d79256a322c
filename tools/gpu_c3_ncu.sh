#!/bin/bash
mkdir -p gpurun_out
A="--config c3 --batches 1 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --soak-seconds 0 --no-graph"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"update|pool|probe|pass|hist|classify|check" -c 60 --csv --log-file gpurun_out/launches_c3.csv python bench.py $A > gpurun_out/ncu_c3.log 2>&1
echo rc=$? > gpurun_out/rc_c3ncu.txt
