#!/bin/bash
mkdir -p gpurun_out
A="--steps 50 --warmup 5 --e2e-steps 0 --no-cpu-baseline --soak-seconds 0"
for i in 1 2; do
timeout 300 python bench.py $A > gpurun_out/ab_cond_$i.log 2>&1
HPS_NO_COND=1 timeout 300 python bench.py $A > gpurun_out/ab_nocond_$i.log 2>&1
done
echo done > gpurun_out/rc_ab.txt
