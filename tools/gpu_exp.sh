#!/bin/bash
mkdir -p gpurun_out
A="--steps 50 --warmup 5 --e2e-steps 0 --no-cpu-baseline --soak-seconds 0"
for v in base old base old; do
  if [ $v = base ]; then L=""; else L=tools/exp/libhps_$v.so; fi
  HPS_LIB=$L timeout 300 python bench.py $A >> gpurun_out/exp_$v.log 2>&1
done
echo done > gpurun_out/rc_exp.txt
