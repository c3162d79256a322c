#!/bin/bash
# A/B of an environment toggle on the C2 bench (one GPU), after the GPU parity tests:
#   gpurun -- 'bash tools/gpu_ab.sh VAR [tag]'   runs VAR=1 vs VAR=0, twice each
VAR=${1:-HPS_PDL}
TAG=${2:-ab}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 240 -p no:cacheprovider -x > gpurun_out/pytest_$TAG.log 2>&1; echo pytest=$? > gpurun_out/rc_$TAG.txt
A="--steps 50 --warmup 5 --e2e-steps 0 --no-cpu-baseline --soak-seconds 0"
for i in 1 2; do
env $VAR=1 timeout 300 python bench.py $A > gpurun_out/${TAG}_on_$i.log 2>&1
env $VAR=0 timeout 300 python bench.py $A > gpurun_out/${TAG}_off_$i.log 2>&1
done
for f in gpurun_out/${TAG}_*.log; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f)"; done >> gpurun_out/rc_$TAG.txt
