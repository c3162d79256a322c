#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-c2ab}
bash tools/gpu_ab_build.sh $TAG "" "-DHPS_AUX_PRIORITY=0" "" "-DHPS_AUX_PRIORITY=0"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --soak-seconds 0 --timeline gpurun_out/timeline_${TAG}.txt > /dev/null 2>&1
timeout 600 python bench.py --config c3 --batches 2 --steps 6 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c3_${TAG}.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest=$? >> gpurun_out/ab_${TAG}.txt
