#!/bin/bash
# C3 update_runs profile + multi-rank tests on one GPU
mkdir -p gpurun_out
TAG=${1:-rp}
make -C paper_2111_05897_b200/csrc -s -j8 > gpurun_out/build_${TAG}.log 2>&1 || exit 3
ARGS="--config c3 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --soak-seconds 0 --batches 2 --no-graph"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"update_runs" -c 1 \
  -o gpurun_out/prof_runs_${TAG} python bench.py $ARGS > gpurun_out/ncu_runs_${TAG}.log 2>&1
echo ncu=$? > gpurun_out/rc_${TAG}.txt
timeout 900 python -m pytest tests/test_sharded.py -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/pytest_sharded_${TAG}.log 2>&1; echo pytest=$? >> gpurun_out/rc_${TAG}.txt
