#!/bin/bash
# C3: ncu full of update_runs + update_single (one step), hot-row parity tests, LRU tests
mkdir -p gpurun_out
TAG=${1:-c3p}
make -C paper_2111_05897_b200/csrc -s -j8 > gpurun_out/build_${TAG}.log 2>&1 || exit 3
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -p no:cacheprovider -k "hot or c3 or multi or large or lru" > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest=$? > gpurun_out/rc_${TAG}.txt
ARGS="--config c3 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --soak-seconds 0 --batches 2 --no-graph"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"update_runs|update_single" -c 2 \
  -o gpurun_out/prof_${TAG} python bench.py $ARGS > gpurun_out/ncu_${TAG}.log 2>&1
echo ncu=$? >> gpurun_out/rc_${TAG}.txt
timeout 600 python bench.py --config c3 --batches 2 --steps 6 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c3_${TAG}.log 2>&1; echo c3=$? >> gpurun_out/rc_${TAG}.txt
