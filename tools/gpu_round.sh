#!/bin/bash
# tests + C2 bench x2 + timeline + C3 bench
mkdir -p gpurun_out
TAG=${1:-rd}
make -C paper_2111_05897_b200/csrc -s -j8 > gpurun_out/build_${TAG}.log 2>&1 || exit 3
timeout 1500 python -m pytest tests -m gpu -q --timeout 1300 -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest=$? > gpurun_out/rc_${TAG}.txt
for r in 1 2; do timeout 500 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 5 > gpurun_out/bench_${TAG}_$r.log 2>&1; done; echo bench=$? >> gpurun_out/rc_${TAG}.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --soak-seconds 0 --timeline gpurun_out/timeline_${TAG}.txt > /dev/null 2>&1
timeout 600 python bench.py --config c3 --batches 2 --steps 6 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c3_${TAG}.log 2>&1; echo c3=$? >> gpurun_out/rc_${TAG}.txt
