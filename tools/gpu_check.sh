#!/bin/bash
# One GPU round trip: smoke, GPU parity tests, bench, launch list, ncu capture.
#   gpurun --timeout 2400 -- 'bash tools/gpu_check.sh [tag] [ncu-kernel-regex]'
TAG=${1:-r2}
KRE=${2:-"update_single|update_multi|pool_kernel|probe_kernel|check_batch|classify"}
mkdir -p gpurun_out
make -C paper_2111_05897_b200/csrc -s -j8 > gpurun_out/build_${TAG}.log 2>&1
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke=$? > gpurun_out/rc_${TAG}.txt
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo pytest=$? >> gpurun_out/rc_${TAG}.txt
timeout 500 python bench.py --steps 30 --warmup 5 --cpu-seconds 8 > gpurun_out/bench_${TAG}.log 2>&1; echo bench=$? >> gpurun_out/rc_${TAG}.txt
ARGS="--steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --soak-seconds 0 --batches 2"
timeout 300 python bench.py $ARGS > gpurun_out/plain_${TAG}.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py $ARGS > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo ncu1=$? >> gpurun_out/rc_${TAG}.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 20 -c 12 \
  -o gpurun_out/prof_${TAG} python bench.py $ARGS > gpurun_out/ncu_full_${TAG}.log 2>&1
echo ncu2=$? >> gpurun_out/rc_${TAG}.txt
