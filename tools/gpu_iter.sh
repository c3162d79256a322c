#!/bin/bash
# Iteration round trip: build, GPU tests, C2 bench + launch list, C3 bench + launch list,
# ncu full of the top C2 kernels.
#   gpurun --timeout 2400 -- 'bash tools/gpu_iter.sh TAG'
TAG=${1:-it}
mkdir -p gpurun_out
make -C paper_2111_05897_b200/csrc -s -j8 > gpurun_out/build_${TAG}.log 2>&1 || exit 3
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo pytest=$? > gpurun_out/rc_${TAG}.txt
timeout 500 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_${TAG}.log 2>&1; echo bench=$? >> gpurun_out/rc_${TAG}.txt
ARGS="--steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --soak-seconds 0 --batches 2"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py $ARGS > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo ncu1=$? >> gpurun_out/rc_${TAG}.txt
timeout 900 python bench.py --config c3 --batches 2 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c3_${TAG}.log 2>&1; echo c3=$? >> gpurun_out/rc_${TAG}.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_c3_${TAG}.csv python bench.py --config c3 $ARGS > gpurun_out/ncu_launch_c3_${TAG}.log 2>&1
echo ncu3=$? >> gpurun_out/rc_${TAG}.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"update_single|pool_warp|check_stream|probe_kernel" -s 12 -c 8 \
  -o gpurun_out/prof_${TAG} python bench.py $ARGS > gpurun_out/ncu_full_${TAG}.log 2>&1
echo ncu2=$? >> gpurun_out/rc_${TAG}.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --soak-seconds 0 --timeline gpurun_out/timeline_${TAG}.txt > gpurun_out/bench_tl_${TAG}.log 2>&1; echo tl=$? >> gpurun_out/rc_${TAG}.txt
