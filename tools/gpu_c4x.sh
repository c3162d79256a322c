#!/bin/bash
# sharded parity tests + C4 bench (and timeline) at N ranks
mkdir -p gpurun_out
N=${1:-2}; TAG=${2:-c4x}
make -C paper_2111_05897_b200/csrc -s -j8 > gpurun_out/build_${TAG}.log 2>&1 || exit 3
timeout 900 python -m pytest tests/test_sharded.py -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest=$? > gpurun_out/rc_${TAG}.txt
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29581"
timeout 600 $R bench.py --gpus $N --steps 32 --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_${TAG}_n${N}.log 2>&1; echo c4=$? >> gpurun_out/rc_${TAG}.txt
timeout 600 $R bench.py --gpus $N --steps 32 --warmup 5 --no-cpu-baseline --e2e-steps 0 --codec-kappa 1024 > gpurun_out/bench_${TAG}codec_n${N}.log 2>&1; echo c4codec=$? >> gpurun_out/rc_${TAG}.txt
timeout 600 $R bench.py --gpus $N --steps 16 --warmup 5 --no-cpu-baseline --e2e-steps 0 --timeline gpurun_out/timeline_${TAG}_n${N} > /dev/null 2>&1
