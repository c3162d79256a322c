#!/bin/bash
# C4 at N ranks: bench (cycle graphs) + a per-rank kernel timeline of the replayed steps
mkdir -p gpurun_out
N=${1:-2}; TAG=${2:-c4tl}
make -C paper_2111_05897_b200/csrc -s -j8 > /dev/null 2>&1 || exit 3
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29571"
timeout 600 $R bench.py --gpus $N --steps 32 --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_${TAG}_n${N}.log 2>&1
timeout 600 $R bench.py --gpus $N --steps 16 --warmup 5 --no-cpu-baseline --e2e-steps 0 --timeline gpurun_out/timeline_${TAG}_n${N} > gpurun_out/bench_${TAG}_tl_n${N}.log 2>&1
echo done > gpurun_out/rc_${TAG}.txt
