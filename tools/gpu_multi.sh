#!/bin/bash
# Multi-GPU check on one box: gpurun --gpus N --timeout 1800 -- 'bash tools/gpu_multi.sh N'
# sharded parity tests (all GPUs visible), the p2p bench line, and the per-region phases.
N=${1:-2}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sharded.py -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_multi_$N.log 2>&1; echo pytest=$? > gpurun_out/rc_multi_$N.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N \
  bench.py --gpus $N --steps 30 --warmup 3 --e2e-steps 5 > gpurun_out/bench_multi_$N.log 2>&1; echo bench=$? >> gpurun_out/rc_multi_$N.txt
TRANSPORT=p2p timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N \
  tools/sharded_phases.py > gpurun_out/phases_multi_$N.log 2>&1; echo phases=$? >> gpurun_out/rc_multi_$N.txt
