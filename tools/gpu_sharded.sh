#!/bin/bash
# Multi-GPU round trip (gpurun --gpus N): sharded parity tests + sharded bench.
#   gpurun --gpus 2 --timeout 1800 -- 'bash tools/gpu_sharded.sh 2'
N=${1:-2}
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 600 python -m pytest tests/test_sharded.py tests/test_abi.py -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_sharded.log 2>&1; echo pytest=$? > gpurun_out/rc_sharded.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus $N --steps 20 --warmup 3 --e2e-steps 5 > gpurun_out/bench_sharded_$N.log 2>&1; echo bench=$? >> gpurun_out/rc_sharded.txt
