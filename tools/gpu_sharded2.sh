#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sharded.py tests/test_gpu_parity.py -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_sharded.log 2>&1; echo pytest=$? > gpurun_out/rc_sharded.txt
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 tools/sharded_phases.py > gpurun_out/phases_2.log 2>&1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29553 tools/sharded_phases.py > gpurun_out/phases_1.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 20 --warmup 3 --e2e-steps 5 > gpurun_out/bench_sharded_2.log 2>&1; echo bench=$? >> gpurun_out/rc_sharded.txt
