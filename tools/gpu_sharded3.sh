#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sharded.py -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_sharded.log 2>&1; echo pytest=$? > gpurun_out/rc_sharded.txt
for T in p2p nccl; do
TRANSPORT=$T timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 tools/sharded_phases.py > gpurun_out/phases_2_$T.log 2>&1
TRANSPORT=$T timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29553 tools/sharded_phases.py > gpurun_out/phases_1_$T.log 2>&1
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 20 --warmup 3 --e2e-steps 5 > gpurun_out/bench_sharded_2.log 2>&1; echo bench=$? >> gpurun_out/rc_sharded.txt
