#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1; echo pytest=$? > gpurun_out/rc_sharded.txt
TRANSPORT=p2p timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 tools/sharded_phases.py > gpurun_out/phases_2_p2p.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 20 --warmup 3 --e2e-steps 5 > gpurun_out/bench_sharded_2.log 2>&1; echo bench=$? >> gpurun_out/rc_sharded.txt
timeout 600 python bench.py --steps 30 --warmup 5 --cpu-seconds 5 > gpurun_out/bench.log 2>&1; echo bench1=$? >> gpurun_out/rc_sharded.txt
