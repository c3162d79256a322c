#!/bin/bash
# Scaling check on one box: gpurun --gpus N --timeout 1800 -- 'bash tools/gpu_scale.sh N'
N=${1:-4}
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo_$N.txt 2>&1
for T in p2p nccl; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N \
  bench.py --gpus $N --steps 20 --warmup 3 --e2e-steps 5 --transport $T > gpurun_out/bench_scale_${N}_$T.log 2>&1; echo $T=$? >> gpurun_out/rc_scale_$N.txt
done
TRANSPORT=p2p timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N tools/sharded_phases.py > gpurun_out/phases_${N}_p2p.log 2>&1
