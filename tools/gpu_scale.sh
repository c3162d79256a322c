#!/bin/bash
# Scaling check on one box: gpurun --gpus N --timeout 1800 -- 'bash tools/gpu_scale.sh N'
# the p2p bench line at N, then the per-region phases.
N=${1:-4}
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo_$N.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N \
  bench.py --gpus $N --steps 30 --warmup 3 --e2e-steps 5 > gpurun_out/bench_scale_${N}_p2p.log 2>&1; echo p2p=$? > gpurun_out/rc_scale_$N.txt
TRANSPORT=p2p timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N \
  tools/sharded_phases.py > gpurun_out/phases_${N}_p2p.log 2>&1; echo phases=$? >> gpurun_out/rc_scale_$N.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N \
  bench.py --gpus $N --config c5 --steps 30 --warmup 5 > gpurun_out/bench_c5_n$N.log 2>&1; echo c5=$? >> gpurun_out/rc_scale_$N.txt
