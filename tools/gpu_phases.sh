#!/bin/bash
mkdir -p gpurun_out
N=${1:-2}
P=29541
run() {  # tag, env...
  local tag=$1; shift
  P=$((P+1))
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P tools/sharded_phases.py > gpurun_out/phases_${N}_$tag.log 2>&1
}
run base X=1
run minch32 NCCL_MIN_P2P_NCHANNELS=32
run ce NCCL_P2P_USE_CUDA_MEMCPY=1
run nvls NCCL_NVLS_ENABLE=1 NCCL_MIN_P2P_NCHANNELS=16 NCCL_P2P_NET_CHUNKSIZE=524288
echo done > gpurun_out/rc_phases.txt
