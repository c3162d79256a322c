#!/bin/bash
# p2p sharded step phases at N ranks + C2 register placement A/B on GPU 0
mkdir -p gpurun_out
N=${1:-2}; TAG=${2:-ph}
make -C paper_2111_05897_b200/csrc -s -j8 > /dev/null 2>&1 || exit 3
TRANSPORT=p2p timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29561 tools/sharded_phases.py > gpurun_out/phases_${TAG}_n${N}.log 2>&1
for after in push pull push pull; do
  CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 0 --soak-seconds 0.5 --register-after $after 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('after $after', round(d['ms_per_step'],4))" >> gpurun_out/ab_${TAG}.txt
done
