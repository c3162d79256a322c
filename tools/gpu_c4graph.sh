#!/bin/bash
mkdir -p gpurun_out
make -C paper_2111_05897_b200/csrc -s -j8 > /dev/null 2>&1 || exit 3
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621"
for F in "" "--no-graph"; do for r in 1 2; do
timeout 600 $R bench.py --gpus 2 --steps 32 --warmup 5 --no-cpu-baseline --e2e-steps 0 $F > gpurun_out/ab.log 2>&1
python3 -c "
import json
l=[x for x in open('gpurun_out/ab.log') if x.startswith('{')][-1]; d=json.loads(l)
print('$F', round(d['ms_per_step'],4))
" >> gpurun_out/ab_c4graph.txt 2>&1
done; done
timeout 600 $R bench.py --gpus 2 --steps 16 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-graph --timeline gpurun_out/timeline_c4eager_n2 > /dev/null 2>&1
