#!/bin/bash
# C4 A/B at N ranks: build variants x bench flag variants
mkdir -p gpurun_out
N=${1:-2}; TAG=${2:-c4ab}; shift 2
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29591"
for V in "$@"; do
  touch paper_2111_05897_b200/csrc/*.cu
  make -C paper_2111_05897_b200/csrc -s -j8 EXTRA="$V" > gpurun_out/ab_build.log 2>&1 || { echo "build $V failed" >> gpurun_out/ab_${TAG}.txt; continue; }
  for F in "" "--prefetch-priority -1"; do
    timeout 600 $R bench.py --gpus $N --steps 32 --warmup 5 --no-cpu-baseline --e2e-steps 0 $F > gpurun_out/ab.log 2>&1
    python3 -c "
import json
l=[x for x in open('gpurun_out/ab.log') if x.startswith('{')][-1]; d=json.loads(l)
print('$V', '$F', round(d['ms_per_step'],4))
" >> gpurun_out/ab_${TAG}.txt 2>&1
  done
done
