#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-prio}
make -C paper_2111_05897_b200/csrc -s -j8 > gpurun_out/build_${TAG}.log 2>&1 || exit 3
for P in 0 -1 0 -1; do
  timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 0 --soak-seconds 0.5 --register-priority $P > gpurun_out/ab.log 2>&1
  python3 -c "
import json
l=[x for x in open('gpurun_out/ab.log') if x.startswith('{')][-1]; d=json.loads(l)
print('prio $P', round(d['ms_per_step'],4))
" >> gpurun_out/ab_${TAG}.txt
done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --soak-seconds 0 --timeline gpurun_out/timeline_${TAG}.txt > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "pipelined or graph or c2 or hot or c3_multi" > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest=$? >> gpurun_out/ab_${TAG}.txt
