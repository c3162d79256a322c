#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-sched}
make -C paper_2111_05897_b200/csrc -s -j8 > gpurun_out/build_${TAG}.log 2>&1 || exit 3
for R in push pull push pull; do
for P in 0 -1; do
  timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 0 --soak-seconds 0.5 --register-priority $P --register-after $R > gpurun_out/ab.log 2>&1
  python3 -c "
import json
l=[x for x in open('gpurun_out/ab.log') if x.startswith('{')][-1]; d=json.loads(l)
print('after $R prio $P', round(d['ms_per_step'],4))
" >> gpurun_out/ab_${TAG}.txt
done; done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --soak-seconds 0 --register-after pull --timeline gpurun_out/timeline_${TAG}.txt > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest=$? >> gpurun_out/ab_${TAG}.txt
timeout 600 python bench.py --config c3 --batches 2 --steps 6 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c3_${TAG}.log 2>&1; echo c3=$? >> gpurun_out/ab_${TAG}.txt
