#!/bin/bash
# Build-time A/B on C3 (and a C2 guard line): for each -D variant rebuild and run both.
#   gpurun -- 'bash tools/gpu_ab_c3.sh TAG "-DX=1" ...'
TAG=$1; shift
mkdir -p gpurun_out
for V in "$@"; do
  touch paper_2111_05897_b200/csrc/*.cu
  make -C paper_2111_05897_b200/csrc -s -j8 EXTRA="$V" > gpurun_out/ab_build.log 2>&1 || { echo "build $V failed" >> gpurun_out/ab_${TAG}.txt; continue; }
  timeout 600 python bench.py --config c3 --batches 2 --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab.log 2>&1
  python3 -c "
import json
l=[x for x in open('gpurun_out/ab.log') if x.startswith('{')][-1]; d=json.loads(l)
print('c3 $V', round(d['ms_per_step'],3), {k: round(v,3) for k, v in d['kernels_ms'].items()})
" >> gpurun_out/ab_${TAG}.txt 2>&1
  timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 0 --soak-seconds 0.5 > gpurun_out/ab.log 2>&1
  python3 -c "
import json
l=[x for x in open('gpurun_out/ab.log') if x.startswith('{')][-1]; d=json.loads(l)
print('c2 $V', round(d['ms_per_step'],4))
" >> gpurun_out/ab_${TAG}.txt 2>&1
done
touch paper_2111_05897_b200/csrc/*.cu
make -C paper_2111_05897_b200/csrc -s -j8 > /dev/null 2>&1
