#!/bin/bash
# Build-time A/B: for each -D variant, rebuild update.cu/pool.cu and run the C2 bench.
#   gpurun -- 'bash tools/gpu_ab_build.sh TAG "-DX=1" "-DX=2" ...'
TAG=$1; shift
mkdir -p gpurun_out
for V in "$@"; do
  touch paper_2111_05897_b200/csrc/*.cu
  make -C paper_2111_05897_b200/csrc -s -j8 EXTRA="$V" > gpurun_out/ab_build.log 2>&1 || { echo "build $V failed"; continue; }
  for rep in 1 2; do
    timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 0 --soak-seconds 0.5 > gpurun_out/ab.log 2>&1
    python3 -c "
import json,sys
l=[x for x in open('gpurun_out/ab.log') if x.startswith('{')][-1]; d=json.loads(l)
print('$V', round(d['ms_per_step'],4), {k: v for k, v in d['kernels_ms'].items() if k in ('pool','check','update','update_multi')})
" >> gpurun_out/ab_${TAG}.txt
  done
done
touch paper_2111_05897_b200/csrc/*.cu
make -C paper_2111_05897_b200/csrc -s -j8 > /dev/null 2>&1
