#!/bin/bash
# C3 parity subset + C3 bench for each build variant
TAG=$1; shift
mkdir -p gpurun_out
for V in "$@"; do
  touch paper_2111_05897_b200/csrc/*.cu
  make -C paper_2111_05897_b200/csrc -s -j8 EXTRA="$V" > gpurun_out/ab_build.log 2>&1 || { echo "build $V failed" >> gpurun_out/ab_${TAG}.txt; continue; }
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "hot or c3 or multi or large" > gpurun_out/pytest_${TAG}.log 2>&1; echo "$V pytest=$?" >> gpurun_out/ab_${TAG}.txt
  for r in 1 2; do
    timeout 600 python bench.py --config c3 --batches 2 --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab.log 2>&1
    python3 -c "
import json
l=[x for x in open('gpurun_out/ab.log') if x.startswith('{')][-1]; d=json.loads(l)
print('c3 $V', round(d['ms_per_step'],3), round(d['kernels_ms']['update'],3), round(d['kernels_ms']['update_multi'],3))
" >> gpurun_out/ab_${TAG}.txt 2>&1
  done
done
touch paper_2111_05897_b200/csrc/*.cu
make -C paper_2111_05897_b200/csrc -s -j8 > /dev/null 2>&1
