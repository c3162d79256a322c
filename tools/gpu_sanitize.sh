#!/bin/bash
mkdir -p gpurun_out
make -C paper_2111_05897_b200/csrc -s -j8 > /dev/null 2>&1 || exit 3
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python tools/sanitize_case.py > gpurun_out/sanitize_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_rc.txt
done
