#!/bin/bash
mkdir -p gpurun_out
make -C paper_2111_05897_b200/csrc -s -j8 >/dev/null 2>&1
for r in 1 2; do for F in "" "--register-after pull" "--register-after pull --step-priority -1" "--register-after pull --register-priority -1"; do
timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 0 --soak-seconds 0.5 $F 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$F', round(d['ms_per_step'],4))" >> gpurun_out/ab_regpos.txt
done; done
