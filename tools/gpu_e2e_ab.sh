#!/bin/bash
mkdir -p gpurun_out
make -C paper_2111_05897_b200/csrc -s -j8 > /dev/null 2>&1
python tools/pcie_probe.py > gpurun_out/pcie2.txt 2>&1
for r in 1 2; do for K in 2 3 4; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 30 --e2e-slots $K --soak-seconds 0 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('slots $K', round(d['e2e']['value']/1e6,3))" >> gpurun_out/ab_e2e.txt
done; done
