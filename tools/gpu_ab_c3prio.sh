mkdir -p gpurun_out
make -C paper_2111_05897_b200/csrc -s -j8 >/dev/null 2>&1
for r in 1 2; do for F in "" "--step-priority -1" "--register-priority -1"; do
timeout 600 python bench.py --config c3 --batches 2 --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 0 $F 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 $F', round(d['ms_per_step'],3))" >> gpurun_out/ab_c3prio.txt
done; done
