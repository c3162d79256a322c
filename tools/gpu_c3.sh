#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --config c3 --batches 2 --steps 10 --warmup 3 --cpu-seconds 5 --e2e-steps 2 > gpurun_out/bench_c3.log 2>&1; echo c3=$? > gpurun_out/rc_c3.txt
timeout 600 python bench.py --config c1 --steps 30 --warmup 5 --cpu-seconds 5 > gpurun_out/bench_c1.log 2>&1; echo c1=$? >> gpurun_out/rc_c3.txt
