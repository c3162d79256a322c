#!/bin/bash
# tests + bench, one GPU
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 240 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/rc_quick.txt
timeout 500 python bench.py --steps 50 --warmup 5 --cpu-seconds 5 > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/rc_quick.txt
