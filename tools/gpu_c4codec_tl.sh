#!/bin/bash
mkdir -p gpurun_out
make -C paper_2111_05897_b200/csrc -s -j8 > /dev/null 2>&1 || exit 3
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29601"
timeout 600 $R bench.py --gpus 2 --steps 16 --warmup 5 --no-cpu-baseline --e2e-steps 0 --codec-kappa 1024 --timeline gpurun_out/timeline_codec_n2 > gpurun_out/bench_codec_tl.log 2>&1
echo done > gpurun_out/rc_codectl.txt
