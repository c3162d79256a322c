#!/bin/bash
# Multi-GPU on one box: sharded tests at world N, C4 bench at N (exact and codec), phases.
#   gpurun --gpus N -- 'bash tools/gpu_multi.sh TAG N'
TAG=${1:-mg}; N=${2:-2}
mkdir -p gpurun_out
make -C paper_2111_05897_b200/csrc -s -j8 > gpurun_out/build_${TAG}.log 2>&1 || exit 3
nvidia-smi topo -m > gpurun_out/topo_${TAG}.txt 2>&1
timeout 900 python -m pytest tests/test_sharded.py tests/test_hybrid.py -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest=$? > gpurun_out/rc_${TAG}.txt
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611"
timeout 900 $R bench.py --gpus $N --steps 30 --warmup 5 > gpurun_out/bench_c4_n${N}_${TAG}.log 2>&1; echo c4=$? >> gpurun_out/rc_${TAG}.txt
timeout 900 $R bench.py --gpus $N --steps 30 --warmup 5 --codec-kappa 1024 > gpurun_out/bench_c4codec_n${N}_${TAG}.log 2>&1; echo c4codec=$? >> gpurun_out/rc_${TAG}.txt
timeout 900 $R bench.py --gpus $N --steps 20 --warmup 4 --config c5 > gpurun_out/bench_c5_n${N}_${TAG}.log 2>&1; echo c5=$? >> gpurun_out/rc_${TAG}.txt
timeout 600 $R bench.py --impl reference --gpus $N --steps 4 --warmup 1 > gpurun_out/bench_ref_n${N}_${TAG}.log 2>&1; echo ref=$? >> gpurun_out/rc_${TAG}.txt
