#!/bin/bash
# C5 hybrid step: parity tests + bench at staleness 4 and 0 (one GPU), and with
# N GPUs visible the sharded hybrid step:  gpurun [--gpus N] -- 'bash tools/gpu_hybrid.sh N'
N=${1:-1}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_hybrid.py -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_hybrid.log 2>&1; echo pytest=$? > gpurun_out/rc_hybrid.txt
for T in 4 0; do
timeout 600 python bench.py --config c5 --steps 40 --warmup 5 --staleness $T > gpurun_out/bench_c5_t$T.log 2>&1; echo bench_t$T=$? >> gpurun_out/rc_hybrid.txt
done
if [ "$N" -gt 1 ]; then
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2971$N \
  bench.py --gpus $N --config c5 --steps 30 --warmup 5 > gpurun_out/bench_c5_n$N.log 2>&1; echo bench_n$N=$? >> gpurun_out/rc_hybrid.txt
fi
for f in gpurun_out/bench_c5_*.log; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"loss_first_last": [^]]*' $f)"; done >> gpurun_out/rc_hybrid.txt
