#!/bin/bash
# sharded hybrid (staleness over tau+1 exchanges) on N GPUs: tests + C5 bench
N=${1:-2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sharded.py -m gpu -q --timeout 400 -p no:cacheprovider -k hybrid > gpurun_out/pytest_hyb2.log 2>&1; echo pytest=$? > gpurun_out/rc_hyb2.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2981$N \
  bench.py --gpus $N --config c5 --steps 30 --warmup 5 > gpurun_out/bench_c5_n$N.log 2>&1; echo c5=$? >> gpurun_out/rc_hyb2.txt
grep -o '"ms_per_step": [0-9.]*\|"value": [0-9.]*\|"staleness": [0-9]*' gpurun_out/bench_c5_n$N.log >> gpurun_out/rc_hyb2.txt
