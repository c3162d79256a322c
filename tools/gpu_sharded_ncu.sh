#!/bin/bash
# Launch list of the sharded (p2p) step at world size 1 (local overheads of the exchange
# plan without NVLink): gpurun -- 'bash tools/gpu_sharded_ncu.sh'
mkdir -p gpurun_out
export WORLD_SIZE=1 RANK=0 LOCAL_RANK=0 MASTER_ADDR=127.0.0.1 MASTER_PORT=29631 TRANSPORT=p2p ROWS_PER_GPU=${ROWS_PER_GPU:-125000000}
timeout 300 python tools/sharded_phases.py > gpurun_out/xphases_1.log 2>&1; echo plain=$? > gpurun_out/rc_xncu.txt
MASTER_PORT=29632 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/xlaunches_1.csv python tools/sharded_phases.py > gpurun_out/xncu.log 2>&1; echo ncu=$? >> gpurun_out/rc_xncu.txt
