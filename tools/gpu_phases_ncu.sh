#!/bin/bash
mkdir -p gpurun_out
export MASTER_ADDR=127.0.0.1 MASTER_PORT=29561 WORLD_SIZE=1 RANK=0 LOCAL_RANK=0 TRANSPORT=${1:-p2p}
timeout 300 python tools/sharded_phases.py > gpurun_out/phases_plain1.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/launches_sharded1.csv python tools/sharded_phases.py > gpurun_out/phases_ncu.log 2>&1
echo rc=$? > gpurun_out/rc_phases.txt
