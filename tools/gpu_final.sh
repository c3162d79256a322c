#!/bin/bash
# round-end check of HEAD on one GPU: the driver's sequence (gpu tests, smoke, default
# bench, reference arm) plus the C3 line
mkdir -p gpurun_out
TAG=${1:-fin}
make -C paper_2111_05897_b200/csrc -s -j8 > gpurun_out/build_${TAG}.log 2>&1 || exit 3
timeout 1500 python -m pytest tests -m gpu -q --timeout 1300 -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest=$? > gpurun_out/rc_${TAG}.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke=$? >> gpurun_out/rc_${TAG}.txt
( time timeout 900 python bench.py ) > gpurun_out/bench_${TAG}.log 2>&1; echo bench=$? >> gpurun_out/rc_${TAG}.txt
( time timeout 900 python bench.py --impl reference ) > gpurun_out/bench_ref_${TAG}.log 2>&1; echo ref=$? >> gpurun_out/rc_${TAG}.txt
timeout 600 python bench.py --config c3 --batches 2 --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c3_${TAG}.log 2>&1; echo c3=$? >> gpurun_out/rc_${TAG}.txt
