#!/bin/bash
# Everything the driver runs at round end, on the GPUs this call got (2 recommended):
# smoke, the whole GPU test suite, the default bench and the reference arm.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1; echo smoke=$? > gpurun_out/rc_full.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/full_pytest.log 2>&1; echo pytest=$? >> gpurun_out/rc_full.txt
timeout 600 python bench.py > gpurun_out/full_bench.log 2>&1; echo bench=$? >> gpurun_out/rc_full.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/full_bench_ref.log 2>&1; echo bench_ref=$? >> gpurun_out/rc_full.txt
