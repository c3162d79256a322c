"""bench.py's CPU-side contract (no GPU): the reference arm runs the reference's own C++
path (oracle/_ref) on the C2 config and prints one JSON line with the fields the driver
reads; the C5 CPU baseline runs the reference's hybrid step on a small sample."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.usefixtures("oracle_built")
def test_reference_arm_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"] == "embedding lookup+update samples/sec"
    assert d["unit"] == "samples/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["value"] == d["cpu_baseline"]["value"]
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "samples/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["global_batch"] == 16384
    legs = d["legs"]
    assert legs["ps_lookup_rows_per_s"] > 0 and legs["ps_apply_rows_per_s"] > 0


@pytest.mark.usefixtures("oracle_built")
def test_hybrid_cpu_baseline_small_sample():
    sys.path.insert(0, ROOT)
    import bench
    from paper_2111_05897_b200 import workloads as W

    v, cores, sample = bench.hybrid_cpu_baseline(W.CONFIGS["c5"], 64, steps=1)
    assert v > 0 and cores >= 1
    assert "DenseNet" in sample and "oracle/_ref" in sample
