# SPDX-License-Identifier: Apache-2.0
"""The bench.py JSON contract (the driver parses these lines): keys, types and
the units the task statement fixes.  The reference arm runs on the CPU; the
GPU arm needs a B200."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRIC = "reconstructed frames/sec at 256^3 grid, 4x512x424 RGB-D views; per-stage ms/frame"


def run_bench(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def check_common(d):
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "e2e"):
        assert key in d, key
    assert d["metric"] == METRIC and d["unit"] == "frames/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["n_gpus"] == 1
    assert d["vs_baseline"] is None  # BASELINE.md has no published number for this metric
    assert "workload" in d["config"] and "model" not in d["config"]
    e = d["e2e"]
    for key in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert key in e, key
    assert e["unit"] == d["unit"] and e["value"] > 0


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "0")
    check_common(d)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert cb["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"]


@pytest.mark.gpu
def test_gpu_arm_line():
    d = run_bench("--steps", "40", "--warmup", "3", "--no-cpu-baseline")
    check_common(d)
    assert d["warmup"] >= 3 and d["steps"] == 40 and d["scaling"] == "weak"
    assert d["e2e"]["h2d_bytes_per_step"] > 5_000_000 and d["e2e"]["d2h_bytes_per_step"] > 0
    # kernels launched inside the timed region: the frame graph's kernels x steps
    assert d["gpu_launches"] >= 15 * d["steps"]
    r = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert r["bound"] in ("hbm", "tensor") and r["unit"] == "GB/s"
    assert 0 < r["frac"] < 1.5 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    c = d["clocks"]
    assert c["sm_mhz"] is None or c["sm_mhz"] > 0
    assert isinstance(c["reasons"], list)
