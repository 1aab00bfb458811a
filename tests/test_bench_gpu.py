"""bench.py's JSON contract on the GPU (a short run without the optional
sections): one line with the base keys and the roofline / e2e / clocks /
gpu_launches extras the driver checks."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def test_bench_line_contract():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "4", "--warmup", "3",
                          "--no-cpu", "--no-sweep", "--no-rn18", "--no-rn50", "--no-baselines"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks",
                "gpu_launches"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] >= 3 and d["value"] > 0
    r = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert 0 < r["frac"] < 1.5 and r["bound"] == "hbm"
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["gpu_launches"] > 0
    assert d["config"]["workload"] == "resnet20_cifar10_lpp_sgd"
    # the headline is at the reference arm's precision; bf16 is a labelled extra
    assert d["dtype"] == "f32" and d["config"]["conv_compute"].startswith("fp32")
    assert d["value_bf16"] > 0 and d["e2e_bf16"]["value"] > 0
    # the step's dominant kernels: the fp32 convolutions vs the measured FFMA peak
    rc = d["roofline_conv"]
    assert rc["unit"] == "TFLOP/s" and 50 < rc["peak"] < 100 and 0.1 < rc["frac"] < 1.0
    assert d["gpu_launches_split"]["in_graph"] > 0
