"""bench.py contract pieces that run without a GPU: the reference arm
(`--impl reference`: the CPU path on the host cores) prints one JSON line
with the required keys, and the optional-section guard records failures
instead of dropping the line."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_prints_one_contract_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "5",
                          "--warmup", "4"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "images/s"
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"] == "resnet20_cifar10_lpp_sgd"


def test_optional_section_guard():
    sys.path.insert(0, str(ROOT))
    import bench

    line = {}
    with bench._Optional(line, "resnet50"):
        raise RuntimeError("CUDA out of memory")
    assert "resnet50" in line["optional_errors"]
    try:
        with bench._Optional(line, "x"):
            raise KeyboardInterrupt
    except KeyboardInterrupt:
        pass
    else:
        raise AssertionError("non-Exception errors must propagate")
