"""Shared test setup.

Markers: ``gpu`` — needs a CUDA device (run on the B200 box with
``pytest -m gpu``); everything else runs on CPU in the build container.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

# the CUDA library and the C oracle are build products (git-ignored): make
# sure they exist before any test loads them (nvcc cross-compiles on CPU)
from paper_2203_06638_b200 import build as _build  # noqa: E402

_build.build()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA device (B200)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_npz(name: str) -> dict:
    with np.load(GOLDEN / name) as f:
        return {k: f[k] for k in f.files}


@pytest.fixture(scope="session")
def golden_scalars():
    import json

    return json.loads((GOLDEN / "scalars.json").read_text())
