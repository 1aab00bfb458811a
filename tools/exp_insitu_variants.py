"""In-situ time of the step's apply kernel inside the bench's fp32 ResNet-20
LPP-SGD run (CUDA events around every launch), for engine variants:
the default (fused K1+K3 with the K5 plan on the high-priority apply stream),
no write tags (plain fused), apply on the updater stream, unfused K3 + K1.
Also images/s.  LPP_FUSED_CTAS=<n> caps the fused grid (run per value)."""
import dataclasses
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2203_06638_b200.engine import Trainer  # noqa: E402
from paper_2203_06638_b200.objectives import ResNetObjective  # noqa: E402

torch.backends.cudnn.benchmark = True
torch.backends.cudnn.allow_tf32 = False
only = sys.argv[1:] or None
obj = ResNetObjective("resnet20", n_samples=50_000, seed=0, autocast=None)
base = bench.build_cfg(obj, 400 * 4)
variants = {
    "default": base,
    "no_tags": dataclasses.replace(base, track_writes=False),
    "apply_on_updater_stream": dataclasses.replace(base, apply_priority=False),
    "unfused": dataclasses.replace(base, fuse_snapshot=False),
}
for name, cfg in variants.items():
    if only and name not in only:
        continue
    tr = Trainer(cfg, time_apply=True)
    tr.run(5 * 4, evaluate=False)
    for rep in range(3):
        res = tr.run(60 * 4, evaluate=False)
        n_, ms, by = res.apply_timing
        q = np.percentile(np.array(res.apply_ms_samples) * 1e3, [10, 50, 90, 99]) if res.apply_ms_samples else []
        print(json.dumps({"variant": name, "ctas_cap": os.environ.get("LPP_FUSED_CTAS", ""), "rep": rep,
                          "img_per_s": round(sum(res.counter_finals) * 128 / (res.device_ms / 1e3)),
                          "apply_avg_us": round(1e3 * ms / n_, 2),
                          "p10_50_90_99_us": [round(float(v), 1) for v in q],
                          "frac": round(by / (ms / 1e3) / 1e9 / 6560.6, 4)}), flush=True)
    tr.close()
