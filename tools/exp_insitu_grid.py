"""In-situ time of the fused apply (K1+K3+K5 plan) inside the bench's fp32
ResNet-20 LPP-SGD run, for a grid-size cap given as LPP_FUSED_CTAS (the
experiment hook in apply_snapshot_launch); also images/s.  Run once per cap:

    for c in 0 148 74 37; do LPP_FUSED_CTAS=$c python tools/exp_insitu_grid.py $c; done
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2203_06638_b200.engine import Trainer  # noqa: E402
from paper_2203_06638_b200.objectives import ResNetObjective  # noqa: E402

torch.backends.cudnn.benchmark = True
torch.backends.cudnn.allow_tf32 = False
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for autocast in (None, "bf16"):
    obj = ResNetObjective("resnet20", n_samples=50_000, seed=0, autocast=autocast)
    cfg = bench.build_cfg(obj, 400 * 4)
    tr = Trainer(cfg, time_apply=True)
    tr.run(5 * 4, evaluate=False)
    for rep in range(2):
        res = tr.run(60 * 4, evaluate=False)
        n_, ms, by = res.apply_timing
        print(json.dumps({"ctas": tag, "compute": autocast or "fp32", "rep": rep,
                          "img_per_s": round(sum(res.counter_finals) * 128 / (res.device_ms / 1e3)),
                          "apply_avg_us": round(1e3 * ms / n_, 2),
                          "frac": round(by / (ms / 1e3) / 1e9 / 6560.6, 4)}), flush=True)
    tr.close()
