"""Does timing every apply (CUDA events around each launch, time_apply=True)
cost the step throughput?  fp32 and bf16 ResNet-20 LPP-SGD, U = 4, A/B in
one process, alternating."""
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
for autocast in (None, "bf16"):
    obj = ResNetObjective("resnet20", n_samples=50_000, seed=0, autocast=autocast)
    trs = {ta: Trainer(bench.build_cfg(obj, 4000 * 4), time_apply=ta) for ta in (False, True)}
    for tr in trs.values():
        tr.run(10 * 4, evaluate=False)
    for rep in range(3):
        for ta, tr in trs.items():
            res = tr.run(200 * 4, evaluate=False)
            print(json.dumps({"compute": autocast or "fp32", "time_apply": ta, "rep": rep,
                              "img_per_s": round(sum(res.counter_finals) * 128 / (res.device_ms / 1e3))}),
                  flush=True)
    for tr in trs.values():
        tr.close()
