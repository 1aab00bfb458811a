"""In-situ fused-apply timing on ResNet-18 / ResNet-50 (the bench's C2/C3
streams), repeated, for A/B of kernel variants (swap the .so between runs,
or set LPP_FUSED_UNR)."""
import dataclasses, json, os, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2203_06638_b200.engine import Trainer
from paper_2203_06638_b200.objectives import ResNetObjective

torch.backends.cudnn.benchmark = True
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for arch, B, K, n in (("resnet18", 128, 40, 8192), ("resnet50", 32, 30, 2048)):
    obj = ResNetObjective(arch, n_samples=n, seed=0)
    cfg = dataclasses.replace(bench.build_cfg(obj, 400 * 4), batch_size=B)
    tr = Trainer(cfg, time_apply=True)
    tr.run(5 * 4, evaluate=False)
    for rep in range(3):
        res = tr.run(K * 4, evaluate=False)
        nn_, ms, by = res.apply_timing
        print(json.dumps({"variant": tag or os.environ.get("LPP_FUSED_UNR", "2 (default)"), "arch": arch, "rep": rep,
                          "img_per_s": round(sum(res.counter_finals) * B / (res.device_ms / 1e3)),
                          "apply_avg_us": round(1e3 * ms / nn_, 1), "frac": round(by / (ms / 1e3) / 1e9 / 6560.6, 3)}),
              flush=True)
    tr.close()
