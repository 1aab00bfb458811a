"""In-situ apply kernel timing with and without a high-priority apply stream."""
import dataclasses, json, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2203_06638_b200.engine import Trainer
from paper_2203_06638_b200.objectives import ResNetObjective

torch.backends.cudnn.benchmark = True
for arch, B, K in (("resnet20", 128, 40), ("resnet50", 32, 10)):
    obj = ResNetObjective(arch, n_samples=50_000 if arch == "resnet20" else 2048, seed=0)
    for prio in (False, True):
        cfg = dataclasses.replace(bench.build_cfg(obj, (K + 5) * 4), batch_size=B, apply_priority=prio)
        tr = Trainer(cfg, time_apply=True)
        tr.run(5 * 4, evaluate=False)
        torch.cuda.synchronize()
        res = tr.run(K * 4, evaluate=False)
        n, ms, by = res.apply_timing
        print(json.dumps({"arch": arch, "apply_priority": prio,
                          "img_per_s": round(sum(res.counter_finals) * B / (res.device_ms / 1e3)),
                          "apply_avg_us": round(1e3 * ms / n, 2), "apply_GBps": round(by / (ms / 1e3) / 1e9)}),
              flush=True)
        tr.close()
