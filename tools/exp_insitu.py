"""In-situ apply timing (CUDA events around every K1/K2 launch inside the
4-stream ResNet-20 step) across execution variants."""
import dataclasses, json, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2203_06638_b200.engine import Trainer
from paper_2203_06638_b200.objectives import ResNetObjective

torch.backends.cudnn.benchmark = True
K = int(sys.argv[1]) if len(sys.argv) > 1 else 60
obj = ResNetObjective("resnet20", n_samples=50_000, seed=0)
variants = [dict(), dict(track_writes=False), dict(fuse_snapshot=False),
            dict(fuse_snapshot=False, track_writes=False), dict(apply_priority=True),
            dict(apply_priority=True, track_writes=False)]
for v in variants:
    cfg = dataclasses.replace(bench.build_cfg(obj, (K + 5) * 4), **v)
    tr = Trainer(cfg, time_apply=True)
    tr.run(5 * 4, evaluate=False)
    torch.cuda.synchronize()
    res = tr.run(K * 4, evaluate=False)
    n, ms, by = res.apply_timing
    print(json.dumps({**v, "fused": tr.eng.fused(),
                      "img_per_s": round(sum(res.counter_finals) * 128 / (res.device_ms / 1e3)),
                      "apply_avg_us": round(1e3 * ms / n, 2), "MB_per_launch": round(by / n / 1e6, 2),
                      "apply_GBps": round(by / (ms / 1e3) / 1e9)}), flush=True)
    tr.close()
