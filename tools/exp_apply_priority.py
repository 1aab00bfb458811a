"""In-situ apply kernel timing with and without a high-priority apply stream
(fused K1+K3, native loop), on the bench's C1/C2/C3 streams; repeated."""
import dataclasses, json, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2203_06638_b200.engine import Trainer
from paper_2203_06638_b200.objectives import ResNetObjective

torch.backends.cudnn.benchmark = True
for arch, B, K, n in (("resnet20", 128, 100, 50_000), ("resnet18", 128, 30, 8192), ("resnet50", 32, 20, 2048)):
    obj = ResNetObjective(arch, n_samples=n, seed=0)
    for prio in (False, True, False, True):
        cfg = dataclasses.replace(bench.build_cfg(obj, (K + 5) * 4), batch_size=B, apply_priority=prio)
        tr = Trainer(cfg, time_apply=True)
        tr.run(5 * 4, evaluate=False)
        torch.cuda.synchronize()
        res = tr.run(K * 4, evaluate=False)
        nn_, ms, by = res.apply_timing
        print(json.dumps({"arch": arch, "apply_priority": prio, "fused": tr.eng.fused(),
                          "native": tr.eng.native_loop(),
                          "img_per_s": round(sum(res.counter_finals) * B / (res.device_ms / 1e3)),
                          "apply_avg_us": round(1e3 * ms / nn_, 2),
                          "frac": round(by / (ms / 1e3) / 1e9 / 6548.5, 3)}), flush=True)
        tr.close()
