"""Gradient write-out A/B inside the captured step: autograd.grad + one
multi-tensor copy into the gradient arena ("copy") vs zero + backward()
accumulation into arena views ("accumulate"), ResNet-20 LPP U=4 images/s."""
import dataclasses, json, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2203_06638_b200 import step as step_mod
from paper_2203_06638_b200.engine import Trainer
from paper_2203_06638_b200.objectives import ResNetObjective

torch.backends.cudnn.benchmark = True
# fp32 parameters under autocast (the accumulate mode needs arena .grad views)
obj = ResNetObjective("resnet20", n_samples=50_000, seed=0, shadow_weights=False)
orig = step_mod.StepProgram.__init__
res = {"copy": [], "accumulate": []}
for rep in range(3):
    for mode in ("accumulate", "copy"):
        def init(self, *a, _mode=mode, **k):
            k["grad_mode"] = _mode
            orig(self, *a, **k)
        step_mod.StepProgram.__init__ = init
        K = 100
        tr = Trainer(bench.build_cfg(obj, (K + 5) * 4))
        tr.run(20, evaluate=False)
        r = tr.run(K * 4, evaluate=False)
        res[mode].append(round(sum(r.counter_finals) * 128 / (r.device_ms / 1e3)))
        tr.close()
print(json.dumps(res))
