"""Small Trainer runs for bisecting an ncu interception failure:
    python tools/ncu_bisect.py <variant>   (tags | notags | python | unfused)"""
import dataclasses
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2203_06638_b200.engine import Trainer  # noqa: E402
from paper_2203_06638_b200.objectives import ResNetObjective  # noqa: E402

v = sys.argv[1]
obj = ResNetObjective("resnet20", n_samples=2048, seed=0, autocast=None)
cfg = bench.build_cfg(obj, 12)
cfg = {"tags": cfg, "notags": dataclasses.replace(cfg, track_writes=False),
       "python": dataclasses.replace(cfg, host_loop="python"),
       "unfused": dataclasses.replace(cfg, fuse_snapshot=False)}[v]
tr = Trainer(cfg)
res = tr.run()
torch.cuda.synchronize()
print(v, "ok", res.counter_finals)
tr.close()
