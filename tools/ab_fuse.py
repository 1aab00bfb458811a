"""A/B: fused apply+snapshot vs separate K3/K1 (interleaved, same process)."""
import dataclasses, json, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2203_06638_b200.engine import Trainer
from paper_2203_06638_b200.objectives import ResNetObjective

torch.backends.cudnn.benchmark = True
K = 60
obj = ResNetObjective("resnet20", n_samples=50_000, seed=0)
trs = {}
for fuse in (False, True):
    cfg = dataclasses.replace(bench.build_cfg(obj, (K + 5) * 4), fuse_snapshot=fuse)
    trs[fuse] = Trainer(cfg)
    trs[fuse].run(20, evaluate=False)
res = {False: [], True: []}
for rep in range(4):
    for fuse in (False, True):
        torch.cuda.synchronize()
        r = trs[fuse].run(K * 4, evaluate=False)
        res[fuse].append(sum(r.counter_finals) * 128 / (r.device_ms / 1e3))
for fuse in (False, True):
    v = sorted(res[fuse])
    print(json.dumps({"fuse_snapshot": fuse, "img_per_s": [round(x) for x in v], "median": round(v[len(v) // 2])}))
