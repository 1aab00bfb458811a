"""CNN-step execution variants for the ResNet-20 LPP/MB workload."""
import json, sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2203_06638_b200.engine import Trainer
from paper_2203_06638_b200.objectives import ResNetObjective

torch.backends.cudnn.benchmark = True
K, W = 30, 5
for cl, ac, tf32, U in [(True, "bf16", False, 4), (False, "bf16", False, 4), (False, None, True, 4),
                        (True, None, True, 4), (True, "bf16", False, 8), (False, "bf16", False, 8),
                        (True, "bf16", False, 2)]:
    torch.backends.cuda.matmul.allow_tf32 = tf32
    torch.backends.cudnn.allow_tf32 = tf32
    obj = ResNetObjective("resnet20", n_samples=50_000, seed=0, channels_last=cl, autocast=ac)
    out = {"channels_last": cl, "autocast": ac, "tf32": tf32, "U": U}
    for algo in ("lpp_sgd", "mb_sgd"):
        if algo == "mb_sgd" and U != 4:
            continue
        cfg = bench.build_cfg(obj, (K + W) * U, algo=algo, updaters=U)
        tr = Trainer(cfg)
        tr.run(W * U, evaluate=False)
        torch.cuda.synchronize()
        res = tr.run(K * U, evaluate=False)
        n = sum(res.counter_finals) if algo == "lpp_sgd" else K * U
        out[algo] = round(n * 128 / (res.device_ms / 1e3))
        tr.close()
    print(json.dumps(out), flush=True)
