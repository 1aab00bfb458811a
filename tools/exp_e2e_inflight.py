"""e2e (host batches + loss read-back) images/s vs in_flight depth."""
import dataclasses, json, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2203_06638_b200.engine import Trainer
from paper_2203_06638_b200.objectives import ResNetObjective

torch.backends.cudnn.benchmark = True
K = 50
hobj = ResNetObjective("resnet20", n_samples=50_000, seed=0, data="host")
for threads in (0, 1, 4):
  if threads:
    torch.set_num_threads(threads)
  for inf in (2,):
      cfg = dataclasses.replace(bench.build_cfg(hobj, (K + 5) * 4, sampling="host"), in_flight=inf)
      tr = Trainer(cfg, host_batches=True, read_loss=True)
      tr.run(5 * 4, evaluate=False)
      r = tr.run(K * 4, evaluate=False)
      print(json.dumps({"threads": torch.get_num_threads(), "in_flight": inf, "e2e_img_per_s": round(sum(r.counter_finals) * 128 / (r.device_ms / 1e3))}), flush=True)
      tr.close()
