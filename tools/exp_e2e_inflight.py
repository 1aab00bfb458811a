"""End-to-end (host batches + loss read-back) images/s vs the framework's
CPU thread-pool size: the host row gather used to go through a framework
index_select that fans out to the intra-op pool from each of the U updater
threads (oversubscription: 151k vs 160k images/s); it now goes through
lpp_host_gather_rows and this script shows the pool size no longer matters."""
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
    for sampling, loop in (("host", "python"), ("device", "native")):
        cfg = dataclasses.replace(bench.build_cfg(hobj, (K + 5) * 4, sampling=sampling), host_loop=loop)
        tr = Trainer(cfg, host_batches=True, read_loss=True)
        tr.run(5 * 4, evaluate=False)
        r = tr.run(K * 4, evaluate=False)
        print(json.dumps({"threads": torch.get_num_threads(), "loop": loop,
                          "e2e_img_per_s": round(sum(r.counter_finals) * 128 / (r.device_ms / 1e3))}),
              flush=True)
        tr.close()
