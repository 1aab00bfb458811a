"""Golden fixture: the reference's OWN asynchronous engine on BASELINE
config 0 (small CNN, LPP-SGD, 2 workers x 2 local updaters, 2-block partial
backprop), 5 seeds -> tests/golden/async_band_cnn.json.

The reference has no CNN; its engine takes any ``Objective``
(objectives.py:33-63).  The small CNN's math (oracle/cnn.py, fp64 torch on
the CPU) is plugged into the reference's Objective ABC unchanged and driven
by the unmodified ``run_experiment`` -> ``_run_async`` (engine.py:466-523):
live threads, so the fixture is a band over seeds, not a trajectory.

    python tests/golden/make_cnn_band.py      (build container: needs /root/reference)
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import torch

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parents[1]))

from make_golden import import_reference  # noqa: E402

N_SAMPLES, PATTERN, DATA_SEED = 512, 0.3, 3
T, B, Q, U = 300, 32, 2, 2


def main() -> None:
    import_reference()
    from asyncsgd import engine as rengine
    from asyncsgd import objectives as robj
    from asyncsgd import partition as rpart
    from asyncsgd import schedules as rsched

    from oracle.cnn import SmallCnnOracle, make_images

    torch.set_num_threads(1)

    class RefCnn(robj.Objective):
        def __init__(self, o):
            self.o, self.dim, self.n_samples = o, o.dim, o.n_samples
            self.layer_param_counts = o.layer_param_counts

        def loss(self, x, batch):
            return self.o.loss(x, batch)

        def init_params(self, seed):
            return self.o.init_params(seed)

        def grad_block(self, x, block, batch):
            self.check_block(block)
            return robj.GradResult(self.o.grad_block(x, block.start, block.stop, batch), 0, 0, len(batch))

    cnn = RefCnn(SmallCnnOracle(*make_images(N_SAMPLES, DATA_SEED, pattern_scale=PATTERN)))
    bounds = rpart.balanced_boundaries(cnn.layer_param_counts, 2)
    band = {"config": f"BASELINE config 0: small CNN, synthetic CIFAR-10-shaped images "
                      f"(n={N_SAMPLES}, class patterns x {PATTERN}, data seed {DATA_SEED}), lpp_sgd "
                      f"Q={Q} U={U}, blocks {list(bounds)}, B={B}, T={T}, cosine 0.05 warmup {T // 10}, "
                      f"T_st {T // 10}, period 16 after T/2, record light; the reference's own "
                      f"engine (live threads)",
            "n_samples": N_SAMPLES, "pattern_scale": PATTERN, "data_seed": DATA_SEED,
            "bounds": list(bounds), "T": T, "B": B, "Q": Q, "U": U,
            "seeds": [], "initial": [], "final": [], "wall_s": [], "p_hat": []}
    for seed in (1, 2, 3, 4, 5):
        cfg = rengine.RunConfig(
            algo="lpp_sgd", objective=cnn, partition=rpart.make_partition(cnn.dim, bounds),
            lr=rsched.LrSchedule(kind="cosine", alpha0=0.05, total=T, warmup=T // 10, batch_local=B,
                                 workers=Q, batch_base=B),
            sync=rsched.SyncScheme(total=T, period=16), budget=T, warm_start_budget=T // 10,
            workers=Q, updaters=U, batch_size=B, seed=seed, record_mode="light")
        t0 = time.perf_counter()
        res = rengine.run_experiment(cfg)
        band["seeds"].append(seed)
        band["initial"].append(res.metrics[0].train_loss)
        band["final"].append(res.metrics[-1].train_loss)
        band["wall_s"].append(time.perf_counter() - t0)
        band["p_hat"].append(res.p_hat)
        print(seed, band["initial"][-1], band["final"][-1], band["wall_s"][-1], flush=True)
    (HERE / "async_band_cnn.json").write_text(json.dumps(band, indent=1) + "\n")


if __name__ == "__main__":
    main()
