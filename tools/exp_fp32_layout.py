"""fp32 (TF32 off) ResNet-20 fwd+bwd throughput on one stream, B = 512:
channels-last vs NCHW, cudnn.benchmark on — which layout the fp32 headline
should use (the convolutions are cuDNN's; the step is a captured graph)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2203_06638_b200.objectives import ResNetObjective  # noqa: E402

torch.backends.cudnn.benchmark = True
torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False
bench_mode = "--no-benchmark" not in sys.argv
torch.backends.cudnn.benchmark = bench_mode
limits = [int(a) for a in sys.argv[1:] if not a.startswith("--")] or [10]
for tf32, cl, lim in [(False, True, l) for l in limits] + ([(False, False, 10), (True, True, 10)] if len(sys.argv) == 1 else []):
    torch.backends.cudnn.allow_tf32 = tf32
    torch.backends.cudnn.benchmark_limit = lim
    if True:
        obj = ResNetObjective("resnet20", n_samples=4096, seed=0, autocast=None, channels_last=cl)
        arena = torch.from_numpy(obj.init_params(0)).float().cuda()
        grads = torch.zeros_like(arena)
        b = obj.bind(arena, grads)
        feats, labs = obj.features_on("cuda"), obj.labels_on("cuda")
        idx = torch.randint(0, 4096, (512,), device="cuda")
        params = b.params

        def step():
            loss = obj.loss_on(b, feats.index_select(0, idx), labs.index_select(0, idx))
            gs = torch.autograd.grad(loss, params)
            torch._foreach_copy_(b.grad_views, list(gs))

        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(3):
                step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        n = 40
        for _ in range(n):
            g.replay()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"tf32={tf32} channels_last={cl} benchmark={bench_mode} limit={lim}: "
              f"{n * 512 / dt:,.0f} images/s")
