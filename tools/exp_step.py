"""Experiment: ResNet-20 fwd/bwd step variants, single stream, CUDA graph.
(a) fp32 params + bf16 autocast + grads accumulated into arena views (current)
(b) bf16 params (no autocast), torch.autograd.grad outputs (no accumulate)
(c) (b) + BN without num_batches_tracked / running stats (track_running_stats=False)
Prints ms per step and kernels per step (graph node count)."""
import sys, time
from pathlib import Path
import torch
import torch.nn as nn
import torch.nn.functional as F
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2203_06638_b200.objectives import CifarResNet20

torch.backends.cudnn.benchmark = True
B = 128
dev = torch.device("cuda")
data = torch.randn(8192, 3, 32, 32, device=dev)
labels = torch.randint(0, 10, (8192,), device=dev)
idx = torch.randint(0, 8192, (B,), device=dev)


def variant(name, dtype, autocast, use_grad, bn_track=True):
    m = CifarResNet20(10).to(dev).to(memory_format=torch.channels_last)
    if not bn_track:
        for mod in m.modules():
            if isinstance(mod, nn.BatchNorm2d):
                mod.track_running_stats = False
                mod.running_mean = None
                mod.running_var = None
                mod.num_batches_tracked = None
    if dtype == torch.bfloat16:
        m = m.to(dtype)
    params = list(m.parameters())
    d = data.to(dtype) if dtype == torch.bfloat16 else data
    if not use_grad:
        for p in params:
            p.grad = torch.zeros_like(p)
    s = torch.cuda.Stream()
    out = [None]

    def body():
        xb = d.index_select(0, idx).contiguous(memory_format=torch.channels_last)
        yb = labels.index_select(0, idx)
        if autocast:
            with torch.autocast("cuda", dtype=torch.bfloat16):
                logits = m(xb)
        else:
            logits = m(xb)
        loss = F.cross_entropy(logits.float(), yb)
        if use_grad:
            out[0] = torch.autograd.grad(loss, params)
        else:
            for p in params:
                p.grad.zero_()
            loss.backward()

    with torch.cuda.stream(s):
        for _ in range(3):
            body()
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        body()
    for _ in range(20):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        g.replay()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 200
    # 4 concurrent streams
    gs = []
    ss = [torch.cuda.Stream() for _ in range(4)]
    for st in ss:
        gg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gg, stream=st):
            body()
        gs.append(gg)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(100):
        for st, gg in zip(ss, gs):
            with torch.cuda.stream(st):
                gg.replay()
    for st in ss:
        torch.cuda.current_stream().wait_stream(st)
    e1.record()
    e1.synchronize()
    ms4 = e0.elapsed_time(e1) / 100
    print(f"{name:40s} 1-stream {ms:.3f} ms/step ({B/ms*1e3:8.0f} img/s)   4-stream {ms4:.3f} ms/4 steps ({4*B/ms4*1e3:8.0f} img/s)", flush=True)


variant("a fp32+autocast+accumulate", torch.float32, True, False)
variant("a' fp32+autocast+autograd.grad", torch.float32, True, True)
variant("b bf16 params+autograd.grad", torch.bfloat16, False, True)
variant("c bf16 params+grad, BN no running stats", torch.bfloat16, False, True, bn_track=False)
