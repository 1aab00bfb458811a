"""Benchmark: LPP-SGD training images/sec on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): ResNet-20 on synthetic CIFAR-10-shaped
data (N(0,1) images, 50,000 x 3x32x32 fp32 = 614 MB resident in HBM, larger
than the 126 MB L2), fp32 convolutions with TF32 off (the reference arm's
precision; the bf16 variant is reported beside it as value_bf16 / e2e_bf16),
LPP-SGD with U = 4 Hogwild CUDA streams per GPU,
B = 128 per stream, 4-block PASSM+ partition (balanced_boundaries),
momentum 0.9, wd 5e-4, cosine lr with warm-up, averaging every tick until
T/2 then every 16 (SyncScheme defaults).  One *step* = one minibatch on
every updater stream (U x B images per GPU); K steps are timed with CUDA
events (max over ranks), after W untimed warm-up steps.

Extra keys beyond the base contract:
  roofline      the fused apply kernel (K1+K3 with the K5 plan), timed live
                with CUDA events around every launch in the timed region,
                algorithmic bytes (block 12 B/elem + 8 momentum, replica
                refresh 4 inside / 8 outside the block; K5 is per-block
                stamps, O(1) bytes) vs MEASURED_PEAKS.json hbm_gbs; + the ncu
                standalone time and DRAM traffic of the same kernel (profiles/)
  e2e           the same metric through Trainer(..., host_batches=True,
                read_loss=True): each step's batch gathered from pinned host
                memory and copied H2D inside the step (native updater loop,
                copy stream), each step's loss copied D2H
  cpu_baseline  oracle/engine_port.py (threaded CPU LPP-SGD, the reference's
                compiled _atomics) on this host, bounded sample, rank 0, N=1
  baselines     the box's own synchronous B1 MB-SGD (same per-GPU B, and
                U x B per GPU) and B2 L-SGD / PL-SGD at the same N (NCCL
                all-reduce for N > 1), and LAP-SGD (same engine, no partial
                backprop), all fp32
  resnet18      config C2 (CIFAR-100-shaped, d = 11.2M): LPP vs MB-SGD images/s
                and the apply kernel's in-situ HBM roofline
  resnet50      config C3 (ImageNet-shaped, d = 25.6M, B = 32 per stream,
                averaging every H = 16 local steps from the start): images/s,
                the apply kernel's in-situ HBM roofline, vs MB-SGD
  kernel_sweep  K1/K3 and the fused apply with its K5 plan alone at 16M/64M
                params, L2 flushed (HBM roofline evidence)
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
# 4 updater + 4 apply + 1 averager (+ 4 copy, end to end) streams per GPU:
# more than the default 8 hardware work queues, which would make unrelated
# streams share a queue (in-situ apply p99 of ms, tools/exp_insitu_variants.py)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "16")

B = 128
U = 4
N_SAMPLES = 50_000


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "src": "measured"}
    return {"hbm_gbs": 6650.0, "src": "fallback"}


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out = ""
        else:
            self.out = ""

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.out.splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


class _Optional:
    """An optional section of the bench line: a failure there (e.g. an
    out-of-memory on a smaller box) is recorded in the line instead of
    losing the headline measurement."""

    def __init__(self, line: dict, key: str):
        self.line, self.key = line, key

    def __enter__(self):
        return self

    def __exit__(self, et, ev, tb):
        if et is None or not issubclass(et, Exception):
            return False
        self.line.setdefault("optional_errors", {})[self.key] = f"{et.__name__}: {ev}"[:300]
        try:
            import torch

            torch.cuda.synchronize()
            torch.cuda.empty_cache()
        except Exception:
            pass
        return True


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def reference_arm(args) -> None:
    """The reference's CPU implementation of the path (oracle port + the
    reference's compiled _atomics), rank 0 only, same metric/config."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    from oracle.engine_port import run_lpp_cpu

    cores = len(os.sched_getaffinity(0))
    # a reference-arm step is ONE minibatch of B images (a bounded sample of
    # the workload: K = 200 steps is ~25 s of CPU work); images/s is the metric
    run_lpp_cpu(slots=max(args.warmup - U, 1), updaters=U, batch_size=B)  # warm-up
    r = run_lpp_cpu(slots=max(args.steps - U, 1), updaters=U, batch_size=B, threads=cores)
    value = r["images"] / r["seconds"]
    steps = r["minibatches"]
    line = {
        "metric": "train_images_per_sec", "value": value, "unit": "images/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * r["seconds"] / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": "resnet20_cifar10_lpp_sgd", "model": "resnet20", "global_batch": B * U,
                   "batch_per_updater": B, "updaters_per_gpu": U, "workers": 1, "blocks": U,
                   "parallelism": f"lpp_sgd_q1_u{U}", "device": "host CPU (reference arm)"},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": r["cores"], "kind": "port",
                         "cpu_count": os.cpu_count(),
                         "sample": f"{r['minibatches']} minibatches x {B} images, one minibatch per "
                                   f"reference-arm step (LPP-SGD, U={U}, "
                                   f"threaded port of engine.py:289-523 incl. the averager and "
                                   f"write tags, torch-CPU ResNet-20 grads, store ops = the "
                                   f"reference's own compiled _atomics ({r['atomics']}))"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def build_cfg(obj, steps_slots: int, algo: str = "lpp_sgd", workers: int = 1, sampling: str = "device",
              updaters: int = U):
    from paper_2203_06638_b200.engine import RunConfig
    from paper_2203_06638_b200.partition import balanced_boundaries, make_partition
    from paper_2203_06638_b200.schedules import LrSchedule, SyncScheme

    total = max(steps_slots, 8)
    nb = max(updaters, 1)
    bounds = balanced_boundaries(obj.layer_param_counts, nb) if algo == "lpp_sgd" else (0, obj.dim)
    return RunConfig(
        algo=algo, objective=obj, partition=make_partition(obj.dim, bounds),
        lr=LrSchedule(kind="cosine", alpha0=0.1, total=total, warmup=max(total // 10, 1),
                      batch_local=B, workers=workers, batch_base=B, boost=(algo == "lpp_sgd")),
        sync=SyncScheme(total=total, period=16), budget=total,
        warm_start_budget=max(total // 10, 1), workers=workers,
        updaters=updaters if algo in ("lap_sgd", "lpp_sgd") else 1, batch_size=B, seed=0,
        momentum=0.9, weight_decay=5e-4, sampling=sampling, evaluate=False, record_mode="off")


def conv_roofline(N) -> dict:
    """The fp32 3x3 convolution kernels (csrc/conv_f32.cu) — most of the
    fp32 step's kernel time — against the FFMA peak measured here
    (lpp_fma_probe): each kernel launched standalone at B = 128 on the
    ResNet-20 shapes, CUDA events, weighted by its launches per minibatch
    (6 / 5 / 5 convolutions x forward, dgrad, wgrad).  Algorithmic flops:
    2 x B x H x W x C x C x 9 per launch."""
    import torch

    from paper_2203_06638_b200 import conv

    def timed(fn, n=20):
        """Device ms per call: n calls captured in one CUDA graph, replayed
        (the kernels are µs-scale; a Python launch loop would time the host)."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(3):
                fn()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, capture_error_mode="thread_local"):
            for _ in range(n):
                fn()
        g.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(5):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        ms_ = a.elapsed_time(b) / (5 * n)
        del g
        return ms_

    sink = torch.empty(148 * 8, device="cuda")
    iters = 2000

    def probe():
        N.check(N.lib.lpp_fma_probe(sink.data_ptr(), 148 * 8, iters, torch.cuda.current_stream().cuda_stream),
                "fma_probe")

    ms = timed(probe, 2)
    peak = 148 * 8 * 256 * iters * 128 * 2 / (ms / 1e3) / 1e12
    B, rows, tot_f, tot_ms = 128, [], 0.0, 0.0
    g = torch.Generator(device="cuda").manual_seed(0)
    for c, hw, cnt in ((16, 32, 6), (32, 16, 5), (64, 8, 5)):
        x = torch.randn(B, c, hw, hw, device="cuda", generator=g).to(memory_format=torch.channels_last)
        w = torch.randn(c, c, 3, 3, device="cuda", generator=g).to(memory_format=torch.channels_last)
        cells = conv.arrival_cells("cuda")
        flop = 2.0 * B * hw * hw * c * c * 9
        for kind, fn in (("fwd", lambda: conv.conv_fwd(x, w)), ("dgrad", lambda: conv.conv_fwd(x, w, dgrad=True)),
                         ("wgrad", lambda: conv.conv_wgrad(x, x, w, cells))):
            t = timed(fn)
            rows.append({"c": c, "hw": hw, "pass": kind, "us": round(1e3 * t, 2),
                         "tflops": round(flop / (t / 1e3) / 1e12, 2)})
            tot_f += cnt * flop
            tot_ms += cnt * t
    ach = tot_f / (tot_ms / 1e3) / 1e12
    return {"bound": "fp32 FFMA (no tensor cores: TF32 is below the reference arm's precision)",
            "kernel": "k_conv3x3 (forward / dgrad) + k_wgrad3x3, 16 stride-1 3x3 convolutions",
            "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
            "peak_src": "measured: lpp_fma_probe (148 x 8 CTAs x 256 threads of dependent-chain FFMA)",
            "flops_per_launch": "2 x 128 x H x W x C x C x 9", "per_kernel": rows,
            "note": "standalone device time (graph-replayed), B = 128, weighted by launches per "
                    "full-backprop minibatch; in the step our kernels are ~93 % of the kernel time "
                    "(profiles/r2_bench_trace_share.txt)"}


def ours(args) -> None:
    import torch
    import torch.distributed as dist

    ws, rank, local = _dist()
    # one process per GPU; LPP_DIST_BACKEND=gloo + fewer GPUs than ranks is the
    # single-GPU validation mode of the N>1 path (no kernel waits on a peer)
    dev = local % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    torch.backends.cudnn.benchmark = True
    group = None
    if ws > 1:
        backend = os.environ.get("LPP_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
        from paper_2203_06638_b200.group import ProcessGroup

        group = ProcessGroup(workers=ws, max_rounds=(args.steps + args.warmup + 4) * U * ws + 64)
    from paper_2203_06638_b200 import _native as N
    from paper_2203_06638_b200.engine import Trainer
    from paper_2203_06638_b200.objectives import ResNetObjective
    from paper_2203_06638_b200.schedules import SyncScheme
    from paper_2203_06638_b200.step import graph_kernel_count

    peaks = _peaks()
    K, W = args.steps, args.warmup

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if ws == 1:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # the headline runs at the reference arm's precision: fp32 convolutions
    # with TF32 off; the bf16 variant is reported beside it
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False

    def lpp_phase(autocast, data="device", host_batches=False, time_apply=False):
        """W warm-up then K timed steps of LPP-SGD ResNet-20 through Trainer;
        returns (images/s, result, trainer facts, launches in the timed phase)."""
        o = ResNetObjective("resnet20", n_samples=N_SAMPLES, seed=0, data=data, autocast=autocast)
        c = build_cfg(o, (K + W) * U, workers=ws)
        t = Trainer(c, group=group, host_batches=host_batches, read_loss=host_batches,
                    time_apply=time_apply)
        facts = {"fused": t.eng.fused(), "native": t.eng.native_loop(), "tracks": c.tracks,
                 "dim": o.dim}
        t.run(W * U, evaluate=False)
        barrier()
        if os.environ.get("LPP_NVTX") and not host_batches and autocast is None:
            t.eng.nvtx = "lpp_timed"   # ncu --nvtx --nvtx-include lpp_timed/ profiles this phase only
        with Clocks(dev) as clk:
            barrier()
            l0, g0 = N.launch_count(), graph_kernel_count()
            r = t.run(K * U, evaluate=False)
            n_l = N.launch_count() - l0
            n_g = graph_kernel_count() - g0
            barrier()
        facts["launches_c_abi"], facts["launches_in_graph"] = n_l, n_g
        t.eng.nvtx = None
        ms = max_over_ranks(r.device_ms)
        v = sum(r.counter_finals) * B * ws / (ms / 1e3)   # claim-then-process: K*U + U per rank
        facts["clocks"] = clk.summary()
        t.close()
        del t
        return v, r, facts, n_l + n_g, ms

    # ---------------- device-resident throughput (value), fp32 ----------------
    value, res, facts, launches, dev_ms = lpp_phase(None, time_apply=True)
    fused, tr_native, dim20 = facts["fused"], facts["native"], facts["dim"]
    n_app, app_ms, app_bytes = res.apply_timing
    k4_rounds, k4_ms = getattr(res, "k4_timing", (0, 0.0))
    achieved = app_bytes / (app_ms / 1e3) / 1e9
    rounds = max((st.round for st in res.stamps), default=0)
    # the per-launch distribution (the native loop's log): the mean above is
    # the contract's number; the median shows the tail's weight
    samples = sorted(1e3 * v for v in getattr(res, "apply_ms_samples", []))
    in_situ_pct = ([round(samples[min(len(samples) - 1, int(q * len(samples)))], 2)
                    for q in (0.10, 0.50, 0.90, 0.99)] if samples else None)

    # traffic: DRAM bytes per launch of the same kernel at the ResNet-20 arena
    # size from the committed ncu --set full capture (profiles/)
    traffic = None
    standalone = None
    tp = ROOT / "profiles" / "r2_kernel_traffic.json"
    if not tp.exists():
        tp = ROOT / "profiles" / "r1_kernel_traffic.json"
    if tp.exists():
        launches_ = json.loads(tp.read_text())["launches"]
        # the plan variant (momentum + wd, K5 plan) at the d20 size: the
        # capture's small-grid launches (the d50 ones run the full grid)
        name = "void k_apply_snapshot<1, 1, 0, 1" if fused else "void k_apply<1, 1, 1>"
        cands = [e for e in launches_ if e["kernel"].startswith(name) and e["grid"] < 148 * 16]
        traffic = sum(e["dram_bytes"] for e in cands) / len(cands) if cands else None
        floor = [e["us"] for e in launches_ if e["kernel"].startswith(("k_gather", "void k_gather"))]
        if cands:
            us = sum(e["us"] for e in cands) / len(cands)
            standalone = {"us": us, "latency_floor_us": min(floor) if floor else None,
                          "src": f"{tp.relative_to(ROOT)}: ncu gpu__time_duration of the same kernel "
                                 "at d20 launched alone (cold L2); latency_floor_us = a 16-element "
                                 "gather kernel (a launch + dependent loads)"}
    line = {
        "metric": "train_images_per_sec", "value": value, "unit": "images/s", "n_gpus": ws,
        "steps": K, "warmup": W, "ms_per_step": dev_ms / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (N(0,1) CIFAR-10-shaped images, uniform labels; random init)",
        "config": {"workload": "resnet20_cifar10_lpp_sgd", "model": "resnet20", "global_batch": B * U * ws,
                   "batch_per_updater": B, "updaters_per_gpu": U, "workers": ws, "blocks": U,
                   "parallelism": f"lpp_sgd_q{ws}_u{U}", "params": dim20,
                   "conv_compute": "fp32 (TF32 off), the reference arm's precision; arena, grads, "
                                   "apply and averaging fp32",
                   "conv_kernels": ("lpp_conv3x3_f32 / lpp_conv3x3_wgrad_f32 (FFMA, NHWC) for the 16 "
                                    "3x3 stride-1 C->C convolutions; cuDNN for the stem, stride-2 and "
                                    "1x1 ones" if os.environ.get("LPP_CONV", "native") != "cudnn"
                                    else "cuDNN (LPP_CONV=cudnn)"),
                   "l2": "inputs larger than L2 (50,000-image dataset, 614 MB fp32, gathered per step)",
                   "sampling": "in-graph device RNG", "host_loop": "native" if tr_native else "python",
                   "momentum": 0.9, "weight_decay": 5e-4,
                   "write_tags": facts["tracks"], "averaging_rounds": rounds},
        "gpu_launches": launches,
        "gpu_launches_note": "lpp_b200 kernels in the timed region on this rank: launched through "
                             "the C ABI (the fused K1+K3+K5 apply per minibatch — its block-stamp "
                             "publication is a stream write, its record a memcpy — the round-stamp "
                             "cell write, and K4 for Q > 1, per averaging round) plus those inside "
                             "the replayed step graphs (the device sampler and the fp32 3x3 "
                             "convolutions: forward, dgrad, wgrad + its reduction), counted per "
                             "graph at capture and summed per replay",
        "gpu_launches_split": {"c_abi": facts["launches_c_abi"], "in_graph": facts["launches_in_graph"]},
        "roofline": {"bound": "hbm",
                     "kernel": ("lpp_apply_snapshot_plan (K1+K3 fused + K5 plan, red.add.v4.f32 + "
                                "re-read)" if fused else
                                "lpp_apply_sgd (K1/K2, red.global.add.v4.f32)"),
                     "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "peak_src": peaks["src"],
                     "traffic": traffic,
                     "traffic_src": "ncu --set full, d20, cold L2 (profiles/)",
                     "launches": n_app, "avg_us": 1e3 * app_ms / max(n_app, 1),
                     "in_situ_us_p10_50_90_99": in_situ_pct,
                     "bytes_per_launch": app_bytes / max(n_app, 1),
                     "standalone": standalone,
                     "note": "d20 arena (1.09 MB) is L2-resident: latency-bound; see kernel_sweep, "
                             "resnet18 / resnet50 apply_roofline for the HBM-sized arenas"},
    }
    line["clocks"] = facts["clocks"]
    if os.environ.get("LPP_CONV", "native") != "cudnn":
        line["roofline_conv"] = conv_roofline(N)

    # ---------------- end to end (host buffers), fp32 ----------------
    if not args.no_e2e:
        # host-drawn batches (the device sampler's stream), pinned row gather,
        # H2D every step, loss D2H every step — inside the native updater loop
        e2e, hres, hfacts, _, _ = lpp_phase(None, data="host", host_batches=True)
        per_img = 3 * 32 * 32 * 4 + 8
        line["e2e"] = {"value": e2e, "unit": "images/s", "h2d_bytes_per_step": U * B * per_img,
                       "d2h_bytes_per_step": U * 4, "api": "Trainer(cfg, host_batches=True, read_loss=True).run",
                       "host_loop": "native" if hfacts["native"] else "python",
                       "losses_read": len(hres.losses),
                       "last_loss": hres.losses[-1] if hres.losses else None}

    # ---------------- the same two measurements with bf16 convolutions ----------------
    if not args.no_bf16:
        with _Optional(line, "bf16"):
            vb, rb, fb, _, _ = lpp_phase("bf16", time_apply=True)
            line["value_bf16"] = vb
            # the same apply kernel timed inside the bf16 step (shorter
            # convolution CTAs: fewer waves to wait through) — round 1's
            # headline condition
            nb_, msb_, byb_ = rb.apply_timing
            if nb_:
                ab_ = byb_ / (msb_ / 1e3) / 1e9
                line["roofline"]["in_situ_bf16_step"] = {
                    "avg_us": 1e3 * msb_ / nb_, "achieved": ab_, "frac": ab_ / peaks["hbm_gbs"],
                    "launches": nb_}
            line["bf16"] = {"conv_compute": "bf16 shadow weights (one cast per step from the fp32 "
                                            "replica), dataset stored NHWC bf16; arena, grads, apply, "
                                            "averaging fp32", "clocks": fb["clocks"]}
            if not args.no_e2e:
                eb, _, _, _, _ = lpp_phase("bf16", data="host", host_batches=True)
                line["e2e_bf16"] = {"value": eb, "unit": "images/s",
                                    "h2d_bytes_per_step": U * B * (3 * 32 * 32 * 4 + 8),
                                    "d2h_bytes_per_step": U * 4}

    # ---------------- averaging bandwidth across the group (N > 1) ----------------
    # BASELINE.json's second metric: K4 over the P2P/NVLink-mapped arenas of
    # all ranks, each rank averaging its owned shard of a d-element group;
    # busbw = 2(Q-1)/Q x 4d bytes per GPU and direction / max-over-ranks time.
    # The denominators: NVLink 5's 900 GB/s per direction (nominal) and a peer
    # copy measured here in the same run (cudaMemcpyPeer-class read of the
    # next rank's arena into local HBM, 256 MB)
    if ws > 1 and not args.no_sweep:
        from paper_2203_06638_b200.arena import Arena
        from paper_2203_06638_b200.engine import shard_bounds

        avg = {}
        peer_gbs = None
        for d in (16_000_000, 64_000_000):
            ar = Arena(d, dev)
            ar.tensor.normal_()
            ptrs = group.attach_arenas(ar)
            lo, hi = shard_bounds(d, ws)[rank]
            st = torch.cuda.current_stream().cuda_stream
            if d == 64_000_000:
                # peer copy: this rank pulls its right neighbour's whole arena
                dst = torch.empty(d, dtype=torch.float32, device="cuda")
                src = ptrs[(rank + 1) % ws]
                for _ in range(3):
                    N.copy_async(dst.data_ptr(), src, 4 * d, st)
                ts = []
                for _ in range(5):
                    barrier()
                    a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a_.record()
                    N.copy_async(dst.data_ptr(), src, 4 * d, st)
                    b_.record()
                    b_.synchronize()
                    ts.append(max_over_ranks(a_.elapsed_time(b_)))
                peer_gbs = 4 * d / (sorted(ts)[len(ts) // 2] / 1e3) / 1e9
                del dst
            for mode_name, mode in (("red", N.MODE_RED), ("bulk", N.MODE_BULK)):
                for _ in range(3):
                    N.average_shard(ptrs, lo, hi, None, mode, st)
                ts = []
                for _ in range(10):
                    barrier()
                    a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a_.record()
                    N.average_shard(ptrs, lo, hi, None, mode, st)
                    b_.record()
                    b_.synchronize()
                    ts.append(max_over_ranks(a_.elapsed_time(b_)))
                t = sorted(ts)[len(ts) // 2] / 1e3
                busbw = 2 * (ws - 1) / ws * 4 * d / t / 1e9
                avg.setdefault(str(d), {})[mode_name] = {"us": t * 1e6, "busbw_gbs": busbw,
                                                         "frac_of_900": busbw / 900.0}
            barrier()
            for pm in group.peers[-(ws - 1):]:
                pm.close()
            del group.peers[-(ws - 1):]
            ar.close()
        if peer_gbs:
            for per in avg.values():
                for v in per.values():
                    v["frac_of_peer_copy"] = v["busbw_gbs"] / peer_gbs
        # the training run's own rounds (native averager, CUDA events around
        # every K4 launch): ResNet-20's 1.09 MB arena, latency-bound
        avg_us = 1e3 * k4_ms / k4_rounds if k4_rounds else 0.0
        avg_us = max_over_ranks(avg_us)
        avg["in_situ_resnet20"] = {
            "rounds": k4_rounds, "avg_us": avg_us,
            "busbw_gbs": (2 * (ws - 1) / ws * 4 * dim20 / (avg_us * 1e-6) / 1e9) if avg_us else None}
        line["averaging"] = {"kernel": "lpp_average_shard (K4, owner-computes over peer arenas; "
                                       "red = LSU loads + red.add, bulk = TMA-staged)",
                             "unit": "GB/s", "sizes": avg, "peer_copy_gbs": peer_gbs,
                             "ranks_share_device": torch.cuda.device_count() < ws,
                             "note": "busbw = 2(Q-1)/Q x 4d per GPU per direction (nccl-tests convention); "
                                     "900 = NVLink 5 nominal per direction; peer_copy_gbs = a 256 MB "
                                     "read of the next rank's arena measured in this run"}

    # ---------------- synchronous baselines on the same box, at the same N ----------------
    # B1 NCCL MB-SGD (engine.py:544-583) and B2 NCCL L-SGD / PL-SGD (period 16
    # after T/2, engine.py:586-629), same fp32 ResNet-20, same per-GPU batch;
    # MB-SGD also at B = U x 128 per GPU (as many images per step as the U
    # LPP updaters); LAP-SGD = the async engine without partial backprop
    if not args.no_baselines:
        with _Optional(line, "baselines"):
            bobj = ResNetObjective("resnet20", n_samples=N_SAMPLES, seed=0, data="device", autocast=None)

            def sync_rate(algo, batch, steps, warm):
                c = dataclasses.replace(build_cfg(bobj, steps + warm, algo=algo, workers=ws),
                                        batch_size=batch)
                t = Trainer(c, group=group)
                t.run(warm, evaluate=False)
                barrier()
                r = t.run(steps, evaluate=False)
                ms = max_over_ranks(r.device_ms)
                t.close()
                return steps * batch * ws / (ms / 1e3)

            base = {}
            coll = f"{dist.get_backend()} all-reduce" if ws > 1 else "none (one worker)"
            mb = sync_rate("mb_sgd", B, K * U, W * U)
            base["mb_sgd"] = {"value": mb, "unit": "images/s", "batch_per_gpu": B, "streams": 1,
                              "collective": coll, "note": "B1: synchronous SGD, same per-GPU batch"}
            mbl = sync_rate("mb_sgd", B * U, K, W)
            base[f"mb_sgd_b{B * U}"] = {"value": mbl, "unit": "images/s", "batch_per_gpu": B * U,
                                        "streams": 1, "collective": coll,
                                        "note": "B1 at U x 128 per GPU: the images per step of the U "
                                                "LPP updaters together, U x fewer model updates"}
            pl = sync_rate("pl_sgd", B, K * U, W * U)
            base["pl_sgd"] = {"value": pl, "unit": "images/s", "batch_per_gpu": B, "streams": 1,
                              "collective": coll,
                              "note": "B2: local SGD, parameter average every step until T/2, then "
                                      "every 16 steps"}
            if ws == 1:
                lcfg = build_cfg(bobj, (K + W) * U, algo="lap_sgd", workers=1)
                ltr = Trainer(lcfg)
                ltr.run(W * U, evaluate=False)
                torch.cuda.synchronize()
                lres = ltr.run(K * U, evaluate=False)
                base["lap_sgd"] = {"value": sum(lres.counter_finals) * B / (lres.device_ms / 1e3),
                                   "unit": "images/s", "streams": U,
                                   "note": "same engine, full backprop every step (no PASSM+ blocks)"}
                ltr.close()
                del ltr
            base["lpp_over_mb"] = value / mb
            base[f"lpp_over_mb_b{B * U}"] = value / mbl
            base["lpp_over_pl"] = value / pl
            base["dtype"] = "f32"
            line["baselines"] = base

    # ---------------- the paper's U = 6 variant ----------------
    if not args.no_baselines and ws == 1:
        with _Optional(line, "lpp_sgd_u6"):
            o6 = ResNetObjective("resnet20", n_samples=N_SAMPLES, seed=0, data="device", autocast=None)
            c6 = build_cfg(o6, (K + W) * 6, workers=1, updaters=6)
            t6 = Trainer(c6)
            t6.run(W * 6, evaluate=False)
            torch.cuda.synchronize()
            r6 = t6.run(K * 6, evaluate=False)
            line["baselines"]["lpp_sgd_u6"] = {
                "value": sum(r6.counter_finals) * B / (r6.device_ms / 1e3), "unit": "images/s",
                "streams": 6, "note": "same workload with 6 updater streams (the paper's best LPP row)"}
            t6.close()
            del t6

    def phase(cfg_, steps, warm, images_per_slot, time_apply=False):
        """warm-up + timed phase of cfg_ over the group; returns (whole-job
        images/s, result); the timed region is max over ranks."""
        t = Trainer(cfg_, group=group, time_apply=time_apply)
        t.run(warm, evaluate=False)
        barrier()
        r = t.run(steps, evaluate=False)
        ms = max_over_ranks(r.device_ms)
        slots = sum(r.counter_finals) if cfg_.algo in ("lap_sgd", "lpp_sgd") else steps
        t.close()
        return slots * images_per_slot * ws / (ms / 1e3), r

    def apply_roofline(r):
        na, msa, bya = r.apply_timing
        a_ = bya / (msa / 1e3) / 1e9
        return {"achieved": a_, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": a_ / peaks["hbm_gbs"],
                "launches": na, "avg_us": 1e3 * msa / max(na, 1), "bytes_per_launch": bya / max(na, 1)}

    # ---------------- ResNet-18 / CIFAR-100 shape (config C2), at every N ----------------
    if not args.no_rn18:
        with _Optional(line, "resnet18"):
            obj18 = ResNetObjective("resnet18", n_samples=N_SAMPLES, seed=0, data="device")
            out18 = {"workload": "resnet18_cifar100_u4_b128", "params": obj18.dim, "unit": "images/s",
                     "workers": ws, "conv_compute": "bf16 shadow weights (all three rows)",
                     "collective": f"{dist.get_backend()} all-reduce (B1/B2)" if ws > 1 else "none"}
            for algo in ("lpp_sgd", "mb_sgd", "pl_sgd"):
                c18 = build_cfg(obj18, (args.rn18_steps + 3) * U, algo=algo, workers=ws)
                lpp = algo == "lpp_sgd"
                v18, r18 = phase(c18, args.rn18_steps * U, 3 * U, B, time_apply=lpp)
                out18[algo] = v18
                if lpp:
                    out18["apply_roofline"] = apply_roofline(r18)
            out18["lpp_over_mb"] = out18["lpp_sgd"] / out18["mb_sgd"]
            out18["lpp_over_pl"] = out18["lpp_sgd"] / out18["pl_sgd"]
            line["resnet18"] = out18

    # ---------------- ResNet-50 / ImageNet shape (config C3), at every N ----------------
    if not args.no_rn50:
        with _Optional(line, "resnet50"):
            obj50 = ResNetObjective("resnet50", n_samples=2048, seed=0, data="device")
            c50 = build_cfg(obj50, 64, workers=ws)
            # C3: B = 32 per stream, non-blocking averaging every H = 16 local
            # steps from the start (switch_point 0)
            c50 = dataclasses.replace(c50, batch_size=32,
                                      sync=SyncScheme(total=c50.sync.total, period=16, switch_point=0))
            v50, r50 = phase(c50, args.rn50_steps * U, 3 * U, 32, time_apply=True)
            line["resnet50"] = {
                "workload": "resnet50_imagenet224_lpp_sgd_u4_b32_h16", "params": obj50.dim, "workers": ws,
                "conv_compute": "bf16 shadow weights (both rows)", "value": v50, "unit": "images/s",
                "apply_roofline": apply_roofline(r50)}
            m50 = dataclasses.replace(build_cfg(obj50, 64, algo="mb_sgd", workers=ws), batch_size=32)
            line["resnet50"]["mb_sgd"], _ = phase(m50, args.rn50_steps * U, 3 * U, 32)
            line["resnet50"]["lpp_over_mb"] = line["resnet50"]["value"] / line["resnet50"]["mb_sgd"]

    # ---------------- kernel sweep (HBM roofline evidence) ----------------
    if not args.no_sweep and rank == 0:
        with _Optional(line, "kernel_sweep"):
            from paper_2203_06638_b200.arena import Arena

            st = torch.cuda.current_stream().cuda_stream
            scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
            sweep = []
            import numpy as np

            # the shipped fused apply with its K5 plan (16 sampled tags,
            # classification, block stamps), as the engine launches it
            kstamps = torch.zeros(5, dtype=torch.int32, device="cuda")
            kcell = torch.zeros(1, dtype=torch.long, device="cuda")
            krec = torch.zeros(64, dtype=torch.long, device="cuda")

            def plan_for(d_, lo_, hi_):
                bnd = np.array([0, lo_, hi_, d_], dtype=np.int64)
                idx = np.sort(np.random.default_rng(0).choice(d_, 16, replace=False)).astype(np.int64)
                return (bnd, idx), N.TagPlan(idx.ctypes.data, krec[32:].data_ptr(), None, krec[4:].data_ptr(),
                                             krec.data_ptr(), kcell.data_ptr(), kstamps.data_ptr(),
                                             bnd.ctypes.data, 3, 2, 16)

            for d in (16_000_000, 64_000_000):
                x, g, m = Arena(d, dev), Arena(d, dev), Arena(d, dev)
                r_ = Arena(d, dev)
                part = (d // 5, d // 5 + 2 * d // 5)      # a partial block of 40 %
                keep_full, plan_full = plan_for(d, 0, d)
                keep_part, plan_part = plan_for(d, *part)
                blen = part[1] - part[0]
                for name, fn, bpe in (
                    ("apply_red", lambda: N.apply_sgd(x.ptr, g.ptr, None, d, 1e-3, None, 0.0, 0.0, N.MODE_RED, st), 12),
                    ("apply_red_mom_wd", lambda: N.apply_sgd(x.ptr, g.ptr, m.ptr, d, 1e-3, None, 0.9, 5e-4, N.MODE_RED, st), 20),
                    ("apply_bulk_mom_wd", lambda: N.apply_sgd(x.ptr, g.ptr, m.ptr, d, 1e-3, None, 0.9, 5e-4, N.MODE_BULK, st), 20),
                    ("snapshot", lambda: N.snapshot(x.ptr, r_.ptr, d, st), 8),
                    ("fused_apply_k5_full_block_mom_wd",
                     lambda: N.apply_snapshot_plan(x.ptr, g.ptr, m.ptr, r_.ptr, None, d, 0, d, 1e-3, None, 0.9,
                                                   5e-4, 3, plan_full, st), 24),
                    ("fused_apply_k5_block40pct_mom_wd",
                     lambda: N.apply_snapshot_plan(x.ptr, g.ptr, m.ptr, r_.ptr, None, d, part[0], part[1], 1e-3,
                                                   None, 0.9, 5e-4, 3, plan_part, st),
                     (24 * blen + 8 * (d - blen)) / d),
                ):
                    for _ in range(5):
                        fn()
                    ts = []
                    for _ in range(10):
                        N.l2_flush(scratch.data_ptr(), scratch.numel(), st)
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record()
                        fn()
                        b.record()
                        b.synchronize()
                        ts.append(a.elapsed_time(b))
                    t = sorted(ts)[len(ts) // 2] / 1e3
                    gbs = bpe * d / t / 1e9
                    sweep.append({"kernel": name, "params": d, "us": t * 1e6, "gbs": gbs,
                                  "frac": gbs / peaks["hbm_gbs"]})
                # K4 over Q=4 arenas in this one HBM (the NVLink path needs >1 GPU):
                # DRAM bytes = read + write-back of every arena element
                ars = [x, r_, Arena(d, dev), Arena(d, dev)]
                for kname, kmode in (("average_q4_local_hbm", N.MODE_RED),
                                     ("average_q4_local_hbm_tma", N.MODE_BULK)):
                    for _ in range(3):
                        N.average_shard([a_.ptr for a_ in ars], 0, d, None, kmode, st)
                    ts = []
                    for _ in range(10):
                        N.l2_flush(scratch.data_ptr(), scratch.numel(), st)
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record()
                        N.average_shard([a_.ptr for a_ in ars], 0, d, None, kmode, st)
                        b.record()
                        b.synchronize()
                        ts.append(a.elapsed_time(b))
                    t = sorted(ts)[len(ts) // 2] / 1e3
                    gbs = 8 * 4 * d / t / 1e9
                    sweep.append({"kernel": kname, "params": d, "us": t * 1e6, "gbs": gbs,
                                  "frac": gbs / peaks["hbm_gbs"]})
                for a_ in (x, g, m, r_) + tuple(ars[2:]):
                    a_.close()
            line["kernel_sweep"] = sweep

    # ---------------- the reference's own store primitives on this host ----------------
    # accum_cas_f64 (the apply) and snapshot_f64 (K3) of the
    # reference's compiled _atomics, 1 thread, at 1M / 4M elements (fp64)
    if not args.no_cpu and rank == 0 and ws == 1:
        with _Optional(line, "cpu_reference_primitives"):
            import numpy as np

            from oracle.native import reference_atomics

            at = reference_atomics()
            if at is not None:
                prims = []
                for d in (1_000_000, 4_000_000):
                    x = np.random.default_rng(0).normal(size=d)
                    g = 1e-3 * np.random.default_rng(1).normal(size=d)
                    out = np.empty(d)
                    for name, fn, nbytes in (("accum_cas_f64", lambda: at.accum_cas_f64(x, 0, g, -1.0), 24 * d),
                                             ("snapshot_f64", lambda: at.snapshot_f64(x, out), 16 * d)):
                        fn()
                        t0 = time.perf_counter()
                        reps = 3
                        for _ in range(reps):
                            fn()
                        sec = (time.perf_counter() - t0) / reps
                        prims.append({"primitive": name, "elements": d, "ms": 1e3 * sec,
                                      "gbs": nbytes / sec / 1e9})
                # one averaging round of the reference at Q = 2 (engine.py:418-421,
                # 199-229): snapshot both stores, fixed-order mean, add_assign
                # (mean - snap) through the reference's CAS accumulate
                d = 1_000_000
                xs = [np.random.default_rng(q).normal(size=d) for q in range(2)]
                snaps = [np.empty(d) for _ in range(2)]
                t0 = time.perf_counter()
                for q in range(2):
                    at.snapshot_f64(xs[q], snaps[q])
                mean = np.mean(np.stack(snaps), axis=0)
                for q in range(2):
                    at.accum_cas_f64(xs[q], 0, mean - snaps[q], 1.0)
                sec = time.perf_counter() - t0
                prims.append({"primitive": "averaging_round_Q2 (snapshot + mean + add_assign)",
                              "elements": d, "ms": 1e3 * sec,
                              "gbs_busbw_convention": 2 * (2 - 1) / 2 * 8 * d / sec / 1e9})
                line["cpu_reference_primitives"] = {
                    "threads": 1, "source": "oracle/_ref (the reference's _atomics.c, compiled from "
                                            "its own source)", "rows": prims}

    # ---------------- CPU baseline (rank 0, N=1) ----------------
    if not args.no_cpu and rank == 0 and ws == 1:
        with _Optional(line, "cpu_baseline"):
            from oracle.engine_port import run_lpp_cpu

            # bounded sample of the same workload: ~100 minibatches, 10-15 s of
            # CPU work on the box's host cores (after a short warm-up)
            run_lpp_cpu(slots=U, updaters=U, batch_size=B)
            r = run_lpp_cpu(slots=25 * U, updaters=U, batch_size=B)
            line["cpu_baseline"] = {"value": r["images"] / r["seconds"], "unit": "images/s",
                                    "cores": r["cores"], "kind": "port", "cpu_count": os.cpu_count(),
                                    "sample": f"{r['minibatches']} minibatches x {B} images, LPP-SGD U={U} "
                                              f"(port of engine.py:289-523 incl. averager + tags), "
                                              f"torch-CPU ResNet-20 grads, store ops via the "
                                              f"reference's compiled _atomics ({r['atomics']})"}
    if rank == 0:
        print(json.dumps(line), flush=True)
        if args.out:
            Path(args.out).write_text(json.dumps(line, indent=1) + "\n")
    if ws > 1:
        group.close()
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)   # timed minibatches = steps x U; ramp-up and drain are <2 % at 200
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-bf16", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-baselines", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-rn50", action="store_true")
    ap.add_argument("--no-rn18", action="store_true")
    ap.add_argument("--rn18-steps", type=int, default=15)
    ap.add_argument("--rn50-steps", type=int, default=10)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        reference_arm(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
