"""Kernel sweep (config C4): achieved GB/s of K1 (3 modes, +momentum/wd), K3
and K4 (Q arenas on one GPU) vs the measured HBM copy peak.  CUDA events on
the launching stream, warm-up, L2 flushed between timed launches."""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2203_06638_b200 import _native as N  # noqa: E402
from paper_2203_06638_b200.arena import Arena  # noqa: E402


def timed(fn, flush, iters=10, warm=3):
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(iters):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1e6,4e6,16e6,64e6,100e6")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6650.0
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    flush = lambda: N.l2_flush(scratch.data_ptr(), scratch.numel(), st)  # noqa: E731
    rows = []
    for d in [int(float(v)) for v in args.sizes.split(",")]:
        x, g, m, r = Arena(d, 0), Arena(d, 0), Arena(d, 0), Arena(d, 0)
        x.tensor.normal_(), g.tensor.normal_().mul_(1e-3)
        for mode in ("plain", "red", "bulk"):
            for mu, wd, bpe in ((0.0, 0.0, 12), (0.9, 5e-4, 20)):
                t = timed(lambda: N.apply_sgd(x.ptr, g.ptr, m.ptr, d, 1e-3, None, mu, wd, N.MODES[mode], st), flush)
                rows.append(dict(kernel=f"apply_{mode}" + ("_mom_wd" if mu else ""), d=d, us=t * 1e6,
                                 gbs=bpe * d / t / 1e9, frac=bpe * d / t / 1e9 / peak))
        t = timed(lambda: N.snapshot(x.ptr, r.ptr, d, st), flush)
        rows.append(dict(kernel="snapshot", d=d, us=t * 1e6, gbs=8 * d / t / 1e9, frac=8 * d / t / 1e9 / peak))
        for Q in (2, 4, 8):
            if Q * d * 4 > 40e9:
                continue
            ars = [x, r] + [Arena(d, 0) for _ in range(Q - 2)]
            t = timed(lambda: N.average_shard([a.ptr for a in ars], 0, d, None, N.MODE_RED, st), flush)
            # single-GPU emulation: all Q arenas in one HBM.  DRAM bytes = one
            # read + one write-back per arena element (the red.add hits the L2
            # line its own load just brought in); the NVLink-facing number of a
            # real Q-GPU group is 2(Q-1)/Q x 4d per GPU and direction.
            hbm = 2 * 4 * d * Q
            rows.append(dict(kernel=f"average_Q{Q}_local", d=d, us=t * 1e6, gbs=hbm / t / 1e9,
                             frac=hbm / t / 1e9 / peak))
            tb = timed(lambda: N.average_shard([a.ptr for a in ars], 0, d, None, N.MODE_BULK, st), flush)
            rows.append(dict(kernel=f"average_Q{Q}_local_bulk", d=d, us=tb * 1e6, gbs=hbm / tb / 1e9,
                             frac=hbm / tb / 1e9 / peak))
            if Q == 4:
                # the same round while 3 updater streams keep applying K1
                # (momentum + wd) into the averaged arena
                side = [torch.cuda.Stream() for _ in range(3)]
                gs = [Arena(d, 0) for _ in range(3)]
                for ga in gs:
                    ga.tensor.normal_().mul_(1e-3)
                ts = []
                for _ in range(5):
                    flush()
                    torch.cuda.synchronize()
                    for sd, ga in zip(side, gs):
                        for _ in range(3):
                            N.apply_sgd(ars[0].ptr, ga.ptr, None, d, 1e-3, None, 0.0, 5e-4,
                                        N.MODE_RED, sd.cuda_stream)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    N.average_shard([a_.ptr for a_ in ars], 0, d, None, N.MODE_RED, st)
                    b.record()
                    b.synchronize()
                    ts.append(a.elapsed_time(b) * 1e-3)
                    torch.cuda.synchronize()
                tc = sorted(ts)[len(ts) // 2]
                rows.append(dict(kernel="average_Q4_local_under_K1", d=d, us=tc * 1e6,
                                 gbs=hbm / tc / 1e9, frac=hbm / tc / 1e9 / peak,
                                 slowdown=tc / t, note="3 streams of K1 (red, wd) into arena 0 "
                                                       "concurrently; frac counts K4's bytes only"))
                for ga in gs:
                    ga.close()
            for a in ars[2:]:
                a.close()
        for a in (x, g, m, r):
            a.close()
    for row in rows:
        print(json.dumps(row))
    if args.out:
        Path(args.out).write_text("\n".join(json.dumps(r) for r in rows) + "\n")


if __name__ == "__main__":
    main()
