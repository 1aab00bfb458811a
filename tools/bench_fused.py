"""Standalone K1+K3 fused apply timing (CUDA events, L2 flushed before each
launch): d20 / d18 / d50 arenas, full block and a partial block, tags on.
"""
import itertools, json, os, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2203_06638_b200 import _native as N  # noqa: E402
from paper_2203_06638_b200.arena import Arena  # noqa: E402

st = torch.cuda.current_stream().cuda_stream
scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6548.5)
out = []
for d in (272_474, 11_220_132, 25_557_032):
    x, g, m, rep, tg = (Arena(d, 0) for _ in range(5))
    x.tensor.normal_(), g.tensor.normal_()
    for (lo, hi), tagged in itertools.product(((0, d), (d // 10, d // 2)), (True, False)):
        L = hi - lo
        # block: g, x, m read + x, m (+ tag) write; rest: x read; replica write
        nbytes = (24 if tagged else 20) * L + 4 * (d - L) + 4 * d
        ts = []
        for rep_i in range(12):
            N.l2_flush(scratch.data_ptr(), scratch.numel(), st)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            N.apply_snapshot(x.ptr, g.ptr, m.ptr, rep.ptr, tg.ptr if tagged else None, d, lo, hi, 1e-3,
                             None, 0.9, 5e-4, 3, st)
            e1.record()
            torch.cuda.synchronize()
            if rep_i >= 2:
                ts.append(e0.elapsed_time(e1) * 1e3)
        us = sorted(ts)[len(ts) // 2]
        out.append({"d": d, "block": [lo, hi], "tags": tagged, "us": round(us, 2), "GBps": round(nbytes / us / 1e3),
                    "frac": round(nbytes / us / 1e3 / peak, 3)})
    for a in (x, g, m, rep, tg):
        a.close()
print(json.dumps({"rows": out}))
