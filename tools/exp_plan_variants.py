"""Standalone timing (CUDA events, 300 back-to-back launches, d20 and d50) of
the fused apply with the K5 plan in variants that isolate its costs:
no plan / plan without outputs / + classification record / + next-step
tags, with the records in device vs host-mapped memory."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2203_06638_b200 import _native as N  # noqa: E402
from paper_2203_06638_b200.arena import Arena  # noqa: E402

st = torch.cuda.current_stream().cuda_stream
hb = N.HostBuffer(4096)
idx = torch.arange(0, 16 * 1000, 1000, dtype=torch.long)   # host: the plan takes indices by value
cell = torch.zeros(1, dtype=torch.long, device="cuda")
tags_dev = torch.zeros(64, dtype=torch.int32, device="cuda")
claim_dev = torch.zeros(4, dtype=torch.long, device="cuda")
done = torch.zeros(1, dtype=torch.int32, device="cuda")
stamps = torch.zeros(5, dtype=torch.int32, device="cuda")
for d, lo, hi in ((272_474, 68_000, 204_000), (25_557_032, 2_000_000, 12_000_000)):
    x, g, m, rep = (Arena(d, 0) for _ in range(4))
    x.tensor.normal_(), g.tensor.normal_()
    bnd = torch.tensor([0, lo, hi, d], dtype=torch.long)   # host boundaries

    def plan(next_idx=True, next_host=False, claim=None):
        return N.TagPlan(idx.data_ptr() if next_idx else None, tags_dev[16:32].data_ptr(),
                         hb.dev + 512 if next_host else None, tags_dev[:16].data_ptr(), claim,
                         cell.data_ptr(), stamps.data_ptr(), bnd.data_ptr(), 3, 2, 16)

    variants = {
        "no plan": None,
        "plan: stamps only": plan(next_idx=False),
        "plan: + next tags (device)": plan(),
        "plan: + next tags (host-mapped)": plan(next_host=True),
        "plan: + claim record (device)": plan(claim=claim_dev.data_ptr()),
        "plan: + claim record (host-mapped)": plan(claim=hb.dev + 1024),
        "plan: engine layout (both host-mapped)": plan(next_host=True, claim=hb.dev + 1024),
    }
    for name, p in variants.items():
        def launch():
            if p is None:
                N.apply_snapshot(x.ptr, g.ptr, m.ptr, rep.ptr, None, d, lo, hi, 1e-3, None, 0.9, 5e-4, 3, st)
            else:
                N.apply_snapshot_plan(x.ptr, g.ptr, m.ptr, rep.ptr, None, d, lo, hi, 1e-3, None, 0.9,
                                      5e-4, 3, p, st)
        for _ in range(20):
            launch()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 300
        a.record()
        for _ in range(n):
            launch()
        b.record()
        b.synchronize()
        print(f"d={d:>9}  {name:<40} {1e3 * a.elapsed_time(b) / n:8.2f} us", flush=True)
    for a_ in (x, g, m, rep):
        a_.close()
