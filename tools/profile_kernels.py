"""Standalone launches of K1/K3/K4 for ncu (one stream, one thread):
d20 = 272,474 (ResNet-20 arena) and 64M (sweep) for apply/snapshot, and
K4 over Q=4 local arenas at 16M.  L2 flushed before every launch."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2203_06638_b200 import _native as N  # noqa: E402
from paper_2203_06638_b200.arena import Arena  # noqa: E402

st = torch.cuda.current_stream().cuda_stream
scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush = lambda: N.l2_flush(scratch.data_ptr(), scratch.numel(), st)  # noqa: E731
for d in (272_474, 64_000_000):
    x, g, m, r = (Arena(d, 0) for _ in range(4))
    x.tensor.normal_(), g.tensor.normal_()
    for _ in range(2):
        flush()
        N.apply_sgd(x.ptr, g.ptr, None, d, 1e-3, None, 0.0, 0.0, N.MODE_RED, st)
        flush()
        N.apply_sgd(x.ptr, g.ptr, m.ptr, d, 1e-3, None, 0.9, 5e-4, N.MODE_RED, st)
        flush()
        N.snapshot(x.ptr, r.ptr, d, st)
    for a in (x, g, m, r):
        a.close()
# K1/K2 + K5 (the engine's default for lap/lpp) at the ResNet-18 / ResNet-50 arena sizes
for d in (11_220_132, 25_557_032):
    x, g, m, tg = (Arena(d, 0) for _ in range(4))
    x.tensor.normal_(), g.tensor.normal_()
    for _ in range(2):
        flush()
        N.apply_sgd_tagged(x.ptr, g.ptr, m.ptr, d, 1e-3, None, 0.9, 5e-4, N.MODE_RED, tg.ptr, 7, st)
    for a in (x, g, m, tg):
        a.close()
# K1+K3 fused (the async default) at d20 and d50 with a partial block: the
# engine's launch with the K5 plan (classify this step, read the next step's
# 16 sampled tags before their values, publish the block stamp from the last
# CTA) — and without K5 for comparison; laid out as the engine does it:
# indices, stamps, the round-stamp cell and the step records on the device
claim = torch.zeros(2, dtype=torch.long, device="cuda")
idx = torch.arange(0, 16 * 1000, 1000, dtype=torch.long)   # host: the plan takes indices by value
cell = torch.zeros(1, dtype=torch.long, device="cuda")
dev_tags = torch.zeros(32, dtype=torch.int32, device="cuda")
done = torch.zeros(1, dtype=torch.int32, device="cuda")
stamps = torch.zeros(5, dtype=torch.int32, device="cuda")


def make_plan(d, lo, hi):
    bnd = torch.tensor([0, lo, hi, d], dtype=torch.long)   # host boundaries
    return bnd, N.TagPlan(idx.data_ptr(), dev_tags[16:].data_ptr(), None,
                          dev_tags[:16].data_ptr(), claim.data_ptr(), cell.data_ptr(),
                          stamps.data_ptr(), bnd.data_ptr(), 3, 2, 16)


for d, lo, hi in ((272_474, 68_000, 204_000), (25_557_032, 2_000_000, 12_000_000)):
    x, g, m, rep, tg = (Arena(d, 0) for _ in range(5))
    x.tensor.normal_(), g.tensor.normal_()
    bnd, plan = make_plan(d, lo, hi)
    for _ in range(2):
        flush()
        N.apply_snapshot_plan(x.ptr, g.ptr, m.ptr, rep.ptr, None, d, lo, hi, 1e-3, None, 0.9, 5e-4,
                              3, plan, st)
        flush()
        N.apply_snapshot(x.ptr, g.ptr, m.ptr, rep.ptr, None, d, lo, hi, 1e-3, None, 0.9, 5e-4, 3, st)
    for a in (x, g, m, rep, tg):
        a.close()
# the latency floor: a 16-element sampled-tag gather (one launch, dependent loads)
idx_dev = idx.cuda()
for _ in range(2):
    flush()
    N.gather_block_stamps(stamps.data_ptr(), torch.tensor([0, 5000, 272_474], device="cuda").data_ptr(), 2,
                          idx_dev.data_ptr(), 16, cell.data_ptr(), dev_tags.data_ptr(), None, st)
d = 16_000_000
ars = [Arena(d, 0) for _ in range(4)]
for _ in range(2):
    flush()
    N.average_shard([a.ptr for a in ars], 0, d, None, N.MODE_RED, st)
for _ in range(2):
    flush()
    N.average_shard([a.ptr for a in ars], 0, d, None, N.MODE_BULK, st)   # TMA-staged K4
torch.cuda.synchronize()
print("ok")
