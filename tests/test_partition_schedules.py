"""Product-side block scheduler and schedules vs the reference (golden
vectors from the reference's own functions) plus the reference's KATs
(test_partition.py:103-188, test_schedules.py:26-175).  CPU only."""

from __future__ import annotations

import itertools

import pytest

from paper_2203_06638_b200.partition import (
    SelectionReason,
    balanced_boundaries,
    even_boundaries,
    make_partition,
    select_block,
)
from paper_2203_06638_b200.schedules import LrSchedule, SyncScheme, constant_schedule, lr_at, sync_every


def test_balanced_matches_reference_golden(golden_scalars):
    for sizes, u, bounds in golden_scalars["partition"]["balanced"]:
        assert list(balanced_boundaries(sizes, u)) == bounds, (sizes, u)


def test_balanced_with_costs_matches_reference_golden(golden_scalars):
    for sizes, u, costs, bounds in golden_scalars["partition"]["costed"]:
        assert list(balanced_boundaries(sizes, u, costs)) == bounds, (sizes, u, costs)
    sizes, u, bounds = golden_scalars["partition"]["c0"]
    assert list(balanced_boundaries(sizes, u)) == bounds


def _brute(sizes, k):
    n = len(sizes)
    suffix = [sum(sizes[i:]) for i in range(n + 1)]
    prefix = [sum(sizes[:i]) for i in range(n + 1)]
    best = None
    for cut in itertools.combinations(range(1, n), k - 1):
        sp = (0, *cut, n)
        key = (max(suffix[sp[i]] for i in range(k)),
               max(prefix[sp[i + 1]] - prefix[sp[i]] for i in range(k)),
               tuple(prefix[c] for c in sp))
        if best is None or key < best:
            best = key
    return best[2]


def test_balanced_fast_path_equals_brute_force_randomised():
    import random

    rnd = random.Random(7)
    for _ in range(400):
        n = rnd.randint(1, 12)
        sizes = [rnd.randint(1, 50) for _ in range(n)]
        k = rnd.randint(1, n)
        assert balanced_boundaries(sizes, k) == _brute(sizes, k)


def test_balanced_kats_and_errors():
    assert balanced_boundaries((4, 4, 4, 4), 2) == (0, 8, 16)
    assert balanced_boundaries((2, 3, 4), 3) == (0, 2, 5, 9)
    assert balanced_boundaries((2, 4, 2), 2) == (0, 2, 8)
    assert balanced_boundaries((2, 2, 4), 2) == (0, 4, 8)
    with pytest.raises(ValueError):
        balanced_boundaries((4, 4), 3)
    with pytest.raises(ValueError):
        balanced_boundaries((4, 0), 1)


def test_balanced_scales_to_resnet50_tensor_count():
    # 161 tensors at U=8: C(160, 7) splits is infeasible for the reference's
    # brute force; the exact fast path answers instantly
    sizes = [((i * 7919) % 5000) + 64 for i in range(161)]
    b = balanced_boundaries(sizes, 8)
    assert len(b) == 9 and b[0] == 0 and b[-1] == sum(sizes)


def test_select_block_matches_reference_golden(golden_scalars):
    for t_st, nb, rank, ids, reasons in golden_scalars["partition"]["select"]:
        for s, (bid, why) in enumerate(zip(ids, reasons)):
            c = select_block(s, t_st, nb, rank)
            assert c.block_id == bid and c.reason.value == why


def test_select_block_kats():
    assert select_block(5, 100, 4, 3).reason is SelectionReason.WARM_START
    assert select_block(101, 100, 4, 3).block_id == 0
    c = select_block(102, 100, 4, 3)
    assert c.block_id == 3 and c.reason is SelectionReason.ALTERNATE_PARTIAL
    for bad in (0, 5):
        with pytest.raises(ValueError):
            select_block(0, 0, 4, bad)
    total, warm = 20000, 2000
    partial = sum(select_block(s, warm, 4, 1).reason is SelectionReason.ALTERNATE_PARTIAL
                  for s in range(1, total + 1))
    assert partial / total == pytest.approx(9 / 20, abs=1 / total)


def test_partition_and_even(golden_scalars):
    for d, k, b in golden_scalars["partition"]["even"]:
        assert list(even_boundaries(d, k)) == b
    p = make_partition(8, (0, 2, 4, 8))
    assert p.block(0) == (0, 8) and p.block(3) == (4, 8) and p.num_blocks == 3
    with pytest.raises(ValueError):
        p.block(4)
    for bad in [(0, 4), (1, 8), (0, 4, 4, 8)]:
        with pytest.raises(ValueError):
            make_partition(8, bad)


def test_lr_traces_bitwise(golden_scalars):
    for name, rec in golden_scalars["schedules"]["lr"].items():
        kw = dict(rec["kw"])
        if "milestones" in kw:
            kw["milestones"] = tuple(kw["milestones"])
        sc = LrSchedule(**kw)
        assert sc.peak == rec["peak"], name
        got = [lr_at(sc, s) for s in rec["s"]]
        assert got == rec["lr"], name


def test_sync_traces(golden_scalars):
    for total, period, sw, sw_res, values in golden_scalars["schedules"]["sync"]:
        sc = SyncScheme(total=total, period=period, switch_point=sw)
        assert sc.switch_point == sw_res
        assert [sync_every(sc, s) for s in range(total + 3)] == values


def test_schedule_validation():
    with pytest.raises(ValueError):
        LrSchedule(kind="linear", alpha0=0.1, total=10)
    with pytest.raises(ValueError):
        LrSchedule(kind="cosine", alpha0=0.1, total=10, warmup=11)
    with pytest.raises(ValueError):
        SyncScheme(total=10, period=0)
    with pytest.raises(ValueError):
        lr_at(constant_schedule(0.1, 10), -1)


def test_product_epoch_sampler_matches_reference(golden_scalars):
    """objectives.py:77-104 / engine.py:294-296 (the product's host sampler)."""
    from paper_2203_06638_b200.sampling import EpochSampler, sample_batch, worker_sampler

    for n, Q, q, rank, seed, bs, batches in golden_scalars["epoch_sampler"]:
        smp = worker_sampler(n, Q, q, rank, seed)
        assert [smp.next_batch(bs).tolist() for _ in batches] == batches
    with pytest.raises(ValueError):
        EpochSampler([], 0)
    import numpy as np

    with pytest.raises(ValueError):
        sample_batch(np.random.default_rng(0), 0, 4)
