"""Property tests (hypothesis): the product's host-side schedule logic agrees
with the oracle's independent restatements and with the reference's brute
force on random inputs, and the round-shard layout covers the arena."""

from __future__ import annotations

import itertools

from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import schedule as osched
from paper_2203_06638_b200.engine import shard_bounds
from paper_2203_06638_b200.partition import balanced_boundaries, select_block
from paper_2203_06638_b200.schedules import LrSchedule, SyncScheme, lr_at, sync_every


def _brute(sizes, k, costs=None):
    n = len(sizes)
    costs = costs or sizes
    suffix = [sum(costs[i:]) for i in range(n + 1)]
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


@settings(max_examples=300, deadline=None)
@given(st.lists(st.integers(1, 60), min_size=1, max_size=11), st.data())
def test_balanced_equals_brute_force(sizes, data):
    k = data.draw(st.integers(1, len(sizes)))
    assert balanced_boundaries(sizes, k) == _brute(sizes, k)


@settings(max_examples=200, deadline=None)
@given(st.lists(st.integers(1, 40), min_size=1, max_size=9), st.data())
def test_balanced_with_nonnegative_costs_equals_brute_force(sizes, data):
    k = data.draw(st.integers(1, len(sizes)))
    costs = data.draw(st.lists(st.floats(0, 100, allow_nan=False), min_size=len(sizes),
                               max_size=len(sizes)))
    assert balanced_boundaries(sizes, k, costs) == _brute(sizes, k, costs)


@settings(max_examples=500, deadline=None)
@given(st.integers(0, 10**6), st.integers(0, 10**5), st.integers(1, 16), st.data())
def test_select_block_equals_oracle(s, t_st, nb, data):
    rank = data.draw(st.integers(1, nb))
    assert select_block(s, t_st, nb, rank).block_id == osched.select_block(s, t_st, nb, rank)


@settings(max_examples=300, deadline=None)
@given(st.sampled_from(["cosine", "multistep"]), st.floats(1e-4, 1.0), st.integers(1, 5000),
       st.data())
def test_lr_equals_oracle(kind, alpha0, total, data):
    warmup = data.draw(st.integers(0, total))
    ms = tuple(sorted(data.draw(st.lists(st.integers(0, total), max_size=3))))
    sc = LrSchedule(kind=kind, alpha0=alpha0, total=total, warmup=warmup,
                    batch_local=data.draw(st.integers(1, 256)), workers=data.draw(st.integers(1, 8)),
                    batch_base=data.draw(st.integers(1, 256)), boost=data.draw(st.booleans()),
                    milestones=ms)
    o = osched.Lr(kind=kind, alpha0=alpha0, total=total, warmup=warmup, peak=sc.peak,
                  milestones=ms, gamma=sc.gamma)
    for s in data.draw(st.lists(st.integers(0, 2 * total), min_size=1, max_size=20)):
        assert lr_at(sc, s) == o.at(s)


@settings(max_examples=200, deadline=None)
@given(st.integers(1, 10**6), st.integers(1, 64), st.data())
def test_sync_every_equals_oracle(total, period, data):
    sw = data.draw(st.one_of(st.none(), st.integers(0, total)))
    sc = SyncScheme(total=total, period=period, switch_point=sw)
    for s in data.draw(st.lists(st.integers(0, 2 * total), min_size=1, max_size=20)):
        assert sync_every(sc, s) == osched.sync_every(s, sc.switch_point, period)


@settings(max_examples=300, deadline=None)
@given(st.integers(0, 10**8), st.integers(1, 8))
def test_owner_shards_cover_the_arena(dim, q):
    sh = shard_bounds(dim, q)
    assert len(sh) == q and sh[0][0] == 0 and sh[-1][1] == dim
    for (a, b), (c, d) in zip(sh, sh[1:]):
        assert b == c and a <= b
    for lo, hi in sh[:-1]:
        assert lo % 4 == 0 and hi % 4 == 0          # 16-byte aligned shard starts


@settings(max_examples=150, deadline=None)
@given(st.lists(st.integers(0, 2**40), min_size=1, max_size=4), st.integers(1, 3_000_000),
       st.integers(1, 64), st.integers(1, 40))
def test_native_numpy_stream_random_cases(entropy, n, b, k):
    """csrc/nprng.cu == numpy for random entropy, population and sizes
    (the draw sequence of a reference updater: choice, then integers)."""
    import numpy as np

    from paper_2203_06638_b200 import _native as N

    g = np.random.default_rng(np.random.SeedSequence(entropy))
    h = N.NpRng(*entropy)
    k = min(k, n)
    assert np.array_equal(g.choice(n, k, replace=False), h.choice(n, k))
    assert np.array_equal(g.integers(0, n, b), h.integers(n, b))
    assert np.array_equal(g.choice(n, k, replace=False), h.choice(n, k))


@settings(max_examples=200, deadline=None)
@given(st.sampled_from(["cosine", "multistep"]), st.floats(1e-4, 1.0), st.integers(1, 5000),
       st.data())
def test_native_lr_at_random_schedules(kind, alpha0, total, data):
    from paper_2203_06638_b200 import _native as N

    warmup = data.draw(st.integers(0, total))
    ms = tuple(sorted(data.draw(st.lists(st.integers(0, total), max_size=4))))
    sched = LrSchedule(kind=kind, alpha0=alpha0, total=total, warmup=warmup, milestones=ms,
                       batch_local=data.draw(st.integers(1, 256)), workers=data.draw(st.integers(1, 8)),
                       batch_base=data.draw(st.integers(1, 256)), boost=data.draw(st.booleans()))
    for s in data.draw(st.lists(st.integers(0, total + 10), min_size=1, max_size=20)):
        assert N.lr_at_native(sched, s) == lr_at(sched, s)
