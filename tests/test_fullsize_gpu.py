"""Parity at BASELINE.json's full sizes (d20 = ResNet-20,
d18 = ResNet-18, d50 = ResNet-50 arenas, and the 100M end of the C4 sweep).

Element-wise kernels are still compared bit-exactly with the C oracle
(oracle/apply_ref.c finishes 25M elements in well under a second); the
averaging round adds the size-independent properties of the domain:
conservation of the worker sum, every arena at the mean after a quiescent
round, write tags stamped on exactly the block."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

D20, D18, D50 = 272_474, 11_220_132, 25_557_032


@pytest.fixture(scope="module")
def N():
    from paper_2203_06638_b200 import _native

    return _native


@pytest.fixture(scope="module")
def orc():
    from oracle import native

    return native


def _arena(a: np.ndarray):
    from paper_2203_06638_b200.arena import Arena

    ar = Arena(len(a), 0)
    ar.tensor.copy_(torch.from_numpy(a).cuda())
    return ar


def _inputs(d, seed):
    gen = np.random.default_rng(seed)
    x = gen.standard_normal(d, dtype=np.float32)
    g = (1e-2 * gen.standard_normal(d, dtype=np.float32)).astype(np.float32)
    m = gen.standard_normal(d, dtype=np.float32)
    return x, g, m


@pytest.mark.parametrize("d", [D20, D18, D50])
@pytest.mark.parametrize("mode", ["red", "bulk"])
def test_apply_momentum_wd_bitexact_at_full_size(N, orc, d, mode):
    x, g, m = _inputs(d, d % 1000)
    ax, ag, am = _arena(x), _arena(g), _arena(m)
    # a layer-aligned partial block of the arena (K2), misaligned start
    lo, hi = d // 7 + 1, d - d // 5
    N.apply_sgd(ax.ptr + 4 * lo, ag.ptr + 4 * lo, am.ptr + 4 * lo, hi - lo, 0.0375, None, 0.9, 5e-4,
                N.MODES[mode], 0)
    torch.cuda.synchronize()
    xv, mv = x[lo:hi].copy(), m[lo:hi].copy()
    orc.apply_sgd(xv, g[lo:hi].copy(), mv, 0.0375, 0.9, 5e-4)
    gx, gm = ax.tensor.cpu().numpy(), am.tensor.cpu().numpy()
    assert np.array_equal(gx[lo:hi], xv) and np.array_equal(gm[lo:hi], mv)
    assert np.array_equal(gx[:lo], x[:lo]) and np.array_equal(gx[hi:], x[hi:])
    for a in (ax, ag, am):
        a.close()


@pytest.mark.parametrize("d", [D20, D50])
def test_fused_apply_snapshot_bitexact_at_full_size(N, orc, d):
    x, g, m = _inputs(d, 5)
    ax, ag, am = _arena(x), _arena(g), _arena(m)
    rep, tg = _arena(np.full(d, -3.0, np.float32)), _arena(np.zeros(d, np.float32))
    lo, hi = d // 10 - 3, d // 2 + 1
    N.apply_snapshot(ax.ptr, ag.ptr, am.ptr, rep.ptr, tg.ptr, d, lo, hi, 0.05, None, 0.9, 5e-4, 77, 0)
    torch.cuda.synchronize()
    xv, mv = x[lo:hi].copy(), m[lo:hi].copy()
    orc.apply_sgd(xv, g[lo:hi].copy(), mv, 0.05, 0.9, 5e-4)
    want = x.copy()
    want[lo:hi] = xv
    assert np.array_equal(ax.tensor.cpu().numpy(), want)
    assert np.array_equal(rep.tensor.cpu().numpy(), want)
    t = tg.tensor.view(torch.int32).cpu().numpy()
    assert (t[lo:hi] == 77).all() and not t[:lo].any() and not t[hi:].any()
    for a in (ax, ag, am, rep, tg):
        a.close()


@pytest.mark.parametrize("d,Q", [(D18, 8), (D50, 4)])
def test_average_round_at_full_size(N, orc, d, Q):
    """K4 owner-computes over Q arenas (local emulation of the group): the
    result matches the oracle bit for bit, every arena holds the mean (to
    fp32 rounding), and the worker sum is conserved up to fp32 rounding of
    Q terms."""
    from paper_2203_06638_b200.engine import shard_bounds

    gen = np.random.default_rng(Q)
    xs = [gen.standard_normal(d, dtype=np.float32) for _ in range(Q)]
    ars = [_arena(a) for a in xs]
    ptrs = [a.ptr for a in ars]
    for lo, hi in shard_bounds(d, Q):      # every owner's shard
        N.average_shard(ptrs, lo, hi, None, N.MODE_RED, 0)
    torch.cuda.synchronize()
    want = [a.copy() for a in xs]
    for lo, hi in shard_bounds(d, Q):
        orc.average(want, lo, hi)
    got = [a.tensor.cpu().numpy() for a in ars]
    for q in range(Q):
        assert np.array_equal(got[q], want[q]), q
    # x_q + (mean - x_q) is the mean up to one fp32 rounding per step
    for q in range(1, Q):
        np.testing.assert_allclose(got[q], got[0], rtol=1e-6, atol=1e-6)
    before = np.sum(np.stack(xs).astype(np.float64), axis=0)
    after = np.sum(np.stack(got).astype(np.float64), axis=0)
    assert np.max(np.abs(after - before)) <= Q * 4 * np.finfo(np.float32).eps * np.max(np.abs(np.stack(xs)))
    for a in ars:
        a.close()


def test_snapshot_and_sampler_at_sweep_size(N):
    """K3 at the 100M end of the C4 sweep is an exact copy; the in-graph
    sampler over the 50,000-image CIFAR set and the 1.28M-image ImageNet
    index range equals its host twin."""
    from paper_2203_06638_b200.arena import Arena

    d = 100_000_000
    src, dst = Arena(d, 0), Arena(d, 0)
    src.tensor.copy_(torch.arange(d, dtype=torch.float32, device="cuda"))
    N.snapshot(src.ptr, dst.ptr, d, 0)
    torch.cuda.synchronize()
    assert torch.equal(src.tensor, dst.tensor)
    src.close(), dst.close()
    for n, b in ((50_000, 128), (1_281_167, 1024)):
        idx = torch.zeros(b, dtype=torch.long, device="cuda")
        step = torch.full((1,), 12345, dtype=torch.long, device="cuda")
        N.sample_indices(idx.data_ptr(), step.data_ptr(), b, n, 99, 0)
        torch.cuda.synchronize()
        assert np.array_equal(idx.cpu().numpy(), N.sample_indices_host(b, n, 99, 12345))


@pytest.mark.parametrize("d", [D20, D18, D50])
def test_fused_apply_with_k5_plan_at_full_size(N, orc, d):
    """The async default at the C1 / C2 / C3 arena sizes (full grid, two
    vectors per thread per round): values bit-exact with the oracle, the
    replica equal to the arena, 32 sampled next-step tags (spread over the
    arena, incl. the tail) by the block-stamp rule, the classification."""
    x, g, m = _inputs(d, 9)
    ax, ag, am = _arena(x), _arena(g), _arena(m)
    rep = _arena(np.full(d, -3.0, np.float32))
    bounds = np.array([0, d // 4, d // 2 + 1, 3 * d // 4, d], dtype=np.int64)
    bid, lo, hi = 2, d // 4, d // 2 + 1
    gen = np.random.default_rng(d)
    idx = np.sort(gen.choice(d, size=32, replace=False)).astype(np.int64)
    idx[-1] = d - 1
    idx = np.unique(idx)
    k = len(idx)
    stamps_h = np.array([11, 5, 30, 7, 9], dtype=np.int32)
    stamps = torch.from_numpy(stamps_h).cuda()
    cell = torch.tensor([8], dtype=torch.long, device="cuda")
    cur = torch.full((k,), 8, dtype=torch.int32, device="cuda")
    nxt = torch.zeros(k, dtype=torch.int32, device="cuda")
    claim = torch.zeros(2, dtype=torch.long, device="cuda")
    plan = N.TagPlan(idx.ctypes.data, nxt.data_ptr(), None, cur.data_ptr(), claim.data_ptr(),
                     cell.data_ptr(), stamps.data_ptr(), bounds.ctypes.data, 4, bid, k)
    N.apply_snapshot_plan(ax.ptr, ag.ptr, am.ptr, rep.ptr, None, d, lo, hi, 0.05, None, 0.9, 5e-4, 77,
                          plan, 0)
    torch.cuda.synchronize()
    xv, mv = x[lo:hi].copy(), m[lo:hi].copy()
    orc.apply_sgd(xv, g[lo:hi].copy(), mv, 0.05, 0.9, 5e-4)
    want = x.copy()
    want[lo:hi] = xv
    assert np.array_equal(ax.tensor.cpu().numpy(), want)
    assert np.array_equal(rep.tensor.cpu().numpy(), want)
    b_of = np.searchsorted(bounds[1:-1], idx, side="right") + 1
    t = np.maximum(np.maximum(stamps_h[0], stamps_h[b_of]), 8)
    t = np.where((idx >= lo) & (idx < hi), np.maximum(t, 77), t)
    assert np.array_equal(nxt.cpu().numpy(), t)
    assert claim.cpu().tolist() == [8, 1]
    for a in (ax, ag, am, rep):
        a.close()
