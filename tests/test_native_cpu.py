"""C-ABI library checks that need no GPU: it loads, exports every symbol
include/lpp_b200.h declares, and its host atomics (K6, the replacement of
_atomics.{load,store,fetch_add}_i64) keep the reference's counter contract
under real thread contention (test_paramstore.py:133-183)."""

from __future__ import annotations

import re
import subprocess
import threading
from pathlib import Path

import numpy as np
import pytest

from paper_2203_06638_b200 import _native as N

ROOT = Path(__file__).resolve().parents[1]


def _declared_symbols() -> set[str]:
    text = (ROOT / "include" / "lpp_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(lpp_[a-z0-9_]+)\s*\(", text))


def test_library_exports_every_declared_symbol():
    declared = _declared_symbols()
    assert len(declared) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (lpp_[a-z0-9_]+)$", out, flags=re.M))
    assert declared <= exported, declared - exported
    assert declared == set(N.EXPORTED), declared ^ set(N.EXPORTED)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_abi_version_and_error_channel():
    assert N.lib.lpp_abi_version() == 4
    with pytest.raises(IndexError):
        # range check happens before any device work
        N.accum(0, 4, 3, 0, 2, 1.0, N.MODE_RED, 0)


def test_counter_semantics():
    from paper_2203_06638_b200.paramstore import AtomicCounter

    c = AtomicCounter(0)
    assert c.read_and_inc() == 0 and c.read_and_inc() == 1 and c.read() == 2
    c = AtomicCounter(5)
    assert c.add(3) == 5 and c.read() == 8
    c.store(-2)
    assert c.read() == -2
    assert c.cas(-2, 7) and not c.cas(-2, 9) and c.read() == 7


def _run_threads(bodies):
    gate = threading.Barrier(len(bodies))

    def wrap(fn):
        def run():
            gate.wait()
            fn()
        return run

    ts = [threading.Thread(target=wrap(b)) for b in bodies]
    for t in ts:
        t.start()
    for t in ts:
        t.join()


def test_concurrent_claims_are_unique():
    from paper_2203_06638_b200.paramstore import AtomicCounter

    c = AtomicCounter(0)
    got = [[] for _ in range(16)]

    def claim(i):
        def body():
            for _ in range(2000):
                got[i].append(c.read_and_inc())
        return body

    _run_threads([claim(i) for i in range(16)])
    flat = sorted(v for g in got for v in g)
    assert flat == list(range(16 * 2000))


def test_cas_elects_exactly_one_opener_per_round():
    cell = np.zeros(1, dtype=np.int64)
    wins = [0] * 8

    def body(i):
        def run():
            for r in range(500):
                # everyone tries to open round r+1 from r; exactly one wins
                while N.atomic_load(cell, 0) < r:
                    pass
                if N.atomic_cas(cell, 0, r, r + 1):
                    wins[i] += 1
        return run

    _run_threads([body(i) for i in range(8)])
    assert sum(wins) == 500 and N.atomic_load(cell, 0) == 500


def test_wait_ge_returns_and_aborts():
    cell = np.zeros(2, dtype=np.int64)
    seen = []

    def waiter():
        seen.append(N.atomic_wait_ge(cell, 0, 3))

    t = threading.Thread(target=waiter)
    t.start()
    for _ in range(3):
        N.atomic_fetch_add(cell, 0, 1)
    t.join(5)
    assert seen == [3]
    N.atomic_store(cell, 1, 1)
    assert N.atomic_wait_ge(cell, 0, 100, abort=cell, abort_i=1) is None


def test_counter_checks_buffer_type_and_range():
    with pytest.raises(ValueError):
        N.atomic_load(np.zeros(1, dtype=np.float64), 0)
    with pytest.raises(IndexError):
        N.atomic_load(np.zeros(1, dtype=np.int64), 1)


def test_updater_cfg_struct_layout_matches_header(tmp_path):
    """The ctypes mirrors of lpp_updater_cfg / lpp_updater_stats /
    lpp_averager_cfg have the C layout (offsets and sizes from the header,
    compiled with gcc)."""
    import ctypes

    structs = (("lpp_updater_cfg", N.UpdaterCfg), ("lpp_updater_stats", N.UpdaterStats),
               ("lpp_averager_cfg", N.AveragerCfg))
    src = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{ROOT / "include" / "lpp_b200.h"}"',
           'int main(void) {']
    want = []
    for cname, py in structs:
        src.append(f'printf(" %zu", sizeof({cname}));')
        want.append(ctypes.sizeof(py))
        for f, _ in py._fields_:
            src.append(f'printf(" %zu", offsetof({cname}, {f}));')
            want.append(getattr(py, f).offset)
    src += ['return 0; }']
    (tmp_path / "off.c").write_text("\n".join(src))
    subprocess.run(["gcc", "-I/usr/local/cuda/include", str(tmp_path / "off.c"), "-o",
                    str(tmp_path / "off")], check=True)
    got = [int(v) for v in subprocess.run([str(tmp_path / "off")], capture_output=True, text=True,
                                          check=True).stdout.split()]
    assert got == want


def test_native_lr_at_is_bit_identical_to_python():
    """lpp_lr_at (the native loop's lr) == schedules.lr_at bit for bit."""
    from paper_2203_06638_b200.schedules import LrSchedule, constant_schedule, lr_at

    scheds = [LrSchedule(kind="cosine", alpha0=0.1, total=997, warmup=97, batch_local=128,
                         workers=8, batch_base=128, boost=True),
              LrSchedule(kind="cosine", alpha0=0.05, total=60, warmup=0),
              LrSchedule(kind="multistep", alpha0=0.1, total=500, warmup=13, milestones=(100, 250, 400),
                         gamma=0.1, batch_local=32, workers=2, batch_base=32),
              constant_schedule(0.05, 50)]
    for sc in scheds:
        for s in list(range(0, sc.total + 5)) + [10**6]:
            assert N.lr_at_native(sc, s) == lr_at(sc, s), (sc, s)


def test_native_select_block_matches_python():
    from paper_2203_06638_b200.partition import select_block

    for t_st in (0, 1, 5, 100):
        for nb in (1, 2, 4):
            for rank in range(1, nb + 1):
                for s in range(0, 240):
                    assert N.select_block_native(s, t_st, nb, rank) == select_block(s, t_st, nb, rank).block_id
    with pytest.raises(ValueError):
        N.select_block_native(3, 0, 4, 5)
    with pytest.raises(ValueError):
        N.select_block_native(3, 0, 4, 0)


def test_device_sampler_host_twin():
    """The in-graph sampler's host twin: indices in [0, n), a deterministic
    function of (key, step), different per step and per key, ~uniform."""
    a = N.sample_indices_host(4096, 1000, 7, 0)
    assert a.min() >= 0 and a.max() < 1000
    assert np.array_equal(a, N.sample_indices_host(4096, 1000, 7, 0))
    assert not np.array_equal(a, N.sample_indices_host(4096, 1000, 7, 1))
    assert not np.array_equal(a, N.sample_indices_host(4096, 1000, 8, 0))
    counts = np.bincount(N.sample_indices_host(100_000, 10, 3, 5), minlength=10)
    assert counts.min() > 9_500 and counts.max() < 10_500


def test_device_sampler_matches_oracle_restatement():
    """oracle/devsample.py (the checker's independent restatement of the
    device sampler) equals the C ABI's host twin bit for bit."""
    from oracle import devsample

    for key, step, b, n in [(42, 0, 100, 5000), (7, 123, 64, 50_000), (2**63 + 5, 9, 33, 10),
                            (devsample.engine_key(0, 0, 0), 0, 128, 50_000),
                            (devsample.engine_key(3, 1, 2), 77, 32, 2048)]:
        assert np.array_equal(devsample.iid_batch(key, step, b, n), N.sample_indices_host(b, n, key, step))


def test_host_gather_rows_and_range_check():
    src = np.arange(40, dtype=np.float32).reshape(10, 4)
    dst = np.zeros((3, 4), dtype=np.float32)
    N.host_gather_rows(dst.ctypes.data, src.ctypes.data, 10, 16, np.array([7, 0, 7]))
    assert np.array_equal(dst, src[[7, 0, 7]])
    with pytest.raises(IndexError):
        N.host_gather_rows(dst.ctypes.data, src.ctypes.data, 10, 16, np.array([1, 10, 2]))
    with pytest.raises(IndexError):
        N.host_gather_rows(dst.ctypes.data, src.ctypes.data, 10, 16, np.array([-1]))


def test_device_epoch_sampler_host_twin_covers_each_epoch():
    """f4 on the device: every epoch of an updater's stream visits each
    element of its worker's shard arange(n)[q::Q] exactly once, epochs are
    reshuffled, batch boundaries may cut an epoch anywhere, and the stream
    is a function of (key, step) only."""
    for m, B, base, stride in ((1000, 64, 3, 8), (37, 5, 0, 1), (2, 3, 1, 2), (50_000, 128, 0, 1)):
        steps = (3 * m + B - 1) // B + 1
        a = np.concatenate([N.sample_epoch_host(B, base, stride, m, 77, t) for t in range(steps)])
        shard = list(range(base, base + stride * m, stride))
        orders = []
        for e in range(3):
            ep = a[e * m:(e + 1) * m]
            assert sorted(ep.tolist()) == shard, (m, e)
            orders.append(ep.tolist())
        if m > 2:
            assert orders[0] != orders[1] != orders[2]
    assert np.array_equal(N.sample_epoch_host(16, 0, 1, 100, 5, 9), N.sample_epoch_host(16, 0, 1, 100, 5, 9))
    assert not np.array_equal(N.sample_epoch_host(16, 0, 1, 100, 5, 9), N.sample_epoch_host(16, 0, 1, 100, 6, 9))


def test_native_loops_validate_before_touching_the_device():
    """The C++ loops reject incomplete configurations with status codes (no
    device work, no crash) — the error channel the engine turns into a
    failed run."""
    with pytest.raises(ValueError, match="null"):
        N.updater_run(N.UpdaterCfg())
    cells = np.zeros(4, dtype=np.int64)
    c = N.UpdaterCfg()
    c.sample_counter = c.update_order = c.stop = c.last_avg_stamp = cells.ctypes.data
    with pytest.raises(ValueError, match="block tables"):
        N.updater_run(c)
    with pytest.raises(ValueError, match="null"):
        N.averager_run(N.AveragerCfg())
    a = N.AveragerCfg()
    a.ctrl = a.sample_counter = a.update_order = a.exited = a.last_avg_stamp = a.synced_at = cells.ctypes.data
    a.arenas = a.mean_out = cells.ctypes.data
    a.workers, a.q = 9, 0
    with pytest.raises(ValueError, match="worker"):
        N.averager_run(a)


def test_native_numpy_stream_is_bit_identical_to_numpy():
    """csrc/nprng.cu restates numpy's default_rng(SeedSequence(entropy)):
    interleaved integers / choice(replace=False) / permutation calls give
    numpy's exact values (the reference's batches, sampled tag indices and
    epoch permutations, engine.py:293, 343-351, objectives.py:70-104)."""
    for ent in ([1, 0, 1], [0, 0, 0], [12345, 3, 2], [2**40 + 7, 1, 4], [7], [99, 1007]):
        g = np.random.default_rng(np.random.SeedSequence(ent))
        h = N.NpRng(*ent)
        for _ in range(3):
            for pop, k in ((272474, 16), (11220132, 16), (5000, 16), (30, 16), (20000, 500), (10001, 300)):
                assert np.array_equal(g.choice(pop, k, replace=False), h.choice(pop, k)), (ent, pop, k)
            for n in (50_000, 2048, 2**40, 2**32, 1):
                assert np.array_equal(g.integers(0, n, 64), h.integers(n, 64)), (ent, n)
            assert np.array_equal(g.permutation(1000), h.permutation(1000))
