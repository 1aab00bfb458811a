"""The CPU baseline arm (oracle/engine_port.py) runs the reference's thread
structure end to end: claim-then-process accounting, aligned averaging
rounds, write-tag classification (CPU only; small sizes)."""

from __future__ import annotations

from oracle.engine_port import run_lpp_cpu


def test_cpu_port_runs_q1_and_q2():
    r1 = run_lpp_cpu(slots=4, updaters=2, batch_size=16, n_samples=256, threads=2)
    assert r1["minibatches"] == 4 + 2 and r1["finite"] and r1["rounds"] >= 1
    assert 0.0 <= r1["p_hat"] <= 1.0
    r2 = run_lpp_cpu(slots=4, updaters=2, batch_size=16, n_samples=256, threads=2, workers=2)
    assert r2["minibatches"] == 2 * (4 + 2) and r2["finite"] and r2["rounds"] >= 1
