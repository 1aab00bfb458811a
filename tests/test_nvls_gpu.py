"""NVLS averaging on the single-GPU pool: the multicast
object / VMM / multimem.ld_reduce / multimem.st path is exercised with a
one-device group (the in-switch sum of one copy is that copy), and the
engine's NVLS round is checked against the oracle in the serialized
schedule at Q = 1.  Multi-GPU reduction needs an NVSwitch box with >1 GPU."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def nv():
    from paper_2203_06638_b200 import nvls

    ok, why = nvls.probe(0)
    if not ok:
        pytest.skip(f"NVSwitch multicast unavailable on this box: {why}")
    return nvls


@pytest.mark.parametrize("d", [5, 4096, 1_000_003])
def test_single_device_multicast_mean_and_apply(nv, d):
    from paper_2203_06638_b200.arena import Arena

    g = nv.NvlsGroup(d, 1, 0)
    try:
        x = Arena(d, 0)
        x.tensor.copy_(torch.randn(d, device="cuda"))
        before = x.tensor.clone()
        s = torch.cuda.current_stream().cuda_stream
        g.stage_copy(x.ptr, s)
        g.reduce_mean(0, d, s)
        torch.cuda.synchronize()
        assert torch.equal(g.mean_tensor, before)          # sum of one copy / 1
        # updates that land between the stage and the apply survive
        x.tensor.add_(1.0)
        g.apply(x.ptr, None, 0, s)
        torch.cuda.synchronize()
        assert torch.equal(x.tensor, before + 1.0)
        x.close()
    finally:
        g.close()


def test_engine_nvls_refuses_cleanly_without_multicast():
    """Where the box cannot create multicast objects, asking for NVLS
    averaging fails loudly at construction (no silent fallback to P2P)."""
    import sys
    from pathlib import Path

    from paper_2203_06638_b200 import nvls

    if nvls.probe(0)[0]:
        pytest.skip("multicast available: covered by the functional tests")
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from test_engine_gpu import _mlp, _tiny
    from paper_2203_06638_b200.engine import run_experiment

    obj = _mlp("deep")[0]
    with pytest.raises(RuntimeError, match="NVSwitch multicast"):
        run_experiment(_tiny(obj, algo="lap_sgd", budget=10, workers=1, updaters=1, averaging="nvls"))


def test_engine_nvls_round_serialized_q1_matches_oracle(nv):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from test_engine_gpu import ATOL, RTOL, _mlp

    from oracle import schedule as osched
    from oracle.mlp import MlpOracle
    from paper_2203_06638_b200.engine import RunConfig, run_experiment
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import SyncScheme, constant_schedule

    obj, X, y, hidden, k = _mlp("deep")
    bounds = (0, obj.edges[2], obj.dim)
    cfg = RunConfig(algo="lpp_sgd", objective=obj, partition=make_partition(obj.dim, bounds),
                    lr=constant_schedule(0.05, 40), sync=SyncScheme(total=40, period=4),
                    budget=40, warm_start_budget=6, workers=1, updaters=2, batch_size=8, seed=1,
                    schedule="serialized", record_mode="full", averaging="nvls", evaluate=False)
    res = run_experiment(cfg)
    o = MlpOracle(X, y, hidden, k)

    class A:
        dim, n_samples = o.dim, o.n_samples
        init_params = staticmethod(o.init_params)
        grad_block = staticmethod(o.grad_block)

    tr = osched.run_serialized(A, algo="lpp_sgd", workers=1, updaters=2, boundaries=bounds,
                               lr=osched.Lr(kind="multistep", alpha0=0.05, total=40, peak=0.05),
                               switch_point=20, period=4, budget=40, warm_start=6, batch_size=8,
                               seed=1)
    np.testing.assert_allclose(res.final_values, tr.final_values, atol=ATOL, rtol=RTOL)
    assert [tuple(r) for r in res.round_trace] == [(a, b, *c) for a, b, c in tr.rounds]


def test_engine_nvls_async_q1_runs(nv):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from test_engine_gpu import _mlp, _tiny
    from paper_2203_06638_b200.engine import run_experiment

    obj = _mlp("deep")[0]
    res = run_experiment(_tiny(obj, algo="lap_sgd", budget=120, workers=1, updaters=3, averaging="nvls"))
    assert res.counter_finals == [123]
    assert len(res.stamps) >= 2 and np.all(np.isfinite(res.final_values))
