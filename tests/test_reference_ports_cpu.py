"""Ports of the reference's configuration-validation tests
(/root/reference/pkg/tests/test_engine.py:341-366) onto this package's
RunConfig: same rules, same messages — host logic, no GPU."""

from __future__ import annotations

import pytest


@pytest.fixture(scope="module")
def quad8():
    from oracle import flat
    from paper_2203_06638_b200.objectives import QuadraticObjective

    return QuadraticObjective(flat.make_linear_targets(32, 8, 1.0, 0.5, 3))


def tiny_config(obj, **kw):
    from paper_2203_06638_b200.engine import RunConfig
    from paper_2203_06638_b200.partition import make_partition
    from paper_2203_06638_b200.schedules import SyncScheme, constant_schedule

    budget = kw.pop("budget", 50)
    d = dict(algo="lap_sgd", objective=obj, partition=make_partition(obj.dim, (0, obj.dim)),
             lr=constant_schedule(0.05, max(budget, 1)),
             sync=SyncScheme(total=max(budget, 1), period=4, switch_point=0), budget=budget,
             warm_start_budget=0, workers=2, updaters=1, batch_size=8, seed=1)
    d.update(kw)
    return RunConfig(**d)


def test_sequential_baselines_reject_extra_updaters(quad8):
    with pytest.raises(ValueError, match="mb_sgd is sequential per worker"):
        tiny_config(quad8, algo="mb_sgd", updaters=4)
    with pytest.raises(ValueError, match="updaters=1"):
        tiny_config(quad8, algo="pl_sgd", updaters=2)


def test_round_budget_rejected_for_sequential_baselines(quad8):
    with pytest.raises(ValueError, match="asynchronous"):
        tiny_config(quad8, algo="mb_sgd", round_budget=10)
    with pytest.raises(ValueError, match="round_budget must be positive"):
        tiny_config(quad8, algo="lap_sgd", round_budget=0)


def test_block_alternation_needs_one_block_per_updater(quad8):
    with pytest.raises(ValueError, match="at least one block per updater"):
        tiny_config(quad8, algo="lpp_sgd", updaters=4)  # single-block partition


def test_unknown_algorithm_and_record_mode_are_rejected(quad8):
    with pytest.raises(ValueError, match="unknown algorithm"):
        tiny_config(quad8, algo="sgd")
    with pytest.raises(ValueError, match="unknown record mode"):
        tiny_config(quad8, record_mode="verbose")
    with pytest.raises(ValueError, match="budget must be positive"):
        tiny_config(quad8, budget=0)


def test_b200_options_are_validated(quad8):
    for field, bad in (("schedule", "eager"), ("apply_mode", "cas"), ("sampling", "gpu"),
                       ("averaging", "ring"), ("host_loop", "rust")):
        with pytest.raises(ValueError, match="unknown"):
            tiny_config(quad8, **{field: bad})
    with pytest.raises(ValueError, match="at most"):
        tiny_config(quad8, workers=10_000)
