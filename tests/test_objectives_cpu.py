"""Objective layouts and the partial-backprop cost model on CPU
(test_objectives.py:237-301 of the reference; SURVEY §2 shapes)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import data as odata
from paper_2203_06638_b200.objectives import MlpObjective, ResNetObjective, flops_savings_ratio
from paper_2203_06638_b200.partition import Block, balanced_boundaries, make_partition


def _mlp(hidden, f, k, seed):
    X, y = odata.make_blobs(16, f, k, 1.0, 0.5, seed)
    return MlpObjective(X, y, hidden, k)


def test_savings_ratio_uniform_layers():
    obj = _mlp((4, 4, 4), 4, 4, 1)               # 4 uniform layers
    for u, want in [(1, 0.0), (2, 0.25), (4, 0.375)]:
        part = make_partition(obj.dim, balanced_boundaries(obj.layer_param_counts, u))
        assert flops_savings_ratio(obj, part) == pytest.approx(want, rel=1e-12)


def test_savings_ratio_formula_matches_uniform_model():
    obj = _mlp((6,) * 5, 6, 6, 2)                # 6 uniform layers: (U-1)/(2U)
    for u in (2, 3, 6):
        part = make_partition(obj.dim, balanced_boundaries(obj.layer_param_counts, u))
        assert flops_savings_ratio(obj, part) == pytest.approx((u - 1) / (2 * u), rel=1e-12)


def test_backward_cost_declines_towards_the_output():
    obj = _mlp((6, 6, 6), 6, 6, 13)
    part = make_partition(obj.dim, balanced_boundaries(obj.layer_param_counts, 4))
    costs = [obj.backward_cost(b) for b in part.blocks()]
    assert costs == sorted(costs, reverse=True)
    assert costs[0] == obj.backward_cost(Block(0, obj.dim))


def test_mlp_layout_and_init_match_the_reference(golden_scalars):
    from conftest import load_npz

    g = load_npz("mlp.npz")
    X, y = odata.make_blobs(48, 4, 3, 2.0, 0.5, 9)
    obj = MlpObjective(X, y, (5,), 3)
    assert obj.layer_param_counts == (25, 18) and obj.dim == 43
    assert np.array_equal(obj.init_params(1), g["small_x0"])
    assert tuple(int(e) for e in g["small_edges"]) == obj.edges
    with pytest.raises(ValueError):
        obj.tensors_of_block(Block(1, 7))


@pytest.mark.parametrize("arch,dim,tensors", [("resnet20", 272_474, 65), ("resnet18", 11_220_132, 62),
                                              ("resnet50", 25_557_032, 161)])
def test_resnet_arena_sizes(arch, dim, tensors):
    """SURVEY §2 notes: d20 / d18 / d50 and their tensor counts."""
    obj = ResNetObjective(arch, n_samples=4)
    assert obj.dim == dim and len(obj.layer_param_counts) == tensors
    part = make_partition(obj.dim, balanced_boundaries(obj.layer_param_counts, 4))
    r = flops_savings_ratio(obj, part)
    assert 0.0 < r < 0.75          # at most (U-1)/U


def test_smallcnn_objective_matches_oracle_layout_data_and_init():
    """The product's config-0 CNN shares the oracle's flat layout, synthetic
    data stream and init (so GPU parity compares like with like)."""
    from oracle.cnn import LAYER_COUNTS, SmallCnnOracle, make_images
    from paper_2203_06638_b200.objectives import ResNetObjective

    obj = ResNetObjective("smallcnn", n_samples=64, seed=3, channels_last=False, autocast=None,
                          data="host")
    X, y = make_images(64, 3)
    assert obj.layer_param_counts == LAYER_COUNTS and obj.dim == 10218
    assert np.array_equal(obj.features.double().numpy(), X)
    assert np.array_equal(obj.labels.numpy(), y)
    assert np.array_equal(obj.init_params(5), SmallCnnOracle(X, y).init_params(5))


def test_small_cnn_learnable_images_match_the_oracle_data():
    """The config-0 band fixture's data (oracle.cnn.make_images with class
    patterns) is the product's host dataset bit for bit."""
    from oracle.cnn import make_images
    from paper_2203_06638_b200.objectives import ResNetObjective

    obj = ResNetObjective("smallcnn", n_samples=64, seed=3, channels_last=False, autocast=None,
                          data="host", pattern_scale=0.3)
    X, y = make_images(64, 3, pattern_scale=0.3)
    assert np.array_equal(obj.labels.numpy(), y)
    assert np.array_equal(obj.features.double().numpy(), X)
