"""The arithmetic-order facts the device kernel relies on,
pinned against the numpy in this image: einsum's (x, z, y) order, the
pairwise-sum tree, the FMA chain of the prescribed-displacement matmul, and
numpy.maximum's zero-tie rule.  Both the oracle's and the product's
independent implementations of the tree are checked against np.sum."""

import numpy as np
import pytest

from oracle import frb_oracle as orc
from paper_2305_07030_b200 import plan as pplan
from paper_2305_07030_b200.network import segment_lengths


def test_einsum_order_is_x_z_y():
    rng = np.random.default_rng(0)
    d = rng.standard_normal((50000, 3)) * np.exp(rng.standard_normal((50000, 3)) * 3)
    e = np.sqrt(np.einsum("ij,ij->i", d, d))
    assert np.array_equal(e, segment_lengths(d))
    assert np.array_equal(e, orc.seg_len(d))


SIZES = list(range(0, 300)) + [450, 1000, 4097, 6591, 10125, 65535, 81000, 98304]


@pytest.mark.parametrize("n", SIZES)
def test_pairwise_tree_equals_np_sum(n):
    rng = np.random.default_rng(n)
    a = rng.standard_normal(n) * np.exp(rng.standard_normal(n) * 6)
    ref = float(np.sum(a))
    assert float(orc.PairwisePlan(n)(a)[0]) == ref
    assert pplan.evaluate(pplan.reduction_plan(n), a) == ref
    if n <= 300:
        assert orc.pairwise_scalar(a) == ref


def test_prescribed_displacement_fma_chain_matches_blas():
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 1, (400, 3))
    F = np.eye(3) + rng.uniform(-0.2, 0.2, (3, 3))
    assert np.array_equal(orc.prescribed_displacement(x, F), x @ (F - np.eye(3)).T)


def test_maximum_zero_tie_returns_positive_zero():
    out = np.maximum(np.full(64, -0.0), 0.0)
    assert not np.signbit(out).any()
    assert np.isnan(np.maximum(np.full(64, np.nan), 0.0)).all()
