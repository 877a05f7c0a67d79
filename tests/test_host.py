"""Host-side logic of the package (no GPU): parameter validation, schedules,
TopK semantics, layout round trips, scalar predicates, estimator params."""
import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2503_04422_b200 as P


def test_schedule_examples():
    assert [b - a for a, b in P.step_schedule(100, 2)] == [2, 4, 8, 16, 32, 38]
    assert [b - a for a, b in P.step_schedule(2, 2)] == [2]
    assert [b - a for a, b in P.step_schedule(3, 2)] == [2, 1]
    assert [b for _, b in P.step_schedule(128)] == [2, 6, 14, 30, 62, 126, 128]
    assert len(P.step_schedule(1536)) == 10


def test_params_validation():
    with pytest.raises(ValueError):
        P.SearchParams(k=0)
    with pytest.raises(ValueError):
        P.SearchParams(k=1, selection_fraction=0.0)
    with pytest.raises(ValueError):
        P.SearchParams(k=1, initial_step=0)
    with pytest.raises(ValueError):
        P.SearchParams(k=1, pruner="bsa?")
    with pytest.raises(ValueError):
        P.SearchParams(k=1, metric=P.Metric.IP, pruner="bond")
    with pytest.raises(ValueError):
        P.SearchParams(k=1, metric=P.Metric.IP, pruner="ads")
    with pytest.raises(ValueError):
        P.SearchParams(k=1, metric=P.Metric.L1, pruner="ads")
    with pytest.raises(ValueError):
        P.AdsPruner(d=4, epsilon0=0)


def test_topk_semantics():
    tk = P.TopK(2)
    assert tk.threshold() == float("inf")
    tk.push(3.0, 1)
    tk.push(1.0, 2)
    tk.push(2.0, 3)
    assert tk.threshold() == 2.0 and tk.items() == [(1.0, 2), (2.0, 3)]
    t1 = P.TopK(1)
    t1.push(1.0, 5)
    t1.push(1.0, 3)
    assert t1.ids() == [3]
    t2 = P.TopK.from_arrays(3, np.array([1, 2, 3], np.float32), np.array([7, 8, 9]), 2)
    assert t2.items() == [(1.0, 7), (2.0, 8)] and t2.threshold() == float("inf")


def test_ads_predicates():
    p = P.AdsPruner(d=128, epsilon0=2.1)
    assert P.ads_should_prune(50.0, 32, p, 100.0) is True
    assert P.ads_should_prune(40.0, 32, p, 100.0) is False
    assert P.ads_should_prune(99.0, 128, p, 100.0) is False
    assert P.ads_should_prune(100.0, 128, p, 100.0) is True
    with pytest.raises(ValueError):
        P.ads_should_prune(1.0, 0, P.AdsPruner(d=8), 1.0)
    assert P.bond_should_prune(10.0, 10.0) is True
    assert P.bond_should_prune(9.999, 10.0) is False
    assert P.default_zone_width(128) == 8 and P.default_zone_width(1536) == 96
    assert P.default_zone_width(4) == 4


@settings(max_examples=60, deadline=None)
@given(n=st.integers(1, 400), d=st.integers(1, 64), bs=st.sampled_from([1, 7, 64, 128]))
def test_layout_round_trip(n, d, bs):
    x = np.random.default_rng(n * 1000 + d).standard_normal((n, d)).astype(np.float32)
    c = P.VectorCollection.from_array(x)
    blocks = P.to_blocks(c, bs)
    assert [b.m for b in blocks][:-1] == [bs] * (len(blocks) - 1)
    back = P.from_blocks(blocks)
    np.testing.assert_array_equal(back.data, x)
    np.testing.assert_array_equal(back.ids, c.ids)
    assert all(b.m_padded == bs for b in blocks)


def test_layout_hand_example():
    c = P.VectorCollection.from_array(np.array([[1, 2, 3], [4, 5, 6]], np.float32))
    b = P.to_blocks(c, 4)[0]
    np.testing.assert_array_equal(b.data, [[1, 4, 0, 0], [2, 5, 0, 0], [3, 6, 0, 0]])
    assert [blk.m for blk in P.to_blocks(P.VectorCollection.from_array(np.zeros((130, 2))), 64)] == [64, 64, 2]
    with pytest.raises(ValueError):
        P.to_blocks(c, 0)


def test_estimator_params_and_unfitted():
    from sklearn.base import clone
    from sklearn.exceptions import NotFittedError
    est = P.IvfNearestNeighbors(pruner="ads", epsilon0=1.5, nprobe=4)
    params = est.get_params()
    assert params["epsilon0"] == 1.5 and params["nprobe"] == 4
    assert clone(est).get_params() == params
    with pytest.raises(NotFittedError):
        P.ExactNearestNeighbors().kneighbors(np.zeros((1, 3), np.float32))
    with pytest.raises(NotFittedError):
        P.IvfNearestNeighbors().kneighbors(np.zeros((1, 3), np.float32))


def test_horizontal_oracle_examples():
    assert P.horizontal_distance([1, 2], [1, 2], P.Metric.L2) == 0.0
    assert P.horizontal_distance([3, 4], [0, 0], P.Metric.L2) == 25.0
    assert P.horizontal_distance([1, 2], [2, 1], P.Metric.L1) == 2.0
    with pytest.raises(ValueError):
        P.horizontal_distance([1, 2], [1, 2, 3], P.Metric.L2)
