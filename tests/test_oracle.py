"""The C oracle against the reference's own outputs (tests/golden, produced
by running the reference) and the reference tests' known answers.  CPU only."""
import numpy as np
import pytest

import recipes
from conftest import GOLDEN, decode_survivors, host_means
from paper_2503_04422_b200.layout import VectorCollection, to_blocks


def _ivf_view(O, arrays, case):
    key = f"i{manifest_index(case)}"
    x = recipes.data(case["kind"], case["n"], case["d"], case["seed"])
    assign = arrays[key + "_assign"]
    cents = arrays[key + "_centroids"]
    chains = []
    for c in range(case["nlist"]):
        mem = np.flatnonzero(assign == c)
        part = VectorCollection(data=x[mem], ids=mem.astype(np.int64))
        chains.append(to_blocks(part, 64) if part.n else [])
    view = O.IvfView(to_blocks(VectorCollection.from_array(cents), 64), chains,
                     arrays[key + "_means"])
    return x, view


def manifest_index(case):
    return case["seed"] - 3000


def test_known_answers(oracle):
    O = oracle
    assert [b - a for a, b in O.step_schedule(100, 2)] == [2, 4, 8, 16, 32, 38]
    assert [b - a for a, b in O.step_schedule(2, 2)] == [2]
    assert [b - a for a, b in O.step_schedule(3, 2)] == [2, 1]
    # ADS formula example: bound = 100*(32/128)*(1+2.1/sqrt(32))^2 ~ 47.0
    b = O.ads_bound(32, 128, 2.1, 100.0)
    assert 46.9 < b < 47.1 and not (40.0 >= b) and (50.0 >= b)
    assert O.ads_bound(128, 128, 2.1, 100.0) == 100.0
    # vertical kernel examples (L2 [0,5], IP [5,0], L1 2)
    blk = np.zeros((2, 64), np.float32)
    blk[:, 0] = [1, 2]
    for metric, want in (("l2", [0.0, 5.0]), ("ip", [5.0, 0.0])):
        acc = np.zeros(64, np.float32)
        O.vertical_accumulate(blk, [1, 2], (0, 2), metric, acc)
        assert acc[0] == want[0] and acc[1] == want[1]
    b1 = np.zeros((2, 64), np.float32)
    b1[:, 0] = [0, 3]
    acc = np.zeros(64, np.float32)
    O.vertical_accumulate(b1, [1, 2], (0, 2), "l1", acc)
    assert acc[0] == 2.0
    # orders examples
    np.testing.assert_array_equal(O.dimension_order([0.5, 1.0, 0.9], [0.5, 0.0, 1.0], "dmeans"), [1, 2, 0])
    np.testing.assert_array_equal(O.dimension_order([3, 1, 2], [0, 0, 0], "decreasing"), [0, 2, 1])
    np.testing.assert_array_equal(O.dimension_order([0, 0, 5, 0], [0, 0, 0, 0], "zones", 2), [2, 3, 0, 1])
    np.testing.assert_array_equal(O.dimension_order([1.0, 1.0, 1.0], [0, 0, 0], "decreasing"), [0, 1, 2])


def test_topk_tie_and_threshold(oracle):
    # two identical vectors: the lower id wins the single slot
    blocks = to_blocks(VectorCollection(data=np.ones((2, 4), np.float32),
                                        ids=np.array([5, 3], np.int64)), 64)
    items, _ = oracle.search(blocks, np.zeros(4, np.float32), 1)
    assert items == [(4.0, 3)]


def test_range_additivity_bit_exact(oracle):
    rng = np.random.default_rng(5)
    rows = rng.standard_normal((40, 100)).astype(np.float32)
    q = rng.standard_normal(100).astype(np.float32)
    blk = to_blocks(VectorCollection.from_array(rows), 64)[0].data
    for metric in ("l2", "l1", "ip"):
        whole = oracle.vertical_accumulate(blk, q, (0, 100), metric, np.zeros(64, np.float32))
        split = np.zeros(64, np.float32)
        for a, c in zip([0, 13, 37, 64], [13, 37, 64, 100]):
            oracle.vertical_accumulate(blk, q, (a, c), metric, split)
        np.testing.assert_array_equal(whole, split)


def test_numpy_sum_association(oracle):
    rng = np.random.default_rng(0)
    for _ in range(3000):
        n = int(rng.integers(0, 700))
        a = np.abs(rng.standard_normal(n) * np.exp(rng.standard_normal(n) * 3))
        assert oracle.numpy_sum(a) == a.sum()


def test_search_cases_match_reference(oracle, golden):
    arrays, manifest = golden
    for case in manifest["search"]:
        x = recipes.data(case["kind"], case["n"], case["d"], case["seed"])
        Q = recipes.queries("near", x, 3, case["seed"] + 1)
        blocks = to_blocks(VectorCollection.from_array(x), case["block_size"])
        mu = host_means(x)
        for qi, qc in enumerate(case["queries"]):
            orders = None
            if case["criteria"] != "sequential":
                orders = oracle.dimension_order(Q[qi], mu, case["criteria"])
            items, st = oracle.search(blocks, Q[qi], case["k"], case["metric"], case["pruner"],
                                      case["sf"], case["step"], case["d"], case["eps"],
                                      orders=orders)
            key = qc["key"]
            assert [i for _, i in items] == arrays[key + "_ids"].tolist(), key
            np.testing.assert_array_equal(np.array([d for d, _ in items], np.float32),
                                          arrays[key + "_dist"], err_msg=key)
            assert st["values_touched"] == qc["touched"], key
            assert st["values_total"] == qc["total"], key
            assert st["survivors"] == decode_survivors(arrays[key + "_surv"]), key


def test_flat_cases_match_reference(oracle, golden):
    arrays, manifest = golden
    for case in manifest["flat"]:
        x = recipes.data(case["kind"], case["n"], case["d"], case["seed"])
        Q = recipes.queries("near", x, 3, case["seed"] + 1)
        blocks = to_blocks(VectorCollection.from_array(x), case["partition_size"], pad=False)
        out = oracle.exact_search_batch(blocks, host_means(x), Q, 10, pruner=case["pruner"],
                                        criteria=case["criteria"], survivors_cap=1 << 16)
        for qi, qc in enumerate(case["queries"]):
            key = qc["key"]
            n = out["count"][qi]
            assert out["ids"][qi, :n].tolist() == arrays[key + "_ids"].tolist(), key
            np.testing.assert_array_equal(out["dist"][qi, :n], arrays[key + "_dist"])
            assert out["touched"][qi] == qc["touched"] and out["total"][qi] == qc["total"]
            assert out["survivor_lists"][qi] == decode_survivors(arrays[key + "_surv"])


def test_ivf_cases_match_reference(oracle, golden):
    arrays, manifest = golden
    for case in manifest["ivf"]:
        x, view = _ivf_view(oracle, arrays, case)
        # bucket means: compute_means of each bucket, float64, sequential rows
        assign = arrays[f"i{manifest_index(case)}_assign"]
        for c in range(case["nlist"]):
            mem = np.flatnonzero(assign == c)
            if mem.size:
                np.testing.assert_array_equal(host_means(x[mem]),
                                              arrays[f"i{manifest_index(case)}_means"][c])
        Q = recipes.queries("near", x, 4, case["seed"] + 1)
        for run in case["runs"]:
            out = oracle.ivf_search_batch(view, Q[run["q"]:run["q"] + 1], 10, run["nprobe"],
                                          pruner=run["pruner"], criteria=run["criteria"],
                                          eps0=run["eps"], survivors_cap=1 << 16)
            key = run["key"]
            n = out["count"][0]
            assert out["selected"][0].tolist() == arrays[key + "_sel"].tolist(), key
            assert out["ids"][0, :n].tolist() == arrays[key + "_ids"].tolist(), key
            np.testing.assert_array_equal(out["dist"][0, :n], arrays[key + "_dist"])
            assert out["touched"][0] == run["touched"] and out["total"][0] == run["total"], key
            assert out["survivor_lists"][0] == decode_survivors(arrays[key + "_surv"]), key


def test_orders_match_reference(oracle, golden):
    arrays, manifest = golden
    for o in manifest["orders"]:
        got = oracle.dimension_order(arrays[o["key"] + "_q"], arrays[o["key"] + "_mu"],
                                     o["criteria"], o["zone_width"])
        np.testing.assert_array_equal(got, arrays[o["key"] + "_order"], err_msg=o["key"])


def test_ads_bounds_match_reference(oracle, golden):
    arrays, _ = golden
    for D, ds_, eps, T, b, b32 in arrays["ads_bounds"]:
        got = oracle.ads_bound(int(ds_), int(D), float(eps), float(T))
        assert got == b
        assert float(np.float32(got)) == b32


@pytest.mark.parametrize("d,seed", [(16, 3), (64, 7), (128, 0)])
def test_orthogonal_matches_reference(golden, d, seed):
    from paper_2503_04422_b200.pruning import generate_orthogonal
    arrays, _ = golden
    np.testing.assert_array_equal(generate_orthogonal(d, seed).matrix, arrays[f"orth_{d}_{seed}"])


def test_oracle_bsa_matches_host_restatement(oracle):
    """BSA (this build's restatement): the C oracle's per-step
    survivors equal a direct host evaluation of the estimate; coef = 2 (the
    Cauchy-Schwarz bound) keeps BOND's results."""
    from paper_2503_04422_b200.pruning import bsa_estimate
    from paper_2503_04422_b200.search import step_schedule
    rng = np.random.default_rng(5)
    d = 16
    x = (rng.standard_normal((600, d)) * np.linspace(3, 0.2, d)).astype(np.float32)
    q = (x[7] + 0.1 * rng.standard_normal(d)).astype(np.float32)
    blocks = to_blocks(VectorCollection.from_array(x), 64, pad=False)
    sched = step_schedule(d, 2)
    coef = np.array([1.6, 1.2, 0.8, 0.0][:len(sched)], np.float32)
    items, st = oracle.search(blocks, q, 5, pruner="bsa", bsa_coef=coef)
    # host replay of the same block-synchronous pass
    import heapq
    heap, trace = [], []
    for bi, blk in enumerate(blocks):
        m = blk.ids.shape[0]
        acc = np.zeros(m, np.float32)
        T = np.inf if len(heap) < 5 else -heap[0][0]
        pos = list(range(m))
        linear = bi == 0 or T == np.inf
        rec = []
        for s, (a, b) in enumerate(sched):
            for j in range(a, b):
                t = (q[j] - blk.data[j, :m]).astype(np.float32)
                acc = (acc + (t * t).astype(np.float32)).astype(np.float32)
            if not linear:
                pos = [i for i in pos if bsa_estimate(acc[i], blk.data[:, i], q, b, coef[s]) < T]
                rec.append(len(pos))
        trace.append([m] if linear else rec)
        for i in (range(m) if linear else pos):
            key = (-float(acc[i]), -int(blk.ids[i]))
            if len(heap) < 5:
                heapq.heappush(heap, key)
            elif key > heap[0]:
                heapq.heapreplace(heap, key)
    want = sorted((-a, -b) for a, b in heap)
    assert [(np.float32(dv), i) for dv, i in items] == [(np.float32(dv), i) for dv, i in want]
    n = len(sched)
    a, sa = oracle.search(blocks, q, 5, pruner="bsa", bsa_coef=np.full(n, 2.0, np.float32))
    b, sb = oracle.search(blocks, q, 5, pruner="bond")
    assert a == b and sa["values_touched"] <= sb["values_touched"]
    with pytest.raises(ValueError):
        oracle.search(blocks, q, 5, pruner="bsa")


def test_oracle_c2_headline_prefix_equals_reference():
    """The bench's headline config (C2, BASELINE configs[1]) on the
    reference-k-means index: the C oracle equals the real reference's
    ivf_search (tests/golden/c2_reference_prefix.npz) bit for bit on the
    query prefix at nprobe 8 / 32 / 128 — the oracle is pinned at full size,
    not only on the small golden cases."""
    import bench
    from oracle import oracle as O
    g = np.load(GOLDEN / "c2_reference_prefix.npz")
    X, _ = bench.make_data(1_000_000, 1000)
    T = bench.rotation(128)
    XR = X @ T.T
    cent, assign, same = bench.load_fixture(XR)
    if not same:
        pytest.skip("this host's BLAS rotated the data differently from the fixture's")
    view = O.IvfView.from_assignment(XR, cent, assign, 1024)
    for npb in (8, 32, 128):
        ref = O.ivf_search_batch(view, g["queries"], 10, npb, pruner="ads", eps0=2.1)
        np.testing.assert_array_equal(ref["ids"], g[f"ids_{npb}"])
        np.testing.assert_array_equal(ref["dist"], g[f"dist_{npb}"])
        np.testing.assert_array_equal(ref["touched"], g[f"touched_{npb}"])
        np.testing.assert_array_equal(ref["total"], g[f"total_{npb}"])


def test_packed_ivf_view_equals_block_list_view():
    """oracle.IvfView.from_assignment (numpy packing, used by the bench's
    reference arm) = the view built from per-bucket to_blocks chains."""
    from oracle import oracle as O
    rng = np.random.default_rng(1)
    n, d, nl = 5000, 24, 37
    x = rng.standard_normal((n, d)).astype(np.float32)
    c = rng.standard_normal((nl, d)).astype(np.float32)
    a = rng.integers(0, nl - 3, n)  # the last buckets stay empty
    chains, means = [], []
    for b in range(nl):
        mem = np.flatnonzero(a == b)
        chains.append(to_blocks(VectorCollection(data=x[mem], ids=mem.astype(np.int64)), 64)
                      if len(mem) else [])
        means.append(x[mem].astype(np.float64).sum(0) / len(mem) if len(mem)
                     else c[b].astype(np.float64))
    v1 = O.IvfView(to_blocks(VectorCollection.from_array(c), 64), chains, means)
    v2 = O.IvfView.from_assignment(x, c, a, nl)
    np.testing.assert_array_equal(v1.means, v2.means)
    q = rng.standard_normal((50, d)).astype(np.float32)
    for pr, cr in (("ads", "sequential"), ("bond", "dmeans"), ("none", "sequential")):
        r1 = O.ivf_search_batch(v1, q, 10, 8, pruner=pr, criteria=cr, survivors_cap=1 << 14)
        r2 = O.ivf_search_batch(v2, q, 10, 8, pruner=pr, criteria=cr, survivors_cap=1 << 14)
        for key in ("ids", "dist", "touched", "total", "selected"):
            np.testing.assert_array_equal(r1[key], r2[key])
        assert r1["survivor_lists"] == r2["survivor_lists"]
