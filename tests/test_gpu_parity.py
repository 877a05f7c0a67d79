"""GPU path (libpdx_b200.so through the package API) against the reference's
golden outputs and the C oracle: identical ids, bit-identical float32
distances, identical values_touched / values_total and survivor traces."""
import numpy as np
from pathlib import Path
import pytest

import recipes
from conftest import decode_survivors, host_means

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2503_04422_b200 as P
    from paper_2503_04422_b200 import _lib
    _lib.lib()
    return P


def _items(tk):
    it = tk.items()
    return [i for _, i in it], np.array([d for d, _ in it], np.float32)


def test_search_cases_match_reference(P, golden):
    arrays, manifest = golden
    for case in manifest["search"]:
        x = recipes.data(case["kind"], case["n"], case["d"], case["seed"])
        Q = recipes.queries("near", x, 3, case["seed"] + 1)
        col = P.VectorCollection.from_array(x)
        blocks = P.to_blocks(col, case["block_size"])
        mu = host_means(x)
        params = P.SearchParams(k=case["k"], metric=case["metric"], pruner=case["pruner"],
                                selection_fraction=case["sf"], initial_step=case["step"],
                                ads=P.AdsPruner(d=case["d"], epsilon0=case["eps"]))
        for qi, qc in enumerate(case["queries"]):
            orders = None
            if case["criteria"] != "sequential":
                orders = P.bond_dimension_order(Q[qi], mu, case["criteria"])
            st = P.SearchStats()
            tk = P.search(blocks, Q[qi], params, orders=orders, stats=st)
            ids, dist = _items(tk)
            key = qc["key"]
            assert ids == arrays[key + "_ids"].tolist(), key
            np.testing.assert_array_equal(dist, arrays[key + "_dist"], err_msg=key)
            assert st.values_touched == qc["touched"], key
            assert st.values_total == qc["total"], key
            assert st.survivors == decode_survivors(arrays[key + "_surv"]), key


@pytest.mark.parametrize("group", [1, 8])
def test_flat_cases_match_reference(P, golden, group):
    arrays, manifest = golden
    for case in manifest["flat"]:
        x = recipes.data(case["kind"], case["n"], case["d"], case["seed"])
        Q = recipes.queries("near", x, 3, case["seed"] + 1)
        flat = P.flat_build(P.VectorCollection.from_array(x), case["partition_size"], group=group)
        np.testing.assert_array_equal(flat.global_means, host_means(x))
        params = P.SearchParams(k=10, pruner=case["pruner"])
        out = P.exact_search_batch(flat, Q, params, criteria=case["criteria"], trace=True)
        for qi, qc in enumerate(case["queries"]):
            key = qc["key"]
            n = out["count"][qi]
            assert out["ids"][qi, :n].tolist() == arrays[key + "_ids"].tolist(), key
            np.testing.assert_array_equal(out["dist"][qi, :n], arrays[key + "_dist"])
            assert out["touched"][qi] == qc["touched"] and out["total"][qi] == qc["total"], key
            assert out["survivors"][qi] == decode_survivors(arrays[key + "_surv"]), key


@pytest.mark.parametrize("group", [1, 8])
def test_ivf_cases_match_reference(P, golden, group):
    arrays, manifest = golden
    for case in manifest["ivf"]:
        key0 = f"i{case['seed'] - 3000}"
        x = recipes.data(case["kind"], case["n"], case["d"], case["seed"])
        col = P.VectorCollection.from_array(x)
        index = P.IvfIndex.from_assignment(col, arrays[key0 + "_centroids"],
                                           arrays[key0 + "_assign"], nlist=case["nlist"],
                                           group=group)
        np.testing.assert_array_equal(index.means_dev.cpu().numpy(), arrays[key0 + "_means"])
        Q = recipes.queries("near", x, 4, case["seed"] + 1)
        for run in case["runs"]:
            params = P.SearchParams(k=10, pruner=run["pruner"],
                                    ads=P.AdsPruner(d=case["d"], epsilon0=run["eps"]))
            out = P.ivf_search_batch(index, Q[run["q"]:run["q"] + 1], params, run["nprobe"],
                                     criteria=run["criteria"], trace=True)
            key = run["key"]
            n = out["count"][0]
            assert out["selected"][0].tolist() == arrays[key + "_sel"].tolist(), key
            assert out["ids"][0, :n].tolist() == arrays[key + "_ids"].tolist(), key
            np.testing.assert_array_equal(out["dist"][0, :n], arrays[key + "_dist"])
            assert out["touched"][0] == run["touched"] and out["total"][0] == run["total"], key
            assert out["survivors"][0] == decode_survivors(arrays[key + "_surv"]), key


def test_orders_match_reference(P, golden):
    arrays, manifest = golden
    for o in manifest["orders"]:
        got = P.bond_dimension_order(arrays[o["key"] + "_q"], arrays[o["key"] + "_mu"],
                                     o["criteria"], o["zone_width"])
        np.testing.assert_array_equal(got, arrays[o["key"] + "_order"], err_msg=o["key"])


# ---------------------------------------------------------- vs the oracle
def _oracle_ivf(O, index, x):
    chains = index.buckets
    return O.IvfView(index.centroid_blocks, chains, index.means_dev.cpu().numpy())


@pytest.mark.parametrize("pruner,criteria", [("none", "sequential"), ("bond", "sequential"),
                                             ("bond", "dmeans"), ("bond", "zones")])
def test_config1_exact_vs_oracle(P, oracle, pruner, criteria):
    """BASELINE config 1 (100K x 128, sigma_j=(j+1)^-0.5, 64-blocks), 40 queries."""
    x = recipes.data("decay", 100_000, 128, 0)
    Q = recipes.data("decay", 40, 128, 1)
    col = P.VectorCollection.from_array(x)
    group = 1 if criteria != "sequential" else 8
    flat = P.flat_build(col, 64, group=group)
    params = P.SearchParams(k=10, pruner=pruner)
    out = P.exact_search_batch(flat, Q, params, criteria=criteria, trace=True)
    ref = oracle.exact_search_batch(P.to_blocks(col, 64), host_means(x), Q, 10, pruner=pruner,
                                    criteria=criteria, survivors_cap=1 << 18)
    np.testing.assert_array_equal(out["ids"], ref["ids"])
    np.testing.assert_array_equal(out["dist"], ref["dist"])
    np.testing.assert_array_equal(out["touched"], ref["touched"])
    np.testing.assert_array_equal(out["total"], ref["total"])
    assert out["survivors"] == ref["survivor_lists"]


@pytest.mark.parametrize("eps,nprobe", [(2.1, 8), (2.1, 32), (0.7, 16)])
def test_ivf_ads_vs_oracle(P, oracle, eps, nprobe):
    """IVF + ADS on rotated mixture data (config-2 recipe, 200K x 128): the
    threshold chain, every decision and the stats equal the oracle's."""
    import torch
    x = recipes.data("mixture", 200_000, 128, 7)
    Q = recipes.queries("near", x, 64, 8)
    T = P.generate_orthogonal(128, 0)
    xr = P.apply_transform(T, x)
    qr = P.apply_transform(T, Q)
    np.testing.assert_allclose(qr, Q @ T.matrix.T, rtol=1e-5, atol=1e-5)
    col = P.VectorCollection.from_array(xr)
    index = P.ivf_build(col, nlist=256, seed=0)
    params = P.SearchParams(k=10, pruner="ads", ads=P.AdsPruner(d=128, epsilon0=eps))
    out = P.ivf_search_batch(index, qr, params, nprobe, trace=True)
    view = _oracle_ivf(oracle, index, xr)
    ref = oracle.ivf_search_batch(view, qr, 10, nprobe, pruner="ads", eps0=eps,
                                  survivors_cap=1 << 18)
    np.testing.assert_array_equal(out["selected"], ref["selected"])
    np.testing.assert_array_equal(out["ids"], ref["ids"])
    np.testing.assert_array_equal(out["dist"], ref["dist"])
    np.testing.assert_array_equal(out["touched"], ref["touched"])
    assert out["survivors"] == ref["survivor_lists"]
    del torch


@pytest.mark.parametrize("metric,pruner,criteria,k", [("l2", "bond", "decreasing", 100),
                                                      ("l1", "bond", "dmeans", 10),
                                                      ("ip", "none", "sequential", 32),
                                                      ("l2", "none", "sequential", 1)])
def test_ivf_metrics_vs_oracle(P, oracle, metric, pruner, criteria, k):
    x = recipes.data("skewed", 30_000, 48, 11)
    Q = recipes.queries("near", x, 32, 12)
    col = P.VectorCollection.from_array(x)
    index = P.ivf_build(col, nlist=64, seed=3, block_size=64,
                        group=1 if criteria != "sequential" else 8)
    params = P.SearchParams(k=k, metric=metric, pruner=pruner)
    out = P.ivf_search_batch(index, Q, params, 12, criteria=criteria, trace=True)
    ref = oracle.ivf_search_batch(_oracle_ivf(oracle, index, x), Q, k, 12, metric=metric,
                                  pruner=pruner, criteria=criteria, survivors_cap=1 << 18)
    np.testing.assert_array_equal(out["ids"], ref["ids"])
    np.testing.assert_array_equal(out["dist"], ref["dist"])
    np.testing.assert_array_equal(out["touched"], ref["touched"])
    assert out["survivors"] == ref["survivor_lists"]


def test_wide_partitions_and_block_sizes_vs_oracle(P, oracle):
    """10,000-wide partitions (ExactNearestNeighbors' default), odd block sizes."""
    x = recipes.data("skewed", 23_456, 96, 21)
    Q = recipes.queries("near", x, 16, 22)
    col = P.VectorCollection.from_array(x)
    for psize, step, sf in [(10_000, 2, 0.2), (777, 1, 0.05), (130, 8, 0.4)]:
        flat = P.flat_build(col, psize, group=1)
        params = P.SearchParams(k=10, pruner="bond", initial_step=step, selection_fraction=sf)
        out = P.exact_search_batch(flat, Q, params, criteria="dmeans", trace=True)
        ref = oracle.exact_search_batch(P.to_blocks(col, psize, pad=False), host_means(x), Q, 10,
                                        pruner="bond", criteria="dmeans", initial_step=step,
                                        selection_fraction=sf, survivors_cap=1 << 18)
        np.testing.assert_array_equal(out["ids"], ref["ids"])
        np.testing.assert_array_equal(out["dist"], ref["dist"])
        np.testing.assert_array_equal(out["touched"], ref["touched"])
        assert out["survivors"] == ref["survivor_lists"]


# ------------------------------------------------------------ edge cases
def test_edge_cases(P, oracle):
    # empty list, single vector, k > n, d = 1
    assert len(P.search([], np.zeros(4, np.float32), P.SearchParams(k=5))) == 0
    x = np.array([[3.0]], np.float32)
    tk = P.search(P.to_blocks(P.VectorCollection.from_array(x), 64), np.array([1.0], np.float32),
                  P.SearchParams(k=4, pruner="bond"))
    assert tk.items() == [(4.0, 0)]
    x = recipes.data("normal", 70, 1, 3)
    blocks = P.to_blocks(P.VectorCollection.from_array(x), 64)
    q = np.array([0.1], np.float32)
    for k in (1, 69, 70, 200):
        got = P.search(blocks, q, P.SearchParams(k=k, pruner="bond")).items()
        ref, _ = oracle.search(blocks, q, k, pruner="bond")
        assert got == ref
    with pytest.raises(ValueError):
        P.search(blocks, np.zeros(2, np.float32), P.SearchParams(k=1))
    # identical vectors: ties resolve to the lower id
    dup = np.ones((300, 8), np.float32)
    tk = P.search(P.to_blocks(P.VectorCollection.from_array(dup), 64), np.zeros(8, np.float32),
                  P.SearchParams(k=10, pruner="bond"))
    assert tk.ids() == list(range(10))


def test_large_k_vs_oracle(P, oracle):
    x = recipes.data("normal", 20_000, 32, 31)
    Q = recipes.queries("near", x, 4, 32)
    blocks = P.to_blocks(P.VectorCollection.from_array(x), 64)
    for k in (1000, 4096):
        for q in Q:
            got = P.search(blocks, q, P.SearchParams(k=k, pruner="bond")).items()
            ref, _ = oracle.search(blocks, q, k, pruner="bond")
            assert got == ref


def test_select_buckets_vs_oracle(P, oracle):
    x = recipes.data("mixture", 50_000, 64, 41)
    col = P.VectorCollection.from_array(x)
    index = P.ivf_build(col, nlist=3000, seed=0)
    Q = recipes.queries("near", x, 16, 42)
    view = _oracle_ivf(oracle, index, x)
    for metric in ("l2", "ip", "l1"):
        for nprobe in (1, 100, 3000):
            got = P.index.select_buckets_device(index, P.store.to_device(Q), nprobe, metric)
            got = got.cpu().numpy()
            for i, q in enumerate(Q):
                ref = oracle.select_buckets(view.cent, index.nlist, q, metric, nprobe)
                np.testing.assert_array_equal(got[i], ref)


@pytest.mark.parametrize("nlist", [1024, 700, 40, 32, 20])
def test_select_buckets_warp_path_vs_oracle(P, oracle, nlist):
    """nlist <= 1024, nprobe <= 32: the one-warp-per-query selection (lane
    minima threshold, candidates ranked), incl. nprobe == nlist (nlist 32,
    20) and nlist < 32, where some lanes hold no keys."""
    x = recipes.data("mixture", 20_000, 32, 43)
    col = P.VectorCollection.from_array(x)
    index = P.ivf_build(col, nlist=nlist, seed=0)
    Q = np.concatenate([recipes.queries("near", x, 96, 44), recipes.queries("skewed", x, 32, 45)])
    view = _oracle_ivf(oracle, index, x)
    for metric in ("l2", "ip", "l1"):
        for nprobe in sorted(p for p in {1, 7, 32, min(32, nlist)} if p <= nlist):
            got = P.index.select_buckets_device(index, P.store.to_device(Q), nprobe, metric)
            got = got.cpu().numpy()
            for i, q in enumerate(Q):
                ref = oracle.select_buckets(view.cent, index.nlist, q, metric, nprobe)
                np.testing.assert_array_equal(got[i], ref)


def test_merge_topk_matches_host(P):
    import torch
    from paper_2503_04422_b200 import _lib
    rng = np.random.default_rng(0)
    parts, nq, k = 5, 33, 17
    dist = np.sort(rng.integers(0, 20, (parts, nq, k)).astype(np.float32), axis=2)
    ids = rng.permutation(parts * nq * k).reshape(parts, nq, k).astype(np.int64)
    ids[:, :, -3:] = -1
    dist[:, :, -3:] = np.inf
    D = torch.from_numpy(dist).cuda()
    I = torch.from_numpy(ids).cuda()
    od = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    oi = torch.empty((nq, k), dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().pdx_merge_topk(_lib.ptr(D), _lib.ptr(I), parts, nq, k, _lib.ptr(od),
                                         _lib.ptr(oi), _lib.stream_handle()))
    for q in range(nq):
        pairs = sorted((float(dist[p, q, j]), int(ids[p, q, j])) for p in range(parts)
                       for j in range(k) if ids[p, q, j] >= 0)[:k]
        assert oi[q].cpu().tolist()[:len(pairs)] == [i for _, i in pairs]


def test_ground_truth_and_estimators(P):
    x = recipes.data("clustered", 20_000, 32, 51)
    Q = recipes.queries("near", x, 20, 52)
    col = P.VectorCollection.from_array(x)
    gt = P.compute_ground_truth(col, Q, 10)
    for i, q in enumerate(Q):
        d = ((x.astype(np.float64) - q.astype(np.float64)) ** 2).sum(1)
        ref = np.argsort(d, kind="stable")[:10]
        assert sorted(gt.ids[i].tolist()) == sorted(ref.tolist())
    est = P.ExactNearestNeighbors(partition_size=2000).fit(x)
    dist, ids = est.kneighbors(Q, 10)
    assert dist.dtype == np.float64 and ids.dtype == np.int64
    for i in range(len(Q)):
        assert sorted(ids[i].tolist()) == sorted(gt.ids[i].tolist())
    assert np.all(np.diff(dist, axis=1) >= 0)
    ivf = P.IvfNearestNeighbors(pruner="bond", criteria="dmeans", nlist=30, nprobe=30).fit(x)
    _, ids = ivf.kneighbors(Q, 10)
    for i in range(len(Q)):
        assert sorted(ids[i].tolist()) == sorted(gt.ids[i].tolist())
    ads = P.IvfNearestNeighbors(pruner="ads", nlist=40, seed=7).fit(x)
    _, ids = ads.kneighbors(Q, 10, nprobe=40)
    rec = np.mean([P.recall_at_k(gt.ids[i], ids[i], 10) for i in range(len(Q))])
    assert rec >= 0.95
    # padding when k exceeds the probed vectors
    d2, i2 = P.ExactNearestNeighbors(partition_size=64).fit(x[:5]).kneighbors(Q[:2], 8)
    assert np.all(i2[:, 5:] == -1) and np.all(np.isinf(d2[:, 5:]))


def test_sharded_index_merge_exact(P):
    """Two bucket shards scanned separately on one GPU and merged by K7 equal
    the unsharded search for BOND (exact); ADS keeps its recall."""
    import torch
    from paper_2503_04422_b200.sharded import merge_device, shard_index
    x = recipes.data("mixture", 40_000, 32, 91)
    Q = recipes.queries("near", x, 24, 92)
    col = P.VectorCollection.from_array(x)
    index = P.ivf_build(col, nlist=64, seed=1)
    for pruner in ("bond", "none"):
        params = P.SearchParams(k=10, pruner=pruner)
        full = P.ivf_search_batch(index, Q, params, 16)
        dl, il = [], []
        for rank in range(2):
            sh = shard_index(index, col, rank, 2)
            r = P.ivf_search_batch(sh, Q, params, 16)
            dl.append(torch.from_numpy(r["dist"]))
            il.append(torch.from_numpy(r["ids"]))
        d, i = merge_device(torch.stack(dl).cuda(), torch.stack(il).cuda(), 10)
        np.testing.assert_array_equal(i.cpu().numpy(), full["ids"])
        np.testing.assert_array_equal(d.cpu().numpy(), full["dist"])


# ----------------------------------------------------------------- BSA
# BSA is this build's restatement (not in the reference):
# parity is GPU vs the C oracle restatement, not vs reference output.

def _bsa_setup(P, n=100_000, d=96, nq=48):
    x = recipes.data("mixture", n, d, 31)
    Q = recipes.queries("near", x, nq, 32)
    T = P.fit_pca(x, seed=0)
    m = T.matrix.astype(np.float64)
    np.testing.assert_allclose(m @ m.T, np.eye(d), atol=1e-5)
    xr = P.apply_transform(T, x)
    qr = P.apply_transform(T, Q)
    return x, Q, xr, qr


@pytest.mark.parametrize("quantile,multiplier", [(0.99, 1.0), (0.9, 1.0), (0.5, 0.7)])
def test_ivf_bsa_vs_oracle(P, oracle, quantile, multiplier):
    """Learned coefficients (aggressive ones included): results, every
    decision and the stats equal the oracle's BSA restatement."""
    import torch
    x, Q, xr, qr = _bsa_setup(P)
    bsa = P.fit_bsa(torch.from_numpy(xr).cuda(), quantile=quantile, multiplier=multiplier)
    assert bsa.coef[-1] == 0.0 and len(bsa.coef) == len(P.step_schedule(96, 2))
    index = P.ivf_build(P.VectorCollection.from_array(xr), nlist=128, seed=0)
    params = P.SearchParams(k=10, pruner="bsa", bsa=bsa)
    out = P.ivf_search_batch(index, qr, params, 16, trace=True)
    ref = oracle.ivf_search_batch(_oracle_ivf(oracle, index, xr), qr, 10, 16, pruner="bsa",
                                  bsa_coef=np.asarray(bsa.coef, np.float32),
                                  survivors_cap=1 << 18)
    np.testing.assert_array_equal(out["ids"], ref["ids"])
    np.testing.assert_array_equal(out["dist"], ref["dist"])
    np.testing.assert_array_equal(out["touched"], ref["touched"])
    assert out["survivors"] == ref["survivor_lists"]


@pytest.mark.parametrize("group", [1, 8])
def test_bsa_exact_bound_and_residuals(P, oracle, group):
    """coef = 2 is the Cauchy-Schwarz bound: BOND's results with fewer values
    touched; the store's residual energies equal the sequential host sums."""
    import torch
    x, Q, xr, qr = _bsa_setup(P, n=30_000, d=64, nq=32)
    nsteps = len(P.step_schedule(64, 2))
    bsa = P.BsaPruner(coef=(2.0,) * nsteps, d=64)
    col = P.VectorCollection.from_array(xr)
    index = P.ivf_build(col, nlist=64, seed=0, group=group)
    a = P.ivf_search_batch(index, qr, P.SearchParams(k=10, pruner="bsa", bsa=bsa), 8, trace=True)
    b = P.ivf_search_batch(index, qr, P.SearchParams(k=10, pruner="bond"), 8, trace=True)
    np.testing.assert_array_equal(a["ids"], b["ids"])
    np.testing.assert_array_equal(a["dist"], b["dist"])
    assert (a["touched"] <= b["touched"]).all() and a["touched"].sum() < b["touched"].sum()
    ref = oracle.ivf_search_batch(_oracle_ivf(oracle, index, xr), qr, 10, 8, pruner="bsa",
                                  bsa_coef=np.full(nsteps, 2.0, np.float32),
                                  survivors_cap=1 << 18)
    assert a["survivors"] == ref["survivor_lists"]
    st = index.store
    resid = st.ensure_bsa_residuals(2).cpu().numpy()
    ids = st.tile_ids.cpu().numpy().reshape(-1, 64)
    ends = [e for _, e in P.step_schedule(64, 2)]
    rng = np.random.default_rng(0)
    for t in rng.integers(0, st.ntiles, 6):
        for i in range(64):
            if ids[t, i] < 0:
                continue
            row = xr[ids[t, i]]
            for s, e in enumerate(ends):
                r = np.float32(0)
                for v in row[e:]:
                    r = np.float32(r + np.float32(v * v))
                assert resid[t, s, i] == r
    del torch


def test_bsa_estimator_recall(P):
    """BSA prunes harder than BOND yet keeps recall on clustered data."""
    x = recipes.data("mixture", 100_000, 128, 41)
    Q = recipes.queries("near", x, 200, 42)
    gt = P.compute_ground_truth(P.VectorCollection.from_array(x), Q, 10)
    stats = {}
    for pruner in ("bond", "bsa"):
        est = P.IvfNearestNeighbors(pruner=pruner, nlist=128, nprobe=128).fit(x)
        _, ids = est.kneighbors(Q, 10)
        out = P.ivf_search_batch(est.index_, P.apply_transform(est.transform_, Q)
                                 if est.transform_ is not None else Q,
                                 est.searcher(10).params, 128, stats=True)
        rec = float(np.mean([P.recall_at_k(gt.ids[i], ids[i], 10) for i in range(len(Q))]))
        stats[pruner] = (rec, int(out["touched"].sum()))
    assert stats["bond"][0] == 1.0
    assert stats["bsa"][0] >= 0.97, stats
    assert stats["bsa"][1] < stats["bond"][1], stats


# ------------------------------------------------------------ split mode
@pytest.mark.parametrize("metric,pruner,k,splits", [("l2", "bond", 10, 7), ("l2", "none", 100, 100),
                                                    ("ip", "none", 10, 300), ("l1", "bond", 5, 3)])
def test_split_mode_exact(P, metric, pruner, k, splits):
    """Split ranges + K7 merge (two levels when splits * k > 8192) return the
    exact top-k of the single-chain scan; values_total is unchanged and
    values_touched is the split run's own (>= BOND's single chain)."""
    x = recipes.data("skewed", 40_000, 40, 51)
    Q = recipes.queries("near", x, 12, 52)
    col = P.VectorCollection.from_array(x)
    flat = P.flat_build(col, 64, group=8)
    params = P.SearchParams(k=k, metric=metric, pruner=pruner)
    one = P.exact_search_batch(flat, Q, params, stats=True)
    many = P.exact_search_batch(flat, Q, params, stats=True, splits=splits)
    np.testing.assert_array_equal(many["ids"], one["ids"])
    np.testing.assert_array_equal(many["dist"], one["dist"])
    np.testing.assert_array_equal(many["count"], one["count"])
    np.testing.assert_array_equal(many["total"], one["total"])
    if pruner == "none":
        np.testing.assert_array_equal(many["touched"], one["touched"])
    else:
        assert (many["touched"] >= one["touched"]).all()
    with pytest.raises(ValueError, match="traces"):
        P.exact_search_batch(flat, Q[:1], params, trace=True, splits=4)


# ------------------------------------------------------- K8 tensor cores
@pytest.mark.parametrize("metric,k,normalize,n,d,nq", [
    ("ip", 100, True, 30_000, 96, 200), ("l2", 10, False, 30_000, 96, 200),
    ("l2", 100, True, 30_000, 96, 200), ("ip", 7, False, 30_000, 96, 200),
    ("l2", 10, False, 600_000, 40, 300), ("ip", 50, True, 300_000, 100, 129),
    ("l2", 100, False, 140_000, 37, 64)])
def test_tensor_core_exact_equals_scan(P, metric, k, normalize, n, d, nq):
    """tcgen05 candidate generation (dense first chunk, then the fused
    filter waves with tau tightening) + exact rescoring returns the scan's
    exact top-k bit for bit (ids, float32 keys, counts): across the first
    chunk (8,192 rows) and wave (32K doubling to 256K rows) edges, partial query tiles
    (nq not a multiple of 128), d not a multiple of 32 or of 4 (zero-padded
    TMA rows), partitions that are not multiples of 64."""
    import torch
    rng = np.random.default_rng(61 + n + d)
    c = rng.standard_normal((64, d)).astype(np.float32)
    x = c[rng.integers(0, 64, n)] + 0.5 * rng.standard_normal((n, d)).astype(np.float32)
    q = c[rng.integers(0, 64, nq)] + 0.5 * rng.standard_normal((nq, d)).astype(np.float32)
    if normalize:
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        q /= np.linalg.norm(q, axis=1, keepdims=True)
    col = P.VectorCollection.from_array(x)
    for psize, group in ((64, 8), (1000, 1)):
        flat = P.flat_build(col, psize, group=group)
        params = P.SearchParams(k=k, metric=metric)
        Qd = torch.from_numpy(q).cuda()
        ref = P.ExactSearcher(flat, params).run(Qd)
        for precision in ("tf32", "bf16", "auto"):
            tc = P.TensorCoreExactSearcher(flat, params, precision=precision)
            out = tc.run(Qd)
            if precision != "bf16":
                assert tc.overflow == 0
            np.testing.assert_array_equal(out.ids.cpu().numpy(), ref.ids.cpu().numpy())
            np.testing.assert_array_equal(out.dist.cpu().numpy(), ref.dist.cpu().numpy())
            np.testing.assert_array_equal(out.count.cpu().numpy(), ref.count.cpu().numpy())
        if n > 100_000:
            break  # the 1000-wide partitions repeat the same rows


def test_tensor_core_cta_pair_mode(P):
    """The cta_group::2 variant of the K8 kernel (PDX_K8_PAIR=1: a CTA pair
    per 256 x 256 tile, leader-issued MMAs, multicast commits) returns the
    scan's results too (run in a subprocess: the mode is read once)."""
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, sys\n"
        "sys.path.insert(0, '.')\n"
        "import paper_2503_04422_b200 as P\n"
        "rng = np.random.default_rng(3)\n"
        "x = rng.standard_normal((90000, 72)).astype(np.float32)\n"
        "q = torch.from_numpy(rng.standard_normal((300, 72)).astype(np.float32)).cuda()\n"
        "flat = P.flat_build(P.VectorCollection.from_array(x), 64)\n"
        "for m in ('l2', 'ip'):\n"
        "    prm = P.SearchParams(k=20, metric=m)\n"
        "    a = P.TensorCoreExactSearcher(flat, prm).run(q)\n"
        "    b = P.ExactSearcher(flat, prm).run(q)\n"
        "    assert torch.equal(a.ids, b.ids) and torch.equal(a.dist, b.dist), m\n"
        "print('ok')\n")
    import os
    env = dict(os.environ, PDX_K8_PAIR="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300, cwd=str(Path(__file__).resolve().parents[1]))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_tensor_core_dense_mode_scores(P):
    """Small collections (n = 3,000 < 8,192: the tcgen05 kernel's dense
    mode and pdx_k8_filter decide every candidate; n = 5,000: one fused
    wave), up to k = n."""
    import torch
    rng = np.random.default_rng(5)
    for n, d, nq, k in ((5000, 64, 130, 500), (3000, 37, 20, 3000)):
        x = rng.standard_normal((n, d)).astype(np.float32)
        q = rng.standard_normal((nq, d)).astype(np.float32)
        flat = P.flat_build(P.VectorCollection.from_array(x), 64)
        tc = P.TensorCoreExactSearcher(flat, P.SearchParams(k=k, metric="ip"),
                                       candidates=max(4096 if k < n else n, k))
        out = tc.run(torch.from_numpy(q).cuda())
        assert tc.overflow == 0
        ref = P.ExactSearcher(flat, P.SearchParams(k=k, metric="ip")).run(torch.from_numpy(q).cuda())
        np.testing.assert_array_equal(out.ids.cpu().numpy(), ref.ids.cpu().numpy())


def test_exact_estimator_tensor_core_auto(P):
    x = recipes.data("skewed", 20_000, 48, 71)
    Q = recipes.queries("near", x, 80, 72)
    a = P.ExactNearestNeighbors(pruner="none", criteria="sequential", tensor_cores=True).fit(x)
    b = P.ExactNearestNeighbors(pruner="none", criteria="sequential", tensor_cores=False).fit(x)
    da, ia = a.kneighbors(Q, 10)
    db, ib = b.kneighbors(Q, 10)
    np.testing.assert_array_equal(ia, ib)
    np.testing.assert_array_equal(da, db)


def _np_vertical(data, q, a, b, metric, acc, positions=None, order=None):
    """kernels.py:41-91 restated with numpy float32 ufuncs (each op rounded)."""
    dims = range(a, b) if order is None else order[a:b]
    sl = slice(None) if positions is None else np.unique(positions)
    for j in dims:
        col = data[j, sl]
        if metric == "l2":
            t = q[j] - col
            acc[sl] += t * t
        elif metric == "l1":
            acc[sl] += np.abs(q[j] - col)
        else:
            acc[sl] += q[j] * col
    return acc


@pytest.mark.parametrize("metric", ["l2", "l1", "ip"])
def test_vertical_accumulate_ops(P, metric):
    """The exported vertical kernels (pdx_vertical_accumulate) = numpy's
    per-op rounding, natural and permuted orders, selected slots with
    duplicates, and bit-exact range additivity (tests/test_kernels.py:54-65
    of the reference)."""
    rng = np.random.default_rng(5)
    x = rng.standard_normal((50, 37)).astype(np.float32) * 3
    blk = P.to_blocks(P.VectorCollection.from_array(x), 64)[0]
    q = rng.standard_normal(37).astype(np.float32)
    order = rng.permutation(37)
    for o in (None, order):
        acc = P.new_accumulator(64)
        P.vertical_accumulate(blk, q, (0, 37), metric, acc, order=o)
        ref = _np_vertical(blk.data, q, 0, 37, metric, P.new_accumulator(64), order=o)
        np.testing.assert_array_equal(acc, ref)
        split = P.new_accumulator(64)
        P.vertical_accumulate(blk, q, (0, 11), metric, split, order=o)
        P.vertical_accumulate(blk, q, (11, 37), metric, split, order=o)
        np.testing.assert_array_equal(split, acc)
        pos = np.array([3, 9, 9, 0, 49])
        sel = np.full(64, 0.5, np.float32)
        P.vertical_accumulate_selected(blk, q, (2, 30), metric, sel, pos, order=o)
        ref = _np_vertical(blk.data, q, 2, 30, metric, np.full(64, 0.5, np.float32), pos, o)
        np.testing.assert_array_equal(sel, ref)
    with pytest.raises(ValueError):
        P.vertical_accumulate(blk, q, (5, 38), metric, P.new_accumulator(64))
    with pytest.raises(ValueError):
        P.vertical_accumulate_selected(blk, q, (0, 3), metric, P.new_accumulator(64), [50])


@pytest.mark.parametrize("metric", ["l2", "ip"])
def test_select_buckets_tensor_cores_equal_k2(P, oracle, metric):
    """Bucket selection through K8 (tcgen05 candidates + the reference's
    exact centroid keys) = K2 = the oracle's stable argsort, incl. nprobe 1,
    d not a multiple of 4 and duplicated centroids (ties -> lower bucket)."""
    import torch
    rng = np.random.default_rng(8)
    for nlist, d, nq in ((5000, 100, 300), (9000, 37, 140)):
        cents = rng.standard_normal((nlist, d)).astype(np.float32)
        cents[7] = cents[3]
        x = np.repeat(cents, 2, 0) + 0.01 * rng.standard_normal((2 * nlist, d)).astype(np.float32)
        index = P.IvfIndex.from_assignment(P.VectorCollection.from_array(x), cents,
                                           np.repeat(np.arange(nlist), 2), nlist=nlist)
        Q = torch.from_numpy(cents[rng.integers(0, nlist, nq)] +
                             0.5 * rng.standard_normal((nq, d)).astype(np.float32)).cuda()
        for nprobe in (1, 64, 256):
            a = P.index.select_buckets_device(index, Q, nprobe, metric, tensor_cores=True)
            b = P.index.select_buckets_device(index, Q, nprobe, metric, tensor_cores=False)
            np.testing.assert_array_equal(a.cpu().numpy(), b.cpu().numpy())
        view = _oracle_ivf(oracle, index, x)
        qh = Q.cpu().numpy()
        for i in range(0, nq, 37):
            ref = oracle.select_buckets(view.cent, nlist, qh[i], metric, 256)
            np.testing.assert_array_equal(a[i].cpu().numpy(), ref)


@pytest.mark.parametrize("metric,k,d,psize,splits", [("l1", 7, 37, 1000, 50), ("l2", 300, 24, 64, 37),
                                                     ("ip", 1, 130, 333, 148)])
def test_split_mode_streaming_exact(P, metric, k, d, psize, splits):
    """Unpruned split scans take the streaming kernel (pdx_linear.cu): the
    exact top-k of the single-chain scan with the same stats, incl. d not a
    multiple of 8, wide partitions whose last tile is partly padding, k up to
    300 and more splits than blocks in some ranges."""
    x = recipes.data("normal", 30_000, d, 53)
    Q = recipes.queries("near", x, 9, 54)
    flat = P.flat_build(P.VectorCollection.from_array(x), psize, group=8)
    params = P.SearchParams(k=k, metric=metric, pruner="none")
    one = P.exact_search_batch(flat, Q, params, stats=True)
    many = P.exact_search_batch(flat, Q, params, stats=True, splits=splits)
    for key in ("ids", "dist", "count", "touched", "total"):
        np.testing.assert_array_equal(many[key], one[key])
