"""The bucket-major batched IVF pipeline (pdx_batch.cu) against the
per-query scan and the C oracle: ids, float32 distances, values_touched /
values_total and every survivor trace identical (no tolerance)."""
import numpy as np
import pytest

import recipes
from test_gpu_parity import P, _bsa_setup, _oracle_ivf  # noqa: F401 (P is a fixture)

pytestmark = pytest.mark.gpu


def _run(P, index, q, params, nprobe, batched):
    return P.ivf_search_batch(index, q, params, nprobe, trace=True, batched=batched)


def _same(a, b):
    np.testing.assert_array_equal(a["ids"], b["ids"])
    np.testing.assert_array_equal(a["dist"], b["dist"])
    np.testing.assert_array_equal(a["count"], b["count"])
    np.testing.assert_array_equal(a["touched"], b["touched"])
    np.testing.assert_array_equal(a["total"], b["total"])
    assert a["survivors"] == b["survivors"]


@pytest.fixture(scope="module")
def rotated(P):
    x = recipes.data("mixture", 200_000, 128, 7)
    Q = recipes.queries("near", x, 96, 8)
    T = P.generate_orthogonal(128, 0)
    xr, qr = P.apply_transform(T, x), P.apply_transform(T, Q)
    index = P.ivf_build(P.VectorCollection.from_array(xr), nlist=256, seed=0)
    return xr, qr, index


@pytest.mark.parametrize("eps,nprobe,k", [(2.1, 8, 10), (2.1, 32, 10), (0.7, 16, 10),
                                          (0.3, 16, 10), (2.1, 16, 1), (2.1, 16, 100)])
def test_batched_ads_equals_per_query_and_oracle(P, oracle, rotated, eps, nprobe, k):
    xr, qr, index = rotated
    params = P.SearchParams(k=k, pruner="ads", ads=P.AdsPruner(d=128, epsilon0=eps))
    a = _run(P, index, qr, params, nprobe, 2)
    b = _run(P, index, qr, params, nprobe, 1)
    _same(a, b)
    ref = oracle.ivf_search_batch(_oracle_ivf(oracle, index, xr), qr, k, nprobe, pruner="ads",
                                  eps0=eps, survivors_cap=1 << 18)
    np.testing.assert_array_equal(a["ids"], ref["ids"])
    np.testing.assert_array_equal(a["dist"], ref["dist"])
    np.testing.assert_array_equal(a["touched"], ref["touched"])
    assert a["survivors"] == ref["survivor_lists"]


@pytest.mark.parametrize("initial_step,sf", [(1, 0.2), (2, 0.05), (8, 0.4), (16, 0.2)])
def test_batched_schedules_bond(P, rotated, initial_step, sf):
    _, qr, index = rotated
    params = P.SearchParams(k=10, pruner="bond", initial_step=initial_step,
                            selection_fraction=sf)
    _same(_run(P, index, qr, params, 12, 2), _run(P, index, qr, params, 12, 1))


@pytest.mark.parametrize("quantile,multiplier", [(0.99, 1.0), (0.5, 0.7)])
def test_batched_bsa(P, oracle, quantile, multiplier):
    import torch
    x, Q, xr, qr = _bsa_setup(P)
    bsa = P.fit_bsa(torch.from_numpy(xr).cuda(), quantile=quantile, multiplier=multiplier)
    index = P.ivf_build(P.VectorCollection.from_array(xr), nlist=128, seed=0)
    params = P.SearchParams(k=10, pruner="bsa", bsa=bsa)
    a = _run(P, index, qr, params, 16, 2)
    _same(a, _run(P, index, qr, params, 16, 1))
    ref = oracle.ivf_search_batch(_oracle_ivf(oracle, index, xr), qr, 10, 16, pruner="bsa",
                                  bsa_coef=np.asarray(bsa.coef, np.float32),
                                  survivors_cap=1 << 18)
    np.testing.assert_array_equal(a["ids"], ref["ids"])
    np.testing.assert_array_equal(a["touched"], ref["touched"])
    assert a["survivors"] == ref["survivor_lists"]


def test_batched_small_buckets_and_tiny_batches(P):
    """Buckets smaller than k (phase-1 heap not full: fallback), a single
    query, ragged bucket sizes, d not a multiple of 8 and d <= 16."""
    for n, d, nlist, k, nq in [(3000, 37, 300, 20, 40), (5000, 12, 64, 10, 1),
                               (20000, 16, 128, 5, 33), (4000, 9, 50, 10, 64)]:
        rng = np.random.default_rng(n + d)
        x = (rng.standard_normal((n, d)) * (1 + rng.integers(0, 4, (n, 1)))).astype(np.float32)
        q = x[rng.choice(n, nq, replace=False)] + 0.1 * rng.standard_normal((nq, d)).astype(
            np.float32)
        index = P.ivf_build(P.VectorCollection.from_array(x), nlist=nlist, seed=0)
        for pruner in ("ads", "bond"):
            params = P.SearchParams(k=k, pruner=pruner)
            _same(_run(P, index, q, params, min(nlist, 24), 2),
                  _run(P, index, q, params, min(nlist, 24), 1))


def test_batched_duplicates_and_ties(P):
    """Exact duplicate vectors (distance ties, T^ = 0 chains) keep the lower id."""
    rng = np.random.default_rng(5)
    base = rng.standard_normal((500, 32)).astype(np.float32)
    x = np.concatenate([base] * 20)
    q = base[:40] + 0.0
    index = P.ivf_build(P.VectorCollection.from_array(x), nlist=40, seed=0)
    for pruner in ("ads", "bond"):
        params = P.SearchParams(k=10, pruner=pruner)
        _same(_run(P, index, q, params, 8, 2), _run(P, index, q, params, 8, 1))


def test_batched_bucket_shards_and_empty_buckets(P):
    """Queries whose nearest selected buckets are empty (a bucket shard of a
    multi-GPU index: the other ranks' buckets are empty here) — phase 1
    takes the first selected bucket that has blocks."""
    import torch
    from paper_2503_04422_b200.sharded import shard_index
    x = recipes.data("mixture", 60_000, 64, 11)
    q = recipes.queries("near", x, 64, 12)
    col = P.VectorCollection.from_array(x)
    index = P.ivf_build(col, nlist=128, seed=0)
    for rank in range(3):
        sh = shard_index(index, col, rank, 3)
        for pruner in ("ads", "bond"):
            params = P.SearchParams(k=10, pruner=pruner)
            _same(_run(P, sh, q, params, 24, 2), _run(P, sh, q, params, 24, 1))
    del torch


def test_warp_bucket_selection_vs_oracle(P, oracle):
    """K2's warp top-k path (nlist <= 1024, nprobe <= 32): the nprobe smallest
    (distance, bucket) pairs in stable-argsort order, ties included (zero
    queries under IP: every distance equal), a query count that is not a
    multiple of 8, nlist below and at 1024's lane layout."""
    from test_gpu_parity import _oracle_ivf
    x = recipes.data("mixture", 20_000, 48, 43)
    col = P.VectorCollection.from_array(x)
    index = P.ivf_build(col, nlist=500, seed=0)
    index2 = P.ivf_build(col, nlist=1000, seed=0)
    for ix in (index, index2):
        Q = np.concatenate([recipes.queries("near", x, 13, 44),
                            np.zeros((2, 48), np.float32)])
        view = _oracle_ivf(oracle, ix, x)
        for metric in ("l2", "ip", "l1"):
            for nprobe in (1, 7, 32):
                got = P.index.select_buckets_device(ix, P.store.to_device(Q), nprobe, metric)
                got = (got[0] if isinstance(got, tuple) else got).cpu().numpy()
                for i, q in enumerate(Q):
                    ref = oracle.select_buckets(view.cent, ix.nlist, q, metric, nprobe)
                    np.testing.assert_array_equal(got[i], ref)


def test_batched_stats_without_traces(P, rotated):
    """The bench's mode: values_touched / values_total with no survivor
    traces (the pipeline then keeps no per-step counts) equal the per-query
    scan's, for ADS and BOND at several nprobe."""
    _, qr, index = rotated
    for pruner, nprobe in (("ads", 32), ("ads", 8), ("bond", 16)):
        params = P.SearchParams(k=10, pruner=pruner)
        a = P.ivf_search_batch(index, qr, params, nprobe, stats=True, batched=2)
        b = P.ivf_search_batch(index, qr, params, nprobe, stats=True, batched=1)
        for key in ("ids", "dist", "count", "touched", "total"):
            np.testing.assert_array_equal(a[key], b[key])


@pytest.mark.parametrize("d", [300, 392])
def test_batched_dense_continuation_wide(P, oracle, d):
    """d > 256: the dense-continuation variant (every live query of a tile
    advances group by group together, then one lane per survivor) — results,
    decisions, values_touched and traces equal the per-query scan's and the
    oracle's, for ADS, BOND and BSA."""
    import torch
    x = recipes.data("mixture", 30_000, d, 51)
    q = recipes.queries("near", x, 40, 52)
    T = P.generate_orthogonal(d, 3)
    xr, qr = P.apply_transform(T, x), P.apply_transform(T, q)
    index = P.ivf_build(P.VectorCollection.from_array(xr), nlist=48, seed=0)
    for params in (P.SearchParams(k=10, pruner="ads"), P.SearchParams(k=10, pruner="bond"),
                   P.SearchParams(k=5, pruner="ads", ads=P.AdsPruner(d=d, epsilon0=0.8))):
        a = _run(P, index, qr, params, 12, 2)
        _same(a, _run(P, index, qr, params, 12, 1))
    ref = oracle.ivf_search_batch(_oracle_ivf(oracle, index, xr), qr, 10, 12, pruner="ads",
                                  survivors_cap=1 << 18)
    a = _run(P, index, qr, P.SearchParams(k=10, pruner="ads"), 12, 2)
    np.testing.assert_array_equal(a["ids"], ref["ids"])
    np.testing.assert_array_equal(a["touched"], ref["touched"])
    assert a["survivors"] == ref["survivor_lists"]
    bsa = P.fit_bsa(torch.from_numpy(xr).cuda())
    pb = P.SearchParams(k=10, pruner="bsa", bsa=bsa)
    _same(_run(P, index, qr, pb, 12, 2), _run(P, index, qr, pb, 12, 1))


def test_warp_bucket_selection_overflow(P):
    """Rows whose lane minima bound admits > 256 candidates (every 32nd
    bucket far away) take the warp kernel's round-by-round minimum: same
    stable-argsort selection as numpy on the per-op-rounded distances."""
    import torch
    from paper_2503_04422_b200 import _lib
    rng = np.random.default_rng(7)
    nlist, d = 1024, 16
    cent = rng.standard_normal((nlist, d)).astype(np.float32)
    cent[31::32] += 50.0
    cent[5] = cent[9]  # a tie: the lower bucket first
    Q = np.concatenate([np.zeros((3, d), np.float32),
                        rng.standard_normal((6, d)).astype(np.float32)])
    for metric, code in (("l2", 0), ("ip", 2)):
        for nprobe in (1, 17, 32):
            qd, cd = P.store.to_device(Q), P.store.to_device(cent)
            scratch = torch.empty((Q.shape[0] * nlist,), dtype=torch.float32, device="cuda")
            sel = torch.empty((Q.shape[0], nprobe), dtype=torch.int32, device="cuda")
            _lib.check(_lib.lib().pdx_select_buckets(_lib.ptr(qd), Q.shape[0], d, _lib.ptr(cd),
                                                     nlist, code, nprobe, _lib.ptr(scratch),
                                                     _lib.ptr(sel), _lib.stream_handle()))
            for i, q in enumerate(Q):
                acc = np.zeros(nlist, np.float32)
                for j in range(d):  # kernels.py:55-61 order and rounding
                    if metric == "l2":
                        t = (q[j] - cent[:, j]).astype(np.float32)
                        acc = (acc + (t * t).astype(np.float32)).astype(np.float32)
                    else:
                        acc = (acc + (q[j] * cent[:, j]).astype(np.float32)).astype(np.float32)
                key = -acc if metric == "ip" else acc
                ref = np.argsort(key, kind="stable")[:nprobe]
                np.testing.assert_array_equal(sel[i].cpu().numpy(), ref)


def test_batched_concurrent_threads(P, rotated):
    """Two host threads searching on their own streams (the C-ABI allows it;
    ctypes drops the GIL): each result equals the serial search's."""
    import threading

    import torch
    _, qr, index = rotated
    params = P.SearchParams(k=10, pruner="ads")
    serial = [P.ivf_search_batch(index, qr[i::2], params, 16, stats=True, batched=2)
              for i in range(2)]
    got = [None, None]

    def work(i):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            s = P.IvfSearcher(index, params, 16, batched=2)
            q = P.store.to_device(qr[i::2])
            for _ in range(3):
                r = s.run(q, stats=True)
            st.synchronize()
            got[i] = (r.ids.cpu().numpy(), r.dist.cpu().numpy(), r.touched.cpu().numpy())

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for i in range(2):
        np.testing.assert_array_equal(got[i][0], serial[i]["ids"])
        np.testing.assert_array_equal(got[i][1], serial[i]["dist"])
        np.testing.assert_array_equal(got[i][2], serial[i]["touched"])


def test_batched_limits_and_trace_overflow(P, rotated):
    """k = 256 (the batched path's limit), 33 queries, selection_fraction
    1.0 and a survivor-trace buffer too small for the visit list (trace_len
    = -1, the per-query scan's convention): identical to the per-query scan."""
    from paper_2503_04422_b200.search import run_search
    from paper_2503_04422_b200.index import select_buckets_device
    _, qr, index = rotated
    q = qr[:33]
    for params in (P.SearchParams(k=256, pruner="ads"),
                   P.SearchParams(k=10, pruner="bond", selection_fraction=1.0)):
        _same(_run(P, index, q, params, 16, 2), _run(P, index, q, params, 16, 1))
    Qd = P.store.to_device(q)
    sel = select_buckets_device(index, Qd, 16, "l2")
    sel = sel[0] if isinstance(sel, tuple) else sel
    params = P.SearchParams(k=10, pruner="ads")
    outs = []
    for batched in (2, 1):
        r = run_search(index.store, Qd, params, seg_bucket=sel.contiguous(), nseg=16,
                       trace_cap=100, batched=batched)
        outs.append((r.ids.cpu().numpy(), r.trace_len.cpu().numpy(),
                     r.touched.cpu().numpy()))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    np.testing.assert_array_equal(outs[0][2], outs[1][2])
    assert (outs[0][1] == -1).all()


@pytest.mark.parametrize("eps,nprobe,k", [(2.1, 32, 10), (0.7, 16, 10), (0.3, 16, 10),
                                          (2.1, 16, 1), (2.1, 16, 100)])
def test_batched_results_only_equals_full(P, oracle, rotated, eps, nprobe, k):
    """Without stats or traces the pipeline replaces the MODE 1 recompute by
    the survivor verification (bverify_kernel): ids and float32 distances
    identical to the full pipeline, the per-query scan and the oracle."""
    xr, qr, index = rotated
    params = P.SearchParams(k=k, pruner="ads", ads=P.AdsPruner(d=128, epsilon0=eps))
    fast = P.ivf_search_batch(index, qr, params, nprobe, batched=2)
    full = P.ivf_search_batch(index, qr, params, nprobe, stats=True, batched=2)
    scan = P.ivf_search_batch(index, qr, params, nprobe, batched=1)
    ref = oracle.ivf_search_batch(_oracle_ivf(oracle, index, xr), qr, k, nprobe, pruner="ads",
                                  eps0=eps)
    for got in (fast, scan):
        np.testing.assert_array_equal(got["ids"], full["ids"])
        np.testing.assert_array_equal(got["dist"], full["dist"])
    np.testing.assert_array_equal(fast["ids"], ref["ids"])
    np.testing.assert_array_equal(fast["dist"], ref["dist"])


def test_batched_results_only_bond_and_bsa(P, oracle):
    import torch
    x, Q, xr, qr = _bsa_setup(P)
    bsa = P.fit_bsa(torch.from_numpy(xr).cuda())
    index = P.ivf_build(P.VectorCollection.from_array(xr), nlist=128, seed=0)
    for params in (P.SearchParams(k=10, pruner="bsa", bsa=bsa),
                   P.SearchParams(k=10, pruner="bond", initial_step=2)):
        fast = P.ivf_search_batch(index, qr, params, 16, batched=2)
        full = P.ivf_search_batch(index, qr, params, 16, stats=True, batched=2)
        np.testing.assert_array_equal(fast["ids"], full["ids"])
        np.testing.assert_array_equal(fast["dist"], full["dist"])


def _results_only_vs_oracle(P, oracle, x, q, nlist, nprobe, params, from_rows=False, **okw):
    if from_rows:  # buckets around sampled rows (float64 assignment): no k-means on wild data
        rng = np.random.default_rng(nlist)
        ok = np.flatnonzero(np.abs(x).max(1) < 100.0)
        cent = x[rng.choice(ok, nlist, replace=False)]
        with np.errstate(over="ignore"):
            x64, c64 = x.astype(np.float64), cent.astype(np.float64)
            d2 = (x64 * x64).sum(1)[:, None] + (c64 * c64).sum(1)[None, :] - 2.0 * (x64 @ c64.T)
        index = P.IvfIndex.from_assignment(P.VectorCollection.from_array(x), cent,
                                           np.argmin(d2, axis=1), nlist=nlist)
    else:
        index = P.ivf_build(P.VectorCollection.from_array(x), nlist=nlist, seed=0)
    fast = P.ivf_search_batch(index, q, params, nprobe, batched=2)
    scan = P.ivf_search_batch(index, q, params, nprobe, batched=1)
    ref = oracle.ivf_search_batch(_oracle_ivf(oracle, index, x), q, params.k, nprobe, **okw)
    np.testing.assert_array_equal(fast["ids"], scan["ids"])
    np.testing.assert_array_equal(fast["dist"], scan["dist"])
    np.testing.assert_array_equal(fast["ids"], ref["ids"])
    np.testing.assert_array_equal(fast["dist"], ref["dist"])


@pytest.mark.parametrize("initial_step", [1, 2, 4, 8])
@pytest.mark.parametrize("pruner", ["ads", "bond"])
def test_filtered_head_schedules(P, oracle, pruner, initial_step):
    """bscan0_kernel (results-only MODE 0: the head as a certainty-margin
    filter, the candidates' exact chains from shared memory) for every
    compile-time head schedule, d not a multiple of 8 included."""
    for d, seed in [(128, 3), (44, 4), (27, 6), (20, 7), (16, 5)]:  # (d < the first deep step's end too)
        x = recipes.data("mixture", 40_000, d, seed)
        q = recipes.queries("near", x, 70, seed + 1)
        params = P.SearchParams(k=10, pruner=pruner, initial_step=initial_step)
        _results_only_vs_oracle(P, oracle, x, q, 64, 12, params, pruner=pruner,
                                initial_step=initial_step)


def test_filtered_head_offset_data_every_slot_a_candidate(P, oracle):
    """A large common offset: norms dwarf the distances, the filter's margin
    exceeds every partial and keeps (nearly) every slot — all decisions come
    from the exact chains, the warp queues overflow and drain mid-tile."""
    rng = np.random.default_rng(21)
    x = (rng.standard_normal((30_000, 64)) + 3000.0).astype(np.float32)
    q = (x[rng.choice(30_000, 48, replace=False)] +
         0.05 * rng.standard_normal((48, 64))).astype(np.float32)
    for pruner in ("ads", "bond"):
        _results_only_vs_oracle(P, oracle, x, q, 32, 8, P.SearchParams(k=10, pruner=pruner),
                                pruner=pruner)


def test_filtered_head_huge_and_nonfinite_norms(P, oracle):
    """Tiles and queries whose head norms are huge (>= 1e30, squares still
    finite) or overflow to +inf skip the filter; the exact chains reproduce
    the reference's float32 arithmetic (inf distances included)."""
    rng = np.random.default_rng(22)
    x = rng.standard_normal((20_000, 32)).astype(np.float32)
    x[::997, 3] = 2e15          # square 4e30: huge, finite
    x[5::1501, 1] = 3e19        # square overflows float32: +inf partials
    q = (x[rng.choice(20_000, 40, replace=False)] +
         0.1 * rng.standard_normal((40, 32))).astype(np.float32)
    q[7, 2] = 1.5e15            # a query with a huge head norm
    q[11] = x[997]              # a query equal to a huge vector
    with np.errstate(over="ignore", invalid="ignore"):
        for pruner in ("ads", "bond"):
            _results_only_vs_oracle(P, oracle, x, q, 40, 10, P.SearchParams(k=10, pruner=pruner),
                                    from_rows=True, pruner=pruner)


def test_phase1_chain_sequential_equals_overlapped(P, rotated):
    """Phase 1 with the chain kernel after the dense kernel (k > 32 takes it;
    so does PDX_P1_OVERLAP=0) and with the chain running underneath the
    dense pass (k <= 32, results only): both equal the per-query scan."""
    _, qr, index = rotated
    for k in (10, 32, 33):
        params = P.SearchParams(k=k, pruner="ads", ads=P.AdsPruner(d=128, epsilon0=2.1))
        fast = P.ivf_search_batch(index, qr, params, 16, batched=2)
        scan = P.ivf_search_batch(index, qr, params, 16, batched=1)
        np.testing.assert_array_equal(fast["ids"], scan["ids"])
        np.testing.assert_array_equal(fast["dist"], scan["dist"])


def test_large_batch_takes_the_sequential_phase1(P, rotated):
    """More than 8 queries per SM: the chain kernel runs after the dense one
    (all its CTAs at once) instead of underneath it."""
    _, qr, index = rotated
    rng = np.random.default_rng(3)
    q = np.concatenate([qr + 0.01 * rng.standard_normal(qr.shape).astype(np.float32)
                        for _ in range(14)])  # 1,344 queries
    params = P.SearchParams(k=10, pruner="ads", ads=P.AdsPruner(d=128, epsilon0=2.1))
    fast = P.ivf_search_batch(index, q, params, 16, batched=2)
    scan = P.ivf_search_batch(index, q, params, 16, batched=1)
    np.testing.assert_array_equal(fast["ids"], scan["ids"])
    np.testing.assert_array_equal(fast["dist"], scan["dist"])


def test_fuzz_batched_equals_per_query_scan(P):
    """A seeded sample of tools/fuzz_batched.py: random shapes, schedules,
    pruners, k, nprobe and data distributions (offsets, denormal-scale values,
    duplicates, integer grids) — the batched pipeline, results only and with
    statistics, equals the per-query scan."""
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, str(root / "tools" / "fuzz_batched.py"), "14", "7"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "14 / 14 identical" in r.stdout
