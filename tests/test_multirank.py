"""Bucket-sharded search across ranks, world size 2 on gloo.

Each rank owns the buckets plan_shards gives it, scans them (the C oracle
stands in for the GPU scan on this CPU-only box), and the per-rank top-k
lists go through the package's gather_merge exchange.  The merged result
must equal the single-process search exactly for the exact pruners (BOND /
none), as the design claims.  CPU only."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import recipes
from paper_2503_04422_b200.layout import VectorCollection, to_blocks
from paper_2503_04422_b200.sharded import gather_merge, owned_rows, plan_shards


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    x = recipes.data("mixture", 6000, 24, 77)
    q = recipes.queries("near", x, 12, 78)
    rng = np.random.default_rng(5)
    cents = x[rng.choice(x.shape[0], 40, replace=False)]
    assign = np.argmin(((x[:, None, :] - cents[None]) ** 2).sum(-1), axis=1)
    return x, q, cents.astype(np.float32), assign


def _view(O, x, cents, assign, rows_allowed):
    chains = []
    for c in range(cents.shape[0]):
        mem = np.flatnonzero((assign == c) & rows_allowed)
        part = VectorCollection(data=x[mem], ids=mem.astype(np.int64))
        chains.append(to_blocks(part, 64) if part.n else [])
    means = np.stack([x[assign == c].astype(np.float64).mean(0) if np.any(assign == c)
                      else cents[c].astype(np.float64) for c in range(cents.shape[0])])
    return O.IvfView(to_blocks(VectorCollection.from_array(cents), 64), chains, means)


def merge_host(dist_all, ids_all, k):
    """Reference semantics of K7 (TopK's (distance, id) order) in numpy."""
    d = dist_all.numpy()
    i = ids_all.numpy()
    out_d = np.full((d.shape[1], k), np.inf, np.float32)
    out_i = np.full((d.shape[1], k), -1, np.int64)
    for qq in range(d.shape[1]):
        pairs = sorted((float(d[r, qq, j]), int(i[r, qq, j])) for r in range(d.shape[0])
                       for j in range(k) if i[r, qq, j] >= 0)[:k]
        for j, (dv, iv) in enumerate(pairs):
            out_d[qq, j], out_i[qq, j] = dv, iv
    return torch.from_numpy(out_d), torch.from_numpy(out_i)


def _worker(rank, world, port, pruner, criteria, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    x, q, cents, assign = _problem()
    sizes = np.bincount(assign, minlength=cents.shape[0])
    owner = plan_shards(sizes, world)
    mine = np.zeros(x.shape[0], bool)
    mine[owned_rows(assign, owner, rank)] = True
    local = O.ivf_search_batch(_view(O, x, cents, assign, mine), q, 10, 40, pruner=pruner,
                               criteria=criteria)
    d, i = gather_merge(torch.from_numpy(local["dist"]), torch.from_numpy(local["ids"]), 10,
                        merge=merge_host)
    if rank == 0:
        ret["dist"] = d.numpy()
        ret["ids"] = i.numpy()
    dist.destroy_process_group()


def test_plan_shards_balanced_and_deterministic():
    sizes = np.random.default_rng(0).integers(1, 5000, 1024)
    for world in (2, 4, 8):
        owner = plan_shards(sizes, world)
        assert np.array_equal(owner, plan_shards(sizes, world))
        loads = np.bincount(owner, weights=sizes, minlength=world)
        assert loads.max() - loads.min() <= sizes.max()
        assert set(owner.tolist()) == set(range(world))


@pytest.mark.parametrize("pruner,criteria", [("bond", "dmeans"), ("none", "sequential")])
def test_sharded_search_equals_single_process(oracle, pruner, criteria):
    port = _free_port()
    with mp.Manager() as mgr:
        ret = mgr.dict()
        mp.spawn(_worker, args=(2, port, pruner, criteria, ret), nprocs=2, join=True)
        got_d, got_i = ret["dist"], ret["ids"]
    x, q, cents, assign = _problem()
    ref = oracle.ivf_search_batch(_view(oracle, x, cents, assign, np.ones(x.shape[0], bool)),
                                  q, 10, 40, pruner=pruner, criteria=criteria)
    np.testing.assert_array_equal(got_i, ref["ids"])
    np.testing.assert_array_equal(got_d, ref["dist"])


# ------------------------------------------ row-chunk shards (C5 layout)
def _c5_problem():
    """A small chunk-seeded mixture with C5's spectrum: 12 chunks of 700."""
    from paper_2503_04422_b200.synthetic import c5_sigma, mixture_centres
    d, nchunks, rows = 32, 12, 700
    centres = mixture_centres(7, 40, d)
    sig = c5_sigma(d)
    return d, nchunks, rows, centres, sig


def _c5_chunk(c, centres, rows, sig):
    from paper_2503_04422_b200.synthetic import mixture_chunk
    return mixture_chunk(7, c, rows, centres, sig)


def _c5_worker(rank, world, port, pruner, ret):
    """Rank r generates ONLY its chunks c = r, r + world, ... (chunk-seeded),
    assigns them to the replicated centroids, scans its rows (the oracle
    stands in for the GPU scan on this CPU box) and joins the single packed
    all-gather + merge."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    d, nchunks, rows, centres, sig = _c5_problem()
    cents = np.ascontiguousarray(_c5_chunk(0, centres, rows, sig)[:24])  # rank 0's sample
    t = torch.from_numpy(cents)
    dist.broadcast(t, src=0)  # the replicated centroids, as build_rank_index does
    cents = t.numpy()
    mine = list(range(rank, nchunks, world))
    xs = [_c5_chunk(c, centres, rows, sig) for c in mine]
    x = np.concatenate(xs)
    gid = np.concatenate([np.arange(c * rows, (c + 1) * rows) for c in mine]).astype(np.int64)
    assign = np.argmin(((x[:, None, :] - cents[None]) ** 2).sum(-1), axis=1)
    view = O.IvfView.from_assignment(x, cents, assign, cents.shape[0])
    view.buckets.ids[:] = gid[view.buckets.ids]  # global row ids
    q = np.ascontiguousarray(_c5_chunk(99, centres, 16, sig))
    local = O.ivf_search_batch(view, q, 10, 8, pruner=pruner)
    d_, i_ = gather_merge(torch.from_numpy(local["dist"]), torch.from_numpy(local["ids"]), 10,
                          merge=merge_host)
    ret[rank] = (d_.numpy(), i_.numpy(), len(mine) * rows)
    dist.destroy_process_group()


@pytest.mark.parametrize("pruner", ["bond", "none"])
def test_row_chunk_shards_world4_equal_single_process(oracle, pruner):
    """World size 4: no rank generates or holds another rank's chunks; the
    merged top-k (one packed all_gather) equals the single-process search
    on the whole collection for the exact pruners, on every rank."""
    port = _free_port()
    world = 4
    with mp.Manager() as mgr:
        ret = mgr.dict()
        mp.spawn(_c5_worker, args=(world, port, pruner, ret), nprocs=world, join=True)
        res = dict(ret)
    d, nchunks, rows, centres, sig = _c5_problem()
    assert sum(res[r][2] for r in range(world)) == nchunks * rows
    x = np.concatenate([_c5_chunk(c, centres, rows, sig) for c in range(nchunks)])
    cents = np.ascontiguousarray(x[:24])
    assign = np.argmin(((x[:, None, :] - cents[None]) ** 2).sum(-1), axis=1)
    q = np.ascontiguousarray(_c5_chunk(99, centres, 16, sig))
    ref = oracle.ivf_search_batch(oracle.IvfView.from_assignment(x, cents, assign, 24), q, 10, 8,
                                  pruner=pruner)
    for r in range(world):
        np.testing.assert_array_equal(res[r][1], ref["ids"])
        np.testing.assert_array_equal(res[r][0], ref["dist"])


def test_pack_unpack_topk_roundtrip():
    from paper_2503_04422_b200.sharded import pack_topk, unpack_topk
    rng = np.random.default_rng(3)
    dd = torch.from_numpy(rng.standard_normal((5, 7)).astype(np.float32))
    ii = torch.from_numpy(rng.integers(-1, 1 << 40, (5, 7)))
    b = pack_topk(dd, ii)
    d2, i2 = unpack_topk(torch.stack([b, b]), 5, 7)
    assert torch.equal(d2[1], dd) and torch.equal(i2[0], ii)
