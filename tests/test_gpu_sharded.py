"""Row-chunk shards on the GPU (sharded.build_rank_index, the C5 path):
world size 4 over gloo, all four ranks on cuda:0 (independent kernels, no
cross-rank waits; the exchange is gloo over host tensors).  Each rank
generates only its chunks, rank 0 trains the centroids with the GPU k-means
and broadcasts them, every rank scans its rows with the batched pipeline and
the per-rank top-k lists meet in one packed all_gather merged by K7
(pdx_merge_topk).  BOND / none: identical to one process searching the whole
collection with the same centroids; ADS: recall."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

D, NCHUNK, ROWS, NLIST, NQ = 48, 16, 2500, 64, 48


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _chunk_fn():
    from paper_2503_04422_b200.synthetic import c5_sigma, mixture_centres, mixture_chunk
    centres = mixture_centres(11, 100, D)
    sig = c5_sigma(D)
    return lambda c: mixture_chunk(11, c, ROWS, centres, sig)


def _queries():
    from paper_2503_04422_b200.synthetic import c5_sigma, mixture_centres, mixture_chunk
    return mixture_chunk(11, 10_000, NQ, mixture_centres(11, 100, D), c5_sigma(D))


def _worker(rank, world, port, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2503_04422_b200 as P
    from paper_2503_04422_b200.sharded import build_rank_index, gather_merge
    T = P.generate_orthogonal(D, 3)
    index, cent = build_rank_index(_chunk_fn(), NCHUNK, rank, world, NLIST, D, train_chunks=2,
                                   transform=T)
    q = P.apply_transform(T, P.store.to_device(_queries()))
    out = {}
    for pruner in ("bond", "ads", "none"):
        r = P.IvfSearcher(index, P.SearchParams(k=10, pruner=pruner), 12).run(q)
        # gloo moves host tensors; K7 merges on the GPU
        dh, ih = r.dist.cpu(), r.ids.cpu()
        from paper_2503_04422_b200.sharded import merge_device

        def merge(da, ia, k):
            return tuple(t.cpu() for t in merge_device(da.cuda(), ia.cuda(), k))
        d_, i_ = gather_merge(dh, ih, 10, merge=merge)
        out[pruner] = (d_.numpy(), i_.numpy())
    ret[rank] = (out, cent.cpu().numpy(), int(index.store.tile_ids.ge(0).sum().item()))
    dist.destroy_process_group()


def test_row_chunk_shards_world4_on_gpu():
    import paper_2503_04422_b200 as P
    world = 4
    with mp.get_context("spawn").Manager() as mgr:
        ret = mgr.dict()
        mp.spawn(_worker, args=(world, _port(), ret), nprocs=world, join=True)
        res = dict(ret)
    assert sum(res[r][2] for r in range(world)) == NCHUNK * ROWS  # every row exactly once
    cent = res[0][1]
    for r in range(world):
        np.testing.assert_array_equal(res[r][1], cent)
    # one process over the whole collection, same centroids
    T = P.generate_orthogonal(D, 3)
    fn = _chunk_fn()
    x = P.apply_transform(T, P.store.to_device(np.concatenate([fn(c) for c in range(NCHUNK)])))
    a = P.index.kmeans_assign(x, P.store.to_device(cent))
    col = P.VectorCollection.from_array(x.cpu().numpy())
    index = P.IvfIndex.from_assignment(col, cent, a, nlist=NLIST, x_dev=x)
    q = P.apply_transform(T, P.store.to_device(_queries()))
    gt = P.synthetic.ground_truth_device(x, q, 10)[0].cpu().numpy()
    for pruner in ("bond", "none", "ads"):
        ref = P.IvfSearcher(index, P.SearchParams(k=10, pruner=pruner), 12).run(q)
        for r in range(world):
            d_, i_ = res[r][0][pruner]
            if pruner == "ads":  # one threshold chain per shard: recall parity
                rec = np.mean([len(set(i_[j]) & set(gt[j])) / 10 for j in range(NQ)])
                ref_rec = np.mean([len(set(ref.ids.cpu().numpy()[j]) & set(gt[j])) / 10
                                   for j in range(NQ)])
                assert rec >= ref_rec - 0.01
            else:
                np.testing.assert_array_equal(i_, ref.ids.cpu().numpy())
                np.testing.assert_array_equal(d_, ref.dist.cpu().numpy())
