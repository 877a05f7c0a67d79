"""Sharded IVF search across the GPUs of one box.

One process per GPU, two ways to split the collection:

* by bucket (``shard_index`` / ``shard_from_assignment``): every rank holds
  the replicated centroids and the block chains of the buckets it owns
  (longest-processing-time assignment by bucket size, deterministic);
* by row chunk (``build_rank_index``, C5): rank r generates only the chunks
  c = r, r + world, ... of a chunk-seeded collection
  (synthetic.mixture_chunk, default_rng([seed, chunk])), assigns them to the
  replicated centroids (trained on a sample by rank 0 and broadcast) and
  packs its own members of every bucket — no rank, and no host, ever holds
  the whole collection.

All ranks select the same global nprobe buckets (K2), scan what they hold
of them in global selection order, then the per-rank top-k lists are
all-gathered in ONE collective (dist + ids packed into one buffer) and
merged on the device with the reference's (distance, id) rule (K7).

Parity: BOND and 'none' return the exact global top-k (a merge of exact
local top-k lists); ADS runs one threshold chain per shard, so its parity
across shards is recall@k (single-GPU runs keep decision-level parity).
"""
from __future__ import annotations

import numpy as np

from . import _lib


def plan_shards(bucket_sizes, world: int) -> np.ndarray:
    """Owner rank per bucket: largest buckets first, each to the least
    loaded rank (ties: lower bucket index first, lower rank first)."""
    sizes = np.asarray(bucket_sizes, dtype=np.int64)
    order = np.lexsort((np.arange(sizes.size), -sizes))
    load = np.zeros(world, dtype=np.int64)
    owner = np.empty(sizes.size, dtype=np.int32)
    for b in order:
        r = int(np.argmin(load))
        owner[b] = r
        load[r] += sizes[b]
    return owner


def owned_rows(assign, owner, rank: int) -> np.ndarray:
    """Rows (ascending) whose bucket this rank owns."""
    assign = np.asarray(assign)
    return np.flatnonzero(np.asarray(owner)[assign] == rank)


def shard_index(index, collection, rank: int, world: int, x_dev=None):
    """This rank's IvfIndex: same nlist and centroids, only owned buckets
    populated (members keep their original ids and ascending order)."""
    import torch
    from .index import IvfIndex
    from .layout import VectorCollection
    from .store import to_device
    counts = np.asarray(index._counts)
    owner = plan_shards(counts, world)
    off = np.concatenate([[0], np.cumsum(counts)])
    assign = np.empty(collection.n, dtype=np.int64)
    for c in range(index.nlist):
        assign[index._order[off[c]:off[c + 1]]] = c
    rows = owned_rows(assign, owner, rank)
    sub = VectorCollection(data=collection.data[rows], ids=collection.ids[rows])
    xd = None
    if x_dev is not None:
        xd = x_dev[to_device(rows, torch.int64)]
    return IvfIndex.from_assignment(sub, index.centroids, assign[rows], nlist=index.nlist,
                                    training_seed=index.training_seed,
                                    block_size=index.block_size, group=index.store.group,
                                    x_dev=xd)


def shard_from_assignment(XR, centroids, assign, rank: int, world: int, x_dev=None, ids=None,
                          nlist=None, group: int = 8):
    """This rank's bucket shard built straight from (data, centroids,
    assignment): only the owned buckets' rows are uploaded and packed."""
    import torch
    from .index import IvfIndex
    from .layout import VectorCollection
    from .store import to_device
    centroids = np.asarray(centroids, np.float32)
    nlist = centroids.shape[0] if nlist is None else nlist
    assign = np.asarray(assign, np.int64)
    owner = plan_shards(np.bincount(assign, minlength=nlist), world)
    rows = owned_rows(assign, owner, rank)
    ids = np.arange(assign.shape[0], dtype=np.int64) if ids is None else np.asarray(ids)
    sub = VectorCollection(data=XR[rows], ids=ids[rows])
    xd = x_dev[to_device(rows, torch.int64)] if x_dev is not None else None
    return IvfIndex.from_assignment(sub, centroids, assign[rows], nlist=nlist, group=group,
                                    x_dev=xd)


class _RowsOnly:
    """A collection handle with ids but no host data (chunk-built shards)."""

    def __init__(self, ids, d):
        self.ids = ids
        self.n = int(ids.shape[0])
        self.d = d
        self.data = None


def build_rank_index(chunk_fn, nchunks: int, rank: int, world: int, nlist: int, d: int,
                     train_chunks: int = 2, seed: int = 0, max_iters: int = 10,
                     transform=None, group: int = 8, rows_per_chunk=None):
    """Row-chunk shard of a chunk-seeded collection (C5).

    chunk_fn(c) -> float32 [rows, d] host array of chunk c (deterministic).
    Rank 0 trains the centroids on chunks [0, train_chunks) with the GPU
    k-means (index.py:27-64 semantics) and broadcasts them (torch.distributed,
    NCCL on GPUs / gloo on CPU tensors); every rank then generates only its
    chunks c = rank, rank + world, ..., rotates them (K3, when a transform
    is given), assigns them (pdx_kmeans_assign) and packs its members of
    every bucket.  Ids are global row numbers.  Returns (index, centroids)."""
    import torch
    import torch.distributed as dist

    from . import _lib
    from .index import IvfIndex, kmeans_assign, lloyd_kmeans_device
    from .store import to_device
    dev = torch.device("cuda", torch.cuda.current_device())
    Tm = None if transform is None else to_device(np.asarray(transform.matrix, np.float32))

    def rotated(c):
        x = to_device(chunk_fn(c))
        if Tm is None:
            return x
        y = torch.empty_like(x)
        _lib.check(_lib.lib().pdx_project(_lib.ptr(x), x.shape[0], d, _lib.ptr(Tm), _lib.ptr(y),
                                          _lib.stream_handle()))
        return y

    cent = torch.empty((nlist, d), dtype=torch.float32, device=dev)
    distributed = world > 1 and dist.is_initialized()
    if rank == 0 or not distributed:  # (an emulated rank trains the same centroids itself)
        sample = torch.cat([rotated(c) for c in range(min(train_chunks, nchunks))])
        cent.copy_(lloyd_kmeans_device(sample, nlist, seed, max_iters)[0])
        del sample
    if distributed:
        if dist.get_backend() == "nccl":
            dist.broadcast(cent, src=0)
        else:
            h = cent.cpu()
            dist.broadcast(h, src=0)
            cent.copy_(h)
    mine = list(range(rank, nchunks, world))
    xs, ids, assign = [], [], []
    row0 = 0
    for c in range(nchunks):
        if c not in mine:
            row0 += rows_per_chunk(c) if rows_per_chunk else 0
            continue
        x = rotated(c)
        n = x.shape[0]
        r0 = row0 if rows_per_chunk else c * n
        xs.append(x)
        ids.append(torch.arange(r0, r0 + n, dtype=torch.int64, device=dev))
        assign.append(kmeans_assign(x, cent))
        row0 += n
    x = torch.cat(xs) if xs else torch.empty((0, d), dtype=torch.float32, device=dev)
    del xs
    a = torch.cat(assign) if assign else torch.empty(0, dtype=torch.int32, device=dev)
    gid = torch.cat(ids) if ids else torch.empty(0, dtype=torch.int64, device=dev)
    col = _RowsOnly(gid, d)
    index = IvfIndex.from_assignment(col, cent.cpu().numpy(), a, nlist=nlist, group=group,
                                     x_dev=x)
    return index, cent


def pack_topk(dist, ids):
    """(dist f32 [nq,k], ids i64 [nq,k]) -> one int32 buffer [3 nq k]:
    ids first (8-byte aligned), then the distances' bits."""
    import torch
    nq, k = dist.shape
    buf = torch.empty(3 * nq * k, dtype=torch.int32, device=dist.device)
    buf[:2 * nq * k].view(torch.int64).copy_(ids.reshape(-1))
    buf[2 * nq * k:].view(torch.float32).copy_(dist.reshape(-1))
    return buf


def unpack_topk(bufs, nq: int, k: int):
    """[world, 3 nq k] int32 -> (dist [world,nq,k] f32, ids [world,nq,k] i64)."""
    import torch
    ids = bufs[:, :2 * nq * k].contiguous().view(torch.int64).reshape(-1, nq, k)
    dist = bufs[:, 2 * nq * k:].contiguous().view(torch.float32).reshape(-1, nq, k)
    return dist, ids


def merge_device(dist_all, ids_all, k: int):
    """K7: [world, nq, k] sorted lists -> [nq, k] (pdx_merge_topk)."""
    import torch
    world, nq, _ = dist_all.shape
    od = torch.empty((nq, k), dtype=torch.float32, device=dist_all.device)
    oi = torch.empty((nq, k), dtype=torch.int64, device=dist_all.device)
    _lib.check(_lib.lib().pdx_merge_topk(_lib.ptr(dist_all.contiguous()),
                                         _lib.ptr(ids_all.contiguous()), world, nq, k,
                                         _lib.ptr(od), _lib.ptr(oi), _lib.stream_handle()))
    return od, oi


def gather_merge(dist, ids, k: int, group=None, merge=merge_device):
    """All-gather every rank's (dist [nq,k], ids [nq,k]) over the process
    group (NCCL on GPUs, gloo on CPU) in ONE collective of the packed
    buffer (pack_topk) and merge; the global (dist, ids) on every rank."""
    import torch
    import torch.distributed as dist_
    world = dist_.get_world_size(group)
    nq = dist.shape[0]
    buf = pack_topk(dist.contiguous(), ids.contiguous())
    dev = buf.device
    if dev.type == "cuda" and dist_.get_backend(group) != "nccl":
        buf = buf.cpu()  # gloo moves host tensors
    out = torch.empty(world * buf.numel(), dtype=torch.int32, device=buf.device)
    dist_.all_gather_into_tensor(out, buf, group=group)
    d_all, i_all = unpack_topk(out.view(world, -1).to(dev), nq, k)
    return merge(d_all, i_all, k)
