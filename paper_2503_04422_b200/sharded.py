"""Bucket-sharded IVF search across the GPUs of one box.

One process per GPU.  Every rank holds the replicated centroids and the
block chains of the buckets it owns (longest-processing-time assignment by
bucket size, deterministic).  All ranks select the same global nprobe
buckets (K2), scan the ones they own in global selection order (K5/K6),
then the per-rank top-k lists are all-gathered over NCCL and merged on the
device with the reference's (distance, id) rule (K7).

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
    group (NCCL on GPUs) and merge; the global (dist, ids) on every rank."""
    import torch
    import torch.distributed as dist_
    world = dist_.get_world_size(group)
    dl = [torch.empty_like(dist) for _ in range(world)]
    il = [torch.empty_like(ids) for _ in range(world)]
    dist_.all_gather(dl, dist.contiguous(), group=group)
    dist_.all_gather(il, ids.contiguous(), group=group)
    return merge(torch.stack(dl), torch.stack(il), k)
