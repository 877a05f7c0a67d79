"""IVF bucket index and flat partitioning over the HBM store (index.py:1-191).

Build (``lloyd_kmeans``/``ivf_build``/``flat_build``) runs on the GPU in
this library's kernels (csrc/pdx_build.cu): a fused float32 distance +
argmin in the reference's expansion form (index.py:67-72), a stable radix
bucket layout, the float64 segment-mean kernel (numpy's order) for every
mean, and kernel K1 for the packing.  Search
(``ivf_search``/``exact_search`` and their batched forms) runs kernels
K2 (bucket selection), K4 (orders) and K5/K6 (pruned scan + top-k).
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .kernels import Metric
from .layout import Block, VectorCollection, to_blocks
from .pruning import OrderCriteria, dimension_orders_device
from .search import (SearchParams, SearchStats, TopK, _fill_stats, _trace_cap, run_search)
from .store import DeviceStore, device, segment_means_rows, to_device

DEFAULT_PARTITION_SIZE = 10_000
DEFAULT_KMEANS_ITERS = 20
KMEANS_SHIFT_TOL = 1e-4


# ------------------------------------------------------------------ k-means
def _empty(shape, dtype, dev):
    import torch
    return torch.empty(shape, dtype=dtype, device=dev)


def row_norms(x):
    """||x_i||^2, float32 (pdx_row_norms; the einsum of index.py:70)."""
    import torch
    out = _empty((x.shape[0],), torch.float32, x.device)
    _lib.check(_lib.lib().pdx_row_norms(_lib.ptr(x), x.shape[0], x.shape[1], _lib.ptr(out),
                                        _lib.stream_handle()))
    return out


def kmeans_assign(x, centroids, xnorm=None, cnorm=None, rows=None, min_dist=False):
    """Nearest centroid of every row (pdx_kmeans_assign: fused float32
    distance max(xx + cc - 2 x.c, 0) of index.py:67-72 + argmin, lowest
    index on ties as np.argmin).  Returns int32 assignments [, distances]."""
    import torch
    n = x.shape[0] if rows is None else rows.shape[0]
    xnorm = row_norms(x) if xnorm is None else xnorm
    if rows is not None and xnorm.shape[0] != n:
        xnorm = xnorm[rows]
    cnorm = row_norms(centroids) if cnorm is None else cnorm
    a = _empty((n,), torch.int32, x.device)
    md = _empty((n,), torch.float32, x.device) if min_dist else None
    _lib.check(_lib.lib().pdx_kmeans_assign(_lib.ptr(x), _lib.ptr(rows), n, x.shape[1],
                                            _lib.ptr(xnorm), _lib.ptr(centroids),
                                            _lib.ptr(cnorm), centroids.shape[0], _lib.ptr(a),
                                            _lib.ptr(md), _lib.stream_handle()))
    return (a, md) if min_dist else a


def bucket_layout(assign, nlist):
    """Members of every bucket in ascending original index (index.py:100):
    (order int64 [n], counts int64 [nlist], offsets int64 [nlist+1]) from a
    stable radix sort (pdx_bucket_layout)."""
    import ctypes as C

    import torch
    if assign.dtype != torch.int32:
        assign = assign.to(torch.int32)
    n, dev = assign.shape[0], assign.device
    wb = C.c_int64(0)
    L = _lib.lib()
    _lib.check(L.pdx_bucket_layout(_lib.ptr(assign), n, nlist, None, None, None, None,
                                   C.cast(C.pointer(wb), C.c_void_p), _lib.stream_handle()))
    work = _empty((max(1, wb.value),), torch.uint8, dev)
    order = _empty((n,), torch.int64, dev)
    counts = _empty((nlist,), torch.int64, dev)
    off = _empty((nlist + 1,), torch.int64, dev)
    _lib.check(L.pdx_bucket_layout(_lib.ptr(assign), n, nlist, _lib.ptr(order), _lib.ptr(counts),
                                   _lib.ptr(off), _lib.ptr(work),
                                   C.cast(C.pointer(wb), C.c_void_p), _lib.stream_handle()))
    return order, counts, off


def _argmin_chunked(x, c, chunk=None):
    """Nearest centroid of every row, int64 (tools' helper; one fused launch)."""
    import torch
    return kmeans_assign(x, c).to(torch.int64)


def _segment_means(x, order, off, nlist, init=None):
    import torch
    means = (init.clone() if init is not None else
             torch.zeros((nlist, x.shape[1]), dtype=torch.float64, device=x.device))
    _lib.check(_lib.lib().pdx_segment_means(_lib.ptr(x), x.shape[1], _lib.ptr(order),
                                            _lib.ptr(off), nlist, _lib.ptr(means),
                                            _lib.stream_handle()))
    return means


def _farthest(x, assign, bucket, centroid):
    """index.py:52-54: members of `bucket`, the one farthest from centroid
    (first on ties).  pdx_kmeans_farthest."""
    import torch
    key = _empty((1,), torch.int64, x.device)
    cn = float(row_norms(centroid[None, :]).item())
    _lib.check(_lib.lib().pdx_kmeans_farthest(_lib.ptr(x), x.shape[0], x.shape[1],
                                              _lib.ptr(assign), int(bucket), _lib.ptr(centroid),
                                              cn, _lib.ptr(key), _lib.stream_handle()))
    k = int(key.item()) & 0xFFFFFFFF
    return 0xFFFFFFFF - k


def lloyd_kmeans_device(x, nlist: int, seed: int, max_iters: int = DEFAULT_KMEANS_ITERS):
    """Lloyd iterations of index.py:27-64 on a device tensor, every step a
    kernel of this library (no cuBLAS / ATen compute): seeded sample init
    (pdx_gather_rows), fused distance + argmin (pdx_kmeans_assign), stable
    bucket layout (pdx_bucket_layout), float64 member means in the
    reference's summation order (pdx_segment_means), centroid update
    (pdx_kmeans_update), largest-cluster split for empty clusters
    (pdx_kmeans_farthest) and the relative-shift stop (pdx_kmeans_shift).
    Returns (centroids f32 [nlist, d], assign int32 [n])."""
    import torch
    n, d = x.shape
    if not 1 <= nlist <= n:
        raise ValueError(f"nlist must be in [1, {n}], got {nlist}")
    dev = x.device
    L = _lib.lib()
    st = _lib.stream_handle()
    rng = np.random.default_rng(seed)
    init = torch.from_numpy(rng.choice(n, size=nlist, replace=False).astype(np.int64)).to(dev)
    centroids = _empty((nlist, d), torch.float32, dev)
    _lib.check(L.pdx_gather_rows(_lib.ptr(x), d, _lib.ptr(init), nlist, _lib.ptr(centroids), st))
    xnorm = row_norms(x)
    shift = _empty((1,), torch.float32, dev)
    for _ in range(max_iters):
        assign = kmeans_assign(x, centroids, xnorm=xnorm)
        order, counts, off = bucket_layout(assign, nlist)
        means = _segment_means(x, order, off, nlist)
        new = _empty((nlist, d), torch.float32, dev)
        _lib.check(L.pdx_kmeans_update(_lib.ptr(means), _lib.ptr(counts), _lib.ptr(centroids),
                                       nlist, d, _lib.ptr(new), st))
        counts_h = counts.cpu().numpy().copy()
        for c in np.flatnonzero(counts_h == 0):  # index.py:49-56, in bucket order
            if counts_h[c] > 0:
                continue
            largest = int(np.argmax(counts_h))
            stray = _farthest(x, assign, largest, new[largest].contiguous())
            new[c] = x[stray]
            assign[stray] = int(c)
            counts_h[largest] -= 1
            counts_h[c] += 1
        _lib.check(L.pdx_kmeans_shift(_lib.ptr(new), _lib.ptr(centroids), nlist, d,
                                      _lib.ptr(shift), st))
        centroids = new
        if float(shift.item()) < KMEANS_SHIFT_TOL:
            break
    assign = kmeans_assign(x, centroids, xnorm=xnorm)
    return centroids, assign


def lloyd_kmeans(data, nlist: int, seed: int, max_iters: int = DEFAULT_KMEANS_ITERS):
    """index.py:27-64 → (centroids float32 (nlist, d), assignments intp (n,))."""
    import torch
    x = to_device(np.asarray(data, np.float32) if not isinstance(data, torch.Tensor) else data,
                  torch.float32)
    c, a = lloyd_kmeans_device(x, nlist, seed, max_iters)
    return c.cpu().numpy(), a.cpu().numpy().astype(np.intp)


# ---------------------------------------------------------------- IvfIndex
class IvfIndex:
    """k-means buckets as block chains in HBM (index.py:75-88).

    Device state: ``store`` (tiles of every bucket chain, buckets in index
    order, members ascending by original row), ``centroids_dev`` (f32
    row-major), ``means_dev`` (f64 per-bucket means).  The reference's host
    views (``centroid_blocks``, ``buckets``, ``bucket_means``) are built on
    first access."""

    def __init__(self, nlist, centroids, store, means_dev, training_seed, block_size,
                 host_data=None, order=None, ids=None, counts=None):
        self.nlist = int(nlist)
        self.centroids = np.ascontiguousarray(centroids, dtype=np.float32)
        self.store = store
        self.centroids_dev = to_device(self.centroids)
        self.means_dev = means_dev
        self.training_seed = training_seed
        self.block_size = int(block_size)
        self._host_data = host_data
        self._order = order
        self._ids = ids
        self._counts = counts
        self._buckets = None

    @property
    def d(self) -> int:
        return self.centroids.shape[1]

    @property
    def centroid_blocks(self) -> list[Block]:
        return to_blocks(VectorCollection.from_array(self.centroids), self.block_size)

    @property
    def bucket_means(self) -> list[np.ndarray]:
        m = self.means_dev.cpu().numpy()
        return [m[c] for c in range(self.nlist)]

    @property
    def buckets(self) -> list[list[Block]]:
        """Host block chains (index.py:99-102), for inspection and the oracle."""
        if self._buckets is None:
            data = self._host_data
            if data is None:
                raise RuntimeError("index was built from device data; no host copy kept")
            order = self._order
            ids = self._ids if self._ids is not None else np.arange(data.shape[0], dtype=np.int64)
            off = np.concatenate([[0], np.cumsum(self._counts)])
            chains = []
            for c in range(self.nlist):
                mem = order[off[c]:off[c + 1]]
                part = VectorCollection(data=data[mem], ids=ids[mem])
                chains.append(to_blocks(part, self.block_size) if part.n else [])
            self._buckets = chains
        return self._buckets

    @classmethod
    def from_assignment(cls, collection: VectorCollection, centroids, assign, nlist=None,
                        training_seed=0, block_size=64, group=8, x_dev=None) -> "IvfIndex":
        """Pack an index from given centroids and bucket assignments
        (index.py:98-108): members ascending by row, blocks of block_size,
        bucket means in float64 (empty bucket: its centroid)."""
        import torch
        centroids = np.asarray(centroids, dtype=np.float32)
        nlist = centroids.shape[0] if nlist is None else nlist
        x = x_dev if x_dev is not None else to_device(collection.data, torch.float32)
        a = to_device(assign if isinstance(assign, torch.Tensor) else np.asarray(assign, np.int32),
                      torch.int32)
        order, counts, off = bucket_layout(a, nlist)
        means = _segment_means(x, order, off, nlist, init=to_device(centroids, torch.float64))
        counts_h = counts.cpu().numpy()
        nblk = (counts_h + block_size - 1) // block_size
        # vectors per logical block, bucket by bucket
        ms = []
        for c in np.flatnonzero(nblk):
            full, rem = divmod(int(counts_h[c]), block_size)
            ms.extend([block_size] * full)
            if rem:
                ms.append(rem)
        ms = np.asarray(ms, dtype=np.int64)
        ids = to_device(collection.ids, torch.int64)
        store = DeviceStore.pack(x, order, ms, nblk.astype(np.int64), ids=ids, group=group)
        return cls(nlist, centroids, store, means, training_seed, block_size,
                   host_data=collection.data, order=order.cpu().numpy(), ids=collection.ids,
                   counts=counts_h)


def ivf_build(collection: VectorCollection, nlist: int | None = None, seed: int = 0,
              max_iters: int = DEFAULT_KMEANS_ITERS, block_size: int = 64, group: int = 8,
              x_dev=None) -> IvfIndex:
    """Cluster and pack (index.py:91-108), all on the GPU."""
    import torch
    if nlist is None:
        nlist = max(1, round(math.sqrt(collection.n)))
    x = x_dev if x_dev is not None else to_device(collection.data, torch.float32)
    centroids, assign = lloyd_kmeans_device(x, nlist, seed, max_iters)
    return IvfIndex.from_assignment(collection, centroids.cpu().numpy(), assign, nlist=nlist,
                                    training_seed=seed, block_size=block_size, group=group,
                                    x_dev=x)


# --------------------------------------------------------------- selection
# Bucket selection on the tensor cores pays once the centroid scan is a real
# GEMM (C5: 10,000 queries x 65,536 centroids x 768 dims).
TC_SELECT_MIN_WORK = 1 << 34  # nq * nlist * d


def _select_tensor_cores(index: IvfIndex, Q, nprobe: int, metric: Metric):
    """ivf_select_buckets (index.py:111-127) for a batch through K8: tcgen05
    TF32 candidates of the nprobe nearest centroids (pdx_k8_candidates), then
    the candidates' exact keys with the reference's arithmetic (the vertical
    kernel over the centroid chain: per-op-rounded sequential float32) and the
    nprobe smallest (key, bucket) — the stable argsort's order
    (pdx_k8_rescore_rows).  Identical to K2.  None when a query's candidates
    overflow (the caller runs K2)."""
    import ctypes as C

    import torch
    L = _lib.lib()
    d, nlist, nq = index.d, index.nlist, Q.shape[0]
    ld = (d + 3) // 4 * 4
    tc = getattr(index, "_tc_select", None)
    if tc is None:
        X = torch.zeros((nlist, ld), dtype=torch.float32, device=Q.device)
        X[:, :d] = index.centroids_dev
        xn2 = torch.empty(nlist, dtype=torch.float32, device=Q.device)
        _lib.check(L.pdx_k8_norms_ld(_lib.ptr(X), nlist, d, ld, _lib.ptr(xn2),
                                     _lib.stream_handle()))
        tc = index._tc_select = {"X": X, "xn2": xn2,
                                 "rowids": torch.arange(nlist, dtype=torch.int64,
                                                        device=Q.device)}
    Qp = Q if ld == d else torch.nn.functional.pad(Q, (0, ld - d))
    Qp = Qp.contiguous()
    cap = max(4096, 4 * nprobe)
    met = _lib.METRIC[metric.value]
    cand = torch.empty((nq, cap), dtype=torch.int64, device=Q.device)
    cnt = torch.zeros(nq, dtype=torch.int32, device=Q.device)
    wb = C.c_int64(0)
    args = (_lib.ptr(tc["X"]), nlist, d, ld, _lib.ptr(tc["xn2"]), _lib.ptr(Qp), nq, met, nprobe,
            _lib.ptr(cand), _lib.ptr(cnt), cap)
    _lib.check(L.pdx_k8_candidates(*args, None, C.cast(C.pointer(wb), C.c_void_p),
                                   _lib.stream_handle()))
    work = tc.get("work")
    if work is None or work.numel() < wb.value:
        work = tc["work"] = torch.empty(max(1, wb.value), dtype=torch.uint8, device=Q.device)
    _lib.check(L.pdx_k8_candidates(*args, _lib.ptr(work), C.cast(C.pointer(wb), C.c_void_p),
                                   _lib.stream_handle()))
    cmax = int(cnt.max().item())
    if cmax > cap:
        return None
    dist = torch.empty((nq, nprobe), dtype=torch.float32, device=Q.device)
    ids = torch.empty((nq, nprobe), dtype=torch.int64, device=Q.device)
    _lib.check(L.pdx_k8_rescore_rows(_lib.ptr(tc["X"]), ld, d, _lib.ptr(tc["rowids"]),
                                     _lib.ptr(Qp), nq, met, nprobe, _lib.ptr(cand), _lib.ptr(cnt),
                                     cap, max(1, cmax), _lib.ptr(dist), _lib.ptr(ids),
                                     _lib.stream_handle()))
    return ids.to(torch.int32)


def select_buckets_device(index: IvfIndex, Q, nprobe: int, metric=Metric.L2, scratch=None,
                          tensor_cores=None):
    """Bucket selection for a device batch: int32 [nq, nprobe] bucket ids —
    K2 (pdx_select_buckets), or, for GEMM-sized batches (tensor_cores None:
    nq * nlist * d >= TC_SELECT_MIN_WORK) over L2 / IP, the tensor-core path
    with identical results (_select_tensor_cores)."""
    import torch
    if not 1 <= nprobe <= index.nlist:
        raise ValueError(f"nprobe must be in [1, {index.nlist}], got {nprobe}")
    nq = Q.shape[0]
    metric = Metric(metric)
    use_tc = tensor_cores if tensor_cores is not None else (
        nq * index.nlist * index.d >= TC_SELECT_MIN_WORK)
    if use_tc and metric in (Metric.L2, Metric.IP) and nq > 0 and index.nlist >= nprobe:
        sel = _select_tensor_cores(index, Q.contiguous(), nprobe, metric)
        if sel is not None:
            return sel
    if scratch is None or scratch.numel() < nq * index.nlist:
        scratch = torch.empty((nq * index.nlist,), dtype=torch.float32, device=Q.device)
    sel = torch.empty((nq, nprobe), dtype=torch.int32, device=Q.device)
    _lib.check(_lib.lib().pdx_select_buckets(_lib.ptr(Q), nq, index.d,
                                             _lib.ptr(index.centroids_dev), index.nlist,
                                             _lib.METRIC[Metric(metric).value], nprobe,
                                             _lib.ptr(scratch), _lib.ptr(sel),
                                             _lib.stream_handle()))
    return sel


def ivf_select_buckets(index: IvfIndex, query, nprobe: int, metric: Metric = Metric.L2) -> np.ndarray:
    """index.py:111-127: the nprobe nearest buckets, ascending distance."""
    import torch
    if not 1 <= nprobe <= index.nlist:
        raise ValueError(f"nprobe must be in [1, {index.nlist}], got {nprobe}")
    q = to_device(np.asarray(query, np.float32)[None, :], torch.float32)
    return select_buckets_device(index, q, nprobe, metric)[0].cpu().numpy().astype(np.intp)


# ------------------------------------------------------------------ search
class IvfSearcher:
    """Batched IVF search with device-resident buffers (ivf_search,
    index.py:130-156, for a whole query batch): K2 selection, K4 orders
    (BOND with a query-aware criterion), K5/K6 scan."""

    def __init__(self, index: IvfIndex, params: SearchParams, nprobe: int,
                 criteria=OrderCriteria.SEQUENTIAL, zone_width=None, warps: int = 0,
                 batched: int = 0):
        if not 1 <= nprobe <= index.nlist:
            raise ValueError(f"nprobe must be in [1, {index.nlist}], got {nprobe}")
        self.index, self.params, self.nprobe = index, params, nprobe
        self.criteria = OrderCriteria(criteria)
        self.zone_width = zone_width
        self.warps = warps
        self.batched = int(batched)  # pdx_search_params.batched: 0 auto, 1 off, 2 forced
        self._buf = {}
        self._scratch = None

    def select(self, Q):
        """K2 only: int32 [nq, nprobe] selected buckets (ivf_select_buckets)."""
        return select_buckets_device(self.index, Q, self.nprobe, self.params.metric,
                                     self._scratch)

    def search(self, Q, sel, stats=False, trace_cap=0, timed=False):
        """The scan for a given selection (device buffers in and out: the call
        a CUDA graph of a fixed batch captures, see bench.py)."""
        orders, oss = None, 0
        if self.params.pruner == "bond" and self.criteria is not OrderCriteria.SEQUENTIAL:
            orders = dimension_orders_device(Q, self.index.means_dev, self.criteria,
                                             self.zone_width, mean_index=sel, nsets=self.nprobe)
            oss = 1
        res = run_search(self.index.store, Q, self.params, seg_bucket=sel, nseg=self.nprobe,
                         orders=orders, order_qstride=self.nprobe, order_sstride=oss,
                         stats=stats, trace_cap=trace_cap, warps=self.warps, out=self._buf,
                         timed=timed, batched=self.batched)
        res.selected = sel
        return res

    def run(self, Q, stats=False, trace_cap=0, timed=False, phase_times=None, scan_events=None):
        import torch
        ev = None
        if phase_times is not None:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record()
        sel = select_buckets_device(self.index, Q, self.nprobe, self.params.metric,
                                    self._scratch)
        orders, oss = None, 0
        if self.params.pruner == "bond" and self.criteria is not OrderCriteria.SEQUENTIAL:
            orders = dimension_orders_device(Q, self.index.means_dev, self.criteria,
                                             self.zone_width, mean_index=sel, nsets=self.nprobe)
            oss = 1
        if ev:
            ev[1].record()
        if scan_events is not None:
            scan_events[1].record()
        res = run_search(self.index.store, Q, self.params, seg_bucket=sel, nseg=self.nprobe,
                         orders=orders, order_qstride=self.nprobe, order_sstride=oss,
                         stats=stats, trace_cap=trace_cap, warps=self.warps, out=self._buf,
                         timed=timed, batched=self.batched)
        if scan_events is not None:
            scan_events[2].record()
        if ev:
            ev[2].record()
            ev[2].synchronize()
            phase_times["find_nearest_buckets"] = ev[0].elapsed_time(ev[1]) / 1e3
            phase_times["distance_calculation"] = ev[1].elapsed_time(ev[2]) / 1e3
            phase_times["bounds_evaluation"] = 0.0
            phase_times.setdefault("query_preprocessing", 0.0)
        res.selected = sel
        return res


def ivf_search(index: IvfIndex, query, params: SearchParams, nprobe: int,
               criteria: OrderCriteria = OrderCriteria.SEQUENTIAL, zone_width: int | None = None,
               stats: SearchStats | None = None, phase_times: dict | None = None) -> TopK:
    """index.py:130-156 for one query (see ivf_search_batch for batches)."""
    import torch
    q = np.asarray(query, np.float32)
    if q.shape != (index.d,):
        raise ValueError(f"query length {q.shape} does not match d={index.d}")
    s = IvfSearcher(index, params, nprobe, criteria, zone_width)
    want = stats is not None
    res = s.run(to_device(q[None, :], torch.float32), stats=want,
                trace_cap=_trace_cap(nprobe * max(1, index.store.max_bucket_blocks), index.d,
                                     params.initial_step) if want else 0,
                timed=want, phase_times=phase_times)
    _fill_stats(stats, res)
    return res.topk(0, params.k)


def ivf_search_batch(index: IvfIndex, queries, params: SearchParams, nprobe: int,
                     criteria=OrderCriteria.SEQUENTIAL, zone_width=None, stats=False,
                     trace=False, batched=0):
    """All queries in one launch per kernel; returns host arrays
    (dist, ids, count[, touched, total, survivors, selected])."""
    import torch
    Q = to_device(np.asarray(queries, np.float32), torch.float32)
    if Q.shape[1] != index.d:
        raise ValueError(f"query dimensionality {Q.shape[1]} != {index.d}")
    s = IvfSearcher(index, params, nprobe, criteria, zone_width, batched=batched)
    cap = _trace_cap(nprobe * max(1, index.store.max_bucket_blocks), index.d,
                     params.initial_step) if trace else 0
    res = s.run(Q, stats=stats or trace, trace_cap=cap)
    out = res.host()
    out["selected"] = res.selected.cpu().numpy()
    return out


# -------------------------------------------------------------------- flat
@dataclass
class FlatPartitioning:
    """Equally sized horizontal partitions, each one wide block (index.py:159-168)."""

    store: DeviceStore
    global_means: np.ndarray
    partition_size: int
    _host: VectorCollection | None = None
    _partitions: list | None = field(default=None, repr=False)

    @property
    def d(self) -> int:
        return self.store.d

    @property
    def partitions(self) -> list[Block]:
        if self._partitions is None:
            if self._host is None:
                raise RuntimeError("no host copy kept")
            self._partitions = to_blocks(self._host, self.partition_size, pad=False)
        return self._partitions


def flat_build(collection: VectorCollection, partition_size: int = DEFAULT_PARTITION_SIZE,
               group: int = 8, x_dev=None) -> FlatPartitioning:
    """index.py:171-179: partitions of partition_size (one unpadded wide
    block each), global float64 means."""
    import torch
    if partition_size < 1:
        raise ValueError("partition_size must be >= 1")
    if collection.n == 0:
        raise ValueError("cannot partition an empty collection")
    x = x_dev if x_dev is not None else to_device(collection.data, torch.float32)
    n = collection.n
    full, rem = divmod(n, partition_size)
    ms = np.array([partition_size] * full + ([rem] if rem else []), dtype=np.int64)
    order = torch.arange(n, dtype=torch.int64, device=x.device)
    store = DeviceStore.pack(x, order, ms, np.array([len(ms)], np.int64),
                             ids=to_device(collection.ids, torch.int64), group=group)
    means = segment_means_rows(x)
    return FlatPartitioning(store=store, global_means=means, partition_size=partition_size,
                            _host=collection)


class ExactSearcher:
    """Batched exact_search (index.py:182-191) with device buffers.

    ``splits`` > 1 cuts each query's partition list into that many ranges
    scanned by separate CTAs and merged (pdx_search_params.splits): exact
    results for none / BOND with the split run's own values_touched, so one
    query can use the whole GPU."""

    def __init__(self, part: FlatPartitioning, params: SearchParams,
                 criteria=OrderCriteria.SEQUENTIAL, zone_width=None, warps: int = 0,
                 splits: int = 0):
        self.part, self.params = part, params
        self.splits = int(splits)
        self.criteria = OrderCriteria(criteria)
        self.zone_width = zone_width
        self.warps = warps
        self._buf = {}
        self._means = None

    def run(self, Q, stats=False, trace_cap=0, timed=False):
        orders = None
        if self.params.pruner == "bond" and self.criteria is not OrderCriteria.SEQUENTIAL:
            if self._means is None:
                self._means = to_device(self.part.global_means[None, :])
            orders = dimension_orders_device(Q, self._means, self.criteria, self.zone_width)
        return run_search(self.part.store, Q, self.params, nseg=1, orders=orders,
                          order_qstride=1, order_sstride=0, stats=stats, trace_cap=trace_cap,
                          warps=self.warps, out=self._buf, timed=timed, splits=self.splits)


def exact_search(partitioning: FlatPartitioning, query, params: SearchParams,
                 criteria: OrderCriteria = OrderCriteria.SEQUENTIAL, zone_width: int | None = None,
                 stats: SearchStats | None = None) -> TopK:
    """index.py:182-191 for one query."""
    import torch
    q = np.asarray(query, np.float32)
    if q.shape != (partitioning.d,):
        raise ValueError(f"query length {q.shape} does not match d={partitioning.d}")
    want = stats is not None
    s = ExactSearcher(partitioning, params, criteria, zone_width)
    res = s.run(to_device(q[None, :], torch.float32), stats=want,
                trace_cap=_trace_cap(partitioning.store.nblocks, partitioning.d,
                                     params.initial_step) if want else 0, timed=want)
    _fill_stats(stats, res)
    return res.topk(0, params.k)


def exact_search_batch(partitioning: FlatPartitioning, queries, params: SearchParams,
                       criteria=OrderCriteria.SEQUENTIAL, zone_width=None, stats=False,
                       trace=False, splits=0):
    import torch
    Q = to_device(np.asarray(queries, np.float32), torch.float32)
    if Q.shape[1] != partitioning.d:
        raise ValueError(f"query dimensionality {Q.shape[1]} != {partitioning.d}")
    s = ExactSearcher(partitioning, params, criteria, zone_width, splits=splits)
    cap = _trace_cap(partitioning.store.nblocks, partitioning.d, params.initial_step) if trace else 0
    return s.run(Q, stats=stats or trace, trace_cap=cap).host()
