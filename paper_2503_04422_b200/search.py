"""PDXearch front-end (search.py:1-213 of the reference) over the sm_100a scan.

The reference searches one query at a time in the interpreter.  Here every
entry point batches queries and runs the whole search — START/WARMUP/PRUNE,
the block-synchronous threshold chain, ADS / BOND decisions, the top-k and
the work accounting — inside one kernel launch per batch (pdx_search,
csrc/pdx_scan.cu).  Results, decisions and SearchStats counters equal the
reference's; ``TopK``/``SearchParams``/``SearchStats`` keep the reference's
names, fields and errors.
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .kernels import Metric
from .pruning import AdsPruner, BsaPruner

DEFAULT_SELECTION_FRACTION = 0.20
DEFAULT_INITIAL_STEP = 2


class TopK:
    """Bounded max-heap of (distance, id) (search.py:27-58).  Search results
    come back from the GPU already reduced; the heap API is kept so callers
    can inspect or extend results exactly as with the reference."""

    def __init__(self, k: int):
        if k < 1:
            raise ValueError("k must be >= 1")
        self.k = k
        self._heap: list[tuple[float, int]] = []

    @classmethod
    def from_arrays(cls, k, dist, ids, count) -> "TopK":
        tk = cls(k)
        tk._heap = [(-float(dist[i]), -int(ids[i])) for i in range(int(count))]
        heapq.heapify(tk._heap)
        return tk

    def __len__(self) -> int:
        return len(self._heap)

    def threshold(self) -> float:
        if len(self._heap) < self.k:
            return float("inf")
        return -self._heap[0][0]

    def push(self, distance: float, vid: int):
        item = (-distance, -vid)
        if len(self._heap) < self.k:
            heapq.heappush(self._heap, item)
        elif item > self._heap[0]:
            heapq.heapreplace(self._heap, item)

    def items(self) -> list[tuple[float, int]]:
        return sorted((-d, -i) for d, i in self._heap)

    def ids(self) -> list[int]:
        return [i for _, i in self.items()]


@dataclass
class SearchParams:
    """search.py:61-85 (same fields, defaults and ValueErrors)."""

    k: int
    metric: Metric = Metric.L2
    pruner: str = "none"
    selection_fraction: float = DEFAULT_SELECTION_FRACTION
    initial_step: int = DEFAULT_INITIAL_STEP
    ads: AdsPruner | None = None
    bsa: BsaPruner | None = None  # pruner="bsa" (this build's restatement)

    def __post_init__(self):
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if not 0.0 < self.selection_fraction <= 1.0:
            raise ValueError("selection_fraction must be in (0, 1]")
        if self.initial_step < 1:
            raise ValueError("initial_step must be >= 1")
        self.metric = Metric(self.metric)
        if self.pruner not in ("none", "ads", "bond", "bsa"):
            raise ValueError(f"unknown pruner: {self.pruner!r}")
        if self.pruner == "bsa":
            if self.metric is not Metric.L2:
                raise ValueError("the bsa pruner applies to squared L2 only")
            if self.bsa is None:
                raise ValueError("pruner='bsa' needs a fitted BsaPruner (pruning.fit_bsa)")
            if self.bsa.initial_step != self.initial_step:
                raise ValueError("the BsaPruner was fitted for another initial_step")
        if self.pruner == "bond" and self.metric is Metric.IP:
            raise ValueError("inner product has no monotone lower bound; "
                             "use pruner='none' for IP searches")
        if self.pruner == "ads":
            if self.metric is not Metric.L2:
                raise ValueError("the ads pruner applies to squared L2 only")


@dataclass
class SearchStats:
    """search.py:88-103.  ``distance_seconds`` holds the scan kernel's device
    time (distance and bound passes are one fused kernel, so
    ``bounds_seconds`` stays 0)."""

    distance_seconds: float = 0.0
    bounds_seconds: float = 0.0
    values_touched: int = 0
    values_total: int = 0
    survivors: list[list[int]] = field(default_factory=list)

    @property
    def pruning_power(self) -> float:
        if self.values_total == 0:
            return 0.0
        return 1.0 - self.values_touched / self.values_total


def step_schedule(d: int, initial_step: int = DEFAULT_INITIAL_STEP) -> list[tuple[int, int]]:
    """search.py:106-117."""
    if d < 1:
        raise ValueError("dimensionality must be >= 1")
    ranges = []
    start, width = 0, initial_step
    while start < d:
        end = min(start + width, d)
        ranges.append((start, end))
        start = end
        width *= 2
    return ranges


# ---------------------------------------------------------------- engine
class SearchResult:
    """Device outputs of one batched search (torch tensors on the GPU)."""

    def __init__(self, dist, ids, count, touched=None, total=None, trace=None, trace_len=None,
                 seconds=0.0):
        self.dist, self.ids, self.count = dist, ids, count
        self.touched, self.total = touched, total
        self.trace, self.trace_len = trace, trace_len
        self.seconds = seconds

    def host(self):
        out = {"dist": self.dist.cpu().numpy(), "ids": self.ids.cpu().numpy(),
               "count": self.count.cpu().numpy()}
        if self.touched is not None:
            out["touched"] = self.touched.cpu().numpy()
            out["total"] = self.total.cpu().numpy()
        if self.trace is not None:
            tr, tl = self.trace.cpu().numpy(), self.trace_len.cpu().numpy()
            out["survivors"] = [None if tl[i] < 0 else decode_trace(tr[i], tl[i])
                                for i in range(tr.shape[0])]
        return out

    def topk(self, i: int, k: int) -> TopK:
        d = self.dist[i].cpu().numpy()
        ids = self.ids[i].cpu().numpy()
        return TopK.from_arrays(k, d, ids, int(self.count[i].item()))


def decode_trace(buf, n):
    out, i = [], 0
    while i < n:
        ln = int(buf[i])
        out.append([int(v) for v in buf[i + 1:i + 1 + ln]])
        i += 1 + ln
    return out


def make_params(params: SearchParams, d: int, warps=0, device=None,
                splits: int = 0, batched: int = 0) -> _lib.PdxSearchParams:
    """``warps``: compute warps per query CTA, or (warps, tiles_per_warp[,
    ring_slots]); 0 = auto.  ``batched``: 0 auto, 1 per-query scan only, 2
    the bucket-major batched pipeline whenever eligible (pdx_b200.h)."""
    ads = params.ads if params.ads is not None else AdsPruner(d=d)
    w, tpw, rb = (tuple(warps) + (0, 0))[:3] if isinstance(warps, tuple) else (warps, 0, 0)
    coef = None
    if params.pruner == "bsa":
        if params.bsa.d != d:
            raise ValueError(f"the BsaPruner was fitted for d={params.bsa.d}, not {d}")
        coef = params.bsa.device_coef(device if device is not None else "cuda")
    return _lib.PdxSearchParams(int(params.k), _lib.METRIC[Metric(params.metric).value],
                                _lib.PRUNER[params.pruner], int(params.initial_step),
                                float(params.selection_fraction), int(ads.d), int(w),
                                float(ads.epsilon0), int(tpw), int(rb), _lib.ptr(coef),
                                int(splits), int(batched))


def run_search(store, queries, params: SearchParams, seg_bucket=None, nseg=None, orders=None,
               order_qstride=0, order_sstride=0, stats=False, trace_cap=0, warps=0, out=None,
               timed=False, splits=0, batched=0):
    """Launch pdx_search over ``store`` for a device batch ``queries`` (nq x d).

    seg_bucket: int32 [nq, nseg] bucket per visit segment (None: segment s
    is bucket s for s < nseg).  orders: uint16 permutations (see
    pdx_b200.h) or None for the natural order."""
    import torch
    q = queries.contiguous()
    nq = int(q.shape[0])
    if q.shape[1] != store.d:
        raise ValueError(f"query length {q.shape[1]} does not match d={store.d}")
    if nseg is None:
        nseg = int(seg_bucket.shape[1]) if seg_bucket is not None else store.nbuckets
    dev = q.device
    k = int(params.k)
    if out is None:
        out = {}
    dist = out.get("dist")
    if dist is None or dist.shape != (nq, k):
        dist = torch.empty((nq, k), dtype=torch.float32, device=dev)
        ids = torch.empty((nq, k), dtype=torch.int64, device=dev)
        count = torch.empty((nq,), dtype=torch.int32, device=dev)
        out.update(dist=dist, ids=ids, count=count)
    ids, count = out["ids"], out["count"]
    touched = total = trace = trace_len = None
    if stats or trace_cap:
        touched = torch.zeros((nq,), dtype=torch.int64, device=dev)
        total = torch.zeros((nq,), dtype=torch.int64, device=dev)
    if trace_cap:
        trace = torch.zeros((nq, trace_cap), dtype=torch.int32, device=dev)
        trace_len = torch.zeros((nq,), dtype=torch.int64, device=dev)
    debug = out.get("debug_buf")
    if debug is not None and debug.shape != (nq, 16):
        debug = None
    so = _lib.PdxSearchOut(_lib.ptr(dist), _lib.ptr(ids), _lib.ptr(count), _lib.ptr(touched),
                           _lib.ptr(total), _lib.ptr(trace), int(trace_cap), _lib.ptr(trace_len),
                           _lib.ptr(debug))
    L = _lib.lib()
    nlists = nq if seg_bucket is not None else 1
    wb = int(L.pdx_search_workspace(store.ref, nlists, nseg))
    work = out.get("work")
    if work is None or work.numel() < wb:
        work = torch.empty((wb,), dtype=torch.uint8, device=dev)
        out["work"] = work
    if params.pruner == "bsa":
        store.ensure_bsa_residuals(params.initial_step)
    p = make_params(params, store.d, warps, dev, splits, batched)
    sb = None if seg_bucket is None else seg_bucket.contiguous()
    st = _lib.stream_handle()
    ev0 = ev1 = None
    if timed:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
    _lib.check(L.pdx_search(store.ref, C_byref(p), _lib.ptr(q), nq, _lib.ptr(sb), int(nseg),
                            _lib.ptr(orders), int(order_qstride), int(order_sstride),
                            C_byref(so), _lib.ptr(work), wb, st))
    secs = 0.0
    if timed:
        ev1.record()
        ev1.synchronize()
        secs = ev0.elapsed_time(ev1) / 1e3
    return SearchResult(dist, ids, count, touched, total, trace, trace_len, secs)


def C_byref(x):
    import ctypes
    return ctypes.byref(x)


def _fill_stats(stats: SearchStats | None, res: SearchResult, i: int = 0):
    if stats is None:
        return
    h_t = int(res.touched[i].item())
    h_n = int(res.total[i].item())
    stats.values_touched += h_t
    stats.values_total += h_n
    stats.distance_seconds += res.seconds
    if res.trace is not None:
        ln = int(res.trace_len[i].item())
        if ln >= 0:
            stats.survivors.extend(decode_trace(res.trace[i].cpu().numpy(), ln))


def _trace_cap(nblocks: int, d: int, initial_step: int) -> int:
    return max(16, nblocks * (1 + len(step_schedule(d, initial_step))))


def _resolve_orders(orders, nblocks, d):
    """orders: None, one permutation, or one (or None) per block."""
    import torch
    from .store import to_device
    if orders is None:
        return None, 0, 0
    if isinstance(orders, (list, tuple)):
        if len(orders) != nblocks:
            raise ValueError("per-block orders must match the block count")
        if all(o is None for o in orders):
            return None, 0, 0
        ident = np.arange(d)
        arr = np.stack([np.arange(d) if o is None else np.asarray(o) for o in orders])
        _check_perm(arr, d)
        del ident
        return to_device(arr.astype(np.uint16), torch.uint16), 0, d
    arr = np.asarray(orders)
    _check_perm(arr[None, :], d)
    return to_device(arr.astype(np.uint16), torch.uint16), 0, 0


def _check_perm(arr, d):
    if arr.shape[-1] != d:
        raise ValueError(f"order length {arr.shape[-1]} != d={d}")
    if arr.size and (arr.min() < 0 or arr.max() >= d):
        raise ValueError("order entries out of range")


def search(blocks, query, params: SearchParams, orders=None, stats: SearchStats | None = None) -> TopK:
    """Search an ordered block sequence (search.py:177-205) on the GPU.

    ``blocks``: list of Blocks (uploaded once per ``to_blocks`` result and
    cached) or a ``DeviceStore``.  ``orders``: one permutation shared by all
    blocks or one per block (None = natural order)."""
    from .store import DeviceStore, to_device
    import torch
    topk = TopK(params.k)
    if isinstance(blocks, DeviceStore):
        store = blocks
    else:
        if not blocks:
            return topk
        store = getattr(blocks, "_device_store", None)
        if store is None:
            store = DeviceStore.from_blocks(blocks, group=8)
            try:
                blocks._device_store = store
            except AttributeError:
                pass
    q = np.asarray(query, dtype=np.float32)
    if q.shape != (store.d,):
        raise ValueError(f"query length {q.shape} does not match d={store.d}")
    if store.nblocks == 0:
        return topk
    if store.nbuckets != store.nblocks:
        store = store.per_block_buckets()
    ordt, oqs, oss = _resolve_orders(orders, store.nblocks, store.d)
    want = stats is not None
    res = run_search(store, to_device(q[None, :], torch.float32), params, nseg=store.nblocks,
                     orders=ordt, order_qstride=oqs, order_sstride=oss, stats=want,
                     trace_cap=_trace_cap(store.nblocks, store.d, params.initial_step) if want else 0,
                     timed=want)
    _fill_stats(stats, res)
    return res.topk(0, params.k)


def search_batch(store, queries, params: SearchParams, orders=None, stats=False, trace=False):
    """Batched :func:`search` over a DeviceStore (one bucket per block or
    one bucket for all); returns host arrays."""
    from .store import to_device
    import torch
    Q = to_device(np.asarray(queries, np.float32), torch.float32)
    ordt, oqs, oss = _resolve_orders(orders, store.nblocks, store.d)
    res = run_search(store, Q, params, nseg=store.nbuckets, orders=ordt, order_qstride=oqs,
                     order_sstride=oss, stats=stats or trace,
                     trace_cap=_trace_cap(store.nblocks, store.d, params.initial_step) if trace else 0)
    return res.host()


def pruning_power_trace(blocks, query, params: SearchParams, orders=None) -> SearchStats:
    """search.py:208-213."""
    stats = SearchStats()
    search(blocks, query, params, orders=orders, stats=stats)
    return stats
