"""ctypes front-end of the C oracle (oracle/pdx_oracle.c).

TEST INFRASTRUCTURE ONLY: the parity checker for the B200 path.  Only
tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module; the product package never does.

The oracle restates the reference ``dimscan`` package (pure Python/numpy,
/root/reference/pkg/src/dimscan) in C; this wrapper takes plain numpy
structures (anything with ``.data (d, m_padded) f32``, ``.ids (m,) i64`` and
``.m`` per block, i.e. a reference ``Block`` or the package's own) so that
tests can feed the oracle and the GPU identical inputs.

Pinned against the reference: see tests/golden/make_golden.py and
tests/test_oracle.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libpdx_oracle.so"

METRICS = {"l2": 0, "l1": 1, "ip": 2}
PRUNERS = {"none": 0, "ads": 1, "bond": 2, "bsa": 3}
CRITERIA = {"sequential": 0, "decreasing": 1, "dmeans": 2, "zones": 3}


def build(force: bool = False) -> Path:
    """Compile the oracle with gcc (no FMA contraction: numpy rounds each op)."""
    src = HERE / "pdx_oracle.c"
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.check_call(["make", "-s", "-C", str(HERE)])
    return LIB_PATH


class _Blocks(C.Structure):
    _fields_ = [("d", C.c_int32), ("nblocks", C.c_int64), ("data", C.c_void_p),
                ("data_off", C.c_void_p), ("m", C.c_void_p), ("mp", C.c_void_p),
                ("ids", C.c_void_p), ("id_off", C.c_void_p)]


class _Params(C.Structure):
    _fields_ = [("k", C.c_int32), ("metric", C.c_int32), ("pruner", C.c_int32),
                ("initial_step", C.c_int32), ("selection_fraction", C.c_double),
                ("ads_d", C.c_int32), ("_pad", C.c_int32), ("ads_eps0", C.c_double),
                ("bsa_coef", C.c_void_p)]


class _Stats(C.Structure):
    _fields_ = [("values_touched", C.c_int64), ("values_total", C.c_int64),
                ("survivors", C.c_void_p), ("survivors_cap", C.c_int64),
                ("survivors_len", C.c_int64), ("overflow", C.c_int32), ("_pad", C.c_int32)]


class _Ivf(C.Structure):
    _fields_ = [("nlist", C.c_int32), ("_pad", C.c_int32), ("centroids", C.c_void_p),
                ("buckets", C.c_void_p), ("bucket_off", C.c_void_p),
                ("bucket_means", C.c_void_p)]


class _BatchOut(C.Structure):
    _fields_ = [("dist", C.c_void_p), ("ids", C.c_void_p), ("count", C.c_void_p),
                ("touched", C.c_void_p), ("total", C.c_void_p), ("survivors", C.c_void_p),
                ("surv_cap", C.c_int64), ("surv_len", C.c_void_p), ("selected", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB_PATH))
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.orc_search.argtypes = [vp, vp, i64, vp, vp, vp, vp, vp, vp, vp]
        L.orc_vertical_accumulate.argtypes = [vp, i32, i32, vp, i32, i32, i32, vp, vp]
        L.orc_step_schedule.argtypes = [i32, i32, vp, i32]
        L.orc_step_schedule.restype = i32
        L.orc_ads_bound.argtypes = [i32, i32, C.c_double, C.c_double]
        L.orc_ads_bound.restype = C.c_double
        L.orc_numpy_sum.argtypes = [vp, i64]
        L.orc_numpy_sum.restype = C.c_double
        L.orc_dimension_order.argtypes = [vp, vp, i32, i32, i32, vp]
        L.orc_select_buckets.argtypes = [vp, i32, vp, i32, i32, vp]
        L.orc_ivf_search_batch.argtypes = [vp, vp, i64, vp, i32, i32, i32, vp, i32]
        L.orc_exact_search_batch.argtypes = [vp, vp, vp, i64, vp, i32, i32, vp, i32]
        _lib = L
    return _lib


def _p(a) -> int:
    return a.ctypes.data if a is not None else 0


class BlockList:
    """A packed sequence of dimension-major blocks (reference layout.py:53-83)."""

    def __init__(self, blocks, d: int | None = None):
        blocks = list(blocks)
        if d is None:
            d = int(blocks[0].data.shape[0]) if blocks else 1
        self.d = d
        self.nblocks = len(blocks)
        self.m = np.array([int(b.m) for b in blocks], dtype=np.int32)
        self.mp = np.array([int(b.data.shape[1]) for b in blocks], dtype=np.int32)
        sizes = self.mp.astype(np.int64) * d
        self.data_off = np.zeros(max(1, self.nblocks), dtype=np.int64)
        self.id_off = np.zeros(max(1, self.nblocks), dtype=np.int64)
        if self.nblocks:
            self.data_off[1:self.nblocks] = np.cumsum(sizes)[:-1]
            self.id_off[1:self.nblocks] = np.cumsum(self.m.astype(np.int64))[:-1]
            self.data = np.ascontiguousarray(np.concatenate(
                [np.ascontiguousarray(b.data, dtype=np.float32).ravel() for b in blocks]))
            self.ids = np.ascontiguousarray(np.concatenate(
                [np.asarray(b.ids, dtype=np.int64) for b in blocks]))
        else:
            self.data = np.zeros(1, np.float32)
            self.ids = np.zeros(1, np.int64)
        if self.m.size == 0:
            self.m = np.zeros(1, np.int32)
            self.mp = np.zeros(1, np.int32)
        self.c = _Blocks(d, self.nblocks, _p(self.data), _p(self.data_off), _p(self.m),
                         _p(self.mp), _p(self.ids), _p(self.id_off))


class PackedBlocks:
    """A packed block sequence built straight from arrays (no per-block
    objects): ``data`` float32 [nblocks][d][mp] (dimension-major, padding
    slots zero), ``m`` int [nblocks], ``ids`` int64 [sum(m)] in block order."""

    def __init__(self, data, m, ids):
        data = np.ascontiguousarray(data, dtype=np.float32)
        nb, d, mp = data.shape
        self.d, self.nblocks = int(d), int(nb)
        self.data = data.reshape(-1) if nb else np.zeros(1, np.float32)
        self.m = np.ascontiguousarray(m, dtype=np.int32) if nb else np.zeros(1, np.int32)
        self.mp = np.full(max(1, nb), mp, dtype=np.int32)
        self.data_off = np.arange(max(1, nb), dtype=np.int64) * (d * mp)
        self.id_off = np.zeros(max(1, nb), dtype=np.int64)
        if nb:
            self.id_off[1:] = np.cumsum(self.m.astype(np.int64))[:-1]
        self.ids = np.ascontiguousarray(ids, dtype=np.int64) if nb else np.zeros(1, np.int64)
        self.c = _Blocks(self.d, self.nblocks, _p(self.data), _p(self.data_off), _p(self.m),
                         _p(self.mp), _p(self.ids), _p(self.id_off))


def pack_rows(x, rows, block_size=64):
    """to_blocks (layout.py:93-110) of x[rows] in numpy: consecutive
    block_size-row chunks, transposed to [d][block_size], zero padded.
    Returns (data [nb][d][bs], m [nb], ids = rows)."""
    rows = np.asarray(rows, dtype=np.int64)
    n, d = rows.shape[0], x.shape[1]
    nb = (n + block_size - 1) // block_size
    src = np.full(nb * block_size, -1, dtype=np.int64)
    src[:n] = rows
    g = x[np.maximum(src, 0)].astype(np.float32, copy=True)
    g[src < 0] = 0.0
    data = np.ascontiguousarray(g.reshape(nb, block_size, d).transpose(0, 2, 1))
    m = np.full(nb, block_size, dtype=np.int32)
    if nb and n % block_size:
        m[-1] = n % block_size
    return data, m, rows


def _params(k, metric, pruner, selection_fraction, initial_step, ads_d, eps0, bsa_coef=None):
    beta = None
    if str(pruner) == "bsa":
        if bsa_coef is None:
            raise ValueError("pruner='bsa' needs bsa_coef (one coefficient per schedule step)")
        beta = np.ascontiguousarray(bsa_coef, dtype=np.float32)
    p = _Params(int(k), METRICS[str(metric)], PRUNERS[str(pruner)], int(initial_step),
                float(selection_fraction), int(ads_d), 0, float(eps0), _p(beta))
    p._keep = beta
    return p


def _check(rc):
    if rc == 1:
        raise ValueError("oracle: invalid argument")
    if rc:
        raise MemoryError("oracle: allocation failed")


def step_schedule(d: int, initial_step: int = 2):
    ends = np.zeros(64, np.int32)
    n = lib().orc_step_schedule(d, initial_step, _p(ends), 64)
    if n < 0:
        raise ValueError("bad schedule arguments")
    out, a = [], 0
    for b in ends[:n]:
        out.append((a, int(b)))
        a = int(b)
    return out


def ads_bound(dims_seen: int, d: int, eps0: float, threshold: float) -> float:
    return lib().orc_ads_bound(dims_seen, d, eps0, threshold)


def numpy_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().orc_numpy_sum(_p(a), a.size)


def vertical_accumulate(data, query, dim_range, metric, acc, order=None):
    data = np.ascontiguousarray(data, dtype=np.float32)
    q = np.ascontiguousarray(query, dtype=np.float32)
    order = None if order is None else np.ascontiguousarray(order, dtype=np.int32)
    _check(lib().orc_vertical_accumulate(_p(data), data.shape[0], data.shape[1], _p(q),
                                         dim_range[0], dim_range[1], METRICS[str(metric)],
                                         _p(acc), _p(order)))
    return acc


def dimension_order(query, means, criteria, zone_width=None):
    q = np.ascontiguousarray(query, dtype=np.float64)
    mu = np.ascontiguousarray(means, dtype=np.float64)
    if q.shape != mu.shape:
        raise ValueError("length mismatch")
    out = np.zeros(q.shape[0], np.int32)
    _check(lib().orc_dimension_order(_p(q), _p(mu), q.shape[0], CRITERIA[str(criteria)],
                                     int(zone_width or 0), _p(out)))
    return out


def _decode_survivors(buf, n):
    out, i = [], 0
    while i < n:
        ln = int(buf[i])
        out.append([int(v) for v in buf[i + 1:i + 1 + ln]])
        i += 1 + ln
    return out


def search(blocks, query, k, metric="l2", pruner="none", selection_fraction=0.2,
           initial_step=2, ads_d=None, eps0=2.1, orders=None, survivors_cap=1 << 20,
           bsa_coef=None):
    """search (search.py:177-205).  Returns (items, stats dict)."""
    bl = blocks if isinstance(blocks, (BlockList, PackedBlocks)) else BlockList(blocks)
    q = np.ascontiguousarray(query, dtype=np.float32)
    p = _params(k, metric, pruner, selection_fraction, initial_step,
                ads_d if ads_d is not None else bl.d, eps0, bsa_coef)
    n = bl.nblocks
    ord_arrays, ord_ptrs = [], None
    if orders is not None:
        per_block = isinstance(orders, (list, tuple))
        ord_ptrs = (C.c_void_p * max(1, n))()
        for i in range(n):
            o = orders[i] if per_block else orders
            if o is None:
                ord_ptrs[i] = None
            else:
                a = np.ascontiguousarray(o, dtype=np.int32)
                ord_arrays.append(a)
                ord_ptrs[i] = a.ctypes.data
    dist = np.zeros(k, np.float32)
    ids = np.zeros(k, np.int64)
    cnt = np.zeros(1, np.int32)
    surv = np.zeros(survivors_cap, np.int32)
    st = _Stats(0, 0, _p(surv), survivors_cap, 0, 0, 0)
    _check(lib().orc_search(C.addressof(bl.c), None, n,
                            C.addressof(ord_ptrs) if ord_ptrs is not None else None,
                            _p(q), C.addressof(p), _p(dist), _p(ids), _p(cnt),
                            C.addressof(st)))
    items = [(float(dist[i]), int(ids[i])) for i in range(int(cnt[0]))]
    stats = {"values_touched": st.values_touched, "values_total": st.values_total,
             "survivors": None if st.overflow else _decode_survivors(surv, st.survivors_len)}
    return items, stats


def select_buckets(centroid_blocks, nlist, query, metric, nprobe):
    bl = centroid_blocks if isinstance(centroid_blocks, BlockList) else BlockList(centroid_blocks)
    q = np.ascontiguousarray(query, dtype=np.float32)
    out = np.zeros(nprobe, np.int32)
    _check(lib().orc_select_buckets(C.addressof(bl.c), nlist, _p(q), METRICS[str(metric)],
                                    nprobe, _p(out)))
    return out


class IvfView:
    """Oracle view of an IVF index: centroid chain, bucket chains back to
    back with block offsets, per-bucket float64 means (index.py:75-88)."""

    def __init__(self, centroid_blocks, bucket_chains, bucket_means):
        self.cent = BlockList(centroid_blocks)
        d = self.cent.d
        flat, off = [], [0]
        for chain in bucket_chains:
            flat.extend(chain)
            off.append(off[-1] + len(chain))
        self.buckets = BlockList(flat, d=d)
        self.bucket_off = np.asarray(off, dtype=np.int64)
        self.means = np.ascontiguousarray(np.asarray(bucket_means, dtype=np.float64).reshape(-1, d))
        self.nlist = len(bucket_chains)
        self.c = _Ivf(self.nlist, 0, C.addressof(self.cent.c), C.addressof(self.buckets.c),
                      _p(self.bucket_off), _p(self.means))


    @classmethod
    def from_assignment(cls, x, centroids, assign, nlist=None, block_size=64):
        """The reference's ivf_build packing (index.py:98-108) of given
        centroids and assignments, in numpy: members of each bucket in
        ascending row order, block_size blocks, float64 means
        (layout.py:126-138; an empty bucket takes its centroid)."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        centroids = np.ascontiguousarray(centroids, dtype=np.float32)
        nlist = centroids.shape[0] if nlist is None else int(nlist)
        assign = np.asarray(assign, dtype=np.int64)
        order = np.argsort(assign, kind="stable")
        counts = np.bincount(assign, minlength=nlist)
        off = np.concatenate([[0], np.cumsum(counts)])
        nblk = (counts + block_size - 1) // block_size
        # per-slot source row of every bucket's chain, back to back
        slot = np.full(int(nblk.sum()) * block_size, -1, dtype=np.int64)
        boff = np.concatenate([[0], np.cumsum(nblk)]) * block_size
        for c in np.flatnonzero(counts):
            slot[boff[c]:boff[c] + counts[c]] = order[off[c]:off[c + 1]]
        nb = int(nblk.sum())
        g = x[np.maximum(slot, 0)]
        g[slot < 0] = 0.0
        data = g.reshape(nb, block_size, x.shape[1]).transpose(0, 2, 1)
        m = np.full(nb, block_size, dtype=np.int32)
        last = boff[1:] // block_size - 1
        rem = counts % block_size
        m[last[(counts > 0) & (rem > 0)]] = rem[(counts > 0) & (rem > 0)]
        means = centroids.astype(np.float64).copy()
        for c in np.flatnonzero(counts):
            means[c] = x[order[off[c]:off[c + 1]]].astype(np.float64).sum(axis=0) / counts[c]
        self = cls.__new__(cls)
        cd, cm, cids = pack_rows(centroids, np.arange(nlist), block_size)
        self.cent = PackedBlocks(cd, cm, cids)
        self.buckets = PackedBlocks(data, m, order)
        self.bucket_off = np.concatenate([[0], np.cumsum(nblk)]).astype(np.int64)
        self.means = np.ascontiguousarray(means)
        self.nlist = nlist
        self.c = _Ivf(self.nlist, 0, C.addressof(self.cent.c), C.addressof(self.buckets.c),
                      _p(self.bucket_off), _p(self.means))
        return self


def _batch(nq, k, nprobe, surv_cap):
    out = {"dist": np.zeros((nq, k), np.float32), "ids": np.zeros((nq, k), np.int64),
           "count": np.zeros(nq, np.int32), "touched": np.zeros(nq, np.int64),
           "total": np.zeros(nq, np.int64)}
    if surv_cap:
        out["survivors"] = np.zeros((nq, surv_cap), np.int32)
        out["surv_len"] = np.zeros(nq, np.int64)
    if nprobe:
        out["selected"] = np.zeros((nq, nprobe), np.int32)
    c = _BatchOut(_p(out["dist"]), _p(out["ids"]), _p(out["count"]), _p(out["touched"]),
                  _p(out["total"]), _p(out.get("survivors")), surv_cap,
                  _p(out.get("surv_len")), _p(out.get("selected")))
    return out, c


def _finish(out):
    if "survivors" in out:
        out["survivor_lists"] = [
            None if out["surv_len"][i] < 0 else _decode_survivors(out["survivors"][i],
                                                                 out["surv_len"][i])
            for i in range(out["count"].shape[0])]
    return out


def ivf_search_batch(ivf: IvfView, queries, k, nprobe, metric="l2", pruner="none",
                     criteria="sequential", zone_width=None, selection_fraction=0.2,
                     initial_step=2, ads_d=None, eps0=2.1, nthreads=None, survivors_cap=0,
                     bsa_coef=None):
    Q = np.ascontiguousarray(queries, dtype=np.float32)
    nq = Q.shape[0]
    p = _params(k, metric, pruner, selection_fraction, initial_step,
                ads_d if ads_d is not None else ivf.cent.d, eps0, bsa_coef)
    out, c = _batch(nq, k, nprobe, survivors_cap)
    _check(lib().orc_ivf_search_batch(C.addressof(ivf.c), _p(Q), nq, C.addressof(p), nprobe,
                                      CRITERIA[str(criteria)], int(zone_width or 0),
                                      C.addressof(c), int(nthreads or os.cpu_count() or 1)))
    return _finish(out)


def exact_search_batch(blocks, global_means, queries, k, metric="l2", pruner="none",
                       criteria="sequential", zone_width=None, selection_fraction=0.2,
                       initial_step=2, ads_d=None, eps0=2.1, nthreads=None, survivors_cap=0,
                       bsa_coef=None):
    bl = blocks if isinstance(blocks, (BlockList, PackedBlocks)) else BlockList(blocks)
    Q = np.ascontiguousarray(queries, dtype=np.float32)
    mu = np.ascontiguousarray(global_means, dtype=np.float64)
    nq = Q.shape[0]
    p = _params(k, metric, pruner, selection_fraction, initial_step,
                ads_d if ads_d is not None else bl.d, eps0, bsa_coef)
    out, c = _batch(nq, k, 0, survivors_cap)
    _check(lib().orc_exact_search_batch(C.addressof(bl.c), _p(mu), _p(Q), nq, C.addressof(p),
                                        CRITERIA[str(criteria)], int(zone_width or 0),
                                        C.addressof(c), int(nthreads or os.cpu_count() or 1)))
    return _finish(out)
