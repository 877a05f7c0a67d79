"""The owning native index handle (pdx_index_* in include/pdx_b200.h).

``PdxIndex`` is the boundary a non-Python caller binds:
create it from host blocks, a .pdx file or an already resident index, then
``search`` a whole query batch in ONE library call — projection, bucket
selection, orders and the pruned scan run inside the library, with the
host<->device copies at its ends.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .kernels import Metric


class PdxIndex:
    def __init__(self, handle: C.c_void_p, d: int, nlist: int, keep=()):
        self._h = handle
        self.d = int(d)
        self.nlist = int(nlist)
        self._keep = keep  # objects whose device memory the handle borrows
        self._pcache = {}  # PdxQueryParams of repeated calls (search)

    # ------------------------------------------------------------ creation
    @classmethod
    def open(cls, path, group: int = 8) -> "PdxIndex":
        """pdx_index_open: a .pdx file straight into HBM."""
        from .storage import probe
        info = probe(path)
        h = C.c_void_p()
        _lib.check(_lib.lib().pdx_index_open(str(path).encode(), int(group), C.byref(h)))
        return cls(h, info["d"], info["nlist"])

    @classmethod
    def from_blocks(cls, blocks, global_means=None, rotation=None, nlist=0, centroids=None,
                    bucket_offsets=None, bucket_means=None, group: int = 8) -> "PdxIndex":
        """pdx_index_create from host Blocks (the reference's list[Block])."""
        d = blocks[0].d if blocks else int(np.asarray(global_means).shape[0])
        imgs = np.ascontiguousarray(np.concatenate([np.asarray(b.data, np.float32).ravel()
                                                    for b in blocks]) if blocks else
                                    np.zeros(1, np.float32))
        bm = np.asarray([b.m for b in blocks] or [0], np.int32)
        bmp = np.asarray([b.data.shape[1] for b in blocks] or [0], np.int32)
        ids = np.ascontiguousarray(np.concatenate([np.asarray(b.ids, np.int64) for b in blocks])
                                   if blocks else np.zeros(1, np.int64))
        gm = None if global_means is None else np.ascontiguousarray(global_means, np.float64)
        rot = None if rotation is None else np.ascontiguousarray(rotation, np.float32)
        cen = None if centroids is None else np.ascontiguousarray(centroids, np.float32)
        off = None if bucket_offsets is None else np.ascontiguousarray(bucket_offsets, np.int64)
        bme = None if bucket_means is None else np.ascontiguousarray(bucket_means, np.float64)
        desc = _lib.PdxIndexDesc(None, d, int(group), len(blocks), _lib.ptr(imgs), _lib.ptr(bm),
                                 _lib.ptr(bmp), _lib.ptr(ids), _lib.ptr(gm), _lib.ptr(rot),
                                 int(nlist), _lib.ptr(cen), _lib.ptr(off), _lib.ptr(bme))
        h = C.c_void_p()
        _lib.check(_lib.lib().pdx_index_create(C.byref(desc), C.byref(h)))
        return cls(h, d, nlist)

    @classmethod
    def from_index(cls, index, transform=None) -> "PdxIndex":
        """Borrow the HBM store of an IvfIndex / FlatPartitioning (no copy)."""
        tf = transform if transform is not None else getattr(index, "transform", None)
        rot = None if tf is None else np.ascontiguousarray(tf.matrix, np.float32)
        nlist = int(getattr(index, "nlist", 0))
        gm = getattr(index, "global_means", None)
        gm = None if gm is None else np.ascontiguousarray(gm, np.float64)
        cen = bme = None
        if nlist:
            cen = np.ascontiguousarray(index.centroids, np.float32)
            bme = np.ascontiguousarray(index.means_dev.cpu().numpy(), np.float64)
        desc = _lib.PdxIndexDesc(C.addressof(index.store.c), index.d, 0, 0, None, None,
                                 None, None, _lib.ptr(gm), _lib.ptr(rot), nlist, _lib.ptr(cen),
                                 None, _lib.ptr(bme))
        h = C.c_void_p()
        _lib.check(_lib.lib().pdx_index_create(C.byref(desc), C.byref(h)))
        return cls(h, index.d, nlist, keep=(index,))

    # -------------------------------------------------------------- search
    def search(self, Q, k: int = 10, metric="l2", pruner="none", criteria="sequential",
               nprobe: int = 8, selection_fraction: float = 0.2, initial_step: int = 2,
               epsilon0: float = 2.1, rotate: bool | None = None, bsa=None, stats=False,
               out=None, stream=None, tensor_cores: bool = True):
        """One pdx_index_search call.  Q: host array (numpy / CPU tensor,
        pinned for overlap) or a CUDA tensor; outputs live where Q lives
        (or in ``out`` = dict of preallocated dist/ids[/touched/total])."""
        import torch
        from .pruning import OrderCriteria
        on_dev = isinstance(Q, torch.Tensor) and Q.is_cuda
        if not isinstance(Q, torch.Tensor):
            Q = torch.from_numpy(np.ascontiguousarray(Q, np.float32))
        Q = Q.contiguous()
        nq = int(Q.shape[0])
        if Q.shape[1] != self.d:
            raise ValueError(f"query dimensionality {Q.shape[1]} != {self.d}")
        if out is None:
            kw = {"device": Q.device} if on_dev else {"pin_memory": torch.cuda.is_available()}
            out = {"dist": torch.empty((nq, k), dtype=torch.float32, **kw),
                   "ids": torch.empty((nq, k), dtype=torch.int64, **kw)}
            if stats:
                out["touched"] = torch.empty((nq,), dtype=torch.int64, **kw)
                out["total"] = torch.empty((nq,), dtype=torch.int64, **kw)
        coef = None
        if pruner == "bsa":
            coef = np.ascontiguousarray(bsa.coef, np.float32)
        rot = bool(rotate) if rotate is not None else False
        # (the parameter struct of a repeated call is reused: building it is a
        # measurable part of a 0.5 ms call)
        pkey = (k, metric, pruner, criteria, nprobe, selection_fraction, initial_step, rot,
                epsilon0, on_dev, tensor_cores) if coef is None else None
        p = self._pcache.get(pkey) if pkey is not None else None
        if p is None:
            p = _lib.PdxQueryParams(int(k), _lib.METRIC[Metric(metric).value],
                                    _lib.PRUNER[pruner],
                                    _lib.CRITERIA[OrderCriteria(criteria).value], 0,
                                    int(nprobe) if self.nlist else 0, float(selection_fraction),
                                    int(initial_step), int(rot), float(epsilon0), _lib.ptr(coef),
                                    int(on_dev), int(on_dev), int(bool(tensor_cores)))
            if pkey is not None:
                if len(self._pcache) > 64:
                    self._pcache.clear()
                self._pcache[pkey] = p
        _lib.check(_lib.lib().pdx_index_search(
            self._h, C.byref(p), _lib.ptr(Q), nq, _lib.ptr(out["dist"]), _lib.ptr(out["ids"]),
            _lib.ptr(out.get("touched")), _lib.ptr(out.get("total")),
            _lib.stream_handle(stream) if torch.cuda.is_available() else None))
        return out

    def close(self):
        if self._h:
            _lib.lib().pdx_index_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
