"""K8 — batched exact search with tensor-core candidate generation.

For a batch of queries over a flat store (exact_search, index.py:182-191,
pruner "none", L2 or IP) the dense part Q X^T runs as a TF32 GEMM on the
tensor cores (cuBLAS — a plain library GEMM, chunk by chunk); everything
that decides the result is this package's CUDA: an error bound turns each
approximate score into an interval around the reference's key,
pdx_k8_filter keeps every vector that could still be in the top-k, and
pdx_k8_rescore recomputes those candidates with the scan's exact arithmetic.
The results therefore equal the scan's (and the reference's) bit for bit;
queries whose candidates overflow fall back to the scan.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .index import ExactSearcher, FlatPartitioning
from .kernels import Metric
from .search import SearchParams, SearchResult


class TensorCoreExactSearcher:
    """Exact top-k for query batches over ``part`` via the tensor cores."""

    def __init__(self, part: FlatPartitioning, params: SearchParams, chunk: int = 65536,
                 candidates: int = 4096):
        import torch
        metric = Metric(params.metric)
        if params.pruner != "none" or metric not in (Metric.L2, Metric.IP):
            raise ValueError("the tensor-core path covers exact L2 / IP search (pruner 'none')")
        st = part.store
        self.part, self.params, self.metric = part, params, metric
        self.k = int(params.k)
        self.chunk = int(chunk)
        self.cap = max(int(candidates), self.k)
        # row r = vector r of partition r // partition_size, as pdx_k8_rescore maps it
        t = st.tiles
        rows = t.permute(0, 2, 1, 3).reshape(-1, t.shape[1] * t.shape[3])[:, :st.d]
        self.X = rows[st.tile_ids.reshape(-1) >= 0].contiguous()
        self.n = int(self.X.shape[0])
        self.xn2 = torch.empty(self.n, dtype=torch.float32, device=t.device)
        _lib.check(_lib.lib().pdx_k8_norms(_lib.ptr(self.X), self.n, st.d, _lib.ptr(self.xn2),
                                           _lib.stream_handle()))
        self._fallback = ExactSearcher(part, params)

    def run(self, Q, stats=False):
        import torch
        L = _lib.lib()
        st = self.part.store
        dev = Q.device
        Q = Q.contiguous()
        nq, k, cap = int(Q.shape[0]), self.k, self.cap
        qn2 = torch.empty(nq, dtype=torch.float32, device=dev)
        _lib.check(L.pdx_k8_norms(_lib.ptr(Q), nq, st.d, _lib.ptr(qn2), _lib.stream_handle()))
        prev = torch.full((nq, k), float("inf"), dtype=torch.float32, device=dev)
        nxt = torch.empty_like(prev)
        cand = torch.empty((nq, cap), dtype=torch.int64, device=dev)
        ccount = torch.zeros(nq, dtype=torch.int32, device=dev)
        met = _lib.METRIC[self.metric.value]
        old = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = True
        try:
            for r0 in range(0, self.n, self.chunk):
                Xc = self.X[r0:r0 + self.chunk]
                S = Q @ Xc.T  # TF32 tensor cores, fp32 out
                _lib.check(L.pdx_k8_filter(_lib.ptr(S), S.shape[1], nq, int(S.shape[1]), r0,
                                           _lib.ptr(self.xn2[r0:r0 + Xc.shape[0]]),
                                           _lib.ptr(qn2), met, st.d, k, _lib.ptr(prev),
                                           _lib.ptr(nxt), _lib.ptr(cand), _lib.ptr(ccount), cap,
                                           _lib.stream_handle()))
                prev, nxt = nxt, prev
        finally:
            torch.backends.cuda.matmul.allow_tf32 = old
        dist = torch.empty((nq, k), dtype=torch.float32, device=dev)
        ids = torch.empty((nq, k), dtype=torch.int64, device=dev)
        _lib.check(L.pdx_k8_rescore(st.ref, int(self.part.partition_size), _lib.ptr(Q), nq, met,
                                    k, _lib.ptr(cand), _lib.ptr(ccount), cap, _lib.ptr(dist),
                                    _lib.ptr(ids), _lib.stream_handle()))
        over = torch.nonzero(ccount > cap).flatten()
        self.overflow = int(over.numel())
        if self.overflow:
            fb = self._fallback.run(Q[over])
            dist[over] = fb.dist
            ids[over] = fb.ids
        count = (ids >= 0).sum(1).to(torch.int32)
        touched = total = None
        if stats:  # an exact scan without pruning touches every value
            total = torch.full((nq,), self.n * st.d, dtype=torch.int64, device=dev)
            touched = total.clone()
        self.candidates = ccount
        return SearchResult(dist, ids, count, touched, total)
