"""K8 — batched exact search with tensor-core candidate generation.

For a batch of queries over a flat store (exact_search, index.py:182-191,
pruner "none", L2 or IP) the dense part Q X^T runs on the 5th-generation
tensor cores in this library's own kernel (csrc/pdx_k8tc.cu: tcgen05.mma
kind::tf32, TMEM accumulators, TMA-staged operands) with the candidate
filter fused into the TMEM epilogue: an error bound turns each approximate
score into an interval around the reference's key, and a vector stays a
candidate only while its interval can still reach the top-k
(pdx_k8_candidates); pdx_k8_rescore recomputes the candidates with the
scan's exact arithmetic.  The results therefore equal the scan's (and the
reference's) bit for bit; queries whose candidates overflow fall back to
the scan.
"""
from __future__ import annotations

import ctypes as C


from . import _lib
from .index import ExactSearcher, FlatPartitioning
from .kernels import Metric
from .search import SearchParams, SearchResult


class TensorCoreExactSearcher:
    """Exact top-k for query batches over ``part`` via the tensor cores."""

    def __init__(self, part: FlatPartitioning, params: SearchParams, candidates: int = 4096,
                 precision: str = "tf32"):
        """precision: "tf32" (kind::tf32 operands), "bf16" (kind::f16 with bf16
        operands: twice the MMA rate, a wider interval, more candidates) or
        "auto" (bf16, and the tf32 pass for any query whose bf16 candidates
        overflow).  Results are exact in every mode."""
        import torch
        metric = Metric(params.metric)
        if params.pruner != "none" or metric not in (Metric.L2, Metric.IP):
            raise ValueError("the tensor-core path covers exact L2 / IP search (pruner 'none')")
        st = part.store
        self.part, self.params, self.metric = part, params, metric
        self.k = int(params.k)
        self.cap = max(int(candidates), self.k)
        self.d = st.d
        self.ld = (st.d + 3) // 4 * 4  # TMA rows: 16-byte multiples, zero padded
        # row r = vector r of partition r // partition_size, as pdx_k8_rescore maps it
        t = st.tiles
        rows = t.permute(0, 2, 1, 3).reshape(-1, t.shape[1] * t.shape[3])[:, :self.ld]
        valid = st.tile_ids.reshape(-1) >= 0
        X = rows[valid]
        self.rowids = st.tile_ids.reshape(-1)[valid].contiguous()
        if X.shape[1] < self.ld:
            X = torch.nn.functional.pad(X, (0, self.ld - X.shape[1]))
        X[:, st.d:] = 0
        self.X = X.contiguous()
        self.n = int(self.X.shape[0])
        self.xn2 = torch.empty(self.n, dtype=torch.float32, device=t.device)
        _lib.check(_lib.lib().pdx_k8_norms_ld(_lib.ptr(self.X), self.n, st.d, self.ld,
                                              _lib.ptr(self.xn2), _lib.stream_handle()))
        if precision not in ("tf32", "bf16", "auto"):
            raise ValueError(f"unknown precision {precision!r}")
        self.precision = precision
        self.ld16 = (st.d + 7) // 8 * 8
        self.X16 = None
        if precision != "tf32":
            self.X16 = torch.empty((self.n, self.ld16), dtype=torch.bfloat16, device=t.device)
            _lib.check(_lib.lib().pdx_k8_to_bf16(_lib.ptr(self.X), self.n, st.d, self.ld, self.ld16,
                                                 _lib.ptr(self.X16), _lib.stream_handle()))
        self._fallback = ExactSearcher(part, params)
        self._work = None

    def _candidates(self, Qp, nq, met, bf16):
        import torch
        L = _lib.lib()
        k, cap = self.k, self.cap
        cand = torch.empty((nq, cap), dtype=torch.int64, device=Qp.device)
        ccount = torch.zeros(nq, dtype=torch.int32, device=Qp.device)
        wb = C.c_int64(0)
        if bf16:
            Q16 = torch.empty((nq, self.ld16), dtype=torch.bfloat16, device=Qp.device)
            _lib.check(L.pdx_k8_to_bf16(_lib.ptr(Qp), nq, self.d, self.ld, self.ld16, _lib.ptr(Q16),
                                        _lib.stream_handle()))
            args = (_lib.ptr(self.X16), self.n, self.d, self.ld16, _lib.ptr(self.xn2),
                    _lib.ptr(Q16), _lib.ptr(Qp), self.ld, nq, met, k, _lib.ptr(cand),
                    _lib.ptr(ccount), cap)
            fn = L.pdx_k8_candidates_bf16
        else:
            args = (_lib.ptr(self.X), self.n, self.d, self.ld, _lib.ptr(self.xn2), _lib.ptr(Qp),
                    nq, met, k, _lib.ptr(cand), _lib.ptr(ccount), cap)
            fn = L.pdx_k8_candidates
        _lib.check(fn(*args, None, C.cast(C.pointer(wb), C.c_void_p), _lib.stream_handle()))
        if self._work is None or self._work.numel() < wb.value:
            self._work = torch.empty(max(1, wb.value), dtype=torch.uint8, device=Qp.device)
        _lib.check(fn(*args, _lib.ptr(self._work), C.cast(C.pointer(wb), C.c_void_p),
                      _lib.stream_handle()))
        return cand, ccount

    def run(self, Q, stats=False):
        import torch
        L = _lib.lib()
        st = self.part.store
        dev = Q.device
        Q = Q.contiguous()
        nq, k, cap = int(Q.shape[0]), self.k, self.cap
        Qp = Q if self.ld == self.d else torch.nn.functional.pad(Q, (0, self.ld - self.d))
        Qp = Qp.contiguous()
        met = _lib.METRIC[self.metric.value]
        cand, ccount = self._candidates(Qp, nq, met, self.precision != "tf32")
        if self.precision == "auto":  # bf16 overflow: those queries through the tf32 pass
            over = torch.nonzero(ccount > cap).flatten()
            if over.numel():
                c2, n2 = self._candidates(Qp[over].contiguous(), int(over.numel()), met, False)
                cand[over] = c2
                ccount[over] = n2
        dist = torch.empty((nq, k), dtype=torch.float32, device=dev)
        ids = torch.empty((nq, k), dtype=torch.int64, device=dev)
        cmax = min(int(ccount.max().item()) if nq else 0, cap)
        _lib.check(L.pdx_k8_rescore_rows(_lib.ptr(self.X), self.ld, self.d, _lib.ptr(self.rowids),
                                         _lib.ptr(Qp), nq, met, k, _lib.ptr(cand),
                                         _lib.ptr(ccount), cap, max(cmax, 1), _lib.ptr(dist),
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
