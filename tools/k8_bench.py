#!/usr/bin/env python
"""K8 at C4: 2M x 1536 unit-normalised 4,096-centre mixture,
exact top-100, batch of 1,024 queries, IP and L2 — the tcgen05 candidate pass
(pdx_k8_candidates) + exact rescoring, timed with CUDA events (L2 flushed
between reps), split into the two phases, checked bit for bit against the
pruned-scan kernel on a query prefix.  One JSON line per metric.
"""
from __future__ import annotations

import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import paper_2503_04422_b200 as P  # noqa: E402
from bench_configs import mixture  # noqa: E402
from paper_2503_04422_b200 import _lib  # noqa: E402


def main():
    n, d, k, nq = 2_000_000, 1536, 100, 1024
    xq, _ = mixture(n + nq, d, 4096, 4, spread=0.5, centre_scale=1.0, normalize=True)
    x, q = xq[:n].contiguous(), xq[n:].contiguous()
    del xq
    ids = torch.arange(n, dtype=torch.int64, device="cuda")
    nb = (n + 63) // 64
    ms = np.full(nb, 64, np.int64)
    ms[-1] = n - 64 * (nb - 1)
    store = P.DeviceStore.pack(x, ids, ms, np.array([nb], np.int64), ids=ids, group=8)
    flat = P.FlatPartitioning(store=store, global_means=P.store.segment_means_rows(x),
                              partition_size=64)
    del x
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    L = _lib.lib()
    import os
    prof = bool(os.environ.get("K8_PROF"))
    precs = os.environ.get("K8_PRECISION", "tf32,bf16,auto").split(",")
    for metric, precision in [(m, p) for m in (("ip",) if prof else ("ip", "l2")) for p in precs]:
        params = P.SearchParams(k=k, metric=metric)
        tc = P.TensorCoreExactSearcher(flat, params, precision=precision)
        for _ in range(2):
            tc.run(q)
        torch.cuda.synchronize()
        if prof:  # one candidate pass inside the profiler range
            torch.cuda.cudart().cudaProfilerStart()
            tc.run(q)
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStop()
            return
        tot, cand = [], []
        for _ in range(5):
            flush.fill_(1)
            e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            e[0].record()
            r = tc.run(q)
            e[1].record()
            torch.cuda.synchronize()
            tot.append(e[0].elapsed_time(e[1]))
        # the candidate pass alone
        for _ in range(5):
            flush.fill_(1)
            e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            e[0].record()
            tc._candidates(q, nq, _lib.METRIC[metric], precision != "tf32")
            e[1].record()
            torch.cuda.synchronize()
            cand.append(e[0].elapsed_time(e[1]))
        pre = 64
        ref = P.ExactSearcher(flat, params).run(q[:pre])
        same = bool(torch.equal(r.ids[:pre], ref.ids) and torch.equal(r.dist[:pre], ref.dist))
        t, tcand = float(np.median(tot)), float(np.median(cand))
        flops = 2.0 * nq * n * d
        print(json.dumps({
            "config": "C4", "metric": metric, "batch": nq, "k": k, "n": n, "d": d,
            "precision": precision,
            "path": f"K8: tcgen05 {precision} candidates (fused filter) + exact rescoring",
            "qps": nq / (t / 1e3), "batch_ms": t, "candidate_pass_ms": tcand,
            "rescore_ms": t - tcand,
            "tensor_TFLOPs": flops / (tcand / 1e3) / 1e12,
            "candidates_mean": float(tc.candidates.float().mean().item()),
            "candidates_max": int(tc.candidates.max().item()),
            "fallback_queries": tc.overflow,
            f"identical_to_scan_on_first_{pre}": same}), flush=True)


if __name__ == "__main__":
    main()
