#!/usr/bin/env python
"""C4 batch 1: one query over the whole GPU, exact top-100,
pruner none, split mode (pdx_search_params.splits), IP and L2 — the
streaming split kernel (pdx_linear.cu) against the pruned-scan kernel on the
same ranges (PDX_NO_LINEAR), results compared bit for bit; one JSON line per
(metric, kernel)."""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import paper_2503_04422_b200 as P  # noqa: E402
from bench_configs import mixture  # noqa: E402


def main():
    n, d, k = 2_000_000, 1536, 100
    xq, _ = mixture(n + 16, d, 4096, 4, spread=0.5, centre_scale=1.0, normalize=True)
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
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for metric in ("ip", "l2"):
        params = P.SearchParams(k=k, metric=metric)
        res = {}
        for name, env in (("streaming", None), ("pruned-scan kernel", "1")):
            if env:
                os.environ["PDX_NO_LINEAR"] = env
            else:
                os.environ.pop("PDX_NO_LINEAR", None)
            for splits in ((sms, 2 * sms, 3 * sms) if env is None else (3 * sms,)):
                s = P.ExactSearcher(flat, params, splits=splits)
                for _ in range(2):
                    s.run(q[:1])
                torch.cuda.synchronize()
                ts = []
                for i in range(8):
                    flush.fill_(1)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    r = s.run(q[i:i + 1])
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
                rr = s.run(q[:8], stats=True)
                res[(name, splits)] = rr
                ms_ = float(np.median(ts))
                print(json.dumps({"config": "C4", "metric": metric, "batch": 1, "k": k,
                                  "kernel": name, "splits": splits, "latency_ms": ms_,
                                  "qps": 1e3 / ms_,
                                  "streamed_GBps": 4.0 * n * d / (ms_ / 1e3) / 1e9,
                                  "touched_eq_total": bool(torch.equal(rr.touched, rr.total))}),
                      flush=True)
        a, b = res[("streaming", 3 * sms)], res[("pruned-scan kernel", 3 * sms)]
        print(json.dumps({"config": "C4", "metric": metric, "identical_ids": bool(torch.equal(a.ids, b.ids)),
                          "identical_dist": bool(torch.equal(a.dist, b.dist)),
                          "identical_touched": bool(torch.equal(a.touched, b.touched))}), flush=True)


if __name__ == "__main__":
    main()
