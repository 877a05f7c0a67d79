#!/usr/bin/env python
"""One C2 search (the bench's headline step) bracketed by cudaProfilerStart /
Stop, for ncu's per-launch capture (`ncu --profile-from-start off ...`):
warm-up searches first, then exactly one search (K3 projection + K2
selection + the batched pipeline) in the profiled range.

    python tools/one_search.py [--nprobe 32] [--queries 1000]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    import paper_2503_04422_b200 as P
    from paper_2503_04422_b200 import _lib
    ap = argparse.ArgumentParser()
    ap.add_argument("--nprobe", type=int, default=32)
    ap.add_argument("--queries", type=int, default=1000)
    a = ap.parse_args()
    X, Q = bench.make_data(1_000_000, a.queries)
    T = P.generate_orthogonal(128, 0)
    XR = X @ T.matrix.T
    cent, assign, _ = bench.load_fixture(XR)
    index = P.IvfIndex.from_assignment(P.VectorCollection.from_array(XR), cent, assign,
                                       nlist=1024)
    params = P.SearchParams(k=10, pruner="ads", ads=P.AdsPruner(d=128, epsilon0=2.1))
    s = P.IvfSearcher(index, params, a.nprobe)
    Qd = P.store.to_device(Q)
    Tm = P.store.to_device(T.matrix)
    Qr = torch.empty_like(Qd)

    def step():
        _lib.check(_lib.lib().pdx_project(_lib.ptr(Qd), Qd.shape[0], 128, _lib.ptr(Tm),
                                          _lib.ptr(Qr), _lib.stream_handle()))
        return s.run(Qr)
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    r = step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("one search done:", int((r.ids.cpu().numpy() >= 0).sum()), "ids")


if __name__ == "__main__":
    main()
