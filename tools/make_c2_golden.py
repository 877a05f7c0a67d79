#!/usr/bin/env python
"""Golden outputs of the REAL reference on the bench's headline config (C2).

Builds the reference's own ``IvfIndex`` from the committed k-means fixture
(``tests/golden/c2_ivf_reference.npz``, made by tools/make_c2_index.py) with
the reference's packing code (index.py:98-108: ``to_blocks`` of each bucket's
members, ``compute_means``), then runs ``dimscan.ivf_search`` (ADS,
epsilon0 2.1, K 10) on a prefix of the host-rotated queries at nprobe 8, 32
and 128, recording ids, float32 distances, values_touched and
values_total.  ``tests/test_gpu_c2.py`` replays the same queries through the
GPU path and compares bit for bit.

Run (build container only; the reference does not travel):
    PYTHONPATH=/root/reference/pkg/src python tools/make_c2_golden.py [nq]
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")


def reference_index(XR, cent, assign, nlist):
    import dimscan
    from dimscan.index import IvfIndex
    col = dimscan.VectorCollection.from_array(XR)
    buckets, means = [], []
    for c in range(nlist):  # index.py:98-104
        members = np.flatnonzero(assign == c)
        part = dimscan.VectorCollection(data=col.data[members], ids=col.ids[members])
        buckets.append(dimscan.to_blocks(part, 64))
        means.append(dimscan.compute_means(part).means if part.n else cent[c].astype(np.float64))
    chain = dimscan.to_blocks(dimscan.VectorCollection.from_array(cent), 64)
    return IvfIndex(nlist=nlist, centroid_blocks=chain, centroids=cent, buckets=buckets,
                    bucket_means=means, training_seed=0)


def main():
    import dimscan

    from bench import D, EPS, K, NLIST, make_data
    nq = int(sys.argv[1]) if len(sys.argv) > 1 else 48
    X, Q = make_data(1_000_000, 1000)
    T = dimscan.generate_orthogonal(D, 0)
    XR = dimscan.apply_transform(T, X)
    QR = dimscan.apply_transform(T, Q[:nq])
    f = np.load(ROOT / "tests" / "golden" / "c2_ivf_reference.npz")
    index = reference_index(XR, f["centroids"], f["assign"].astype(np.int64), NLIST)
    params = dimscan.SearchParams(k=K, pruner="ads", ads=dimscan.AdsPruner(d=D, epsilon0=EPS))
    out = {"queries": QR}
    for npb in (8, 32, 128):
        ids = np.full((nq, K), -1, np.int64)
        dist = np.full((nq, K), np.inf, np.float32)
        touched = np.zeros(nq, np.int64)
        total = np.zeros(nq, np.int64)
        t0 = time.time()
        for i in range(nq):
            st = dimscan.SearchStats()
            top = dimscan.ivf_search(index, QR[i], params, npb, stats=st)
            items = top.items()
            dist[i, :len(items)] = [d for d, _ in items]
            ids[i, :len(items)] = [v for _, v in items]
            touched[i], total[i] = st.values_touched, st.values_total
        print(f"nprobe {npb}: {nq} queries in {time.time() - t0:.0f} s")
        out[f"ids_{npb}"], out[f"dist_{npb}"] = ids, dist
        out[f"touched_{npb}"], out[f"total_{npb}"] = touched, total
    dst = ROOT / "tests" / "golden" / "c2_reference_prefix.npz"
    np.savez_compressed(dst, **out)
    print(f"wrote {dst}")


if __name__ == "__main__":
    main()
