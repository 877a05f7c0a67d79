#!/usr/bin/env python
"""Build the bench's C2 index (BASELINE configs[1]) ONCE with the reference's
own k-means, in this container, and commit the result as a fixture.

Both bench arms load it: the GPU arm packs it with
``IvfIndex.from_assignment`` (K1), the reference arm (``bench.py --impl
reference``) packs it in numpy for the C oracle — so neither arm builds an
index with this repo's GPU code, and both search the identical index.

Recipe: ``bench.make_data`` (seeded mixture), rotation
``dimscan.generate_orthogonal(128, 0)`` applied with
``dimscan.apply_transform`` (pruning.py:36-53), then
``dimscan.index.lloyd_kmeans(XR, 1024, seed=0)`` (index.py:27-64; ~5 min on
one core).  Output ``tests/golden/c2_ivf_reference.npz``: centroids float32
[1024][128], assignment uint16 [1M], and a fingerprint of the rotated data
(the box recomputes the rotation with numpy; an assignment is a valid
partition of any data, so a BLAS-dependent last-bit difference would not
invalidate the index, but the fingerprint lets the bench say whether it
occurred).

Run:  PYTHONPATH=/root/reference/pkg/src python tools/make_c2_index.py
"""
from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")


def main():
    import dimscan
    from dimscan.index import lloyd_kmeans

    from bench import D, NLIST, make_data

    X, Q = make_data(1_000_000, 1000)
    T = dimscan.generate_orthogonal(D, 0)
    XR = dimscan.apply_transform(T, X)
    t0 = time.time()
    cent, assign = lloyd_kmeans(XR, NLIST, seed=0)
    secs = time.time() - t0
    out = ROOT / "tests" / "golden" / "c2_ivf_reference.npz"
    np.savez_compressed(
        out, centroids=cent.astype(np.float32), assign=assign.astype(np.uint16),
        rotation=T.matrix, xr_sha=np.frombuffer(hashlib.sha256(XR.tobytes()).digest(), np.uint8),
        kmeans_seconds=np.float64(secs))
    sizes = np.bincount(assign, minlength=NLIST)
    print(f"wrote {out} ({out.stat().st_size / 1e6:.1f} MB); k-means {secs:.0f} s; "
          f"bucket sizes min {sizes.min()} median {int(np.median(sizes))} max {sizes.max()}")


if __name__ == "__main__":
    main()
