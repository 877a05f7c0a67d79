#!/usr/bin/env python
"""Full-size configurations against the C oracle on a query prefix
("oracle only on a query subset"): the GPU answers the
whole batch; the oracle (the reference's algorithm restated in C, pinned to
the reference by tests/golden) answers the first --prefix queries on the
SAME index and the SAME float32 inputs (downloaded from the device); ids,
float32 distances and values_touched are compared bit for bit.

    python tools/oracle_configs.py c3 c4 c5 [--prefix 100]

C3: 1M x 960, 2,048 buckets (this repo's GPU k-means), nprobe 64, ADS on the
    rotated data and BOND on the same index; batched pipeline.
C4: 2M x 1536 unit-normalised, flat 64-blocks, K = 100: BOND (L2) through
    the pruned scan and L2 / IP through K8 (tcgen05 candidates + rescoring).
C5: one rank's shard of 8 (6.3M x 768 of the chunk-seeded 50M collection,
    65,536 buckets, nprobe 256): ADS and BOND.
One JSON line per (config, path).
"""
from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import paper_2503_04422_b200 as P  # noqa: E402
from bench_configs import mixture  # noqa: E402
from oracle import oracle as O  # noqa: E402

PREFIX = 100
THREADS = os.cpu_count() or 1


def host_assign(index):
    a = np.empty(int(np.sum(index._counts)), dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(index._counts)])
    for c in range(index.nlist):
        a[index._order[off[c]:off[c + 1]]] = c
    return a


def compare(name, path, got, ref, extra=None, fast=None):
    """fast: the results-only run of the same searcher (no stats: the
    batched pipeline's verification path), compared too."""
    line = {"config": name, "path": path, "prefix_queries": int(ref["ids"].shape[0]),
            "ids_equal": bool(np.array_equal(got["ids"], ref["ids"])),
            "dist_equal": bool(np.array_equal(got["dist"], ref["dist"])),
            "queries_differing": int(np.sum(np.any(got["ids"] != ref["ids"], axis=1)))}
    if fast is not None:
        line["results_only_ids_equal"] = bool(np.array_equal(fast["ids"], ref["ids"]))
        line["results_only_dist_equal"] = bool(np.array_equal(fast["dist"], ref["dist"]))
    if "touched" in got and got["touched"] is not None:
        line["touched_equal"] = bool(np.array_equal(got["touched"], ref["touched"]))
    line.update(extra or {})
    print(json.dumps(line), flush=True)


def c3():
    n, d, nlist, nprobe, nq, k = 1_000_000, 960, 2048, 64, 1000, 10
    sigma = (torch.arange(d, device="cuda", dtype=torch.float32) + 1) ** -0.5
    xq, _ = mixture(n + nq, d, 1000, 3, centre_scale=2.0, sigma=sigma)
    R = P.generate_orthogonal(d, 1)
    x, q = P.apply_transform(R, xq[:n].contiguous()), P.apply_transform(R, xq[n:].contiguous())
    del xq
    cent, a = P.index.lloyd_kmeans_device(x, nlist, 0)
    xh = x.cpu().numpy()
    ix = P.IvfIndex.from_assignment(P.VectorCollection.from_array(xh), cent.cpu().numpy(), a,
                                    nlist=nlist, x_dev=x)
    view = O.IvfView.from_assignment(xh, ix.centroids, host_assign(ix), nlist)
    qh = q.cpu().numpy()[:PREFIX]
    for pruner in ("ads", "bond"):
        prm = P.SearchParams(k=k, pruner=pruner, ads=P.AdsPruner(d=d))
        sr = P.IvfSearcher(ix, prm, nprobe)
        r = sr.run(q, stats=True)
        got = {"ids": r.ids.cpu().numpy()[:PREFIX], "dist": r.dist.cpu().numpy()[:PREFIX],
               "touched": r.touched.cpu().numpy()[:PREFIX]}
        r0 = sr.run(q)
        fast = {"ids": r0.ids.cpu().numpy()[:PREFIX], "dist": r0.dist.cpu().numpy()[:PREFIX]}
        t0 = time.perf_counter()
        ref = O.ivf_search_batch(view, qh, k, nprobe, pruner=pruner, nthreads=THREADS)
        compare("C3 1M x 960, nlist 2048, nprobe 64", f"batched pipeline, {pruner}", got, ref,
                {"oracle_s": round(time.perf_counter() - t0, 1), "gpu_batch_queries": nq}, fast)


def c4():
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
    xh = x.cpu().numpy()
    del x
    # the oracle's 64-blocks, transposed chunk by chunk (host memory: 2 copies)
    data = np.zeros((nb, d, 64), np.float32)
    for b0 in range(0, nb, 4096):
        b1 = min(nb, b0 + 4096)
        r1 = min(n, b1 * 64)
        blk = np.zeros(((b1 - b0) * 64, d), np.float32)
        blk[:r1 - b0 * 64] = xh[b0 * 64:r1]
        data[b0:b1] = blk.reshape(b1 - b0, 64, d).transpose(0, 2, 1)
    del xh
    m = ms.astype(np.int32)
    blocks = O.PackedBlocks(data, m, np.arange(n, dtype=np.int64))
    mu = flat.global_means
    qh = q.cpu().numpy()[:PREFIX]
    r = P.ExactSearcher(flat, P.SearchParams(k=k, pruner="bond")).run(q[:PREFIX], stats=True)
    got = {"ids": r.ids.cpu().numpy(), "dist": r.dist.cpu().numpy(),
           "touched": r.touched.cpu().numpy()}
    t0 = time.perf_counter()
    ref = O.exact_search_batch(blocks, mu, qh, k, pruner="bond", nthreads=THREADS)
    compare("C4 2M x 1536 exact, K 100", "pruned scan, L2 BOND", got, ref,
            {"oracle_s": round(time.perf_counter() - t0, 1)})
    for metric in ("l2", "ip"):
        tc = P.TensorCoreExactSearcher(flat, P.SearchParams(k=k, metric=metric))
        r = tc.run(q)  # the whole 1,024-query batch through tcgen05
        got = {"ids": r.ids.cpu().numpy()[:PREFIX], "dist": r.dist.cpu().numpy()[:PREFIX]}
        t0 = time.perf_counter()
        ref = O.exact_search_batch(blocks, mu, qh, k, metric=metric, pruner="none",
                                   nthreads=THREADS)
        compare("C4 2M x 1536 exact, K 100", f"K8 tcgen05 batch 1024, {metric}", got, ref,
                {"oracle_s": round(time.perf_counter() - t0, 1),
                 "candidates_mean": float(tc.candidates.float().mean().item())})


def c5():
    from paper_2503_04422_b200.sharded import build_rank_index
    from paper_2503_04422_b200.synthetic import c5_sigma, mixture_centres, mixture_chunk
    N, D, nlist, nprobe, rows = 50_000_000, 768, 65536, 256, 65536
    centres, sig = mixture_centres(5, 16384, D), c5_sigma(D)
    nchunks = (N + rows - 1) // rows

    def chunk(c):
        return mixture_chunk(5, c, min(rows, N - c * rows), centres, sig)
    T = P.generate_orthogonal(D, 2)
    ix, cent = build_rank_index(chunk, nchunks, 0, 8, nlist, D, train_chunks=4, transform=T,
                                rows_per_chunk=lambda c: min(rows, N - c * rows))
    q = P.apply_transform(T, P.store.to_device(mixture_chunk(5, 1 << 30, 2000, centres, sig)))
    st = ix.store
    t = st.tiles
    valid = st.tile_ids.reshape(-1) >= 0
    X = t.permute(0, 2, 1, 3).reshape(-1, t.shape[1] * t.shape[3])[:, :D][valid].cpu().numpy()
    gid = st.tile_ids.reshape(-1)[valid].cpu().numpy()
    # the store's rows in tile order are the buckets' members in order: rebuild the view
    bucket_of_tile = np.repeat(np.arange(nlist), np.diff(st.bucket_block.cpu().numpy()))
    tile_bucket = bucket_of_tile  # 64-blocks: one tile per block
    slot_bucket = np.repeat(tile_bucket, 64)[valid.cpu().numpy()]
    view = O.IvfView.from_assignment(X, cent.cpu().numpy(), slot_bucket, nlist)
    view.buckets.ids[:] = gid[view.buckets.ids]
    qh = q.cpu().numpy()[:PREFIX]
    for pruner in ("ads", "bond"):
        prm = P.SearchParams(k=10, pruner=pruner, ads=P.AdsPruner(d=D))
        sr = P.IvfSearcher(ix, prm, nprobe)
        r = sr.run(q, stats=True)
        got = {"ids": r.ids.cpu().numpy()[:PREFIX], "dist": r.dist.cpu().numpy()[:PREFIX],
               "touched": r.touched.cpu().numpy()[:PREFIX]}
        r0 = sr.run(q)
        fast = {"ids": r0.ids.cpu().numpy()[:PREFIX], "dist": r0.dist.cpu().numpy()[:PREFIX]}
        t0 = time.perf_counter()
        ref = O.ivf_search_batch(view, qh, 10, nprobe, pruner=pruner, nthreads=THREADS)
        compare("C5 rank 0 of 8 (6.3M x 768 of 50M, nlist 65536, nprobe 256)",
                f"batched pipeline, {pruner}", got, ref,
                {"oracle_s": round(time.perf_counter() - t0, 1), "gpu_batch_queries": 2000}, fast)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    if "--prefix" in sys.argv:
        PREFIX = int(sys.argv[sys.argv.index("--prefix") + 1])
        args = [a for a in args if a != str(PREFIX)]
    O.build()
    for name in args or ["c3"]:
        {"c3": c3, "c4": c4, "c5": c5}[name]()
        torch.cuda.empty_cache()
