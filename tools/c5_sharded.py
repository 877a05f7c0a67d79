#!/usr/bin/env python
"""C5 (BASELINE configs[4]): 50M x 768 chunk-seeded mixture (16,384 centres,
sigma_j^2 ~ (j+1)^-0.7), seeded rotation, 65,536 buckets, nprobe 256,
10,000 queries, K = 10, ADS and BOND — sharded by row chunk over ranks
(sharded.build_rank_index): rank r generates only chunks r, r + W, ... of
65,536 rows (default_rng([seed, chunk])), rank 0 trains the centroids on a
sample and broadcasts them, each rank packs its members of every bucket,
searches, and one packed all_gather + K7 merge gives the global top-k.

    torchrun --nproc-per-node 8 tools/c5_sharded.py          # the real thing
    python tools/c5_sharded.py --emulate-rank 0 --world 8    # one rank's share on one GPU

With --emulate-rank the process builds exactly the shard rank R of W would
hold and times its search; no collective runs (there is one GPU), so the
line reports the per-rank time, not a whole-job number.  Recall is against
the exact top-10 of the rows this process holds (float64 brute force).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

N, D, NCENT, NLIST, NPROBE, NQ, K = 50_000_000, 768, 16384, 65536, 256, 10_000, 10
ROWS = 65536
SEED = 5


def main():
    import torch
    import torch.distributed as dist

    import paper_2503_04422_b200 as P
    from paper_2503_04422_b200.sharded import build_rank_index, gather_merge
    from paper_2503_04422_b200.synthetic import c5_sigma, mixture_centres, mixture_chunk
    ap = argparse.ArgumentParser()
    ap.add_argument("--emulate-rank", type=int, default=None)
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--n", type=int, default=N)
    ap.add_argument("--nlist", type=int, default=NLIST)
    ap.add_argument("--nprobe", type=int, default=NPROBE)
    ap.add_argument("--nq", type=int, default=NQ)
    ap.add_argument("--train-chunks", type=int, default=4)
    ap.add_argument("--kmeans-iters", type=int, default=10)
    a = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1:
        rank, world = int(os.environ["RANK"]), ws
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    else:
        rank, world = (a.emulate_rank or 0), (a.world if a.emulate_rank is not None else 1)
        torch.cuda.set_device(0)
    nchunks = (a.n + ROWS - 1) // ROWS
    centres = mixture_centres(SEED, NCENT, D)
    sig = c5_sigma(D)

    def chunk(c):
        return mixture_chunk(SEED, c, min(ROWS, a.n - c * ROWS), centres, sig)

    T = P.generate_orthogonal(D, 2)
    t0 = time.perf_counter()
    index, cent = build_rank_index(chunk, nchunks, rank, world, a.nlist, D,
                                   train_chunks=a.train_chunks, seed=0,
                                   max_iters=a.kmeans_iters, transform=T,
                                   rows_per_chunk=lambda c: min(ROWS, a.n - c * ROWS))
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    q = P.apply_transform(T, P.store.to_device(mixture_chunk(SEED, 1 << 30, a.nq, centres, sig)))
    rows_here = int(index.store.tile_ids.ge(0).sum().item())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    # exact top-10 of the rows this rank holds (recall of the local search)
    xs = index.store
    t = xs.tiles
    X = t.permute(0, 2, 1, 3).reshape(-1, t.shape[1] * t.shape[3])[:, :D][xs.tile_ids.reshape(-1) >= 0]
    ids_here = xs.tile_ids.reshape(-1)[xs.tile_ids.reshape(-1) >= 0]
    gt_rows = P.synthetic.ground_truth_device(X.contiguous(), q[:1000], K)[0]
    gt = ids_here[gt_rows].cpu().numpy()
    del X
    out = []
    for pruner in ("ads", "bond"):
        prm = P.SearchParams(k=K, pruner=pruner, ads=P.AdsPruner(d=D))
        s = P.IvfSearcher(index, prm, a.nprobe)
        r = s.run(q, stats=True)
        for _ in range(1):
            s.run(q)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            flush.fill_(1)
            if ws > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rr = s.run(q)
            if ws > 1:
                d_, i_ = gather_merge(rr.dist, rr.ids, K)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t_ms = float(np.median(ts))
        sel_ms = []
        for _ in range(3):  # the bucket-selection part alone (K2)
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s.select(q)
            e1.record()
            torch.cuda.synchronize()
            sel_ms.append(e0.elapsed_time(e1))
        if ws > 1:
            tt = torch.tensor([t_ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_ms = float(tt.item())
        ids = r.ids.cpu().numpy()[:1000]
        rec = float(np.mean([len(set(ids[j]) & set(gt[j])) / K for j in range(1000)]))
        line = {"config": "C5", "n_total": a.n, "d": D, "nlist": a.nlist, "nprobe": a.nprobe,
                "queries": a.nq, "k": K, "pruner": pruner, "world": world, "rank": rank,
                "rows_this_rank": rows_here, "chunks": nchunks, "chunk_rows": ROWS,
                "batch_ms": t_ms, "qps": a.nq / (t_ms / 1e3),
                "selection_ms": float(np.median(sel_ms)),
                "timing": ("whole job: scan + packed all_gather + K7, max over ranks"
                           if ws > 1 else "this rank's scan only (emulated rank; one GPU)"),
                "local_recall_at_10": rec,
                "pruning_power": 1 - r.touched.sum().item() / r.total.sum().item(),
                "algorithmic_GBps": 4 * r.touched.sum().item() / (t_ms / 1e3) / 1e9,
                "build_s": build_s,
                "hbm_GB_peak": torch.cuda.max_memory_allocated() / 1e9}
        out.append(line)
        if rank == 0:
            print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
