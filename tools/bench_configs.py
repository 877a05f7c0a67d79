"""Measure the larger SURVEY.md §8(d) configurations (bench.py runs C2).

    python tools/bench_configs.py c3        # 1M x 960, IVF 2048, nprobe 64: BSA and ADS
    python tools/bench_configs.py c4        # 2M x 1536 exact: batch 1 (split mode) and batched
    python tools/bench_configs.py c1        # 100K x 128 exact, BOND orders, vs the C oracle

Synthetic data with the recipes' shapes and distributions, generated on the
GPU with seeded torch generators (the datasets are not in the image).  Each
line is JSON: throughput from CUDA events with inputs resident in HBM, recall
against the float64 GPU brute force, pruning power from the kernel's exact
values_touched accounting.
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2503_04422_b200 as P  # noqa: E402

import os  # noqa: E402

# pdx_search_params.batched for the IVF configs: 0 auto (the batched pipeline
# for batches of 32+ queries), 1 the per-query scan, 2 batched whenever eligible
BATCHED = int(os.environ.get("PDX_CFG_BATCHED", "0"))


def same_as_per_query(ix, params, nprobe, q, r):
    """The per-query scan on the same batch: identical ids, distances and
    values_touched (the batched pipeline's exactness, at full size)."""
    r1 = P.IvfSearcher(ix, params, nprobe, batched=1).run(q, stats=True)
    return bool(torch.equal(r1.ids, r.ids) and torch.equal(r1.dist, r.dist)
                and torch.equal(r1.touched, r.touched))


def mixture(n, d, centres, seed, spread=1.0, centre_scale=2.0, sigma=None, normalize=False,
            device="cuda"):
    g = torch.Generator(device=device).manual_seed(seed)
    c = torch.randn((centres, d), generator=g, device=device) * centre_scale
    lab = torch.randint(0, centres, (n,), generator=g, device=device)
    x = c[lab] + spread * torch.randn((n, d), generator=g, device=device)
    if sigma is not None:
        x = x * sigma
    if normalize:
        x = x / x.norm(dim=1, keepdim=True)
    return x.contiguous(), c


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return float(np.median(ts))


def recall(gt_ids, ids, k):
    return float(np.mean([len(set(gt_ids[i, :k].tolist()) & set(ids[i, :k].tolist())) / k
                          for i in range(gt_ids.shape[0])]))


def c3():
    n, d, nlist, nprobe, nq, k = 1_000_000, 960, 2048, 64, 1000, 10
    sigma = (torch.arange(d, device="cuda", dtype=torch.float32) + 1) ** -0.5
    xq, _ = mixture(n + nq, d, 1000, 3, centre_scale=2.0, sigma=sigma)
    x, q = xq[:n].contiguous(), xq[n:].contiguous()
    R = P.generate_orthogonal(d, 1)
    x = P.apply_transform(R, x)
    q = P.apply_transform(R, q)
    gt, _ = P.synthetic.ground_truth_device(x, q, k)
    gt = gt.cpu().numpy()
    out = []
    # ADS on the rotated data
    t0 = time.perf_counter()
    ix = P.ivf_build(P.VectorCollection.from_array(x.cpu().numpy()), nlist=nlist, seed=0, x_dev=x)
    build_s = time.perf_counter() - t0
    prm = P.SearchParams(k=k, pruner="ads", ads=P.AdsPruner(d=d))
    s = P.IvfSearcher(ix, prm, nprobe, batched=BATCHED)
    r = s.run(q, stats=True)
    pp = 1 - r.touched.sum().item() / r.total.sum().item()
    sec = timed(lambda: s.run(q))
    out.append({"config": "C3", "pruner": "ads", "batched": BATCHED,
                "same_as_per_query": same_as_per_query(ix, prm, nprobe, q, r),
                "n": n, "d": d, "nlist": nlist, "nprobe": nprobe,
                "queries": nq, "k": k, "qps": nq / sec, "scan_batch_s": sec,
                "recall_at_10": recall(gt, r.ids.cpu().numpy(), k), "pruning_power": pp,
                "algorithmic_GBps": 4 * r.touched.sum().item() / sec / 1e9,
                "index_build_s": build_s})
    del ix, s
    # BSA on the principal axes
    T = P.fit_pca(x, seed=0)
    xp = P.apply_transform(T, x)
    qp = P.apply_transform(T, q)
    ix = P.ivf_build(P.VectorCollection.from_array(xp.cpu().numpy()), nlist=nlist, seed=0, x_dev=xp)
    bsa = P.fit_bsa(xp)
    prm = P.SearchParams(k=k, pruner="bsa", bsa=bsa)
    s = P.IvfSearcher(ix, prm, nprobe, batched=BATCHED)
    r = s.run(qp, stats=True)
    pp = 1 - r.touched.sum().item() / r.total.sum().item()
    sec = timed(lambda: s.run(qp))
    out.append({"config": "C3", "pruner": "bsa", "batched": BATCHED,
                "same_as_per_query": same_as_per_query(ix, prm, nprobe, qp, r),
                "n": n, "d": d, "nlist": nlist,
                "nprobe": nprobe, "queries": nq, "k": k, "qps": nq / sec, "scan_batch_s": sec,
                "recall_at_10": recall(gt, r.ids.cpu().numpy(), k), "pruning_power": pp,
                "algorithmic_GBps": 4 * r.touched.sum().item() / sec / 1e9,
                "bsa_cosine_quantiles": [round(c, 4) for c in bsa.cosines]})
    s = P.IvfSearcher(ix, P.SearchParams(k=k, pruner="bond"), nprobe, batched=BATCHED)
    r = s.run(qp, stats=True)
    sec = timed(lambda: s.run(qp))
    out.append({"config": "C3", "pruner": "bond (same PCA index)", "batched": BATCHED,
                "qps": nq / sec,
                "recall_at_10": recall(gt, r.ids.cpu().numpy(), k),
                "pruning_power": 1 - r.touched.sum().item() / r.total.sum().item()})
    return out


def c4():
    n, d, k = 2_000_000, 1536, 100
    xq, _ = mixture(n + 1024, d, 4096, 4, spread=0.5, centre_scale=1.0, normalize=True)
    x, q = xq[:n].contiguous(), xq[n:].contiguous()
    out = []
    ids = torch.arange(n, dtype=torch.int64, device="cuda")
    order = torch.arange(n, dtype=torch.int64, device="cuda")
    nb = (n + 63) // 64
    ms = np.full(nb, 64, np.int64)
    ms[-1] = n - 64 * (nb - 1)
    store = P.DeviceStore.pack(x, order, ms, np.array([nb], np.int64), ids=ids, group=8)
    flat = P.FlatPartitioning(store=store, global_means=P.store.segment_means_rows(x),
                              partition_size=64)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for metric, pruner in (("ip", "none"), ("l2", "none"), ("l2", "bond")):
        gt, _ = P.synthetic.ground_truth_device(x, q[:8], 10, P.Metric(metric))
        params = P.SearchParams(k=k, metric=metric, pruner=pruner)
        # batch 1: one query over the whole GPU (split mode)
        s1 = P.ExactSearcher(flat, params, splits=3 * sms)
        lat = [timed(lambda i=i: s1.run(q[i:i + 1]), reps=3, warm=1) for i in range(8)]
        r1 = s1.run(q[:8], stats=True)
        out.append({"config": "C4", "metric": metric, "pruner": pruner, "batch": 1, "k": k,
                    "splits": 3 * sms, "latency_ms": 1e3 * float(np.mean(lat)),
                    "qps": 1 / float(np.mean(lat)),
                    "algorithmic_GBps": 4 * n * d / float(np.mean(lat)) / 1e9
                    * (r1.touched.sum().item() / r1.total.sum().item()),
                    "recall_at_10_of_100": recall(gt.cpu().numpy(), r1.ids.cpu().numpy(), 10),
                    "pruning_power": 1 - r1.touched.sum().item() / r1.total.sum().item()})
        # batched: 256 queries, one CTA each
        nb_q = 256
        sb = P.ExactSearcher(flat, params)
        sec = timed(lambda: sb.run(q[:nb_q]), reps=2, warm=1)
        rb = sb.run(q[:nb_q], stats=True)
        out.append({"config": "C4", "metric": metric, "pruner": pruner, "batch": nb_q, "k": k,
                    "qps": nb_q / sec, "batch_s": sec,
                    "algorithmic_GBps": 4 * rb.touched.sum().item() / sec / 1e9,
                    "pruning_power": 1 - rb.touched.sum().item() / rb.total.sum().item()})
        if pruner == "none":  # K8: tensor-core candidates + exact rescoring, batch 1024
            tc = P.TensorCoreExactSearcher(flat, params)
            sec = timed(lambda: tc.run(q), reps=3, warm=1)
            rt = tc.run(q)
            same = bool((rt.ids[:nb_q] == rb.ids).all().item() and
                        (rt.dist[:nb_q] == rb.dist).all().item())
            flops = 2.0 * 1024 * n * d
            out.append({"config": "C4", "metric": metric, "pruner": pruner, "batch": 1024, "k": k,
                        "path": "K8 TF32 tensor-core candidates + exact rescoring",
                        "qps": 1024 / sec, "batch_s": sec, "gemm_TFLOPs_effective": flops / sec / 1e12,
                        "candidates_mean": float(tc.candidates.float().mean().item()),
                        "candidates_max": int(tc.candidates.max().item()),
                        "fallback_queries": tc.overflow,
                        "identical_to_scan_on_first_256": same})
    return out


def c5(n=10_000_000, d=768, nlist=8192, nprobe=128, nq=10_000, k=10):
    """C5's recipe scaled to one GPU (the sharded run splits buckets the same
    way per GPU): sigma_j^2 ~ (j+1)^-0.7, 16,384 centres, seeded rotation,
    k-means on a 500K sample then one assignment pass, ADS and BOND."""
    from types import SimpleNamespace
    from paper_2503_04422_b200.index import IvfIndex, _argmin_chunked, lloyd_kmeans_device
    sigma = (torch.arange(d, device="cuda", dtype=torch.float32) + 1) ** -0.35
    xq, _ = mixture(n + nq, d, 16384, 5, centre_scale=2.0, sigma=sigma)
    R = P.generate_orthogonal(d, 2)
    for r0 in range(0, n + nq, 1 << 20):  # rotate in place, chunk by chunk
        xq[r0:r0 + (1 << 20)] = P.apply_transform(R, xq[r0:r0 + (1 << 20)])
    x, q = xq[:n], xq[n:].contiguous()
    t0 = time.perf_counter()
    g = torch.Generator(device="cpu").manual_seed(0)
    sample = x[torch.randperm(n, generator=g)[:500_000].cuda()].contiguous()
    cent, _ = lloyd_kmeans_device(sample, nlist, 0, max_iters=10)
    del sample
    assign = _argmin_chunked(x, cent, chunk=1 << 16)
    col = SimpleNamespace(ids=np.arange(n, dtype=np.int64), data=None, n=n, d=d)
    ix = IvfIndex.from_assignment(col, cent.cpu().numpy(), assign, nlist=nlist, x_dev=x)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    gt, _ = P.synthetic.ground_truth_device(x, q, k)
    gt = gt.cpu().numpy()
    out = []
    for pruner in ("ads", "bond"):
        prm = P.SearchParams(k=k, pruner=pruner, ads=P.AdsPruner(d=d))
        s = P.IvfSearcher(ix, prm, nprobe, batched=BATCHED)
        r = s.run(q, stats=True)
        sec = timed(lambda: s.run(q), reps=3, warm=1)
        out.append({"config": "C5-scaled (1 GPU)", "batched": BATCHED,
                    "same_as_per_query": same_as_per_query(ix, prm, nprobe, q, r),
                    "n": n, "d": d, "nlist": nlist,
                    "nprobe": nprobe, "queries": nq, "k": k, "pruner": pruner,
                    "qps": nq / sec, "batch_s": sec,
                    "recall_at_10": recall(gt, r.ids.cpu().numpy(), k),
                    "pruning_power": 1 - r.touched.sum().item() / r.total.sum().item(),
                    "algorithmic_GBps": 4 * r.touched.sum().item() / sec / 1e9,
                    "index_build_s": build_s, "hbm_GB_used": torch.cuda.max_memory_allocated() / 1e9})
    return out


def c1():
    n, d, k, nq = 100_000, 128, 10, 100
    rng = np.random.default_rng(0)
    sig = (np.arange(d) + 1) ** -0.5
    X = (rng.standard_normal((n, d)) * sig).astype(np.float32)
    Q = (rng.standard_normal((nq, d)) * sig).astype(np.float32)
    col = P.VectorCollection.from_array(X)
    out = []
    for pruner, crit in (("none", "sequential"), ("bond", "sequential"), ("bond", "dmeans"),
                         ("bond", "zones")):
        flat = P.flat_build(col, 64, group=1 if crit != "sequential" else 8)
        s = P.ExactSearcher(flat, P.SearchParams(k=k, pruner=pruner), crit)
        Qd = P.store.to_device(Q)
        r = s.run(Qd, stats=True)
        sec = timed(lambda: s.run(Qd))
        out.append({"config": "C1", "pruner": pruner, "criteria": crit, "queries": nq,
                    "qps": nq / sec, "pruning_power":
                    1 - r.touched.sum().item() / r.total.sum().item()})
        # throughput mode: each query's blocks over 8 CTAs (exact results, own stats)
        s8 = P.ExactSearcher(flat, P.SearchParams(k=k, pruner=pruner), crit, splits=8)
        r8 = s8.run(Qd, stats=True)
        same = bool((r8.ids == r.ids).all().item() and (r8.dist == r.dist).all().item())
        sec8 = timed(lambda: s8.run(Qd))
        out.append({"config": "C1", "pruner": pruner, "criteria": crit, "queries": nq,
                    "splits": 8, "qps": nq / sec8, "same_results": same,
                    "pruning_power": 1 - r8.touched.sum().item() / r8.total.sum().item()})
    return out


if __name__ == "__main__":
    for name in sys.argv[1:] or ["c1"]:
        for line in {"c1": c1, "c3": c3, "c4": c4, "c5": c5}[name]():
            print(json.dumps(line), flush=True)
