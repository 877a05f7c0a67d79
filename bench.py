#!/usr/bin/env python
"""Benchmark: IVF + ADSampling search (BASELINE.json configs[1]) on B200.

Workload: N = 1,000,000 float32 vectors, D = 128, drawn from a 1,000-centre
Gaussian mixture (centres ~ N(0, 4I), noise ~ N(0, I)), rotated by the
seeded orthogonal projection, 1,024 k-means buckets, epsilon0 = 2.1, K = 10,
1,000 queries from the same mixture, nprobe = 32 (8 and 128 reported as
extras).  Synthetic data of the paper-dataset shape (the real datasets are
not in the container).  A step = one pass of the whole query batch through
the search hot path: query projection (K3), bucket selection (K2), pruned
PDX scan + top-k (K5/K6).

Arms:
  default            our sm_100a path.  `value`: inputs resident in HBM;
                     `e2e`: IvfNearestNeighbors.kneighbors on host arrays.
  --impl reference   the reference algorithm on the host CPU (the C oracle
                     port of dimscan, all host threads), same index/queries.
Multi-GPU (torchrun): buckets are sharded over ranks (LPT by size), each
rank scans its buckets of the globally selected probes, per-rank top-k are
all-gathered over NCCL and merged on device (K7).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_DEFAULT, D, NCENT, NLIST, NQ, K, EPS = 1_000_000, 128, 1000, 1024, 1000, 10, 2.1


def make_data(n, nq, seed=0):
    """BASELINE configs[1] recipe: centres N(0, 4I), labels
    uniform, noise N(0, I); queries from the same mixture."""
    rng = np.random.default_rng(seed)
    C = rng.standard_normal((NCENT, D)) * 2.0
    lab = rng.integers(0, NCENT, n)
    X = (C[lab] + rng.standard_normal((n, D))).astype(np.float32)
    lq = rng.integers(0, NCENT, nq)
    Q = (C[lq] + rng.standard_normal((nq, D))).astype(np.float32)
    return X, Q


class Clocks:
    """SM clock and clock-event reasons sampled through NVML every 10 ms
    during the timed region (the same counters nvidia-smi reports)."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, gpu=0):
        self.samples, self.gpu, self._stop = [], gpu, threading.Event()
        self.max_mhz = None

    def _run(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        except Exception:
            return
        while not self._stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, [n for n, a in self.REASONS.items()
                                          if rs & getattr(N, a)]))
            except Exception:
                pass
            self._stop.wait(0.01)

    def __enter__(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        reasons = sorted({r for s in self.samples for r in s[1]})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


def ncu_traffic():
    """DRAM bytes per launch of the scan kernel from the committed ncu
    capture summary (profiles/ncu_scan.json, written by tools/ncu_summary.py)."""
    try:
        return json.loads((ROOT / "profiles" / "ncu_scan.json").read_text())
    except Exception:
        return None


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def build_index(X, nlist, seed=0):
    import torch
    import paper_2503_04422_b200 as P
    T = P.generate_orthogonal(D, seed)
    xr = P.apply_transform(T, P.store.to_device(X))
    col = P.VectorCollection(data=np.empty((0, D), np.float32), ids=np.empty(0, np.int64))
    # the collection's host copy is only needed for the oracle views
    col = P.VectorCollection.from_array(xr.cpu().numpy())
    t0 = time.perf_counter()
    index = P.ivf_build(col, nlist=nlist, seed=seed, x_dev=xr)
    torch.cuda.synchronize()
    return T, col, index, time.perf_counter() - t0


def cpu_oracle_qps(index, Qr, nprobe, budget_s=12.0, max_q=None, threads=None):
    """The C oracle (dimscan restated) over a bounded prefix of the queries."""
    from oracle import oracle as O
    O.build()
    view = O.IvfView(index.centroid_blocks, index.buckets, index.means_dev.cpu().numpy())
    threads = threads or os.cpu_count() or 1
    done, t_total, chunk = 0, 0.0, max(4 * threads, 64)
    limit = Qr.shape[0] if max_q is None else min(max_q, Qr.shape[0])
    # untimed warm query (cli.py:171-172)
    O.ivf_search_batch(view, Qr[:1], K, nprobe, pruner="ads", eps0=EPS, nthreads=1)
    # passes over the query set (wrapping around) until the time budget is spent
    while t_total < budget_s:
        s = done % limit
        q = Qr[s:min(limit, s + chunk)]
        t0 = time.perf_counter()
        O.ivf_search_batch(view, q, K, nprobe, pruner="ads", eps0=EPS, nthreads=threads)
        t_total += time.perf_counter() - t0
        done += q.shape[0]
    return done / t_total, done, t_total, threads, view


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_DEFAULT)
    ap.add_argument("--nq", type=int, default=NQ)
    ap.add_argument("--nprobe", type=int, default=32)
    ap.add_argument("--warps", default="0", help="compute warps per query CTA, or W,tiles_per_warp")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--debug", action="store_true", help="print kernel diagnostics to stderr")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--batched", type=int, default=0,
                    help="pdx_search_params.batched: 0 auto, 1 per-query scan, 2 batched")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    args.warps = tuple(int(v) for v in str(args.warps).split(",")) if "," in str(args.warps) else int(args.warps)

    ws, rank, local = dist_env()
    import torch
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    X, Q = make_data(args.n, args.nq)
    config = {"workload": f"ivf-ads N={args.n} D={D} nlist={NLIST} nprobe={args.nprobe} "
                          f"nq={args.nq} K={K} eps0={EPS}",
              "n": args.n, "d": D, "nlist": NLIST, "nprobe": args.nprobe, "queries": args.nq,
              "k": K, "epsilon0": EPS, "pruner": "ads", "layout": "tiles [D/8][64][8] f32",
              "l2_flush": "256 MiB write between timed steps", "parallelism": f"buckets x{ws}"}

    if args.impl == "reference":
        if rank != 0:
            return
        import paper_2503_04422_b200 as P
        T, col, index, _ = build_index(X, NLIST)
        Qr = Q @ T.matrix.T
        threads = os.cpu_count() or 1
        from oracle import oracle as O
        O.build()
        view = O.IvfView(index.centroid_blocks, index.buckets, index.means_dev.cpu().numpy())
        sample = min(args.nq, 100)
        O.ivf_search_batch(view, Qr[:1], K, args.nprobe, pruner="ads", eps0=EPS, nthreads=1)
        times = []
        for s in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            O.ivf_search_batch(view, Qr[:sample], K, args.nprobe, pruner="ads", eps0=EPS,
                               nthreads=threads)
            if s >= args.warmup:
                times.append(time.perf_counter() - t0)
        qps = sample * len(times) / sum(times)
        print(json.dumps({
            "impl": "reference", "metric": "queries/sec at recall@10", "value": qps,
            "unit": "queries/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": config,
            "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads, "kind": "port",
                             "sample": f"first {sample} queries per step; index built once "
                                       "(build not timed)"},
            "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}))
        return

    import paper_2503_04422_b200 as P
    from paper_2503_04422_b200 import _lib
    _lib.lib()
    dev = torch.device("cuda", local)
    T, col, index, build_s = build_index(X, NLIST)
    if ws > 1:
        from paper_2503_04422_b200.sharded import shard_index
        index = shard_index(index, col, rank, ws)
    params = P.SearchParams(k=K, pruner="ads", ads=P.AdsPruner(d=D, epsilon0=EPS))
    searcher = P.IvfSearcher(index, params, args.nprobe, warps=args.warps, batched=args.batched)
    Qd = P.store.to_device(Q)
    Tm = P.store.to_device(T.matrix)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step(Qin, ev=None):
        Qr = torch.empty_like(Qin)
        _lib.check(_lib.lib().pdx_project(_lib.ptr(Qin), Qin.shape[0], D, _lib.ptr(Tm),
                                          _lib.ptr(Qr), _lib.stream_handle()))
        res = searcher.run(Qr, scan_events=ev)
        if ws > 1:
            from paper_2503_04422_b200.sharded import gather_merge
            return gather_merge(res.dist, res.ids, K)
        return res.dist, res.ids

    # exactness of the kernel's stats pass and the algorithmic byte count
    Qr_dev = P.apply_transform(T, Qd)
    st_res = searcher.run(Qr_dev, stats=True)
    touched = int(st_res.touched.sum().item())
    total = int(st_res.total.sum().item())
    alg_bytes = 4 * touched
    if args.debug:
        dbg = torch.zeros((args.nq, 16), dtype=torch.int64, device=dev)
        searcher._buf["debug_buf"] = dbg
        searcher.run(Qr_dev)
        torch.cuda.synchronize()
        del searcher._buf["debug_buf"]
        d = dbg.cpu().numpy().astype(np.float64)
        names = ["cycles", "tiles", "fast", "serial", "replay", "commit_idle", "ring_waits",
                 "sparse_items", "cw_wait", "cw_dense", "cw_sparse", "cw_rest", "commit_busy"]
        print("DEBUG per-query mean:", {n: round(float(d[:, i].mean()), 1)
                                        for i, n in enumerate(names)},
              "max cycles", int(d[:, 0].max()), file=sys.stderr)

    for _ in range(args.warmup):
        step(Qd)
    torch.cuda.synchronize()
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    # One GPU: the step as two CUDA graphs (fixed device buffers, inputs
    # resident) — projection + bucket selection, then the search — so the
    # ~30 launches of a step leave no host gaps; events between the replays
    # time the search.  The replayed results are checked against the direct
    # path.  (Multi-GPU steps end in an NCCL gather: launched directly.)
    graphs = None
    if ws == 1:
        gs = torch.cuda.Stream()
        gs.wait_stream(torch.cuda.current_stream())
        Qr_g = torch.empty_like(Qd)

        def pre():
            _lib.check(_lib.lib().pdx_project(_lib.ptr(Qd), Qd.shape[0], D, _lib.ptr(Tm),
                                              _lib.ptr(Qr_g), _lib.stream_handle()))
            return searcher.select(Qr_g)

        with torch.cuda.stream(gs):
            searcher.search(Qr_g, pre())  # warm on the capture stream
            torch.cuda.synchronize()
            g1, g2 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(g1, stream=gs):
                sel_g = pre()
            with torch.cuda.graph(g2, stream=gs):
                res_g = searcher.search(Qr_g, sel_g)
        torch.cuda.synchronize()
        g1.replay()
        g2.replay()
        torch.cuda.synchronize()
        d_ref, i_ref = step(Qd)
        torch.cuda.synchronize()
        assert torch.equal(res_g.ids, i_ref) and torch.equal(res_g.dist, d_ref), \
            "graph replay differs from the direct search"
        graphs = (g1, g2)
    step_ms, scan_ms = [], []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            torch.cuda.synchronize()
            ev[0].record()
            if graphs:
                graphs[0].replay()
                ev[1].record()
                graphs[1].replay()
                ev[2].record()
            else:
                step(Qd, ev=ev)
            ev[3].record()
            torch.cuda.synchronize()
            step_ms.append(ev[0].elapsed_time(ev[3]))
            scan_ms.append(ev[1].elapsed_time(ev[2]))
    t_step = float(np.mean(step_ms))
    t_scan = float(np.mean(scan_ms))
    if ws > 1:
        import torch.distributed as dist
        tt = torch.tensor([t_step, t_scan], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, t_scan = float(tt[0]), float(tt[1])
    qps = args.nq / (t_step / 1e3)

    # e2e through the C-ABI handle with HOST buffers: one pdx_index_search
    # call per batch (H2D of the queries, projection, selection, scan, D2H
    # of the results, all inside the library)
    handle = P.PdxIndex.from_index(index, transform=T)
    Qpin = torch.from_numpy(Q).pin_memory()
    hout = {"dist": torch.empty((args.nq, K), dtype=torch.float32, pin_memory=True),
            "ids": torch.empty((args.nq, K), dtype=torch.int64, pin_memory=True)}

    def e2e_call():
        if ws == 1:
            return handle.search(Qpin, k=K, pruner="ads", nprobe=args.nprobe, epsilon0=EPS,
                                 rotate=True, out=hout)
        # sharded: host queries -> every rank's scan -> NCCL gather + merge -> host
        d_, i_ = step(Qpin.to(dev, non_blocking=True))
        hout["dist"].copy_(d_, non_blocking=True)
        hout["ids"].copy_(i_, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return hout
    for _ in range(2):
        e2e_call()
    torch.cuda.synchronize()
    e2e_ms = []
    for _ in range(max(3, args.steps // 2)):
        flush.fill_(1)
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        e2e_call()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_mean = float(np.mean(e2e_ms))
    if ws > 1:  # the slowest rank
        tt = torch.tensor([e2e_mean], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_mean = float(tt[0])
    e2e_qps = args.nq / (e2e_mean / 1e3)
    # results for recall: the e2e call's output (merged over ranks when sharded)
    i_h = hout["ids"].numpy()

    if rank != 0:
        if ws > 1:
            torch.distributed.barrier()
        return
    # recall@10 against float64 brute force on the unrotated data
    gt = P.compute_ground_truth(P.VectorCollection.from_array(X), Q, K)
    recall = float(np.mean([P.recall_at_k(gt.ids[i], i_h[i], K) for i in range(args.nq)]))
    peak = 6556.2
    try:
        peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
        peak_src = "measured"
    except Exception:
        peak_src = "fallback"
    achieved = alg_bytes / (t_scan / 1e3) / 1e9
    prof = ncu_traffic()
    traffic = None
    if prof and prof.get("workload") == config["workload"]:
        traffic = prof.get("dram_bytes_per_search")
    line = {
        "metric": "queries/sec at recall@10", "value": qps, "unit": "queries/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded Gaussian mixture, BASELINE configs[1] recipe)",
        "config": config, "recall_at_10": recall,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_source": peak_src, "traffic": traffic,
                     "traffic_source": (prof or {}).get("source"),
                     "kernel": "pdx_search (batched pipeline, pdx_batch.cu); achieved = "
                               "algorithmic bytes / the whole search call",
                     "dominant_kernel": (prof or {}).get("dominant_kernel"),
                     "dominant_time_share_ncu": (prof or {}).get("dominant_time_share"),
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "full_scan_bytes_per_launch": 4 * total,
                     "pruning_power": 1 - touched / total, "scan_ms": t_scan},
        "e2e": {"value": e2e_qps, "unit": "queries/s",
                "h2d_bytes_per_step": int(Q.nbytes),
                "d2h_bytes_per_step": int(args.nq * K * (4 + 8)),
                "path": ("pdx_index_search (C-ABI handle, pinned host buffers)" if ws == 1 else
                         "pinned host queries -> sharded scan -> NCCL gather + merge -> host")},
        # per step: the projection + every launch of one search (ncu launch list)
        "gpu_launches": (1 + int((prof or {}).get("launches_per_search") or 0)) * args.steps,
        "index_build_s": build_s,
    }
    line["clocks"] = clk.summary()
    if not args.no_extras:
        extras = {}
        for npb in (8, 128):
            s2 = P.IvfSearcher(index, params, npb, warps=args.warps)
            for _ in range(3):
                s2.run(Qr_dev)
            torch.cuda.synchronize()
            ts = []
            for _ in range(9):
                flush.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                r2 = s2.run(Qr_dev)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ids2 = r2.ids.cpu().numpy()
            rec2 = float(np.mean([P.recall_at_k(gt.ids[i], ids2[i], K) for i in range(args.nq)]))
            extras[f"nprobe_{npb}"] = {"qps": args.nq / (np.median(ts) / 1e3), "recall_at_10": rec2,
                                       "timing": "median of 9 L2-flushed searches"}
        # BSA (this build's restatement) on the same data and nprobe
        est = P.IvfNearestNeighbors(pruner="bsa", nlist=NLIST, nprobe=args.nprobe, seed=0).fit(X)
        sb = est.searcher(K)
        Qb = P.apply_transform(est.transform_, Qd)
        rs = sb.run(Qb, stats=True)
        pp_b = 1 - int(rs.touched.sum().item()) / int(rs.total.sum().item())
        for _ in range(3):
            sb.run(Qb)
        torch.cuda.synchronize()
        ts = []
        for _ in range(9):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rb = sb.run(Qb)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        idsb = rb.ids.cpu().numpy()
        recb = float(np.mean([P.recall_at_k(gt.ids[i], idsb[i], K) for i in range(args.nq)]))
        extras[f"bsa_nprobe_{args.nprobe}"] = {
            "qps": args.nq / (np.median(ts) / 1e3), "recall_at_10": recb,
            "pruning_power": pp_b, "coef": [round(c, 4) for c in est.bsa_.coef]}
        line["extras"] = extras
    if ws == 1:
        cq, done, secs, threads, _ = cpu_oracle_qps(index, Qr_dev.cpu().numpy(), args.nprobe,
                                                    budget_s=args.cpu_budget)
        line["cpu_baseline"] = {"value": cq, "unit": "queries/s", "cores": threads, "kind": "port",
                                "sample": f"{done} query searches ({secs:.1f} s wall; passes over "
                                          f"the {args.nq} queries) of the same workload and "
                                          "index, C oracle of the reference, one query per "
                                          "host thread"}
    print(json.dumps(line))
    if ws > 1:
        torch.distributed.barrier()


if __name__ == "__main__":
    main()
