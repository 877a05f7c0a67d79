#!/usr/bin/env python
"""Benchmark: IVF + ADSampling search (BASELINE.json configs[1]) on B200.

Workload: N = 1,000,000 float32 vectors, D = 128, drawn from a 1,000-centre
Gaussian mixture (centres ~ N(0, 4I), noise ~ N(0, I)), rotated by the
seeded orthogonal projection, 1,024 k-means buckets, epsilon0 = 2.1, K = 10,
1,000 queries from the same mixture, nprobe = 32 (8 and 128 reported as
extras).  Synthetic data of the paper-dataset shape (the real datasets are
not in the container).  A step = one pass of the whole query batch through
the search hot path: query projection (K3), bucket selection (K2), pruned
PDX scan + top-k (the batched pipeline, csrc/pdx_batch.cu).

The index is the REFERENCE's: ``tests/golden/c2_ivf_reference.npz`` holds
the centroids and assignment that ``dimscan.index.lloyd_kmeans`` produced
for this data (tools/make_c2_index.py, run once in the build container).
Both arms pack it themselves — the GPU arm with K1
(``IvfIndex.from_assignment``), the reference arm in numpy — so neither arm
runs this repo's k-means and both search the identical index.

Arms:
  default            our sm_100a path.  `value`: inputs resident in HBM;
                     `e2e`: one pdx_index_search call (C-ABI) per batch with
                     page-locked host buffers.  `parity`: ids, distances,
                     values_touched of all 1000 queries at nprobe 8/32/128
                     against the C oracle on the same index and queries.
  --impl reference   the reference algorithm on the host CPU (the C oracle
                     port of dimscan, all host threads), same index/queries;
                     never loads libpdx_b200.so.
Multi-GPU (torchrun): buckets are sharded over ranks (LPT by size), each
rank scans its buckets of the globally selected probes, per-rank top-k are
all-gathered over NCCL and merged on device (K7).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_DEFAULT, D, NCENT, NLIST, NQ, K, EPS = 1_000_000, 128, 1000, 1024, 1000, 10, 2.1
FIXTURE = ROOT / "tests" / "golden" / "c2_ivf_reference.npz"


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


def rotation(d, seed=0):
    """generate_orthogonal (pruning.py:36-45): seeded Gaussian, QR, sign fix."""
    g = np.random.default_rng(seed).standard_normal((d, d))
    q, r = np.linalg.qr(g)
    return (q * np.sign(np.diag(r))).astype(np.float32)


def load_fixture(XR):
    """(centroids, assignment, data fingerprint matches) of the reference
    k-means index, or None when the fixture does not fit the data."""
    if not FIXTURE.exists():
        return None
    f = np.load(FIXTURE)
    if f["assign"].shape[0] != XR.shape[0]:
        return None
    same = hashlib.sha256(XR.tobytes()).digest() == f["xr_sha"].tobytes()
    return f["centroids"], f["assign"].astype(np.int64), bool(same)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


class Clocks:
    """SM clock and clock-event reasons sampled through NVML during the
    timed region (the counters nvidia-smi reports).  NVML is initialised
    before the region; one sample is taken synchronously at its start and
    one at its end, and a thread samples every 2 ms in between."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, gpu=0):
        self.samples, self._stop = [], threading.Event()
        self.max_mhz, self.h, self.N, self.err = None, None, None, None
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            idx = int(vis.split(",")[gpu]) if vis and vis.split(",")[0].isdigit() else gpu
            self.h = N.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001 - reported in the line
            self.err = repr(e)

    def sample(self):
        if self.h is None:
            return
        N = self.N
        try:
            sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
            rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            self.samples.append((sm, [n for n, a in self.REASONS.items() if rs & getattr(N, a)]))
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)

    def _run(self):
        while not self._stop.wait(0.002):
            self.sample()

    def __enter__(self):
        self.sample()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=6)
        self.sample()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"],
                    "error": self.err}
        sm = [s[0] for s in self.samples]
        reasons = sorted({r for s in self.samples for r in s[1]})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "NVML"}


def ncu_profile():
    """Per-kernel DRAM bytes / issue activity of one search from the
    committed ncu capture (profiles/r02_kernels.json, tools/ncu_kernels.py)."""
    try:
        return json.loads((ROOT / "profiles" / "r02_kernels.json").read_text())
    except Exception:
        return None


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def oracle_qps(view, Qr, nprobe, budget_s, threads):
    """The C oracle (dimscan restated) in passes over the queries until the
    time budget is spent (one untimed warm query first, cli.py:171-172)."""
    from oracle import oracle as O
    O.ivf_search_batch(view, Qr[:1], K, nprobe, pruner="ads", eps0=EPS, nthreads=1)
    done, t_total, chunk = 0, 0.0, max(4 * threads, 16)
    while t_total < budget_s:
        s = done % Qr.shape[0]
        q = Qr[s:min(Qr.shape[0], s + chunk)]
        t0 = time.perf_counter()
        O.ivf_search_batch(view, q, K, nprobe, pruner="ads", eps0=EPS, nthreads=threads)
        t_total += time.perf_counter() - t0
        done += q.shape[0]
    return done / t_total, done, t_total


def reference_arm(args, config):
    """The reference algorithm (C oracle port of dimscan) on the host cores,
    on the reference k-means index; no GPU code is loaded."""
    from oracle import oracle as O
    X, Q = make_data(args.n, args.nq)
    T = rotation(D)
    XR, QR = X @ T.T, Q @ T.T  # apply_transform (pruning.py:48-53)
    fx = load_fixture(XR)
    if fx is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"no reference k-means fixture for n={args.n} (tools/make_c2_index.py)"}))
        return
    cent, assign, _ = fx
    O.build()
    view = O.IvfView.from_assignment(XR, cent, assign, NLIST)
    threads = os.cpu_count() or 1
    O.ivf_search_batch(view, QR[:1], K, args.nprobe, pruner="ads", eps0=EPS, nthreads=1)
    times = []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        O.ivf_search_batch(view, QR, K, args.nprobe, pruner="ads", eps0=EPS, nthreads=threads)
        if s >= args.warmup:
            times.append(time.perf_counter() - t0)
    qps = args.nq * len(times) / sum(times)
    print(json.dumps({
        "impl": "reference", "metric": "queries/sec at recall@10", "value": qps,
        "unit": "queries/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": config,
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"all {args.nq} queries per step, {args.steps} timed steps; "
                                   "the reference's k-means index (fixture), packed in numpy"},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}))


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
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=8.0)
    ap.add_argument("--batched", type=int, default=0,
                    help="pdx_search_params.batched: 0 auto, 1 per-query scan, 2 batched")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        args.no_extras = True  # the extras (BSA index, GPU build) are single-GPU measurements
    args.warps = tuple(int(v) for v in str(args.warps).split(",")) if "," in str(args.warps) else int(args.warps)

    ws, rank, local = dist_env()
    config = {"workload": f"ivf-ads N={args.n} D={D} nlist={NLIST} nprobe={args.nprobe} "
                          f"nq={args.nq} K={K} eps0={EPS}",
              "n": args.n, "d": D, "nlist": NLIST, "nprobe": args.nprobe, "queries": args.nq,
              "k": K, "epsilon0": EPS, "pruner": "ads", "layout": "tiles [D/8][64][8] f32",
              "index": "reference lloyd_kmeans (tests/golden/c2_ivf_reference.npz)",
              "l2_flush": "256 MiB write between timed steps", "parallelism": f"buckets x{ws}",
              "outputs": "ids + distances per query (as kneighbors / ivf_search without "
                         "SearchStats); values_touched comes from a separate stats pass"}

    if args.impl == "reference":
        if rank == 0:
            reference_arm(args, config)
        return

    import torch
    if torch.cuda.is_available():
        local = local % torch.cuda.device_count()  # (ranks share a GPU only in a gloo smoke run)
        torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        backend = os.environ.get("PDX_DIST_BACKEND", "nccl")  # gloo: a one-GPU smoke test
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    import paper_2503_04422_b200 as P
    from paper_2503_04422_b200 import _lib
    _lib.lib()
    dev = torch.device("cuda", local)

    X, Q = make_data(args.n, args.nq)
    T = P.generate_orthogonal(D, 0)
    XR = X @ T.matrix.T  # the index data: apply_transform on the host, as the reference
    x_dev = P.store.to_device(XR)
    col = P.VectorCollection.from_array(XR)
    fx = load_fixture(XR)
    t0 = time.perf_counter()
    if fx is None:  # other sizes: this repo's GPU k-means (same algorithm, index.py:27-64)
        cent, assign = P.index.lloyd_kmeans_device(x_dev, NLIST, 0)
        cent, assign = cent.cpu().numpy(), assign.cpu().numpy().astype(np.int64)
        config["index"] = "GPU lloyd_kmeans (no reference fixture for this n)"
    else:
        cent, assign, same = fx
        config["index_data_fingerprint_match"] = same
    if ws > 1:  # this rank packs only the buckets it owns (LPT by size)
        from paper_2503_04422_b200.sharded import shard_from_assignment
        index = shard_from_assignment(XR, cent, assign, rank, ws, x_dev=x_dev, nlist=NLIST)
    else:
        index = P.IvfIndex.from_assignment(col, cent, assign, nlist=NLIST, x_dev=x_dev)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    del x_dev
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

    for _ in range(args.warmup):
        step(Qd)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    # One GPU: the step as one CUDA graph (fixed device buffers, inputs
    # resident: projection + bucket selection + the search), so the ~30
    # launches of a step leave no host gaps; the search alone is timed from a
    # two-graph split (events between the replays).  The replayed results are
    # checked against the direct path.  (Multi-GPU steps end in an NCCL
    # gather: launched directly.)
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
            g1, g2, gall = (torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(),
                            torch.cuda.CUDAGraph())
            with torch.cuda.graph(g1, stream=gs):
                sel_g = pre()
            with torch.cuda.graph(g2, stream=gs):
                res_g = searcher.search(Qr_g, sel_g)
            with torch.cuda.graph(gall, stream=gs):  # the whole step as one launch
                res_all = searcher.search(Qr_g, pre())
        torch.cuda.synchronize()
        g1.replay()
        g2.replay()
        gall.replay()
        torch.cuda.synchronize()
        d_ref, i_ref = step(Qd)
        torch.cuda.synchronize()
        assert torch.equal(res_g.ids, i_ref) and torch.equal(res_g.dist, d_ref), \
            "graph replay differs from the direct search"
        assert torch.equal(res_all.ids, i_ref) and torch.equal(res_all.dist, d_ref), \
            "graph replay differs from the direct search"
        graphs = (g1, g2, gall)
    step_ms, scan_ms = [], []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            torch.cuda.synchronize()
            ev[0].record()
            if graphs:
                graphs[2].replay()
            else:
                step(Qd, ev=ev)
            ev[3].record()
            torch.cuda.synchronize()
            step_ms.append(ev[0].elapsed_time(ev[3]))
            if not graphs:
                scan_ms.append(ev[1].elapsed_time(ev[2]))
    if graphs:  # the search part alone: the two-graph split, events between
        for _ in range(max(5, args.steps // 2)):
            flush.fill_(1)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            torch.cuda.synchronize()
            graphs[0].replay()
            ev[0].record()
            graphs[1].replay()
            ev[1].record()
            torch.cuda.synchronize()
            scan_ms.append(ev[0].elapsed_time(ev[1]))
    t_step = float(np.mean(step_ms))
    t_scan = float(np.mean(scan_ms))
    if ws > 1:
        tt = torch.tensor([t_step, t_scan], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_step, t_scan = float(tt[0]), float(tt[1])
    qps = args.nq / (t_step / 1e3)

    # live per-phase device time of the search (CUDA events on the search
    # stream inside the library; same L2 flush; direct launches)
    phase_names = ["plan", "phase1_bdense_bchain1", "tprime_join", "bscan_mode0", "chain",
                   "bscan_mode1", "final", "fallback"]
    phases = None
    if ws == 1:
        import ctypes as C
        L = _lib.lib()
        L.pdx_batch_profile(1, None, 0, None)
        for _ in range(20):
            flush.fill_(1)
            searcher.run(Qr_dev)
        torch.cuda.synchronize()
        acc = (C.c_double * 8)()
        calls = C.c_int64()
        L.pdx_batch_profile(0, C.cast(acc, C.c_void_p), 8, C.cast(C.pointer(calls), C.c_void_p))
        if calls.value:
            phases = {n: acc[i] / calls.value for i, n in enumerate(phase_names)}

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
    i_h = hout["ids"].numpy().copy()

    if rank != 0:
        if ws > 1:
            torch.distributed.barrier()
        return
    # recall@10 against float64 brute force on the unrotated data
    gt = P.compute_ground_truth(P.VectorCollection.from_array(X), Q, K)
    recall = float(np.mean([P.recall_at_k(gt.ids[i], i_h[i], K) for i in range(args.nq)]))
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        peak, peak_src = peaks["hbm_gbs"], "measured"
    except Exception:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    prof = ncu_profile()
    if prof and prof.get("workload") != config["workload"]:
        prof = None
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = 148 * 128 * sm_mhz * 1e6 / 1e12  # FADD/FMUL lane ops per s (no FMA: 1 op)
    fp32_ops = 3.0 * touched  # sub, mul, add per value touched (search.py:132, :169)
    kernels = []
    if prof:
        live = {"bscan_mode0": "bscan_mode0", "bscan_mode1": "bscan_mode1",
                "bdense": "phase1_bdense_bchain1", "bchain1": "phase1_bdense_bchain1"}
        for kk in prof.get("kernels", []):
            e = dict(kk)
            ph = live.get(kk.get("role", ""))
            if phases and ph and kk.get("role") in ("bscan_mode0", "bscan_mode1"):
                e["live_ms"] = phases[ph]
                e["dram_gbs_live"] = kk["dram_bytes"] / (phases[ph] / 1e3) / 1e9
                e["dram_frac_live"] = e["dram_gbs_live"] / peak
            kernels.append(e)
    dram = (prof or {}).get("dram_bytes_per_search")
    line = {
        "metric": "queries/sec at recall@10", "value": qps, "unit": "queries/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded Gaussian mixture, BASELINE configs[1] recipe)",
        "config": config, "recall_at_10": recall,
        "roofline": {
            "bound": "issue",
            "achieved": fp32_ops / (t_scan / 1e3) / 1e12, "peak": fp32_peak, "unit": "TFLOP/s",
            "frac": fp32_ops / (t_scan / 1e3) / 1e12 / fp32_peak,
            "peak_source": f"148 SMs x 128 FP32 lanes x {sm_mhz:.0f} MHz (FADD/FMUL, computed)",
            "what": "the whole search (25 launches, pdx_batch.cu): 3 FP32 ops per value touched "
                    "(the reference's values_touched) / search time; the pipeline is "
                    "instruction-issue bound (decisions + bookkeeping), not HBM- or tensor-bound",
            "traffic": dram, "traffic_source": (prof or {}).get("source"),
            "algorithmic_bytes_per_launch": alg_bytes, "full_scan_bytes_per_launch": 4 * total,
            "pruning_power": 1 - touched / total, "scan_ms": t_scan,
            "hbm": {"peak_gbs": peak, "peak_source": peak_src,
                    "bytes_touched_gbs": alg_bytes / (t_scan / 1e3) / 1e9,
                    "bytes_touched_frac": alg_bytes / (t_scan / 1e3) / 1e9 / peak,
                    "bytes_touched_note": "north_star's 'bytes touched / time': a tile is read "
                                          "once per work item and shared by ~31 queries, so this "
                                          "is not DRAM traffic",
                    "dram_gbs": dram / (t_scan / 1e3) / 1e9 if dram else None,
                    "dram_frac": dram / (t_scan / 1e3) / 1e9 / peak if dram else None},
            "phases_ms_live": phases,
            "kernels": kernels,
            "dominant_kernel": (prof or {}).get("dominant_kernel")},
        "e2e": {"value": e2e_qps, "unit": "queries/s",
                "h2d_bytes_per_step": int(Q.nbytes),
                "d2h_bytes_per_step": int(args.nq * K * (4 + 8)),
                "path": ("pdx_index_search (C-ABI handle, pinned host buffers)" if ws == 1 else
                         "pinned host queries -> sharded scan -> NCCL gather + merge -> host")},
        # per step: the projection + every launch of one search (ncu launch list)
        "gpu_launches": (1 + int((prof or {}).get("launches_per_search") or 25)) * args.steps,
        "index_pack_s": build_s,
    }
    line["clocks"] = clk.summary()
    view = None
    if ws == 1:  # the oracle's view of the very index the GPU searched
        from oracle import oracle as O
        O.build()
        view = O.IvfView.from_assignment(index._host_data, index.centroids, index_assign(index),
                                         index.nlist)
    if ws == 1 and not args.no_parity:
        line["parity"] = parity_block(P, view, index, params, Qr_dev, args, i_h)
    if not args.no_extras:
        line["extras"] = extras_block(P, index, params, Qr_dev, Qd, X, args, gt, flush)
    if ws == 1:
        Qh = Qr_dev.cpu().numpy()
        threads = os.cpu_count() or 1
        cq, done, secs = oracle_qps(view, Qh, args.nprobe, args.cpu_budget, threads)
        c1, done1, secs1 = oracle_qps(view, Qh, args.nprobe, args.cpu_budget / 2, 1)
        line["cpu_baseline"] = {
            "value": cq, "unit": "queries/s", "cores": threads, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"{done} query searches ({secs:.1f} s) in passes over the {args.nq} "
                      "queries of the same workload and index; C oracle of the reference, one "
                      "query per host thread",
            "single_thread": {"value": c1, "cores": 1,
                              "sample": f"{done1} query searches ({secs1:.1f} s), 1 thread "
                                        "(the reference's single-threaded semantics)"}}
    print(json.dumps(line))
    if ws > 1:
        torch.distributed.barrier()


def index_assign(index):
    """Row -> bucket of a GPU-built index (for the oracle view)."""
    a = np.empty(int(np.sum(index._counts)), dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(index._counts)])
    for c in range(index.nlist):
        a[index._order[off[c]:off[c + 1]]] = c
    return a


def parity_block(P, view, index, params, Qr_dev, args, i_h):
    """Headline-config parity: ids, f32 distances and values_touched of all
    queries against the C oracle on the same index and the same (device-
    projected) queries, at nprobe 8 / 32 / 128; plus the e2e call's output
    against the device path."""
    import torch
    from oracle import oracle as O
    Qh = Qr_dev.cpu().numpy()
    out = {"queries": int(Qh.shape[0]), "reference": "C oracle (oracle/pdx_oracle.c), pinned "
                                                       "to the reference by tests/golden"}
    ok = True
    for npb in (8, 32, 128):
        s = P.IvfSearcher(index, params, npb)
        r = s.run(Qr_dev, stats=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ref = O.ivf_search_batch(view, Qh, K, npb, pruner="ads", eps0=EPS,
                                 nthreads=os.cpu_count() or 1)
        e = {"ids_equal": bool(np.array_equal(r.ids.cpu().numpy(), ref["ids"])),
             "dist_equal": bool(np.array_equal(r.dist.cpu().numpy(), ref["dist"])),
             "touched_equal": bool(np.array_equal(r.touched.cpu().numpy(), ref["touched"])),
             "total_equal": bool(np.array_equal(r.total.cpu().numpy(), ref["total"])),
             "selection_equal": bool(np.array_equal(r.selected.cpu().numpy(), ref["selected"])),
             "oracle_s": round(time.perf_counter() - t0, 2)}
        e["queries_differing"] = int(np.sum(np.any(r.ids.cpu().numpy() != ref["ids"], axis=1)))
        # the timed step's own path: results only (no stats: the survivor
        # verification instead of the MODE 1 recompute)
        r0 = s.run(Qr_dev)
        e["results_only_ids_equal"] = bool(np.array_equal(r0.ids.cpu().numpy(), ref["ids"]))
        e["results_only_dist_equal"] = bool(np.array_equal(r0.dist.cpu().numpy(), ref["dist"]))
        ok = (ok and e["ids_equal"] and e["dist_equal"] and e["touched_equal"]
              and e["results_only_ids_equal"] and e["results_only_dist_equal"])
        out[f"nprobe_{npb}"] = e
        if npb == args.nprobe:  # the e2e handle's answer (host rotation path) vs device path
            out["e2e_ids_equal_device"] = bool(np.array_equal(i_h, r.ids.cpu().numpy()))
    out["ids_equal"] = out["dist_equal"] = out["touched_equal"] = ok
    return out


def extras_block(P, index, params, Qr_dev, Qd, X, args, gt, flush):
    import torch
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
    # the GPU IVF build (csrc/pdx_build.cu) of the same data vs the
    # reference's k-means (the fixture: 252 s on one host core)
    fx = load_fixture(index._host_data)
    if fx is not None:
        xr = P.store.to_device(index._host_data)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cent_g, assign_g = P.index.lloyd_kmeans_device(xr, NLIST, 0)
        torch.cuda.synchronize()
        tb = time.perf_counter() - t0
        a_g = assign_g.cpu().numpy()
        extras["gpu_ivf_build"] = {
            "kmeans_s": tb, "reference_kmeans_s": float(np.load(FIXTURE)["kmeans_seconds"]),
            "assignment_agreement_with_reference": float(np.mean(a_g == fx[1])),
            "max_centroid_abs_diff": float(np.abs(cent_g.cpu().numpy() - fx[0]).max()),
            "what": "lloyd_kmeans_device (fused f32 distance+argmin, radix bucket layout, f64 "
                    "means, 20 iterations max) on the C2 data"}
        del xr
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
        "pruning_power": pp_b, "coef": [round(c, 4) for c in est.bsa_.coef],
        "index": "GPU k-means of this repo (BSA needs its PCA-space index)"}
    return extras


if __name__ == "__main__":
    main()
