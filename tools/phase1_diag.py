"""Phase-1 diagnostics on the bench workload: tiles in each query's first
selected bucket and the per-query cycles of the per-query scan over it."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2503_04422_b200 as P  # noqa: E402
from paper_2503_04422_b200.index import select_buckets_device  # noqa: E402
from paper_2503_04422_b200.search import run_search  # noqa: E402

X, Q = bench.make_data(bench.N_DEFAULT, bench.NQ)
T, col, index, _ = bench.build_index(X, bench.NLIST)
params = P.SearchParams(k=bench.K, pruner="ads", ads=P.AdsPruner(d=bench.D, epsilon0=bench.EPS))
Qr = P.store.to_device(Q @ T.matrix.T)
sel = select_buckets_device(index, Qr, 32, params.metric)
sel = sel[0] if isinstance(sel, tuple) else sel
s0 = sel[:, :1].contiguous()
sizes = np.diff(index.store.bucket_block.cpu().numpy())
first = sizes[s0.cpu().numpy()[:, 0]]
print("bucket blocks: max", sizes.max(), "mean", sizes.mean().round(1))
print("first-bucket blocks per query: mean", first.mean().round(1), "p50/p90/p99/max",
      np.percentile(first, [50, 90, 99, 100]))
allb = sizes[sel.cpu().numpy()].sum(1)
print("window blocks per query: mean", allb.mean().round(1), "max", allb.max())
for w in ((8, 4, 32),):
    buf = {"debug_buf": torch.zeros((Qr.shape[0], 16), dtype=torch.int64, device="cuda")}
    for _ in range(3):
        run_search(index.store, Qr, params, seg_bucket=s0, nseg=1, warps=w, out=buf, batched=1)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    run_search(index.store, Qr, params, seg_bucket=s0, nseg=1, warps=w, out=buf, batched=1)
    ev[1].record()
    torch.cuda.synchronize()
    cyc = buf["debug_buf"][:, 0].cpu().numpy()
    print(f"warps={w}: {ev[0].elapsed_time(ev[1]) * 1e3:.0f} us; per-query kcycles p50/p90/p99/max",
          np.percentile(cyc / 1e3, [50, 90, 99, 100]).round(0),
          "corr(cycles, blocks)", np.corrcoef(cyc, first)[0, 1].round(2))
