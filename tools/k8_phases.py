"""Phase times of the K8 path at C4 size (GEMM vs filter vs rescore)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import paper_2503_04422_b200 as P  # noqa: E402
from paper_2503_04422_b200 import _lib  # noqa: E402
from bench_configs import mixture  # noqa: E402

n, d, k, nq = 2_000_000, 1536, 100, 1024
xq, _ = mixture(n + nq, d, 4096, 4, spread=0.5, centre_scale=1.0, normalize=True)
x, q = xq[:n].contiguous(), xq[n:].contiguous()
import numpy as np  # noqa: E402
nb = (n + 63) // 64
ms = np.full(nb, 64, np.int64)
ms[-1] = n - 64 * (nb - 1)
store = P.DeviceStore.pack(x, torch.arange(n, device="cuda"), ms, np.array([nb], np.int64),
                           ids=torch.arange(n, device="cuda"), group=8)
flat = P.FlatPartitioning(store=store, global_means=np.zeros(d), partition_size=64)
tc = P.TensorCoreExactSearcher(flat, P.SearchParams(k=k, metric="ip"))
tc.run(q)
torch.cuda.synchronize()
L = _lib.lib()
qn2 = torch.empty(nq, device="cuda")
L.pdx_k8_norms(_lib.ptr(q), nq, d, _lib.ptr(qn2), None)
prev = torch.full((nq, k), float("inf"), device="cuda")
nxt = torch.empty_like(prev)
cand = torch.empty((nq, 4096), dtype=torch.int64, device="cuda")
cc = torch.zeros(nq, dtype=torch.int32, device="cuda")
torch.backends.cuda.matmul.allow_tf32 = True
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
tg = tf = 0.0
per = []
for r0 in range(0, n, 65536):
    Xc = tc.X[r0:r0 + 65536]
    ev[0].record()
    S = q @ Xc.T
    ev[1].record()
    L.pdx_k8_filter(_lib.ptr(S), S.shape[1], nq, S.shape[1], r0, _lib.ptr(tc.xn2[r0:]), _lib.ptr(qn2),
                    2, d, k, _lib.ptr(prev), _lib.ptr(nxt), _lib.ptr(cand), _lib.ptr(cc), 4096, None)
    ev[2].record()
    ev[2].synchronize()
    tg += ev[0].elapsed_time(ev[1])
    tf += ev[1].elapsed_time(ev[2])
    per.append(round(ev[1].elapsed_time(ev[2]), 2))
    prev, nxt = nxt, prev
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
dist = torch.empty((nq, k), device="cuda")
ids = torch.empty((nq, k), dtype=torch.int64, device="cuda")
e0.record()
L.pdx_k8_rescore(store.ref, 64, _lib.ptr(q), nq, 2, k, _lib.ptr(cand), _lib.ptr(cc), 4096,
                 _lib.ptr(dist), _lib.ptr(ids), None)
e1.record()
e1.synchronize()
print("filter per chunk ms:", per)
print(f"gemm {tg:.2f} ms ({2*nq*n*d/tg/1e9:.0f} TF/s)  filter {tf:.2f} ms  rescore {e0.elapsed_time(e1):.2f} ms")
