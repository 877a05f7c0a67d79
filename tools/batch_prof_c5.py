"""C5-scaled (tools/bench_configs.py c5) search for ncu launch lists:
argv[1] = pruner (ads|bond), argv[2] = batched mode."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench_configs as BC  # noqa: E402
import paper_2503_04422_b200 as P  # noqa: E402
from types import SimpleNamespace  # noqa: E402
from paper_2503_04422_b200.index import IvfIndex, _argmin_chunked, lloyd_kmeans_device  # noqa: E402

pruner, batched = sys.argv[1], int(sys.argv[2])
n, d, nlist, nprobe, nq, k = 10_000_000, 768, 8192, 128, 10_000, 10
sigma = (torch.arange(d, device="cuda", dtype=torch.float32) + 1) ** -0.35
xq, _ = BC.mixture(n + nq, d, 16384, 5, centre_scale=2.0, sigma=sigma)
R = P.generate_orthogonal(d, 2)
for r0 in range(0, n + nq, 1 << 20):
    xq[r0:r0 + (1 << 20)] = P.apply_transform(R, xq[r0:r0 + (1 << 20)])
x, q = xq[:n], xq[n:].contiguous()
g = torch.Generator(device="cpu").manual_seed(0)
sample = x[torch.randperm(n, generator=g)[:500_000].cuda()].contiguous()
cent, _ = lloyd_kmeans_device(sample, nlist, 0, max_iters=10)
del sample
assign = _argmin_chunked(x, cent, chunk=1 << 16)
col = SimpleNamespace(ids=np.arange(n, dtype=np.int64), data=None, n=n, d=d)
ix = IvfIndex.from_assignment(col, cent.cpu().numpy(), assign, nlist=nlist, x_dev=x)
s = P.IvfSearcher(ix, P.SearchParams(k=k, pruner=pruner, ads=P.AdsPruner(d=d)), nprobe,
                  batched=batched)
s.run(q)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
s.run(q)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
