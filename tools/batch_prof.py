"""One C2 search step (bench.py's workload) bracketed by cudaProfilerStart/
Stop, for `ncu --profile-from-start off` launch lists of the pipeline."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2503_04422_b200 as P  # noqa: E402

batched = int(sys.argv[1]) if len(sys.argv) > 1 else 0
nprobe = int(sys.argv[2]) if len(sys.argv) > 2 else 32
X, Q = bench.make_data(bench.N_DEFAULT, bench.NQ)
T, col, index, _ = bench.build_index(X, bench.NLIST)
params = P.SearchParams(k=bench.K, pruner="ads", ads=P.AdsPruner(d=bench.D, epsilon0=bench.EPS))
s = P.IvfSearcher(index, params, nprobe, batched=batched)
Qr = P.store.to_device(Q @ T.matrix.T)
for _ in range(3):
    s.run(Qr)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
s.run(Qr)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(20):
    s.run(Qr)
ev[1].record()
torch.cuda.synchronize()
print(f"batched={batched} nprobe={nprobe}: {ev[0].elapsed_time(ev[1]) / 20:.3f} ms per search")
