"""Does a CUDA graph of one batched search (bench workload) replay with the
same results, and how much host launch overhead does it remove?"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2503_04422_b200 as P  # noqa: E402

X, Q = bench.make_data(bench.N_DEFAULT, bench.NQ)
T, col, index, _ = bench.build_index(X, bench.NLIST)
params = P.SearchParams(k=bench.K, pruner="ads", ads=P.AdsPruner(d=bench.D, epsilon0=bench.EPS))
s = P.IvfSearcher(index, params, 32)
Qr = P.store.to_device(Q @ T.matrix.T)
ref = s.run(Qr)
ref_ids = ref.ids.clone()
ref_d = ref.dist.clone()
for _ in range(3):
    s.run(Qr)
torch.cuda.synchronize()


def timeit(fn, n=50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


print(f"direct: {timeit(lambda: s.run(Qr)):.3f} ms per search")
g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(st):
    s.run(Qr)  # warm on the capture stream
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=st):
        out = s.run(Qr)
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
same = torch.equal(out.ids, ref_ids) and torch.equal(out.dist, ref_d)
print(f"graph replay identical: {same}")
print(f"graph: {timeit(g.replay):.3f} ms per search")
