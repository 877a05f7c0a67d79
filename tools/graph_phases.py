#!/usr/bin/env python
"""Per-phase device time of the batched search INSIDE a replayed CUDA graph
(the bench's timed configuration): the library's phase events are captured
as external event nodes and read after each replay (pdx_batch_profile(2))."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    import paper_2503_04422_b200 as P
    from paper_2503_04422_b200 import _lib
    X, Q = bench.make_data(1_000_000, 1000)
    T = P.generate_orthogonal(128, 0)
    XR = X @ T.matrix.T
    cent, assign, _ = bench.load_fixture(XR)
    index = P.IvfIndex.from_assignment(P.VectorCollection.from_array(XR), cent, assign, nlist=1024)
    params = P.SearchParams(k=10, pruner="ads", ads=P.AdsPruner(d=128, epsilon0=2.1))
    s = P.IvfSearcher(index, params, 32)
    Qr = P.store.to_device((Q @ T.matrix.T).astype(np.float32))
    L = _lib.lib()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    gs = torch.cuda.Stream()
    gs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(gs):
        sel = s.select(Qr)
        s.search(Qr, sel)
        torch.cuda.synchronize()
        L.pdx_batch_profile(1, None, 0, None)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=gs):
            s.search(Qr, sel)
    torch.cuda.synchronize()
    names = ["plan", "phase1", "tprime_join", "mode0", "chain", "verify", "final", "fallback"]
    tot = []
    for _ in range(20):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        tot.append(e0.elapsed_time(e1))
        L.pdx_batch_profile(2, None, 0, None)
    acc = (C.c_double * 8)()
    calls = C.c_int64()
    L.pdx_batch_profile(-1, C.cast(acc, C.c_void_p), 8, C.cast(C.pointer(calls), C.c_void_p))
    print("graph replay: search", round(float(np.mean(tot)) * 1000, 1), "us;",
          {n: round(acc[i] / max(1, calls.value) * 1000, 1) for i, n in enumerate(names)})


if __name__ == "__main__":
    main()
