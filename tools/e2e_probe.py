"""Where the e2e call's time goes: handle.search (Python + ctypes + library)
vs the bare ctypes call with prebuilt arguments vs the device time of the
replayed graph (events around the call)."""
import ctypes as C
import sys
import time
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
    h = P.PdxIndex.from_index(index, transform=T)
    Qpin = torch.from_numpy(Q).pin_memory()
    out = {"dist": torch.empty((1000, 10), dtype=torch.float32, pin_memory=True),
           "ids": torch.empty((1000, 10), dtype=torch.int64, pin_memory=True)}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def call():
        return h.search(Qpin, k=10, pruner="ads", nprobe=32, epsilon0=2.1, rotate=True, out=out)
    for _ in range(5):
        call()
    torch.cuda.synchronize()
    for fl in (True, False):
        ts = []
        for _ in range(30):
            if fl:
                flush.fill_(1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            call()
            ts.append((time.perf_counter() - t0) * 1e6)
        print("handle.search wall us (L2 flush %s): mean %.1f min %.1f" % (fl, np.mean(ts), np.min(ts)))
    # bare ctypes call
    from paper_2503_04422_b200.kernels import Metric
    from paper_2503_04422_b200.pruning import OrderCriteria
    p = _lib.PdxQueryParams(10, _lib.METRIC[Metric("l2").value], _lib.PRUNER["ads"],
                            _lib.CRITERIA[OrderCriteria("sequential").value], 0, 32, 0.2, 2, 1, 2.1,
                            None, 0, 0, 1)
    L = _lib.lib()
    args = (h._h, C.byref(p), _lib.ptr(Qpin), 1000, _lib.ptr(out["dist"]), _lib.ptr(out["ids"]),
            None, None, _lib.stream_handle(None))
    for _ in range(3):
        L.pdx_index_search(*args)
    ts = []
    for _ in range(30):
        flush.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        L.pdx_index_search(*args)
        ts.append((time.perf_counter() - t0) * 1e6)
    print("bare pdx_index_search wall us: mean %.1f min %.1f" % (np.mean(ts), np.min(ts)))
    ts = []
    for _ in range(30):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        L.pdx_index_search(*args)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print("device time around the call us: mean %.1f min %.1f" % (np.mean(ts), np.min(ts)))


if __name__ == "__main__":
    main()
