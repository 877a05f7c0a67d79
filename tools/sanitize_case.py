#!/usr/bin/env python
"""A small case through every search kernel, for compute-sanitizer
(memcheck / racecheck / synccheck): the batched IVF pipeline (bprep ...
bdense, bchain1, bscan MODE 0/1, bchain, bfinal) with ADS and BOND, the
per-query scan (pdx_scan_kernel, forced with batched = 1), the exact
scan, K2 selection, the k-means build and K8 (tcgen05) candidates +
rescoring.  Results are checked against the C oracle so a run that
'passes' the tool also computed the right answer."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))


def main():
    import torch

    import paper_2503_04422_b200 as P
    import recipes
    from oracle import oracle as O
    O.build()
    x = recipes.data("mixture", 12_000, 40, 3)
    q = recipes.queries("near", x, 40, 4)
    index = P.ivf_build(P.VectorCollection.from_array(x), nlist=48, seed=0)
    view = O.IvfView(index.centroid_blocks, index.buckets, index.means_dev.cpu().numpy())
    for pruner in ("ads", "bond"):
        for batched in (2, 1):
            out = P.ivf_search_batch(index, q, P.SearchParams(k=10, pruner=pruner), 6,
                                     batched=batched)
            ref = O.ivf_search_batch(view, q, 10, 6, pruner=pruner)
            assert np.array_equal(out["ids"], ref["ids"]), (pruner, batched)
    flat = P.flat_build(P.VectorCollection.from_array(x), 64)
    out = P.exact_search_batch(flat, q, P.SearchParams(k=10, pruner="bond"))
    tc = P.TensorCoreExactSearcher(flat, P.SearchParams(k=10, metric="l2"))
    r = tc.run(torch.from_numpy(q).cuda())
    ref = P.ExactSearcher(flat, P.SearchParams(k=10)).run(torch.from_numpy(q).cuda())
    assert torch.equal(r.ids, ref.ids)
    torch.cuda.synchronize()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
