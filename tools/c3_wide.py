"""C3 (1M x 960, nlist 2048, nprobe 64) results-only ADS / BOND: the batched
pipeline's MODE 0 variant for wide vectors (PDX_BSCAN_FILTER_WIDE=0/1),
checked against the per-query scan."""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import paper_2503_04422_b200 as P  # noqa: E402
from bench_configs import mixture, recall, timed  # noqa: E402

n, d, nlist, nprobe, nq, k = 1_000_000, 960, 2048, 64, 1000, 10
sigma = (torch.arange(d, device="cuda", dtype=torch.float32) + 1) ** -0.5
xq, _ = mixture(n + nq, d, 1000, 3, centre_scale=2.0, sigma=sigma)
x, q = xq[:n].contiguous(), xq[n:].contiguous()
R = P.generate_orthogonal(d, 1)
x = P.apply_transform(R, x)
q = P.apply_transform(R, q)
gt, _ = P.synthetic.ground_truth_device(x, q, k)
gt = gt.cpu().numpy()
ix = P.ivf_build(P.VectorCollection.from_array(x.cpu().numpy()), nlist=nlist, seed=0, x_dev=x)
for name, prm in (("ads", P.SearchParams(k=k, pruner="ads", ads=P.AdsPruner(d=d))),
                  ("bond", P.SearchParams(k=k, pruner="bond"))):
    s = P.IvfSearcher(ix, prm, nprobe, batched=0)
    r = s.run(q)
    r1 = P.IvfSearcher(ix, prm, nprobe, batched=1).run(q)
    same = bool(torch.equal(r.ids, r1.ids) and torch.equal(r.dist, r1.dist))
    sec = timed(lambda: s.run(q))
    print(json.dumps({"config": "C3", "pruner": name, "wide_filter": os.environ.get("PDX_BSCAN_FILTER_WIDE", "0"),
                      "qps": nq / sec, "scan_batch_s": sec, "same_as_per_query": same,
                      "recall_at_10": recall(gt, r.ids.cpu().numpy(), k)}))
