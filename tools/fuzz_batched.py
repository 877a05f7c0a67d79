#!/usr/bin/env python
"""Randomised comparison of the batched pipeline (results only and with
statistics) with the per-query scan: ids and float32 distances must be
identical.  Shapes, schedules, pruners, k, nprobe and data distributions are
drawn from a seeded generator.

    python tools/fuzz_batched.py [cases] [seed]
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def make(rng, n, d, kind):
    if kind == "mixture":
        c = rng.standard_normal((max(2, n // 400), d)) * rng.uniform(1.0, 4.0)
        x = c[rng.integers(0, len(c), n)] + rng.standard_normal((n, d))
    elif kind == "offset":
        x = rng.standard_normal((n, d)) + rng.uniform(50.0, 5000.0)
    elif kind == "scaled":
        x = rng.standard_normal((n, d)) * (np.arange(d) + 1.0) ** -rng.uniform(0.2, 1.0)
    elif kind == "tiny":
        x = rng.standard_normal((n, d)) * 1e-18
    elif kind == "dups":
        base = rng.standard_normal((max(8, n // 16), d))
        x = base[rng.integers(0, len(base), n)]
    else:  # integer grid: many exact ties
        x = rng.integers(-3, 4, (n, d)).astype(np.float64)
    return x.astype(np.float32)


def main():
    import paper_2503_04422_b200 as P
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    rng = np.random.default_rng(seed)
    bad = 0
    for ci in range(cases):
        d = int(rng.choice([16, 17, 24, 31, 32, 40, 64, 96, 128, 200, 300]))
        n = int(rng.integers(3_000, 60_000))
        nlist = int(rng.integers(8, 200))
        nprobe = int(rng.integers(2, min(nlist, 48) + 1))
        k = int(rng.choice([1, 3, 10, 20, 32, 33, 50]))
        nq = int(rng.choice([32, 33, 64, 100, 257]))
        kind = str(rng.choice(["mixture", "offset", "scaled", "tiny", "dups", "grid"]))
        pruner = str(rng.choice(["ads", "bond"]))
        istep = int(rng.choice([1, 2, 4, 8]))
        eps0 = float(rng.choice([0.3, 1.0, 2.1, 4.0]))
        x = make(rng, n, d, kind)
        q = (x[rng.choice(n, nq)] + (0.0 if kind in ("dups", "grid") else 1.0) *
             rng.standard_normal((nq, d)).astype(np.float32) * np.float32(np.abs(x).mean() * 0.1))
        q = q.astype(np.float32)
        cent = x[rng.choice(n, nlist, replace=False)].astype(np.float64)
        x64 = x.astype(np.float64)
        d2 = (x64 * x64).sum(1)[:, None] + (cent * cent).sum(1)[None, :] - 2.0 * (x64 @ cent.T)
        index = P.IvfIndex.from_assignment(P.VectorCollection.from_array(x),
                                           cent.astype(np.float32), np.argmin(d2, axis=1),
                                           nlist=nlist)
        kw = dict(k=k, pruner=pruner, initial_step=istep)
        if pruner == "ads":
            kw["ads"] = P.AdsPruner(d=d, epsilon0=eps0)
        params = P.SearchParams(**kw)
        scan = P.ivf_search_batch(index, q, params, nprobe, batched=1)
        fast = P.ivf_search_batch(index, q, params, nprobe, batched=2)
        full = P.ivf_search_batch(index, q, params, nprobe, stats=True, batched=2)
        ok = all(np.array_equal(a["ids"], scan["ids"]) and
                 np.array_equal(a["dist"], scan["dist"], equal_nan=True) for a in (fast, full))
        if not ok:
            bad += 1
        print(f"case {ci}: d={d} n={n} nlist={nlist} nprobe={nprobe} k={k} nq={nq} {kind} "
              f"{pruner} is={istep} eps0={eps0}: {'ok' if ok else 'DIFFERENT'}", flush=True)
    print(f"{cases - bad} / {cases} identical")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
