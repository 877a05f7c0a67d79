"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the reference package ``dimscan``, feeds it the seeded inputs of
recipes.py and records its outputs: TopK items (ids and float32 distances),
SearchStats (values_touched / values_total / survivors), dimension orders,
ADS bounds, bucket selections, IVF indexes (assignments + centroids) and
bucket means.  The fixtures pin both the C oracle (tests/test_oracle.py)
and the GPU path (tests/test_gpu_parity.py).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
import recipes  # noqa: E402

import dimscan as ds  # noqa: E402  (the reference)
import dimscan.pruning  # noqa: E402,F401


def flatten_survivors(surv):
    out = []
    for rec in surv:
        out.append(len(rec))
        out.extend(int(v) for v in rec)
    return np.asarray(out, dtype=np.int32)


def run_case(blocks, q, params, orders=None):
    st = ds.SearchStats()
    tk = ds.search(blocks, q, params, orders=orders, stats=st)
    items = tk.items()
    return (np.array([i for _, i in items], np.int64), np.array([d for d, _ in items], np.float32),
            st.values_touched, st.values_total, flatten_survivors(st.survivors))


def main():
    rng = np.random.default_rng(20250304)
    arrays, manifest = {}, {"search": [], "flat": [], "ivf": [], "orders": [], "ads": []}

    # ---- block-list searches (search.py:177) over to_blocks(..., block_size)
    kinds = ["normal", "skewed", "clustered", "decay", "mixture"]
    combos = [("none", "l2"), ("none", "l1"), ("none", "ip"), ("bond", "l2"), ("bond", "l1"),
              ("ads", "l2")]
    for ci in range(72):
        kind = kinds[ci % len(kinds)]
        pruner, metric = combos[ci % len(combos)]
        n = int(rng.choice([1, 40, 64, 65, 700, 3000, 5000]))
        d = int(rng.choice([1, 3, 8, 24, 64, 100, 128, 200]))
        bs = int(rng.choice([64, 64, 64, 32, 128, 7]))
        k = int(rng.choice([1, 10, 10, 10, 100]))
        sf = float(rng.choice([0.05, 0.2, 0.2, 0.4]))
        step = int(rng.choice([1, 2, 2, 8]))
        eps = float(rng.choice([2.1, 2.1, 1.0, 0.3]))
        crit = "sequential"
        if pruner == "bond":
            crit = str(rng.choice(["sequential", "decreasing", "dmeans", "zones"]))
        seed = 1000 + ci
        x = recipes.data(kind, n, d, seed)
        Q = recipes.queries("near", x, 3, seed + 1)
        col = ds.VectorCollection.from_array(x)
        blocks = ds.to_blocks(col, bs)
        means = ds.compute_means(col).means
        params = ds.SearchParams(k=k, metric=metric, pruner=pruner, selection_fraction=sf,
                                 initial_step=step,
                                 ads=ds.AdsPruner(d=d, epsilon0=eps) if pruner == "ads" else None)
        case = dict(kind=kind, n=n, d=d, block_size=bs, k=k, metric=metric, pruner=pruner,
                    criteria=crit, sf=sf, step=step, eps=eps, seed=seed, queries=[])
        for qi, q in enumerate(Q):
            orders = None
            if crit != "sequential":
                orders = ds.bond_dimension_order(q, means, crit)
            ids, dist, touched, total, surv = run_case(blocks, q, params, orders)
            key = f"s{ci}_{qi}"
            arrays[key + "_ids"], arrays[key + "_dist"], arrays[key + "_surv"] = ids, dist, surv
            case["queries"].append(dict(key=key, touched=int(touched), total=int(total)))
        manifest["search"].append(case)

    # ---- exact_search over flat partitions (index.py:182-191)
    for fi in range(12):
        kind = ["normal", "skewed", "decay"][fi % 3]
        n = int(rng.choice([500, 2500, 6000]))
        d = int(rng.choice([16, 48, 128]))
        psize = int(rng.choice([300, 700, 2500, 10000]))
        crit = ["sequential", "decreasing", "dmeans", "zones"][fi % 4]
        pruner = "bond" if fi % 6 else "none"
        seed = 2000 + fi
        x = recipes.data(kind, n, d, seed)
        Q = recipes.queries("near", x, 3, seed + 1)
        flat = ds.flat_build(ds.VectorCollection.from_array(x), psize)
        params = ds.SearchParams(k=10, pruner=pruner)
        case = dict(kind=kind, n=n, d=d, partition_size=psize, criteria=crit, pruner=pruner,
                    seed=seed, queries=[])
        for qi, q in enumerate(Q):
            st = ds.SearchStats()
            tk = ds.exact_search(flat, q, params, criteria=crit, stats=st)
            items = tk.items()
            key = f"f{fi}_{qi}"
            arrays[key + "_ids"] = np.array([i for _, i in items], np.int64)
            arrays[key + "_dist"] = np.array([v for v, _ in items], np.float32)
            arrays[key + "_surv"] = flatten_survivors(st.survivors)
            case["queries"].append(dict(key=key, touched=int(st.values_touched),
                                        total=int(st.values_total)))
        manifest["flat"].append(case)

    # ---- IVF: reference k-means index + ivf_search (index.py:91-156)
    for ii in range(6):
        kind = ["mixture", "clustered", "skewed"][ii % 3]
        n = [3000, 5000, 2000, 4000, 3000, 2500][ii]
        d = [32, 16, 64, 24, 128, 8][ii]
        nlist = [20, 40, 15, 30, 12, 25][ii]
        seed = 3000 + ii
        x = recipes.data(kind, n, d, seed)
        Q = recipes.queries("near", x, 4, seed + 1)
        col = ds.VectorCollection.from_array(x)
        index = ds.ivf_build(col, nlist=nlist, seed=ii)
        assign = np.full(n, -1, np.int32)
        for c, chain in enumerate(index.buckets):
            for b in chain:
                assign[b.ids] = c
        key = f"i{ii}"
        arrays[key + "_assign"] = assign
        arrays[key + "_centroids"] = index.centroids.astype(np.float32)
        arrays[key + "_means"] = np.stack(index.bucket_means).astype(np.float64)
        case = dict(kind=kind, n=n, d=d, nlist=nlist, seed=seed, runs=[])
        for ri, (pruner, crit, nprobe, eps) in enumerate([
                ("none", "sequential", 3, 2.1), ("ads", "sequential", 5, 2.1),
                ("ads", "sequential", nlist, 1.0), ("bond", "dmeans", 4, 2.1),
                ("bond", "zones", 6, 2.1), ("bond", "decreasing", nlist, 2.1),
                ("ads", "sequential", 8, 0.5)]):
            params = ds.SearchParams(k=10, pruner=pruner, ads=ds.AdsPruner(d=d, epsilon0=eps))
            for qi, q in enumerate(Q):
                st = ds.SearchStats()
                tk = ds.ivf_search(index, q, params, nprobe, criteria=crit, stats=st)
                items = tk.items()
                rk = f"{key}_{ri}_{qi}"
                arrays[rk + "_ids"] = np.array([i for _, i in items], np.int64)
                arrays[rk + "_dist"] = np.array([v for v, _ in items], np.float32)
                arrays[rk + "_surv"] = flatten_survivors(st.survivors)
                arrays[rk + "_sel"] = ds.ivf_select_buckets(index, q, nprobe).astype(np.int32)
                case["runs"].append(dict(key=rk, q=qi, pruner=pruner, criteria=crit,
                                         nprobe=nprobe, eps=eps, touched=int(st.values_touched),
                                         total=int(st.values_total)))
        manifest["ivf"].append(case)

    # ---- dimension orders (pruning.py:107-140)
    for oi in range(40):
        d = int(rng.choice([1, 2, 5, 8, 16, 100, 128, 300, 768]))
        crit = ["decreasing", "dmeans", "zones", "zones"][oi % 4]
        zw = None if oi % 8 < 4 else int(rng.choice([1, 3, 8, 60, 200]))
        q = rng.standard_normal(d)
        if oi % 5 == 0:
            q = np.round(q, 1)  # ties
        mu = rng.standard_normal(d) * 0.5
        if oi % 7 == 0:
            mu = np.zeros(d)
        o = ds.bond_dimension_order(q, mu, crit, zw)
        key = f"o{oi}"
        arrays[key + "_q"], arrays[key + "_mu"], arrays[key + "_order"] = q, mu, o.astype(np.int32)
        manifest["orders"].append(dict(key=key, criteria=crit, zone_width=zw))

    # ---- ADS bounds (pruning.py:83-88) and their float32 rounding
    rows = []
    for _ in range(400):
        D = int(rng.integers(1, 2000))
        ds_ = int(rng.integers(1, D + 3))
        eps = float(rng.choice([2.1, 1.0, 0.5, 3.3]))
        T = float(np.float32(np.exp(rng.uniform(-5, 12))))
        b = ds.pruning.ads_bound(ds_, ds.AdsPruner(d=D, epsilon0=eps), T)
        rows.append((D, ds_, eps, T, b, float(np.float32(b))))
    arrays["ads_bounds"] = np.array(rows, dtype=np.float64)

    # ---- orthogonal matrices (pruning.py:36-45)
    for d, seed in [(16, 3), (64, 7), (128, 0)]:
        arrays[f"orth_{d}_{seed}"] = ds.generate_orthogonal(d, seed).matrix

    np.savez_compressed(HERE / "reference_golden.npz", **arrays)
    (HERE / "reference_golden.json").write_text(json.dumps(manifest, indent=1))
    print(f"wrote {len(arrays)} arrays")


if __name__ == "__main__":
    main()
