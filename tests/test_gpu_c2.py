"""The bench's headline configuration (BASELINE configs[1] = C2: 1M x 128
mixture, rotated, 1,024 buckets from the REFERENCE's k-means, ADS eps0 2.1,
K = 10) through the GPU path, compared bit for bit with

* the real reference's own outputs on a query prefix
  (tests/golden/c2_reference_prefix.npz, tools/make_c2_golden.py: dimscan's
  ivf_search on the reference-packed index), and
* the C oracle on all 1,000 queries,

at nprobe 8, 32 and 128.  C2's largest bucket holds 5,055 vectors (79
tiles), so the batched pipeline's first-bucket tail (> kP1Cap = 64 tiles,
pdx_batch.cu) is exercised; test_first_bucket_tail_path forces it on
every query."""
import numpy as np
import pytest

import recipes
from test_gpu_parity import P, _oracle_ivf  # noqa: F401 (P is a fixture)

pytestmark = pytest.mark.gpu
GOLD = recipes.__file__.rsplit("/", 1)[0] + "/c2_reference_prefix.npz"


@pytest.fixture(scope="module")
def c2(P):
    import bench
    X, Q = bench.make_data(1_000_000, 1000)
    T = P.generate_orthogonal(128, 0)
    XR, QR = X @ T.matrix.T, Q @ T.matrix.T
    cent, assign, same = bench.load_fixture(XR)
    index = P.IvfIndex.from_assignment(P.VectorCollection.from_array(XR), cent, assign,
                                       nlist=1024)
    return XR, QR, index, cent, assign, same


def _params(P):
    return P.SearchParams(k=10, pruner="ads", ads=P.AdsPruner(d=128, epsilon0=2.1))


@pytest.mark.parametrize("nprobe", [8, 32, 128])
def test_c2_prefix_equals_reference(P, c2, nprobe):
    XR, QR, index, _, _, same = c2
    if not same:
        pytest.skip("this host's BLAS rotated the data differently from the fixture's")
    g = np.load(GOLD)
    q = g["queries"]
    np.testing.assert_array_equal(q, QR[:q.shape[0]])
    out = P.ivf_search_batch(index, q, _params(P), nprobe, stats=True)
    np.testing.assert_array_equal(out["ids"], g[f"ids_{nprobe}"])
    np.testing.assert_array_equal(out["dist"], g[f"dist_{nprobe}"])
    np.testing.assert_array_equal(out["touched"], g[f"touched_{nprobe}"])
    np.testing.assert_array_equal(out["total"], g[f"total_{nprobe}"])


@pytest.mark.parametrize("nprobe", [8, 32, 128])
def test_c2_all_queries_equal_oracle(P, oracle, c2, nprobe):
    XR, QR, index, cent, assign, _ = c2
    view = oracle.IvfView.from_assignment(XR, cent, assign, 1024)
    out = P.ivf_search_batch(index, QR, _params(P), nprobe, stats=True)
    fast = P.ivf_search_batch(index, QR, _params(P), nprobe)  # results only (bverify path)
    ref = oracle.ivf_search_batch(view, QR, 10, nprobe, pruner="ads", eps0=2.1)
    np.testing.assert_array_equal(fast["ids"], ref["ids"])
    np.testing.assert_array_equal(fast["dist"], ref["dist"])
    np.testing.assert_array_equal(out["selected"], ref["selected"])
    np.testing.assert_array_equal(out["ids"], ref["ids"])
    np.testing.assert_array_equal(out["dist"], ref["dist"])
    np.testing.assert_array_equal(out["touched"], ref["touched"])
    np.testing.assert_array_equal(out["total"], ref["total"])


@pytest.mark.parametrize("pruner,eps", [("ads", 2.1), ("ads", 0.7), ("bond", 0.0)])
def test_first_bucket_tail_path(P, oracle, pruner, eps):
    """nlist 8 over 100K rows: every bucket holds ~195 tiles, so every
    query's first bucket exceeds the phase-1 cap (64 tiles) and its tail
    opens the phase-2 window — forced through the batched pipeline
    (batched = 2) and compared with the oracle incl. survivor traces."""
    x = recipes.data("mixture", 100_000, 64, 51)
    Q = recipes.queries("near", x, 48, 52)
    T = P.generate_orthogonal(64, 3)
    xr, qr = P.apply_transform(T, x), P.apply_transform(T, Q)
    index = P.ivf_build(P.VectorCollection.from_array(xr), nlist=8, seed=0)
    assert index.store.max_bucket_tiles > 64
    params = (P.SearchParams(k=10, pruner="ads", ads=P.AdsPruner(d=64, epsilon0=eps))
              if pruner == "ads" else P.SearchParams(k=10, pruner="bond"))
    for nprobe in (2, 3):
        a = P.ivf_search_batch(index, qr, params, nprobe, trace=True, batched=2)
        b = P.ivf_search_batch(index, qr, params, nprobe, trace=True, batched=1)
        ref = oracle.ivf_search_batch(_oracle_ivf(oracle, index, xr), qr, 10, nprobe,
                                      pruner=pruner, eps0=eps or 2.1, survivors_cap=1 << 20)
        for got in (a, b):
            np.testing.assert_array_equal(got["ids"], ref["ids"])
            np.testing.assert_array_equal(got["dist"], ref["dist"])
            np.testing.assert_array_equal(got["touched"], ref["touched"])
            assert got["survivors"] == ref["survivor_lists"]
