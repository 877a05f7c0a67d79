"""The owning native handle (pdx_index_*): one C call per query batch must
return exactly what the per-kernel Python path and the oracle return."""
from pathlib import Path

import numpy as np
import pytest

import paper_2503_04422_b200 as P
from paper_2503_04422_b200 import _lib

GOLD = Path(__file__).resolve().parent / "golden" / "pdx"


def test_handle_symbols_exported():
    L = _lib.lib()
    for name in ("pdx_index_create", "pdx_index_open", "pdx_index_destroy", "pdx_index_search"):
        assert hasattr(L, name)


@pytest.mark.gpu
@pytest.mark.parametrize("pruner,criteria", [("bond", "dmeans"), ("bond", "zones"),
                                             ("ads", "sequential"), ("none", "sequential")])
def test_open_pdx_matches_python_path_and_oracle(oracle, pruner, criteria):
    st = P.read_pdx(GOLD / "ivf.pdx")
    group = 1 if criteria != "sequential" else 8
    h = P.PdxIndex.open(GOLD / "ivf.pdx", group=group)
    Q = np.random.default_rng(3).standard_normal((40, st.d)).astype(np.float32)
    out = h.search(Q, k=7, pruner=pruner, criteria=criteria, nprobe=5, stats=True)
    idx = P.load_index(GOLD / "ivf.pdx", group=group)
    ref = P.ivf_search_batch(idx, Q, P.SearchParams(k=7, pruner=pruner), 5, criteria=criteria,
                             stats=True)
    np.testing.assert_array_equal(out["ids"].numpy(), ref["ids"])
    np.testing.assert_array_equal(out["dist"].numpy(), ref["dist"])
    np.testing.assert_array_equal(out["touched"].numpy(), ref["touched"])
    chains = [st.blocks[int(st.ivf.bucket_offsets[c]):int(st.ivf.bucket_offsets[c + 1])]
              for c in range(st.ivf.nlist)]
    view = oracle.IvfView(P.to_blocks(P.VectorCollection.from_array(st.ivf.centroids), 64),
                          chains, st.ivf.bucket_means)
    o = oracle.ivf_search_batch(view, Q, 7, 5, pruner=pruner, criteria=criteria)
    np.testing.assert_array_equal(out["ids"].numpy(), o["ids"])
    np.testing.assert_array_equal(out["touched"].numpy(), o["touched"])
    h.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["flat64.pdx", "wide.pdx", "flat128.pdx"])
def test_from_host_blocks_exact_vs_oracle(oracle, name):
    st = P.read_pdx(GOLD / name)
    h = P.PdxIndex.from_blocks(st.blocks, global_means=st.global_means, group=1)
    Q = np.random.default_rng(5).standard_normal((16, st.d)).astype(np.float32)
    out = h.search(Q, k=5, pruner="bond", criteria="dmeans", stats=True)
    ref = oracle.exact_search_batch(st.blocks, st.global_means, Q, 5, pruner="bond",
                                    criteria="dmeans")
    np.testing.assert_array_equal(out["ids"].numpy(), ref["ids"])
    np.testing.assert_array_equal(out["dist"].numpy(), ref["dist"])
    np.testing.assert_array_equal(out["touched"].numpy(), ref["touched"])


@pytest.mark.gpu
def test_borrowed_index_rotation_bsa_and_device_outputs():
    import torch
    x = np.random.default_rng(8).standard_normal((20_000, 48)).astype(np.float32)
    Q = x[:100] + 0.05 * np.random.default_rng(9).standard_normal((100, 48)).astype(np.float32)
    T = P.generate_orthogonal(48, 0)
    xr = P.apply_transform(T, x)
    idx = P.ivf_build(P.VectorCollection.from_array(xr), nlist=64, seed=0)
    h = P.PdxIndex.from_index(idx, transform=T)
    params = P.SearchParams(k=10, pruner="ads")
    ref = P.ivf_search_batch(idx, P.apply_transform(T, Q), params, 12, stats=True)
    out = h.search(Q, k=10, pruner="ads", nprobe=12, rotate=True, stats=True)
    # the handle projects with the same K3 kernel, so the decisions match
    np.testing.assert_array_equal(out["ids"].numpy(), ref["ids"])
    np.testing.assert_array_equal(out["touched"].numpy(), ref["touched"])
    bsa = P.fit_bsa(torch.from_numpy(xr).cuda())
    ref_b = P.ivf_search_batch(idx, P.apply_transform(T, Q),
                               P.SearchParams(k=10, pruner="bsa", bsa=bsa), 12, stats=True)
    Qd = torch.from_numpy(P.apply_transform(T, Q)).cuda()
    out_b = h.search(Qd, k=10, pruner="bsa", bsa=bsa, nprobe=12, stats=True)
    assert out_b["ids"].is_cuda
    np.testing.assert_array_equal(out_b["ids"].cpu().numpy(), ref_b["ids"])
    np.testing.assert_array_equal(out_b["touched"].cpu().numpy(), ref_b["touched"])
    with pytest.raises(ValueError, match="nprobe"):
        h.search(Q, k=10, nprobe=65)
    h.close()


@pytest.mark.gpu
@pytest.mark.parametrize("metric", ["ip", "l2"])
def test_handle_tensor_core_path_identical(metric):
    """pdx_index_search routes large exact batches through K8 (cuBLAS TF32 +
    exact rescoring inside the library): identical to the scan."""
    rng = np.random.default_rng(12)
    x = rng.standard_normal((40_000, 64)).astype(np.float32)
    Q = rng.standard_normal((128, 64)).astype(np.float32)
    blocks = P.to_blocks(P.VectorCollection.from_array(x), 64)
    h = P.PdxIndex.from_blocks(blocks, group=8)
    a = h.search(Q, k=20, metric=metric, stats=True, tensor_cores=True)
    b = h.search(Q, k=20, metric=metric, stats=True, tensor_cores=False)
    for key in ("ids", "dist", "touched", "total"):
        np.testing.assert_array_equal(a[key].numpy(), b[key].numpy())
    flat = P.flat_build(P.VectorCollection.from_array(x), 64)
    hb = P.PdxIndex.from_index(flat)  # borrowed store, same path
    c = hb.search(Q, k=20, metric=metric, tensor_cores=True)
    np.testing.assert_array_equal(c["ids"].numpy(), b["ids"].numpy())


@pytest.mark.gpu
def test_handle_graph_replay_identical():
    """Repeated calls with the same page-locked buffers are captured into a
    CUDA graph and replayed (pdx_index_search): every call's ids, distances
    and stats equal the first (direct) call's, across a parameter change."""
    import torch
    rng = np.random.default_rng(21)
    x = rng.standard_normal((30_000, 32)).astype(np.float32)
    idx = P.ivf_build(P.VectorCollection.from_array(x), nlist=64, seed=0)
    h = P.PdxIndex.from_index(idx)
    Q = torch.from_numpy(x[:64] + 0.1 * rng.standard_normal((64, 32)).astype(np.float32))
    Q = Q.pin_memory()
    out = {"dist": torch.empty((64, 10), dtype=torch.float32).pin_memory(),
           "ids": torch.empty((64, 10), dtype=torch.int64).pin_memory(),
           "touched": torch.empty((64,), dtype=torch.int64).pin_memory(),
           "total": torch.empty((64,), dtype=torch.int64).pin_memory()}
    for nprobe, pruner in ((12, "ads"), (6, "bond"), (12, "ads")):
        first = None
        for _ in range(4):  # direct, capture, replay, replay
            h.search(Q, k=10, pruner=pruner, nprobe=nprobe, stats=True, out=out)
            got = {key: v.clone() for key, v in out.items()}
            if first is None:
                first = got
                ref = P.ivf_search_batch(idx, Q.numpy(), P.SearchParams(k=10, pruner=pruner),
                                         nprobe, stats=True)
                np.testing.assert_array_equal(got["ids"].numpy(), ref["ids"])
                np.testing.assert_array_equal(got["touched"].numpy(), ref["touched"])
            for key in first:
                assert torch.equal(got[key], first[key]), key
    h.close()


@pytest.mark.gpu
def test_handle_graph_not_replayed_after_realloc():
    """A, A (captured), a larger B (the handle's scratch buffers are
    reallocated), then A again: the captured graph of A holds the old
    buffers' pointers, so it must not be replayed (the graph key carries the
    buffer generation); every A answer equals the first."""
    import torch
    rng = np.random.default_rng(22)
    x = rng.standard_normal((40_000, 48)).astype(np.float32)
    idx = P.ivf_build(P.VectorCollection.from_array(x), nlist=100, seed=0)
    h = P.PdxIndex.from_index(idx)

    def bufs(nq, k):
        Q = torch.from_numpy(x[:nq] + 0.1 * rng.standard_normal((nq, 48)).astype(np.float32))
        return Q.pin_memory(), {"dist": torch.empty((nq, k), dtype=torch.float32).pin_memory(),
                                "ids": torch.empty((nq, k), dtype=torch.int64).pin_memory()}
    qa, oa = bufs(64, 10)
    qb, ob = bufs(1024, 100)
    first = None
    for call in ("A", "A", "A", "B", "A", "A", "A", "B", "B", "A"):
        if call == "B":
            h.search(qb, k=100, pruner="ads", nprobe=40, out=ob)
            continue
        h.search(qa, k=10, pruner="ads", nprobe=12, out=oa)
        got = (oa["ids"].clone(), oa["dist"].clone())
        if first is None:
            first = got
        assert torch.equal(got[0], first[0]) and torch.equal(got[1], first[1])
    ref = P.ivf_search_batch(idx, qa.numpy(), P.SearchParams(k=10, pruner="ads"), 12)
    np.testing.assert_array_equal(first[0].numpy(), ref["ids"])
    h.close()
