"""File formats (storage.py of the reference).

CPU: the .pdx golden files written by the REFERENCE's write_pdx
(tests/golden/make_pdx_golden.py) are probed natively and read on the host
exactly as the reference read them back; the host writer reproduces their
bytes; framing errors raise the reference's FormatError / OSError.
GPU (marked): the native loader streams them into HBM and the native saver
writes the identical bytes back; searches over a loaded index equal the
oracle's over the same blocks.
"""
import hashlib
import json
import struct
from pathlib import Path

import numpy as np
import pytest

import paper_2503_04422_b200 as P
from conftest import decode_survivors  # noqa: F401

GOLD = Path(__file__).resolve().parent / "golden" / "pdx"
CASES = json.loads((GOLD / "pdx_golden.json").read_text())


@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_pdx_host_read_and_write(name, tmp_path):
    want = CASES[name]
    path = GOLD / name
    info = P.probe(path)
    assert (info["n"], info["d"], info["nblocks"], info["nlist"]) == \
        (want["n"], want["d"], want["nblocks"], want["nlist"])
    assert info["ntiles"] == sum((m + 63) // 64 for m in want["m"])
    st = P.read_pdx(path)
    assert st.n == want["n"] and st.block_size == want["block_size"]
    assert st.transform_seed == want["transform_seed"]
    assert [b.m for b in st.blocks] == want["m"]
    assert [b.data.shape[1] for b in st.blocks] == want["m_padded"]
    assert [[int(i) for i in b.ids] for b in st.blocks] == want["ids"]
    assert [hashlib.sha256(np.ascontiguousarray(b.data).tobytes()).hexdigest()
            for b in st.blocks] == want["data_sha256"]
    if want["nlist"]:
        assert [int(v) for v in st.ivf.bucket_offsets] == want["bucket_offsets"]
    out = tmp_path / "again.pdx"
    P.write_pdx(st, out)
    assert out.read_bytes() == path.read_bytes()


def _corrupt(tmp_path, name, mutate):
    raw = bytearray((GOLD / "flat64.pdx").read_bytes())
    raw = mutate(raw)
    p = tmp_path / name
    p.write_bytes(bytes(raw))
    return p


def test_pdx_framing_errors(tmp_path):
    bad = _corrupt(tmp_path, "bad.pdx", lambda r: b"NOTPDX00" + r[8:])
    with pytest.raises(P.FormatError, match="magic"):
        P.read_pdx(bad)
    ver = _corrupt(tmp_path, "ver.pdx", lambda r: r[:8] + struct.pack("<I", 9) + r[12:])
    with pytest.raises(P.FormatError, match="version"):
        P.probe(ver)
    cut = _corrupt(tmp_path, "cut.pdx", lambda r: r[:-10])
    with pytest.raises(P.FormatError, match="truncated"):
        P.read_pdx(cut)
    lie = _corrupt(tmp_path, "lie.pdx", lambda r: r[:16] + struct.pack("<Q", 131) + r[24:])
    with pytest.raises(P.FormatError, match="header claims 131 vectors"):
        P.probe(lie)
    with pytest.raises(OSError):
        P.probe(tmp_path / "missing.pdx")
    assert issubclass(P.FormatError, ValueError)


def test_vecs_round_trip_and_errors(tmp_path):
    x = np.random.default_rng(0).standard_normal((37, 5)).astype(np.float32)
    p = tmp_path / "a.fvecs"
    P.write_fvecs(P.VectorCollection.from_array(x), p)
    np.testing.assert_array_equal(P.read_fvecs(p).data, x)
    ids = np.arange(30, dtype=np.int32).reshape(6, 5)
    pi = tmp_path / "a.ivecs"
    P.write_ivecs(ids, pi)
    np.testing.assert_array_equal(P.read_ivecs(pi), ids)
    (tmp_path / "empty.fvecs").write_bytes(b"")
    with pytest.raises(P.FormatError, match="no records"):
        P.read_fvecs(tmp_path / "empty.fvecs")
    raw = p.read_bytes()
    (tmp_path / "cut.fvecs").write_bytes(raw[:-3])
    with pytest.raises(P.FormatError, match="truncated record"):
        P.read_fvecs(tmp_path / "cut.fvecs")
    rec = 4 + 4 * 5
    mixed = raw[:rec] + struct.pack("<I", 4) + raw[rec + 4:]
    (tmp_path / "mixed.fvecs").write_bytes(mixed)
    with pytest.raises(P.FormatError, match="inconsistent dimensionality 4 at record 1"):
        P.read_fvecs(tmp_path / "mixed.fvecs")


# ------------------------------------------------------------------ GPU
def _oracle_view(oracle, st):
    ivf = st.ivf
    chains = [st.blocks[int(ivf.bucket_offsets[c]):int(ivf.bucket_offsets[c + 1])]
              for c in range(ivf.nlist)]
    cent = P.to_blocks(P.VectorCollection.from_array(ivf.centroids), st.block_size)
    return oracle.IvfView(cent, chains, ivf.bucket_means)


@pytest.mark.gpu
@pytest.mark.parametrize("group", [1, 8])
@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_pdx_device_round_trip(name, group, tmp_path):
    idx = P.load_index(GOLD / name, group=group)
    out = tmp_path / "dev.pdx"
    P.save_index(idx, out)
    assert out.read_bytes() == (GOLD / name).read_bytes()


@pytest.mark.gpu
@pytest.mark.parametrize("pruner,criteria", [("bond", "dmeans"), ("none", "sequential"),
                                             ("ads", "sequential")])
def test_loaded_ivf_search_vs_oracle(oracle, pruner, criteria):
    st = P.read_pdx(GOLD / "ivf.pdx")
    idx = P.load_index(GOLD / "ivf.pdx", group=1 if criteria != "sequential" else 8)
    rng = np.random.default_rng(3)
    Q = rng.standard_normal((40, st.d)).astype(np.float32)
    params = P.SearchParams(k=7, pruner=pruner)
    out = P.ivf_search_batch(idx, Q, params, 5, criteria=criteria, trace=True)
    ref = oracle.ivf_search_batch(_oracle_view(oracle, st), Q, 7, 5, pruner=pruner,
                                  criteria=criteria, survivors_cap=1 << 16)
    np.testing.assert_array_equal(out["selected"], ref["selected"])
    np.testing.assert_array_equal(out["ids"], ref["ids"])
    np.testing.assert_array_equal(out["dist"], ref["dist"])
    np.testing.assert_array_equal(out["touched"], ref["touched"])
    assert out["survivors"] == ref["survivor_lists"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["flat64.pdx", "flat128.pdx", "wide.pdx"])
def test_loaded_flat_search_vs_oracle(oracle, name):
    st = P.read_pdx(GOLD / name)
    part = P.load_index(GOLD / name, group=1)
    Q = np.random.default_rng(4).standard_normal((24, st.d)).astype(np.float32)
    params = P.SearchParams(k=5, pruner="bond")
    out = P.exact_search_batch(part, Q, params, criteria="dmeans", trace=True)
    ref = oracle.exact_search_batch(st.blocks, st.global_means, Q, 5, pruner="bond",
                                    criteria="dmeans", survivors_cap=1 << 16)
    np.testing.assert_array_equal(out["ids"], ref["ids"])
    np.testing.assert_array_equal(out["dist"], ref["dist"])
    np.testing.assert_array_equal(out["touched"], ref["touched"])
    assert out["survivors"] == ref["survivor_lists"]


@pytest.mark.gpu
def test_gpu_built_index_saves_reference_layout(tmp_path):
    """An ivf_build index saved from HBM reads back (host) as the same
    bucket chains, means and centroids; reloading it searches identically."""
    x = np.random.default_rng(9).standard_normal((5000, 24)).astype(np.float32)
    col = P.VectorCollection.from_array(x)
    idx = P.ivf_build(col, nlist=40, seed=2)
    p = tmp_path / "built.pdx"
    P.save_index(idx, p)
    st = P.read_pdx(p)
    flat = [b for chain in idx.buckets for b in chain]
    assert len(st.blocks) == len(flat)
    for a, b in zip(st.blocks, flat):
        assert a.m == b.m
        np.testing.assert_array_equal(a.ids, b.ids)
        np.testing.assert_array_equal(a.data, b.data)
    np.testing.assert_array_equal(st.ivf.centroids, idx.centroids)
    np.testing.assert_array_equal(st.ivf.bucket_means, np.stack(idx.bucket_means))
    allv = P.from_blocks(flat)
    np.testing.assert_array_equal(st.global_means, allv.data.astype(np.float64).sum(0) / allv.n)
    back = P.load_index(p)
    Q = x[:64] + 0.01
    params = P.SearchParams(k=10, pruner="bond")
    a = P.ivf_search_batch(idx, Q, params, 6, stats=True)
    b = P.ivf_search_batch(back, Q, params, 6, stats=True)
    for key in ("ids", "dist", "touched"):
        np.testing.assert_array_equal(a[key], b[key])
