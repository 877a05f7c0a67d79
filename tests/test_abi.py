"""The C-ABI library loads and exports every symbol include/pdx_b200.h
declares; argument validation answers without a GPU.  CPU only."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "pdx_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|float)\s+(pdx_\w+)\s*\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def L():
    from paper_2503_04422_b200 import _lib
    _lib.build()
    return _lib.lib()


def test_header_matches_binding_list():
    from paper_2503_04422_b200 import _lib
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(L):
    from paper_2503_04422_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT\s+(pdx_\w+)", out))
    for sym in declared_symbols():
        assert sym in exported, sym
        assert getattr(L, sym) is not None


def test_library_is_sm100a(L):
    from paper_2503_04422_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_errors_without_gpu(L):
    from paper_2503_04422_b200 import _lib
    assert L.pdx_abi_version() == 3
    store = _lib.PdxStore(128, 128, 8, 1, 0, 0, None, None, None, None, None, 0, 0)
    prm = _lib.PdxSearchParams(0, 0, 0, 2, 0.2, 128, 0, 2.1)  # k = 0
    out = _lib.PdxSearchOut()
    rc = L.pdx_search(C.byref(store), C.byref(prm), None, 1, None, 1, None, 0, 0, C.byref(out),
                      None, 0, None)
    assert rc == _lib.PDX_EINVAL
    assert "k must be >= 1" in _lib.last_error()
    with pytest.raises(ValueError, match="inner product"):
        prm = _lib.PdxSearchParams(10, 2, 2, 2, 0.2, 128, 0, 2.1)  # IP + bond
        _lib.check(L.pdx_search(C.byref(store), C.byref(prm), None, 1, None, 1, None, 0, 0,
                                C.byref(out), None, 0, None))
    with pytest.raises(ValueError, match="ads"):
        prm = _lib.PdxSearchParams(10, 1, 1, 2, 0.2, 128, 0, 2.1)  # L1 + ads
        _lib.check(L.pdx_search(C.byref(store), C.byref(prm), None, 1, None, 1, None, 0, 0,
                                C.byref(out), None, 0, None))
    with pytest.raises(ValueError, match="nprobe"):
        _lib.check(L.pdx_select_buckets(None, 1, 8, None, 4, 0, 5, None, None, None))
    assert L.pdx_search_workspace(C.byref(store), 10, 4) > 0


def test_product_has_no_oracle_dependency():
    """The shipped package never imports or links the oracle."""
    pkg = ROOT / "paper_2503_04422_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        text = f.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle\b|libpdx_oracle|pdx_oracle", text,
                             flags=re.M), f
