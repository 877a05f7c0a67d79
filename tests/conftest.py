import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
for p in (str(ROOT), str(GOLDEN)):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    arrays = np.load(GOLDEN / "reference_golden.npz")
    manifest = json.loads((GOLDEN / "reference_golden.json").read_text())
    return arrays, manifest


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


def decode_survivors(buf):
    out, i = [], 0
    buf = [int(v) for v in buf]
    while i < len(buf):
        ln = buf[i]
        out.append(buf[i + 1:i + 1 + ln])
        i += 1 + ln
    return out


def host_means(x):
    """compute_means (layout.py:126-132) — float64 axis-0 sum / n."""
    return x.astype(np.float64).sum(axis=0) / x.shape[0]
