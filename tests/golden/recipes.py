"""Seeded synthetic inputs shared by the golden generator and the tests.

Pure numpy (no reference import), so the tests regenerate exactly the
inputs the fixtures were made from — on this container and on the GPU box.
"""
from __future__ import annotations

import numpy as np


def data(kind: str, n: int, d: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    if kind == "normal":
        x = rng.standard_normal((n, d))
    elif kind == "skewed":
        x = np.exp(rng.standard_normal((n, d)) * np.linspace(0.3, 2.5, d))
    elif kind == "clustered":
        centers = rng.standard_normal((8, d)) * 10.0
        x = centers[rng.integers(0, 8, size=n)] + rng.standard_normal((n, d))
    elif kind == "decay":  # BASELINE config 1 recipe: sigma_j = (j+1)^-0.5
        x = rng.standard_normal((n, d)) * (np.arange(d) + 1.0) ** -0.5
    elif kind == "mixture":  # BASELINE config 2 recipe: centres N(0, 4I) + N(0, I)
        c = rng.standard_normal((max(2, n // 50), d)) * 2.0
        x = c[rng.integers(0, c.shape[0], size=n)] + rng.standard_normal((n, d))
    else:
        raise ValueError(kind)
    return np.ascontiguousarray(x.astype(np.float32))


def queries(kind: str, x: np.ndarray, nq: int, seed: int) -> np.ndarray:
    """Queries near the data (a perturbed sample) or from a fresh draw."""
    rng = np.random.default_rng(seed)
    if kind == "near":
        pick = rng.choice(x.shape[0], nq, replace=x.shape[0] < nq)
        q = x[pick] + rng.standard_normal((nq, x.shape[1])).astype(np.float32) * 0.3
    else:
        q = data(kind, nq, x.shape[1], seed)
    return np.ascontiguousarray(q.astype(np.float32))
