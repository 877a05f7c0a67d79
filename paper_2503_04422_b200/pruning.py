"""Pruners, dimension orders and the orthogonal projection (pruning.py:1-140).

Scalar predicates (``ads_should_prune``, ``bond_should_prune``,
``ads_bound``) are the reference's formulas, kept on the host for callers
and tests; the scan kernel evaluates the same float64 expressions on the
device.  ``bond_dimension_order`` runs kernel K4 and ``apply_transform``
kernel K3; ``generate_orthogonal`` is build-time (seeded numpy QR, as the
reference).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib


@dataclass(frozen=True)
class OrthogonalTransform:
    """Seeded random rotation; preserves L2 distances (pruning.py:24-33)."""

    matrix: np.ndarray  # (d, d) float32
    seed: int

    @property
    def d(self) -> int:
        return self.matrix.shape[0]


def generate_orthogonal(d: int, seed: int) -> OrthogonalTransform:
    """QR of a seeded Gaussian matrix with sign fixing (pruning.py:36-45)."""
    if d < 1:
        raise ValueError("dimensionality must be >= 1")
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((d, d))
    q, r = np.linalg.qr(g)
    q = q * np.sign(np.diag(r))
    return OrthogonalTransform(matrix=q.astype(np.float32), seed=seed)


def apply_transform(transform: OrthogonalTransform, x):
    """x @ M^T on the GPU (kernel K3; pruning.py:48-53).  Accepts numpy
    (returns numpy) or a CUDA tensor (returns a CUDA tensor)."""
    import torch
    from .store import to_device
    is_np = not isinstance(x, torch.Tensor)
    xt = to_device(np.asarray(x, dtype=np.float32) if is_np else x, torch.float32)
    if xt.shape[-1] != transform.d:
        raise ValueError(f"length mismatch: {xt.shape[-1]} vs {transform.d}")
    one = xt.dim() == 1
    x2 = xt.reshape(-1, transform.d).contiguous()
    y = torch.empty_like(x2)
    m = getattr(transform, "_dev_matrix", None)
    if m is None or m.device != x2.device:
        m = to_device(transform.matrix, torch.float32)
        try:
            object.__setattr__(transform, "_dev_matrix", m)
        except (AttributeError, TypeError):
            pass
    _lib.check(_lib.lib().pdx_project(_lib.ptr(x2), x2.shape[0], transform.d, _lib.ptr(m),
                                      _lib.ptr(y), _lib.stream_handle()))
    y = y.reshape(xt.shape) if not one else y[0]
    return y.cpu().numpy() if is_np else y


@dataclass(frozen=True)
class AdsPruner:
    """Hypothesis-test pruner on rotated data, L2 only (pruning.py:56-65)."""

    d: int
    epsilon0: float = 2.1

    def __post_init__(self):
        if self.epsilon0 <= 0:
            raise ValueError("epsilon0 must be positive")


def ads_should_prune(partial_l2: float, dims_seen: int, pruner: AdsPruner,
                     threshold_l2: float) -> bool:
    """pruning.py:68-80."""
    if dims_seen < 1:
        raise ValueError("dims_seen must be >= 1")
    if dims_seen >= pruner.d:
        return partial_l2 >= threshold_l2
    ratio = dims_seen / pruner.d
    band = 1.0 + pruner.epsilon0 / math.sqrt(dims_seen)
    return partial_l2 >= threshold_l2 * ratio * band * band


def ads_bound(dims_seen: int, pruner: AdsPruner, threshold_l2: float) -> float:
    """pruning.py:83-88 (evaluated identically by the scan kernel)."""
    if dims_seen >= pruner.d:
        return threshold_l2
    band = 1.0 + pruner.epsilon0 / math.sqrt(dims_seen)
    return threshold_l2 * (dims_seen / pruner.d) * band * band


class OrderCriteria(str, Enum):
    SEQUENTIAL = "sequential"
    DECREASING = "decreasing"
    DISTANCE_TO_MEANS = "dmeans"
    DIMENSION_ZONES = "zones"


def default_zone_width(d: int) -> int:
    return min(d, max(8, d // 16))


def bond_should_prune(partial: float, threshold: float) -> bool:
    """Exact test: a partial sum at the threshold can no longer improve."""
    return partial >= threshold


def dimension_orders_device(queries, means, criteria, zone_width=None, mean_index=None, nsets=1):
    """Kernel K4 on device tensors: uint16 [nq*nsets, d] permutations."""
    import torch
    from .store import to_device
    criteria = OrderCriteria(criteria)
    Q = queries.contiguous()
    nq, d = Q.shape
    if zone_width is not None and zone_width < 1:
        raise ValueError("zone_width must be >= 1")
    mu = to_device(means, torch.float64)
    out = torch.empty((nq * nsets, d), dtype=torch.uint16, device=Q.device)
    mi = None if mean_index is None else mean_index.contiguous()
    q64 = 1 if Q.dtype == torch.float64 else 0
    if not q64:
        Q = Q.to(torch.float32)
    _lib.check(_lib.lib().pdx_dimension_orders(_lib.ptr(Q), q64, nq, d, _lib.ptr(mu), _lib.ptr(mi),
                                               nsets, _lib.CRITERIA[criteria.value],
                                               int(zone_width or 0), _lib.ptr(out),
                                               _lib.stream_handle()))
    return out


def bond_dimension_order(query, means, criteria: OrderCriteria,
                         zone_width: int | None = None) -> np.ndarray:
    """Visit-order permutation (pruning.py:107-140), computed by kernel K4."""
    import torch
    from .store import to_device
    q = np.asarray(query, dtype=np.float64)
    mu = np.asarray(means, dtype=np.float64)
    if q.shape != mu.shape:
        raise ValueError(f"length mismatch: {q.shape} vs {mu.shape}")
    criteria = OrderCriteria(criteria)
    if zone_width is not None and zone_width < 1:
        raise ValueError("zone_width must be >= 1")
    if criteria is OrderCriteria.SEQUENTIAL:
        return np.arange(q.shape[0], dtype=np.intp)
    Q = to_device(q[None, :], torch.float64)
    out = dimension_orders_device(Q, mu[None, :], criteria, zone_width)
    return out[0].cpu().numpy().astype(np.intp)
