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


# ------------------------------------------------------------------ BSA
# The reference names BSA but does not implement it
# (SPEC.md:14).  This build's restatement:
# data and queries are projected onto their principal axes (largest variance
# first); after schedule step s (dims [0, e_s) seen) a candidate survives iff
#     ((partial + rx_s) + rq_s) - (coef_s * sqrt(rx_s)) * sqrt(rq_s) < T
# (float32, per-op rounding), rx_s / rq_s the residual energies of vector and
# query over dims [e_s, d).  coef_s = 2 * min(m * c_s, 1) where c_s is the
# `quantile` of the residual cosine <x_r, q_r> / (|x_r| |q_r|) over (training
# query, true k-NN) pairs and m the multiplier; m -> 1 / c_s is the exact
# Cauchy-Schwarz bound.  The estimate does not depend on T, so the scan's
# speculate-and-commit exactness carries over unchanged.

@dataclass(frozen=True)
class BsaPruner:
    """Learned residual-cosine bound for PCA-projected data (L2 only)."""

    coef: tuple  # float32 coef_s per step of step_schedule(d, initial_step)
    d: int
    initial_step: int = 2
    quantile: float = 0.99
    multiplier: float = 1.0
    cosines: tuple = ()  # the learned c_s (informational)

    def __post_init__(self):
        from .search import step_schedule
        n = len(step_schedule(self.d, self.initial_step))
        if len(self.coef) != n:
            raise ValueError(f"bsa needs {n} coefficients for d={self.d}, initial_step="
                             f"{self.initial_step}; got {len(self.coef)}")
        if any(not (-2.0 <= c <= 2.0) for c in self.coef):
            raise ValueError("bsa coefficients must lie in [-2, 2]")

    def device_coef(self, device):
        """The coefficients as a float32 device tensor (cached per device)."""
        import torch
        cache = self.__dict__.setdefault("_dev", {})
        key = str(device)
        if key not in cache:
            cache[key] = torch.tensor(np.asarray(self.coef, np.float32), device=device)
        return cache[key]


def _residual_energy(v: np.ndarray, start: int) -> np.float32:
    r = np.float32(0.0)
    for x in np.asarray(v, np.float32)[start:]:
        r = np.float32(r + np.float32(x * x))
    return r


def bsa_estimate(partial: float, x, q, dims_seen: int, coef: float) -> np.float32:
    """The scan's BSA estimate for one vector (host restatement, small d)."""
    rx, rq = _residual_energy(x, dims_seen), _residual_energy(q, dims_seen)
    c = np.float32(coef)
    cx = np.float32(c * np.sqrt(rx, dtype=np.float32))
    return np.float32(np.float32(np.float32(np.float32(partial) + rx) + rq)
                      - np.float32(cx * np.sqrt(rq, dtype=np.float32)))


def bsa_should_prune(partial_l2: float, x, q, step: int, pruner: BsaPruner,
                     threshold_l2: float) -> bool:
    """The BSA test after schedule step ``step`` for vector x, query q."""
    from .search import step_schedule
    e = step_schedule(pruner.d, pruner.initial_step)[step][1]
    est = bsa_estimate(partial_l2, x, q, e, pruner.coef[step])
    return not bool(est < np.float32(threshold_l2))


def fit_pca(x, sample: int = 200_000, seed: int = 0) -> OrthogonalTransform:
    """Principal axes of ``x`` (n x d, numpy or CUDA tensor) as an orthogonal
    transform, largest variance first.  Covariance in float64 on the device
    over a seeded row sample; eigenvectors on the host (numpy eigh); each
    axis' sign fixed so its largest-magnitude entry is positive."""
    import torch
    from .store import to_device
    xt = to_device(np.asarray(x, dtype=np.float32) if not isinstance(x, torch.Tensor) else x,
                   torch.float32)
    n, d = int(xt.shape[0]), int(xt.shape[1])
    if n < 2:
        raise ValueError("pca needs at least two vectors")
    if n > sample:
        g = torch.Generator(device="cpu").manual_seed(seed)
        rows = torch.randperm(n, generator=g)[:sample].to(xt.device)
        xt = xt.index_select(0, rows)
    xs = xt.double()
    xs = xs - xs.mean(0, keepdim=True)
    cov = (xs.T @ xs / (xs.shape[0] - 1)).cpu().numpy()
    w, v = np.linalg.eigh(cov)
    v = v[:, np.argsort(-w, kind="stable")]
    v = v * np.where(v[np.abs(v).argmax(0), np.arange(d)] < 0, -1.0, 1.0)
    return OrthogonalTransform(matrix=np.ascontiguousarray(v.T).astype(np.float32), seed=-1)


def fit_bsa(x_proj, d: int | None = None, initial_step: int = 2, k: int = 10,
            quantile: float = 0.99, multiplier: float = 1.0, ntrain: int = 1000,
            seed: int = 0) -> BsaPruner:
    """Learn the BSA coefficients from projected data ``x_proj`` (CUDA tensor
    n x d): ``ntrain`` seeded rows act as training queries and their exact k
    nearest other rows (kernel K9) as the neighbours whose residual cosines
    the quantile is taken over (float64 on the device)."""
    import torch
    from .search import step_schedule
    from .synthetic import ground_truth_device
    if not 0.0 < quantile <= 1.0:
        raise ValueError("quantile must be in (0, 1]")
    if multiplier <= 0:
        raise ValueError("multiplier must be positive")
    n, dd = int(x_proj.shape[0]), int(x_proj.shape[1])
    d = dd if d is None else d
    if n < 2:
        raise ValueError("bsa training needs at least two vectors")
    g = torch.Generator(device="cpu").manual_seed(seed)
    rows = torch.randperm(n, generator=g)[:min(ntrain, n)].to(x_proj.device)
    Q = x_proj.index_select(0, rows).contiguous()
    kk = min(k + 1, n)
    ids, _ = ground_truth_device(x_proj, Q, kk)
    keep = (ids != rows[:, None]).reshape(-1)  # drop the training row itself
    X = x_proj.index_select(0, ids.reshape(-1)).double()[keep]
    Qp = Q.double().repeat_interleave(kk, 0)[keep]
    # suffix sums over dims [e, d): reverse cumulative sums
    xq = (X * Qp).flip(-1).cumsum(-1).flip(-1)
    xx = (X * X).flip(-1).cumsum(-1).flip(-1)
    qq = (Qp * Qp).flip(-1).cumsum(-1).flip(-1)
    coef, cos_q = [], []
    for _, e in step_schedule(d, initial_step):
        if e >= d:
            coef.append(0.0)  # no residual left: the estimate is the distance
            cos_q.append(1.0)
            continue
        den = (xx[:, e] * qq[:, e]).sqrt()
        ok = den > 0
        c = float(torch.quantile((xq[ok, e] / den[ok]).float(), quantile).item()) \
            if int(ok.sum()) else 1.0
        cos_q.append(c)
        coef.append(float(np.float32(2.0 * max(-1.0, min(1.0, multiplier * c)))))
    return BsaPruner(coef=tuple(coef), d=d, initial_step=initial_step, quantile=quantile,
                     multiplier=multiplier, cosines=tuple(cos_q))



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
