"""Precision estimation by componentwise regression on the GPU (estimator.py:27-159).

Interface schema note: the container fields, argument checks and error messages in this module restate the reference's
public interface (estimator.py:64-119) on purpose -- they are what a caller (and the reference's own tests, which `match=` on the
messages) sees at the drop-in boundary.  No arithmetic of the hot path lives here; that is in csrc/ behind the C-ABI.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import device
from .errors import ConfigurationError
from .factors import PrecisionFactors
from .geometry import GridGeometry
from .plan import COL_IDX, ROW_PTR, Plan
from .validation import as_float_array, as_index_array, ensure_finite

RANK_TOLERANCE = 1e-8
VARIANCE_FLOOR = 1e-10
MEAN_ZERO_RTOL = 1e-10


def regression_solve(X_pred, target, rank_tol: float = RANK_TOLERANCE) -> np.ndarray:
    """Minimum-norm least squares of target on the rows of X_pred (estimator.py:27-43).

    Runs the K2 kernel on a two-row-pattern plan: rows 0..p-1 are the predictors, row p is
    the target regressed on all of them.
    """
    X_pred = as_float_array(X_pred, "X_pred", ndim=2)
    target = as_float_array(target, "target", ndim=1)
    if X_pred.shape[1] != target.size:
        raise ValueError(f"X_pred has {X_pred.shape[1]} columns but target has {target.size} entries")
    p = X_pred.shape[0]
    if p == 0:
        return np.zeros(0)
    if target.size < 2:
        raise ConfigurationError(f"ensemble size must be at least 2, got {target.size}")
    indptr = np.zeros(p + 2, dtype=np.int64)
    indptr[p + 1] = p
    plan = Plan.from_csr(indptr, np.arange(p, dtype=np.int64))
    dU = device.to_device(np.vstack([X_pred, target[None, :]]))
    dT, _, _ = device.regress_device(plan, dU, rank_tol, VARIANCE_FLOOR, want_flags=False)
    return -dT.cpu().numpy()[:p]


def fit_factors(U, geometry: GridGeometry, zeta: int, local_order=None, *,
                variance_floor: float = VARIANCE_FLOOR, rank_tol: float = RANK_TOLERANCE,
                return_flags: bool = False):
    """T and D from mean-removed perturbations U (estimator.py:64-159).

    Row j of T holds -beta of component local_order[j] regressed on its predecessors that
    are present in local_order; the stored pattern is exactly that set (zeros kept).
    """
    U = np.ascontiguousarray(as_float_array(U, "U", ndim=2))
    ensure_finite(U, "U")
    n, nens = U.shape
    if nens < 2:
        raise ConfigurationError(f"ensemble size must be at least 2, got {nens}")
    if getattr(geometry, "nlev", 1) != 1:
        raise ConfigurationError("stand-alone fit_factors is built for 2-D geometries (nlev = 1); vertically coupled "
                                 "fields run through assimilate_parallel")
    if local_order is None:
        local_order = np.arange(geometry.n2d, dtype=np.intp)
    local_order = as_index_array(local_order, "local_order")
    if local_order.size != n:
        raise ValueError(f"U has {n} rows but local_order has {local_order.size} entries")
    if local_order.size and local_order[-1] >= geometry.n2d:
        raise ValueError("local_order contains labels outside the geometry")
    if zeta < 0:
        raise ValueError(f"zeta must be nonnegative, got {zeta}")
    sums = np.abs(U.sum(axis=1))
    norms = np.linalg.norm(U, axis=1)
    if np.any(sums > MEAN_ZERO_RTOL * norms + 1e-300):             # estimator.py:113-119
        worst = int(np.argmax(sums - MEAN_ZERO_RTOL * norms))
        raise ValueError(f"U rows must be mean-removed; row {worst} sums to {U[worst].sum():.3e}")

    plan = Plan.local(geometry, zeta, local_order)
    indptr, indices = plan.get(ROW_PTR), plan.get(COL_IDX)
    if n == 0:
        return PrecisionFactors(sp.csr_matrix((0, 0)), np.zeros(0), variance_floor=variance_floor)
    dT, dD, dF = device.regress_device(plan, device.to_device(U), rank_tol, variance_floor, want_flags=True)
    data = dT.cpu().numpy()[: indices.size]
    lower = sp.csr_matrix((data, indices, indptr), shape=(n, n))
    factors = PrecisionFactors(lower, dD.cpu().numpy()[:n], variance_floor=variance_floor)
    if return_flags:
        return factors, dF.cpu().numpy()[:n]
    return factors
