"""Noise floor of the CPU oracle on a given input (TEST INFRASTRUCTURE ONLY, like the oracle itself).

Three probes of how far the reference's *own* answer moves when nothing mathematical changes:

* ``gesvd``: the same solve with LAPACK dgesvd instead of dgesdd.  Both drivers share the
  bidiagonalisation (dgebrd); only the bidiagonal SVD differs, so this probe does not see the rounding of dgebrd
  and underestimates the distance of the reference from the exact answer (measured on cfg3 rows against an 80-bit
  one-sided Jacobi SVD: dgesdd and dgesvd are both 1.1e-9 from the exact T, and 1.2e-12 from each other).
* ``perm``: the ensemble members (columns of X and Ys) in a different order.  T, D and the analysis (un-permuted)
  are mathematically identical; every rounding error of the reference's path changes.
* ``solver``: the local analysis system solved by LU (dgesv) instead of Cholesky (dpotrf / dpotrs).  Only the analysis
  moves; it matters where A = T^T D^-1 T + H^T R^-1 H is numerically singular (many D on the variance floor: more
  predecessors than members), the regime in which the elimination order decides what the answer is.

The parity gates of the GPU tests are max(north_star gate, 10 x floor) with floor = the largest of the probes
(tests/golden/noise_floors.json, written by tools/make_floors.py from this module).
"""

from __future__ import annotations

import numpy as np

from . import enkf_mc_oracle as orc


def _run(X2d, obs, r, Ys, grid, zeta, tiles, csrs):
    out = []
    for t, c in zip(tiles, csrs):
        out.append(orc.analyse_tile(X2d, obs, r, Ys, grid, zeta, t, c))
    return out


def _diff(base, other, unperm=None):
    t_num = t_den = x_num = x_den = 0.0
    d_max = 0.0
    for a, b in zip(base, other):
        t_num += np.sum((a.factors.data - b.factors.data) ** 2)
        t_den += np.sum(a.factors.data ** 2)
        d_max = max(d_max, float(np.max(np.abs(a.factors.d - b.factors.d) / a.factors.d)))
        pos = a.tile.interior_positions()
        xa, xb = a.xa_local[pos], b.xa_local[pos]
        if unperm is not None:
            xb = xb[:, unperm]
        x_num += np.sum((xa - xb) ** 2)
        x_den += np.sum(xa ** 2)
    return float(np.sqrt(t_num / max(t_den, 1e-300))), d_max, float(np.sqrt(x_num / max(x_den, 1e-300)))


def floors(X2d, obs_idx, r_diag, Ys, grid: orc.Grid, delta: int, zeta: int, tile_ids=None, seed: int = 7):
    """{probe: (T norm-wise, D max relative, Xa norm-wise over the tiles' interiors)} for one 2-D field."""
    tiles = orc.decompose(grid, delta, zeta)
    if tile_ids is not None:
        tiles = [tiles[i] for i in tile_ids]
    csrs = [orc.predecessor_csr(grid, zeta, t.local_order) for t in tiles]
    base = _run(X2d, obs_idx, r_diag, Ys, grid, zeta, tiles, csrs)
    with orc.svd_driver("gesvd"):
        alt = _run(X2d, obs_idx, r_diag, Ys, grid, zeta, tiles, csrs)
    perm = np.random.default_rng(seed).permutation(X2d.shape[1])
    inv = np.argsort(perm)
    alt2 = _run(np.ascontiguousarray(X2d[:, perm]), obs_idx, r_diag, np.ascontiguousarray(Ys[:, perm]), grid, zeta, tiles, csrs)
    with orc.linear_solver("lu"):
        alt3 = _run(X2d, obs_idx, r_diag, Ys, grid, zeta, tiles, csrs)
    return {"gesvd": _diff(base, alt), "perm": _diff(base, alt2, inv), "solver": _diff(base, alt3)}
