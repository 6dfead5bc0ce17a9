"""CPU oracle for the EnKF-MC analysis step.  TEST INFRASTRUCTURE ONLY.

This module is a from-scratch numpy/scipy restatement of the reference
package's analysis hot path (``/root/reference/pkg/src/mcholkf``).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import it; the product package
``paper_1606_00807_b200`` never does (a test enforces this).

Parity pin: every function below is checked bit-for-bit (integers) or to
<= 1e-13 relative (floats; most outputs are bit-identical) against the
unmodified reference imported from ``/root/reference`` -- see
``tests/golden/make_golden.py`` (the generating script) and the fixtures it
wrote, plus the reference's own known-answer cases restated in
``tests/test_oracle.py``.

Third-party arithmetic, exactly as in the reference (not vendored there):
numpy ``linalg.svd`` (LAPACK dgesdd) and scipy ``linalg.cho_factor/cho_solve``
(dpotrf/dpotrs); reference pins only lower bounds (numpy>=1.24, scipy>=1.10,
``pkg/pyproject.toml:10-15``); this container has numpy 2.3.5 / scipy 1.18.1.

Extension beyond the reference (no reference pin, flagged "parity unpinned by
the reference" in DESIGN.md): ``nfields`` independent 2-D fields stacked in one
state vector, label = field * (nx*ny) + 2-D label.  Each field is literally a
reference problem, so the per-field arithmetic *is* pinned.  ``periodic_x`` / ``periodic_y``: one boundary flag per
axis.  ``nlev`` / ``zeta_v``: vertically coupled fields (BASELINE.json configs 3 / 5, "vertical r = 1") -- a field is
nlev stacked levels, label = level * (nx*ny) + 2-D label, the box of a component is its 2-D box on every level within
zeta_v (clipped), predecessors are the box members with a smaller label (the reference's rule, geometry.py:159-162, on
the extended box), sub-domains are the reference's 2-D tiles on every level.  The arithmetic per regression / per local
analysis is the reference's; only the integer maps are new (parity unpinned by the reference).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.linalg import cho_factor, cho_solve

RANK_TOL = 1e-8          # estimator.py:22
VARIANCE_FLOOR = 1e-10   # estimator.py:23
TAG_OBS_PERTURB = 2      # rng.py:15


# --------------------------------------------------------------------------
# geometry (geometry.py:101-222)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Grid:
    """ny rows x nx columns; mirrors GridGeometry (geometry.py:22-66)."""

    nx: int
    ny: int = 1
    row_major: bool = True
    periodic: bool = False
    nfields: int = 1
    # extension (no reference counterpart, "parity unpinned by the reference"): one flag per axis; None = `periodic`
    periodic_x: bool | None = None
    periodic_y: bool | None = None
    # extension: vertically coupled levels
    nlev: int = 1
    zeta_v: int = 0

    @property
    def px(self) -> bool:
        return self.periodic if self.periodic_x is None else self.periodic_x

    @property
    def py(self) -> bool:
        return self.periodic if self.periodic_y is None else self.periodic_y

    @property
    def n2d(self) -> int:
        return self.nx * self.ny

    @property
    def nfield(self) -> int:
        """Rows of one field's block (all levels)."""
        return self.n2d * self.nlev

    @property
    def nstate(self) -> int:
        return self.nfield * self.nfields


def grid_for(nx: int, ny: int, boundary: str, nfields: int = 1, row_major: bool = True, nlev: int = 1, zeta_v: int = 0) -> Grid:
    """Grid of a boundary name: "clipped" / "periodic" (reference), "periodic_x" / "periodic_y" (per-axis extension)."""
    if boundary in ("clipped", "periodic"):
        return Grid(nx, ny, row_major, boundary == "periodic", nfields, nlev=nlev, zeta_v=zeta_v)
    return Grid(nx, ny, row_major, False, nfields, periodic_x=boundary == "periodic_x", periodic_y=boundary == "periodic_y",
                nlev=nlev, zeta_v=zeta_v)


def _lift(grid: Grid, labels2d: np.ndarray, levels=None) -> np.ndarray:
    """2-D labels on the given levels (default: all), ascending."""
    lev = np.arange(grid.nlev, dtype=np.int64) if levels is None else np.asarray(levels, dtype=np.int64)
    return (lev[:, None] * grid.n2d + np.asarray(labels2d, dtype=np.int64)[None, :]).ravel()


def coords(grid: Grid, label: int) -> tuple[int, int]:
    """(row, col) of a 2-D label (geometry.py:112-119)."""
    if grid.row_major:
        return divmod(int(label), grid.nx)
    c, r = divmod(int(label), grid.ny)
    return r, c


def _label_grid(grid: Grid, rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
    """Sorted labels of rows x cols (geometry.py:122-129)."""
    rr = np.asarray(rows, dtype=np.int64)[:, None]
    cc = np.asarray(cols, dtype=np.int64)[None, :]
    lab = rr * grid.nx + cc if grid.row_major else cc * grid.ny + rr
    return np.sort(lab.ravel())


def axis_window(center: int, zeta: int, n: int, periodic: bool) -> np.ndarray:
    """Axis coordinates within zeta of center (geometry.py:132-135)."""
    if periodic:
        return np.unique((center + np.arange(-zeta, zeta + 1)) % n)
    return np.arange(max(0, center - zeta), min(n, center + zeta + 1))


def axis_band(lo: int, hi: int, zeta: int, n: int, periodic: bool) -> np.ndarray:
    """Axis coordinates within zeta of [lo, hi) (geometry.py:138-142)."""
    if periodic:
        return np.unique(np.arange(lo - zeta, hi + zeta) % n)
    return np.arange(max(0, lo - zeta), min(n, hi + zeta))


def local_box(grid: Grid, center: int, zeta: int) -> np.ndarray:
    """Chebyshev box members, ascending (geometry.py:145-156); with levels: on every level within zeta_v."""
    if grid.nlev > 1:
        lev, lab2 = divmod(int(center), grid.n2d)
        flat = Grid(grid.nx, grid.ny, grid.row_major, grid.periodic, 1, grid.periodic_x, grid.periodic_y)
        return _lift(grid, local_box(flat, lab2, zeta), axis_window(lev, grid.zeta_v, grid.nlev, False))
    r, c = coords(grid, center)
    return _label_grid(
        grid,
        axis_window(r, zeta, grid.ny, grid.py),
        axis_window(c, zeta, grid.nx, grid.px),
    )


def predecessors(grid: Grid, center: int, zeta: int) -> np.ndarray:
    """Box members with label < center (geometry.py:159-162)."""
    box = local_box(grid, center, zeta)
    return box[box < center]


def tiling(grid: Grid, delta: int) -> tuple[int, int]:
    """(block rows, block cols): minimise (|pr-pc|, pr) (geometry.py:179-193)."""
    best = None
    for pr in range(1, delta + 1):
        if delta % pr:
            continue
        pc = delta // pr
        if pr > grid.ny or pc > grid.nx:
            continue
        key = (abs(pr - pc), pr)
        if best is None or key < best[0]:
            best = (key, pr, pc)
    if best is None:
        raise ValueError(f"delta={delta} does not tile a {grid.ny}x{grid.nx} grid")
    return best[1], best[2]


def _bands(n: int, parts: int) -> list[tuple[int, int]]:
    """Equal bands, remainder to the last (geometry.py:195-199)."""
    base = n // parts
    out = [(i * base, (i + 1) * base) for i in range(parts - 1)]
    out.append(((parts - 1) * base, n))
    return out


@dataclass(frozen=True)
class Tile:
    id: int
    interior: np.ndarray
    halo: np.ndarray
    local_order: np.ndarray

    def interior_positions(self) -> np.ndarray:
        return np.searchsorted(self.local_order, self.interior)  # geometry.py:96-98


def decompose(grid: Grid, delta: int, zeta: int) -> list[Tile]:
    """Tiles of the 2-D grid with exact zeta-ring halos (geometry.py:165-222)."""
    pr, pc = tiling(grid, delta)
    tiles = []
    for bi, (r0, r1) in enumerate(_bands(grid.ny, pr)):
        for bj, (c0, c1) in enumerate(_bands(grid.nx, pc)):
            interior = _label_grid(grid, np.arange(r0, r1), np.arange(c0, c1))
            covered = _label_grid(
                grid,
                axis_band(r0, r1, zeta, grid.ny, grid.py),
                axis_band(c0, c1, zeta, grid.nx, grid.px),
            )
            halo = np.setdiff1d(covered, interior, assume_unique=True)
            if grid.nlev > 1:                       # the tile on every level (extension)
                interior, halo = _lift(grid, interior), _lift(grid, halo)
            tiles.append(Tile(bi * pc + bj, interior, halo, np.union1d(interior, halo)))
    return tiles


def predecessor_csr(grid: Grid, zeta: int, local_order: np.ndarray):
    """CSR (indptr, indices) of local predecessor positions.

    Row j lists, ascending, the local positions of predecessors(local_order[j])
    that are present in local_order (estimator.py:123-131).  Vectorised, but the
    sets are those of the per-row reference loop (checked in the golden tests).
    """
    lo = np.asarray(local_order, dtype=np.int64)
    n = lo.size
    if grid.nlev > 1:                               # levels (extension): the per-row loop of estimator.py:123-131 as it stands
        indptr, cols = np.zeros(n + 1, dtype=np.int64), []
        for j in range(n):
            pred = predecessors(grid, int(lo[j]), zeta)
            pos = np.searchsorted(lo, pred)
            ok = (pos < n) & (lo[np.minimum(pos, n - 1)] == pred)
            cols.append(pos[ok])
            indptr[j + 1] = indptr[j] + int(ok.sum())
        return indptr, (np.concatenate(cols) if cols else np.zeros(0)).astype(np.int64)
    if n == 0 or zeta == 0:
        return np.zeros(n + 1, dtype=np.int64), np.zeros(0, dtype=np.int64)
    if grid.row_major:
        r, c = np.divmod(lo, grid.nx)
    else:
        c, r = np.divmod(lo, grid.ny)
    off = np.arange(-zeta, zeta + 1)
    rr = (r[:, None, None] + off[None, :, None]) + 0 * off[None, None, :]
    cc = (c[:, None, None] + off[None, None, :]) + 0 * off[None, :, None]
    ok = np.ones(rr.shape, dtype=bool)
    if grid.py:
        rr %= grid.ny
    else:
        ok &= (rr >= 0) & (rr < grid.ny)
    if grid.px:
        cc %= grid.nx
    else:
        ok &= (cc >= 0) & (cc < grid.nx)
    lab = np.where(grid.row_major, rr * grid.nx + cc, cc * grid.ny + rr)
    ok &= lab < lo[:, None, None]
    row_id = np.broadcast_to(np.arange(n)[:, None, None], lab.shape)[ok]
    lab = lab[ok]
    # de-duplicate wrapped repeats, sort by (row, label)
    key = np.unique(row_id * np.int64(grid.n2d) + lab)
    row_id, lab = np.divmod(key, np.int64(grid.n2d))
    pos = np.searchsorted(lo, lab)
    present = (pos < n) & (lo[np.minimum(pos, n - 1)] == lab)
    row_id, pos = row_id[present], pos[present]
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(indptr, row_id + 1, 1)
    return np.cumsum(indptr), pos.astype(np.int64)


# --------------------------------------------------------------------------
# observations (kernels.py:90-144, rng.py:22-32)
# --------------------------------------------------------------------------
def restrict_observations(obs_indices: np.ndarray, members: np.ndarray):
    """(local positions, surviving parent rows) (kernels.py:90-113)."""
    obs_indices = np.asarray(obs_indices, dtype=np.int64)
    members = np.asarray(members, dtype=np.int64)
    if members.size == 0:
        z = np.zeros(0, dtype=np.int64)
        return z, z
    idx = np.searchsorted(members, obs_indices)
    inside = (idx < members.size) & (members[np.minimum(idx, members.size - 1)] == obs_indices)
    return idx[inside], np.flatnonzero(inside)


def perturb_observations(y, r_diag, nens: int, seed: int, cycle: int = 0) -> np.ndarray:
    """Ys = y + sqrt(r) * N(0,1), obs-major draw (kernels.py:130-144, rng.py:32)."""
    g = np.random.default_rng([int(seed) & ((1 << 64) - 1), int(cycle), TAG_OBS_PERTURB])
    noise = g.standard_normal((len(y), nens))
    return np.asarray(y, float)[:, None] + np.sqrt(np.asarray(r_diag, float))[:, None] * noise


# --------------------------------------------------------------------------
# estimation (validation.py:35-39, estimator.py:46-159, factors.py:39-64)
# --------------------------------------------------------------------------
def center_rows(X: np.ndarray) -> np.ndarray:
    """Row means removed twice (validation.py:35-39)."""
    U = X - X.mean(axis=1, keepdims=True)
    U -= U.mean(axis=1, keepdims=True)
    return U


_SVD_DRIVER = ["gesdd"]      # what the reference calls (numpy.linalg.svd); "gesvd" only for the noise-floor probe


class svd_driver:
    """Context manager for the noise-floor probe of SURVEY.md section 8c: the same solve with LAPACK dgesvd
    (scipy.linalg.svd, lapack_driver="gesvd", item by item) instead of the reference's dgesdd."""

    def __init__(self, name: str):
        assert name in ("gesdd", "gesvd")
        self.name = name

    def __enter__(self):
        self.prev = _SVD_DRIVER[0]
        _SVD_DRIVER[0] = self.name

    def __exit__(self, *exc):
        _SVD_DRIVER[0] = self.prev


def _batched_svd(A: np.ndarray):
    if _SVD_DRIVER[0] == "gesdd":
        return np.linalg.svd(A, full_matrices=False)       # estimator.py:53
    from scipy.linalg import svd as _svd
    k, p, m = A.shape
    r = min(p, m)
    u, s, vt = np.empty((k, p, r)), np.empty((k, r)), np.empty((k, r, m))
    for i in range(k):
        u[i], s[i], vt[i] = _svd(A[i], full_matrices=False, lapack_driver="gesvd")
    return u, s, vt


def svd_min_norm(A: np.ndarray, y: np.ndarray, rank_tol: float = RANK_TOL):
    """Batched truncated-SVD minimum-norm LS (estimator.py:46-61).

    A: (k, p, m), y: (k, m) -> beta (k, p), residual (k, m).
    """
    u, s, vt = _batched_svd(A)
    tol = rank_tol * s[:, :1]
    with np.errstate(divide="ignore", invalid="ignore"):
        inv_s = np.where((s >= tol) & (s > 0), 1.0 / s, 0.0)
    proj = np.einsum("krm,km->kr", vt, y)
    beta = np.einsum("kpr,kr->kp", u, proj * inv_s)
    resid = y - np.einsum("kpm,kp->km", A, beta)
    return beta, resid


@dataclass
class Factors:
    """Strictly-lower CSR of T (values = -beta) and floored D."""

    indptr: np.ndarray
    indices: np.ndarray
    data: np.ndarray
    d: np.ndarray
    d_raw: np.ndarray

    @property
    def n(self) -> int:
        return self.d.size

    def dense_unit_lower(self) -> np.ndarray:
        t = np.eye(self.n)
        rows = np.repeat(np.arange(self.n), np.diff(self.indptr))
        t[rows, self.indices] = self.data
        return t


def fit_factors(U, grid: Grid, zeta: int, local_order=None,
                variance_floor: float = VARIANCE_FLOOR, rank_tol: float = RANK_TOL,
                csr=None) -> Factors:
    """T and D of one (sub)domain (estimator.py:64-159).

    ``csr`` may carry a precomputed (indptr, indices) predecessor pattern (the
    multi-field driver shares it across fields).
    """
    U = np.asarray(U, dtype=np.float64)
    n, nens = U.shape
    if local_order is None:
        local_order = np.arange(grid.nfield, dtype=np.int64)
    indptr, indices = csr if csr is not None else predecessor_csr(grid, zeta, local_order)
    counts = np.diff(indptr)
    d = np.empty(n)
    data = np.zeros(indices.size)
    for p in np.unique(counts):                      # ascending, estimator.py:137
        rows = np.flatnonzero(counts == p)
        if p == 0:
            blk = U[rows]
            d[rows] = np.einsum("km,km->k", blk, blk) / (nens - 1)   # :141
            continue
        gather = indptr[rows][:, None] + np.arange(p)[None, :]
        A = U[indices[gather]]                        # (k, p, N), estimator.py:145
        y = U[rows]
        beta, resid = svd_min_norm(A, y, rank_tol)
        d[rows] = np.einsum("km,km->k", resid, resid) / (nens - 1)   # :148
        data[gather] = -beta                          # :150
    return Factors(indptr, indices, data, np.maximum(d, variance_floor), d)  # factors.py:60


# --------------------------------------------------------------------------
# local analysis (factors.py:136-145, kernels.py:163-218)
# --------------------------------------------------------------------------
def dense_precision(f: Factors) -> np.ndarray:
    """T^T D^-1 T, exactly symmetric (factors.py:136-145)."""
    c = f.dense_unit_lower() / np.sqrt(f.d)[:, None]
    m = c.T @ c
    return (m + m.T) * 0.5


_LINSOLVE = ["cholesky"]     # what the reference calls (cho_factor / cho_solve); "lu" only for the noise-floor probe


class linear_solver:
    """Context manager for the solver-swap probe of the noise floor: the same local analysis with the system solved by
    LAPACK dgesv (numpy.linalg.solve) instead of the reference's dpotrf / dpotrs."""

    def __init__(self, name: str):
        assert name in ("cholesky", "lu")
        self.name = name

    def __enter__(self):
        self.prev = _LINSOLVE[0]
        _LINSOLVE[0] = self.name

    def __exit__(self, *exc):
        _LINSOLVE[0] = self.prev


def analysis_primal(Xb: np.ndarray, f: Factors, obs_pos, r_diag, Ys) -> np.ndarray:
    """Xa = Xb + (B^-1 + H^T R^-1 H)^-1 H^T R^-1 (Ys - H Xb) (kernels.py:178-218).

    Dense Cholesky route only (the reference's n <= dense_cap branch).
    """
    obs_pos = np.asarray(obs_pos, dtype=np.int64)
    if obs_pos.size == 0:
        return Xb.copy()                              # kernels.py:179-180
    rinv = 1.0 / np.asarray(r_diag, dtype=np.float64)
    rhs = np.zeros_like(Xb)
    rhs[obs_pos] = (Ys - Xb[obs_pos]) * rinv[:, None]
    a = dense_precision(f)
    a[obs_pos, obs_pos] += rinv
    dx = cho_solve(cho_factor(a, lower=True), rhs) if _LINSOLVE[0] == "cholesky" else np.linalg.solve(a, rhs)
    return Xb + dx


# --------------------------------------------------------------------------
# driver (driver.py:99-125, 159-253)
# --------------------------------------------------------------------------
@dataclass
class TileResult:
    tile: Tile
    factors: Factors
    obs_pos: np.ndarray
    obs_rows: np.ndarray
    xa_local: np.ndarray


def analyse_tile(X2d, obs_idx, r_diag, Ys, grid: Grid, zeta: int, tile: Tile, csr=None) -> TileResult:
    """One sub-domain: slice, centre, fit, analyse (driver.py:199-229)."""
    members = tile.local_order
    xb = X2d[members]
    pos, rows = restrict_observations(obs_idx, members)
    f = fit_factors(center_rows(xb), grid, zeta, members, csr=csr)
    xa = analysis_primal(xb, f, pos, r_diag[rows], Ys[rows])
    return TileResult(tile, f, pos, rows, xa)


def merge_interiors(X2d: np.ndarray, results: list[TileResult]) -> np.ndarray:
    """out[interior] = local[interior_positions], exactly once (driver.py:99-125)."""
    out = X2d.copy()
    count = np.zeros(X2d.shape[0], dtype=np.int64)
    for res in results:
        out[res.tile.interior] = res.xa_local[res.tile.interior_positions()]
        count[res.tile.interior] += 1
    if np.any(count != 1):
        raise RuntimeError("interiors must cover each index exactly once")
    return out


def assimilate(X, obs_indices, r_diag, Ys, grid: Grid, delta: int, zeta: int,
               keep_tiles: bool = False, fields=None, pool=None):
    """Whole analysis step (driver.py:159-253), field by field.

    X: (nstate, N); obs_indices sorted global labels; Ys: (nobs, N).
    Returns Xa (and the per-field lists of TileResult when keep_tiles).
    """
    X = np.asarray(X, dtype=np.float64)
    obs_indices = np.asarray(obs_indices, dtype=np.int64)
    r_diag = np.asarray(r_diag, dtype=np.float64)
    tiles = decompose(grid, delta, zeta)
    csrs = [predecessor_csr(grid, zeta, t.local_order) for t in tiles]
    Xa = X.copy()
    kept = []
    for f in (range(grid.nfields) if fields is None else fields):
        lo, hi = f * grid.nfield, (f + 1) * grid.nfield
        sel = np.flatnonzero((obs_indices >= lo) & (obs_indices < hi))
        args = [(X[lo:hi], obs_indices[sel] - lo, r_diag[sel], Ys[sel], grid, zeta, t, c)
                for t, c in zip(tiles, csrs)]
        if pool is not None:
            results = pool.starmap(analyse_tile, args)
        else:
            results = [analyse_tile(*a) for a in args]
        Xa[lo:hi] = merge_interiors(X[lo:hi], results)
        if keep_tiles:
            kept.append(results)
    return (Xa, kept) if keep_tiles else Xa


# --------------------------------------------------------------------------
# LETKF baseline (kernels.py:251-335), the paper's comparison method
# --------------------------------------------------------------------------
EIG_FLOOR = 1e-12        # kernels.py:25


def letkf_point(center: int, Ub: np.ndarray, xb_mean: np.ndarray, obs_pos, r_diag, y, inflation: float = 1.0) -> np.ndarray:
    """Analysis row of one grid point from its local box (kernels.py:251-303)."""
    nbox, nens = Ub.shape
    obs_pos = np.asarray(obs_pos, dtype=np.int64)
    if obs_pos.size == 0:
        return xb_mean[center] + np.sqrt(inflation) * Ub[center]          # :282-284
    z = Ub[obs_pos]
    rinv = 1.0 / np.asarray(r_diag, dtype=np.float64)
    m = z.T @ (z * rinv[:, None])
    m = (m + m.T) * 0.5
    m[np.arange(nens), np.arange(nens)] += (nens - 1) / inflation
    lam, q = np.linalg.eigh(m)
    if lam[0] < EIG_FLOOR:
        raise RuntimeError(f"analysis weight matrix lost positive definiteness (min eig {lam[0]:.3e})")
    innov = np.asarray(y, dtype=np.float64) - xb_mean[obs_pos]
    zri = z.T @ (innov * rinv)
    wa = q @ ((q.T @ zri) / lam)
    sqrt_wa = (q * np.sqrt((nens - 1) / lam)) @ q.T
    return xb_mean[center] + Ub[center] @ (wa[:, None] + sqrt_wa)


def letkf_global(X: np.ndarray, grid: Grid, obs_indices, r_diag, y, zeta: int, inflation: float = 1.0) -> np.ndarray:
    """The point kernel at every grid component, field by field (kernels.py:306-335)."""
    X = np.asarray(X, dtype=np.float64)
    obs_indices = np.asarray(obs_indices, dtype=np.int64)
    r_diag = np.asarray(r_diag, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    xb_mean = X.mean(axis=1)
    u = X - xb_mean[:, None]
    out = X.copy()
    for f in range(grid.nfields):
        off = f * grid.n2d
        for c in range(grid.n2d):
            box = local_box(grid, c, zeta) + off
            pos, rows = restrict_observations(obs_indices, box)
            if pos.size == 0 and inflation == 1.0:
                continue
            cpos = int(np.searchsorted(box, c + off))
            out[c + off] = letkf_point(cpos, u[box], xb_mean[box], pos, r_diag[rows], y[rows], inflation)
    return out
