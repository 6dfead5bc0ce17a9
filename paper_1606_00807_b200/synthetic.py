"""Seeded synthetic inputs shaped like the BASELINE.json configurations.

They stand in for the paper's SPEEDY T-63 data (not available offline); shapes,
sizes and value distributions follow BASELINE.json / SURVEY.md section 8(d).  All
draws come from ``np.random.default_rng(seed)``; the observation ensemble comes
from the reference's (seed, cycle, tag=2) stream (``rng.py:22-32``,
``kernels.py:130-144``) restated in :func:`perturbed_observations`.

State layout: ``X[(field, row, col), member]``, label = field*(nx*ny) + row*nx + col,
C-order float64 with the member index fastest (``kernels.py:28-33``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

TAG_OBS_PERTURB = 2  # rng.py:15


@dataclass
class Workload:
    name: str
    nx: int
    ny: int
    nfields: int
    boundary: str           # "clipped" | "periodic"
    nens: int
    zeta: int
    delta: int
    X: np.ndarray           # (nstate, nens) background ensemble
    obs_indices: np.ndarray  # sorted global labels, int64
    r_diag: np.ndarray
    y: np.ndarray
    Ys: np.ndarray          # (nobs, nens)
    truth: np.ndarray
    seed: int
    nugget: float = 0.0
    notes: dict = field(default_factory=dict)

    @property
    def n2d(self) -> int:
        return self.nx * self.ny

    @property
    def nstate(self) -> int:
        return self.n2d * self.nfields


def perturbed_observations(y, r_diag, nens: int, seed: int, cycle: int = 0) -> np.ndarray:
    """Host-side Ys = y + sqrt(r)*N(0,1) from the reference stream (kernels.py:130-144)."""
    g = np.random.default_rng([int(seed) & ((1 << 64) - 1), int(cycle), TAG_OBS_PERTURB])
    noise = g.standard_normal((len(y), nens))
    return np.asarray(y, np.float64)[:, None] + np.sqrt(np.asarray(r_diag, np.float64))[:, None] * noise


def _gauss_sqrt(n: int, length: float, periodic: bool) -> np.ndarray:
    """Symmetric square root of C_ij = exp(-d_ij^2 / (2 L^2)), negative eigenvalues clipped."""
    i = np.arange(n)
    d = np.abs(i[:, None] - i[None, :]).astype(np.float64)
    if periodic:
        d = np.minimum(d, n - d)
    c = np.exp(-(d * d) / (2.0 * length * length))
    w, v = np.linalg.eigh(c)
    return (v * np.sqrt(np.clip(w, 0.0, None))) @ v.T


def _sinusoid_field(rng, ny: int, nx: int, nterms: int = 8) -> np.ndarray:
    """Sum of low-order sinusoids with N(0,1) amplitudes."""
    yy, xx = np.meshgrid(np.arange(ny) / ny, np.arange(nx) / nx, indexing="ij")
    out = np.zeros((ny, nx))
    for _ in range(nterms):
        a = rng.standard_normal()
        kx, ky = int(rng.integers(0, 4)), int(rng.integers(0, 4))
        phi = rng.uniform(0.0, 2.0 * np.pi)
        out += a * np.sin(2.0 * np.pi * (kx * xx + ky * yy) + phi)
    return out


def make_workload(name: str, *, nx: int, ny: int, nens: int, corr_len: float, zeta: int, delta: int,
                  obs: str, obs_arg: float, r_rel: float | None, r_abs: float | None,
                  seed: int, boundary: str = "clipped", lon_periodic_corr: bool = False,
                  variables: list[tuple[str, float, int]] | None = None,
                  nugget: float = 0.0) -> Workload:
    """Build one workload.

    variables: [(name, std, nlevels)] -- each level of each variable is one 2-D field;
    levels of one variable are correlated by exp(-dl^2/2), variables are independent.
    obs: "lattice" (every obs_arg-th point both ways) or "random" (fraction obs_arg of the
    horizontal points, same set for every field).  r_abs: obs error std (absolute);
    r_rel: obs error std as a fraction of the variable std.
    """
    rng = np.random.default_rng(seed)
    variables = variables or [("x", 1.0, 1)]
    nfields = sum(nl for _, _, nl in variables)
    n2d = nx * ny
    l_lat = _gauss_sqrt(ny, corr_len, False)
    l_lon = _gauss_sqrt(nx, corr_len, lon_periodic_corr or boundary == "periodic")

    X = np.empty((nfields * n2d, nens))
    truth = np.empty(nfields * n2d)
    field_std = np.empty(nfields)
    f0 = 0
    for _, std, nlev in variables:
        lv = _gauss_sqrt(nlev, 1.0, False) if nlev > 1 else np.ones((1, 1))
        for lev in range(nlev):
            truth[(f0 + lev) * n2d:(f0 + lev + 1) * n2d] = std * _sinusoid_field(rng, ny, nx).ravel()
        mean = np.stack([std * _sinusoid_field(rng, ny, nx) for _ in range(nlev)])
        w = rng.standard_normal((nens, nlev, ny, nx))
        eps = np.einsum("ab,mbij->maij", lv, np.einsum("ik,mbkl,jl->mbij", l_lat, w, l_lon, optimize=True))
        if nugget > 0.0:
            eps = eps + nugget * rng.standard_normal(eps.shape)
        members = mean[None] + std * eps                          # (nens, nlev, ny, nx)
        X[f0 * n2d:(f0 + nlev) * n2d] = members.reshape(nens, nlev * n2d).T
        field_std[f0:f0 + nlev] = std
        f0 += nlev

    if obs == "lattice":
        step = int(obs_arg)
        rr, cc = np.meshgrid(np.arange(0, ny, step), np.arange(0, nx, step), indexing="ij")
        horiz = np.sort((rr * nx + cc).ravel())
    elif obs == "random":
        horiz = np.sort(rng.choice(n2d, size=int(round(obs_arg * n2d)), replace=False))
    else:
        raise ValueError(obs)
    obs_indices = (np.arange(nfields)[:, None] * n2d + horiz[None, :]).ravel().astype(np.int64)
    sig = np.repeat(field_std * r_rel if r_abs is None else np.full(nfields, r_abs), horiz.size)
    r_diag = sig * sig
    y = truth[obs_indices] + sig * rng.standard_normal(obs_indices.size)
    Ys = perturbed_observations(y, r_diag, nens, seed, 0)
    return Workload(name, nx, ny, nfields, boundary, nens, zeta, delta, np.ascontiguousarray(X),
                    obs_indices, r_diag, y, Ys, truth, seed, nugget)


_SPEEDY = [("u", 5.0, 7), ("v", 5.0, 7), ("T", 2.0, 7), ("q", 1e-3, 7), ("ps", 100.0, 1)]
_CFG5 = [("u", 5.0, 8), ("v", 5.0, 8), ("T", 2.0, 8), ("q", 1e-3, 8), ("w", 1.0, 8)]


def config(name: str, *, nugget: float = 0.0, boundary: str | None = None, zeta: int | None = None,
           fields: int | None = None, seed: int | None = None) -> Workload:
    """BASELINE.json configurations cfg1..cfg5 (cfg4 takes zeta=1..6).

    ``fields`` truncates the multi-field configs to their first few fields (parity-test sizing).
    """
    if name == "cfg1":
        return make_workload(name, nx=64, ny=32, nens=20, corr_len=4.0, zeta=zeta or 2, delta=8,
                             obs="lattice", obs_arg=2, r_rel=None, r_abs=0.05, seed=seed or 1001,
                             boundary=boundary or "clipped", lon_periodic_corr=True, nugget=nugget)
    if name == "cfg2":
        return make_workload(name, nx=192, ny=96, nens=40, corr_len=6.0, zeta=zeta or 3, delta=64,
                             obs="random", obs_arg=0.25, r_rel=None, r_abs=0.1, seed=seed or 1002,
                             boundary=boundary or "clipped", nugget=nugget)
    if name == "cfg3":
        var = _SPEEDY if fields is None else _take_fields(_SPEEDY, fields)
        return make_workload(name, nx=192, ny=96, nens=80, corr_len=5.0, zeta=zeta or 4, delta=256,
                             obs="random", obs_arg=0.5, r_rel=0.1, r_abs=None, seed=seed or 1003,
                             boundary=boundary or "clipped", variables=var, nugget=nugget)
    if name == "cfg4":
        return make_workload(name, nx=192, ny=96, nens=80, corr_len=6.0, zeta=zeta or 3, delta=64,
                             obs="random", obs_arg=0.25, r_rel=None, r_abs=0.1, seed=seed or 1004,
                             boundary=boundary or "clipped", nugget=nugget)
    if name == "cfg5":
        var = _CFG5 if fields is None else _take_fields(_CFG5, fields)
        return make_workload(name, nx=384, ny=192, nens=128, corr_len=5.0, zeta=zeta or 5, delta=1024,
                             obs="random", obs_arg=0.3, r_rel=0.1, r_abs=None, seed=seed or 1005,
                             boundary=boundary or "clipped", variables=var, nugget=nugget)
    raise ValueError(f"unknown workload {name!r}")


def _take_fields(variables, nfields: int):
    out, left = [], nfields
    for nm, std, nl in variables:
        if left <= 0:
            break
        out.append((nm, std, min(nl, left)))
        left -= nl
    return out
