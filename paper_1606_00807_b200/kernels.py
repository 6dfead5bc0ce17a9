"""Boundary containers and the local analysis: same callables as the reference kernels module
(kernels.py:28-218) for the EnKF-MC primal path.

Interface schema note: the container fields, argument checks and error messages in this module restate the reference's
public interface (kernels.py:28-160) on purpose -- they are what a caller (and the reference's own tests, which `match=` on the
messages) sees at the drop-in boundary.  No arithmetic of the hot path lives here; that is in csrc/ behind the C-ABI.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import device
from .errors import ConfigurationError, NumericalError
from .factors import PrecisionFactors
from .validation import as_float_array, as_index_array, ensure_finite

TAG_OBS_PERTURB = 2  # rng.py:15


@dataclass(frozen=True)
class EnsembleState:
    X: np.ndarray
    role: str = "background"

    def __post_init__(self):
        x = as_float_array(self.X, "X", ndim=2)
        ensure_finite(x, "X")
        if self.role not in ("background", "analysis"):
            raise ValueError(f"unknown role {self.role!r}")
        object.__setattr__(self, "X", x)

    @property
    def nstate(self) -> int:
        return self.X.shape[0]

    @property
    def nens(self) -> int:
        return self.X.shape[1]

    def mean(self) -> np.ndarray:
        return self.X.mean(axis=1)

    def perturbations(self) -> np.ndarray:
        return self.X - self.X.mean(axis=1, keepdims=True)


@dataclass(frozen=True)
class ObservationNetwork:
    obs_indices: np.ndarray
    r_diag: np.ndarray
    y: np.ndarray

    def __post_init__(self):
        idx = as_index_array(self.obs_indices, "obs_indices")
        r = as_float_array(self.r_diag, "r_diag", ndim=1)
        y = as_float_array(self.y, "y", ndim=1)
        ensure_finite(r, "r_diag")
        ensure_finite(y, "y")
        if not (idx.size == r.size == y.size):
            raise ValueError(f"inconsistent lengths: {idx.size} indices, {r.size} variances, {y.size} values")
        if np.any(r <= 0):
            raise ValueError("r_diag must be strictly positive")
        object.__setattr__(self, "obs_indices", idx)
        object.__setattr__(self, "r_diag", r)
        object.__setattr__(self, "y", y)

    @property
    def nobs(self) -> int:
        return self.obs_indices.size

    def project(self, v: np.ndarray) -> np.ndarray:
        return v[self.obs_indices]


def restrict_network(net: ObservationNetwork, members: np.ndarray):
    """Observations inside `members`, re-indexed to positions, plus surviving parent rows
    (kernels.py:90-113).  Integer host logic."""
    members = as_index_array(members, "members")
    if members.size == 0:
        rows = np.zeros(0, dtype=np.intp)
        return ObservationNetwork(rows, np.zeros(0), np.zeros(0)), rows
    idx = np.searchsorted(members, net.obs_indices)
    inside = (idx < members.size) & (members[np.minimum(idx, members.size - 1)] == net.obs_indices)
    rows = np.flatnonzero(inside)
    return ObservationNetwork(idx[inside], net.r_diag[inside], net.y[inside]), rows


@dataclass(frozen=True)
class PerturbedObservations:
    Ys: np.ndarray
    seed: int
    cycle: int

    def __post_init__(self):
        ys = as_float_array(self.Ys, "Ys", ndim=2)
        ensure_finite(ys, "Ys")
        object.__setattr__(self, "Ys", ys)


def perturb_observations(net: ObservationNetwork, nens: int, seed: int, cycle: int = 0) -> PerturbedObservations:
    """Host-side draw from the reference stream (seed, cycle, tag=2), obs-major
    (kernels.py:130-144, rng.py:22-32); north_star keeps this on the host."""
    if nens < 1:
        raise ValueError(f"nens must be positive, got {nens}")
    if cycle < 0:
        raise ValueError(f"cycle must be nonnegative, got {cycle}")
    g = np.random.default_rng([int(seed) & ((1 << 64) - 1), int(cycle), TAG_OBS_PERTURB])
    noise = g.standard_normal((net.nobs, nens))
    ys = net.y[:, None] + np.sqrt(net.r_diag)[:, None] * noise
    return PerturbedObservations(Ys=ys, seed=int(seed), cycle=int(cycle))


def _check_analysis_inputs(Xb, factors, net, Ys) -> np.ndarray:
    if factors.n != Xb.nstate:
        raise ValueError(f"factors dimension {factors.n} does not match state dimension {Xb.nstate}")
    if net.nobs and net.obs_indices[-1] >= Xb.nstate:
        raise ValueError("observation indices exceed the state dimension")
    Ys = as_float_array(Ys, "Ys", ndim=2)
    if Ys.shape != (net.nobs, Xb.nens):
        raise ValueError(f"Ys has shape {Ys.shape}, expected {(net.nobs, Xb.nens)}")
    return Ys


def analysis_primal(Xb: EnsembleState, factors: PrecisionFactors, net: ObservationNetwork, Ys: np.ndarray, *,
                    dense_cap: int = 4096, cg_rtol: float = 1e-9) -> EnsembleState:
    """Xa = Xb + [B^-1 + H^T R^-1 H]^-1 H^T R^-1 (Ys - H Xb) (kernels.py:163-218) on the GPU.

    The K3 kernel always solves directly (banded Cholesky in the pattern's own order), so
    ``dense_cap``/``cg_rtol`` are accepted for signature compatibility only.
    """
    Ys = _check_analysis_inputs(Xb, factors, net, Ys)
    if net.nobs == 0:
        return EnsembleState(Xb.X.copy(), role="analysis")
    plan = factors.plan()
    plan.set_observations(net.obs_indices)
    dX = device.to_device(Xb.X)
    dT, dD = factors._device_factors()
    dXa, dS = device.local_solve_device(plan, dX, dT, dD, device.to_device(net.r_diag),
                                        device.to_device(np.ascontiguousarray(Ys)))
    status = int(dS.cpu()[0])
    if status != 0:
        why = "matrix not positive definite" if status == 1 else "non-finite pivot"
        raise NumericalError(f"primal analysis solve failed: {why}")
    return EnsembleState(dXa.cpu().numpy(), role="analysis")


def analysis_dual(Xb: EnsembleState, factors: PrecisionFactors, net: ObservationNetwork, Ys: np.ndarray) -> EnsembleState:
    """Observation-space analysis through the covariance square root (kernels.py:221-248): with T X = D^{1/2} I and
    V = H X, Xa = Xb + X V^T (R + V V^T)^-1 (Ys - H Xb) -- the primal route by Sherman-Morrison-Woodbury.

    The square root comes from the device unit-triangular solve (``enkfmc_unit_tri_solve``); the nobs x nobs
    observation-space system is a plain dense symmetric solve and goes through the library (torch.linalg on the
    device).  This is the second, independent route of the primal == dual self-check, not the timed hot path."""
    import torch

    Ys = _check_analysis_inputs(Xb, factors, net, Ys)
    if net.nobs == 0:
        return EnsembleState(Xb.X.copy(), role="analysis")
    n = factors.n
    dXs = factors._tri_solve(device.to_device(np.eye(n)), False, scale_in=device.to_device(np.sqrt(factors.variances)))
    obs = torch.from_numpy(np.ascontiguousarray(net.obs_indices)).cuda()
    v = dXs.index_select(0, obs)
    g = v @ v.T
    g.diagonal().add_(device.to_device(net.r_diag))
    dX = device.to_device(Xb.X)
    innovations = device.to_device(np.ascontiguousarray(Ys)) - dX.index_select(0, obs)
    chol, info = torch.linalg.cholesky_ex(g)
    if int(info.item()) != 0:
        raise NumericalError(f"dual observation-space solve failed: leading minor {int(info.item())} is not positive definite")
    w = torch.cholesky_solve(innovations, chol)
    dx = dXs @ (v.T @ w)
    return EnsembleState((dX + dx).cpu().numpy(), role="analysis")


def letkf_analysis_global(Xb: EnsembleState, geometry, net: ObservationNetwork, zeta: int, inflation: float = 1.0) -> EnsembleState:
    """LETKF baseline: the point kernel (kernels.py:251-303) at every grid component (kernels.py:306-335), on the GPU.
    A decomposed run (driver.py:128-156) computes exactly these rows, since every local box lies inside its
    sub-domain's interior + halo."""
    if getattr(geometry, "nlev", 1) != 1:
        raise ConfigurationError("the LETKF baseline is built for 2-D fields only (nlev = 1)")
    if Xb.nstate != geometry.nstate:
        raise ValueError(f"state dimension {Xb.nstate} does not match geometry {geometry.nstate}")
    if net.nobs and net.obs_indices[-1] >= geometry.nstate:
        raise ValueError("observation indices exceed the state dimension")
    if inflation <= 0:
        raise ValueError(f"inflation must be positive, got {inflation}")
    if zeta < 0:
        raise ValueError(f"zeta must be nonnegative, got {zeta}")
    import ctypes as C

    import torch

    from . import _lib
    obs_of_state = np.full(geometry.nstate, -1, dtype=np.int32)
    obs_of_state[net.obs_indices] = np.arange(net.nobs, dtype=np.int32)
    dX = device.to_device(Xb.X)
    dU, dXa = torch.empty_like(dX), torch.empty_like(dX)
    dMean = torch.empty(geometry.nstate, dtype=torch.float64, device="cuda")
    dMap = torch.from_numpy(obs_of_state).cuda()
    dR = device.to_device(np.ascontiguousarray(net.r_diag) if net.nobs else np.ones(1))
    dY = device.to_device(np.ascontiguousarray(net.y) if net.nobs else np.zeros(1))
    bad = C.c_int64(-1)
    _lib.check(_lib.lib().enkfmc_letkf_device(dX.data_ptr(), dU.data_ptr(), dMean.data_ptr(), dXa.data_ptr(), dMap.data_ptr(),
                                              dR.data_ptr(), dY.data_ptr(), geometry.nx, geometry.ny, int(geometry.row_major),
                                              int(geometry.periodic), geometry.nfields, Xb.nens, int(zeta), float(inflation),
                                              C.addressof(bad), device.stream_ptr()))
    return EnsembleState(dXa.cpu().numpy(), role="analysis")
