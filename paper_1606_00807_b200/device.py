"""Device plumbing: torch owns device memory and streams, libenkfmc.so does the work.

Every function here raises BackendError when CUDA is unavailable -- no CPU fallback.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import BackendError


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise BackendError("no CUDA device: paper_1606_00807_b200 runs on sm_100 GPUs only (no CPU fallback)")
    return torch


def stream_ptr() -> int:
    return _torch().cuda.current_stream().cuda_stream


def to_device(a: np.ndarray):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def empty(shape, dtype="f64"):
    torch = _torch()
    return torch.empty(shape, dtype={"f64": torch.float64, "i32": torch.int32, "i64": torch.int64}[dtype], device="cuda")


def center_rows_device(dX, dU=None):
    """K0 on a device tensor [nrows, nens]."""
    torch = _torch()
    if dU is None:
        dU = torch.empty_like(dX)
    _lib.check(_lib.lib().enkfmc_center_rows(dX.data_ptr(), dU.data_ptr(), dX.shape[0], dX.shape[1], stream_ptr()))
    return dU


def center_rows_host(X: np.ndarray) -> np.ndarray:
    torch = _torch()
    dU = center_rows_device(to_device(X))
    torch.cuda.synchronize()
    return dU.cpu().numpy()


def regress_device(plan, dU, rank_tol: float, variance_floor: float, want_flags: bool = True):
    """K2: returns (dT [nfields*nnz], dD [nfields*sum_nlocal], dflags or None)."""
    nens = dU.shape[1]
    dT = empty((max(plan.nfields * plan.nnz, 1),))
    dD = empty((max(plan.nfields * plan.sum_nlocal, 1),))
    dF = empty((max(plan.nfields * plan.sum_nlocal, 1),), "i32") if want_flags else None
    _lib.check(_lib.lib().enkfmc_regress(plan.handle, dU.data_ptr(), nens, rank_tol, variance_floor, dT.data_ptr(),
                                         dD.data_ptr(), dF.data_ptr() if want_flags else None, stream_ptr()))
    return dT, dD, dF


def local_solve_device(plan, dX, dT, dD, dR, dYs, dXa=None):
    """K3: returns (dXa, dstatus)."""
    torch = _torch()
    nens = dX.shape[1]
    if dXa is None:
        dXa = torch.empty_like(dX)
    dS = torch.zeros((max(plan.nfields * plan.ntiles, 1),), dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().enkfmc_local_solve(plan.handle, dX.data_ptr(), dT.data_ptr(), dD.data_ptr(), dR.data_ptr(),
                                             dYs.data_ptr(), nens, dXa.data_ptr(), dS.data_ptr(), stream_ptr()))
    return dXa, dS


def analysis_device(plan, dX, dR, dYs, dXa, rank_tol: float = 1e-8, variance_floor: float = 1e-10):
    """K0 + K2 + K3 on device-resident tensors, current stream, no synchronisation."""
    _lib.check(_lib.lib().enkfmc_analysis_device(plan.handle, dX.data_ptr(), dR.data_ptr(), dYs.data_ptr(),
                                                 dX.shape[1], rank_tol, variance_floor, dXa.data_ptr(), stream_ptr()))
    return dXa


def check_status(plan) -> int:
    """Outcome of the last analysis on this plan: synchronises; raises NumericalError naming the sub-domain if a
    tile's factorisation failed (kernels.py:192-195); returns the number of clamped Cholesky pivots."""
    _lib.check(_lib.lib().enkfmc_plan_check_status(plan.handle))
    return plan.counter(5)


_PINNED_POOL: list = []   # [tensor, weakref-to-the-array-handed-out]


def pinned_empty(shape) -> np.ndarray:
    """float64 host array in page-locked memory.  Buffers are recycled once the array handed out
    earlier (and every view of it) has been garbage collected, so results stay caller-owned."""
    import weakref

    torch = _torch()
    n = int(np.prod(shape))
    for entry in _PINNED_POOL:
        if entry[0].numel() == n and entry[1]() is None:
            base = entry[0].numpy()          # every view handed out keeps `base` alive (numpy base collapsing)
            entry[1] = weakref.ref(base)
            return base.reshape(shape)
    t = torch.empty(max(n, 1), dtype=torch.float64, pin_memory=True)[:n]
    base = t.numpy()
    if len(_PINNED_POOL) >= 4:
        _PINNED_POOL.pop(0)
    _PINNED_POOL.append([t, weakref.ref(base)])
    return base.reshape(shape)


def analysis_host(plan, X: np.ndarray, r_diag: np.ndarray, Ys: np.ndarray, Xa: np.ndarray | None = None,
                  rank_tol: float = 1e-8, variance_floor: float = 1e-10):
    """Host buffers in, host buffer out; H2D/D2H inside.  Returns (Xa, timings_ms[4])."""
    _torch()
    if Xa is None:
        Xa = pinned_empty(X.shape)
    tm = np.zeros(4)
    _lib.check(_lib.lib().enkfmc_analysis_host(plan.handle, _lib.ptr(X), _lib.ptr(r_diag), _lib.ptr(Ys), X.shape[1],
                                               rank_tol, variance_floor, _lib.ptr(Xa), _lib.ptr(tm)))
    return Xa, tm


def scatter_rows(dDst, dst_rows: np.ndarray, dSrc, src_rows: np.ndarray):
    d_dst_rows, d_src_rows = to_device(_lib.as_i64(dst_rows)), to_device(_lib.as_i64(src_rows))
    _lib.check(_lib.lib().enkfmc_scatter_rows(dDst.data_ptr(), d_dst_rows.data_ptr(), dSrc.data_ptr(),
                                              d_src_rows.data_ptr(), d_src_rows.numel(), dDst.shape[1], stream_ptr()))
    _torch().cuda.synchronize()
    return dDst


def workspace_tensor(plan, what: int, shape, dtype="f64"):
    """Copy of one of the plan's device workspace buffers (U, T, D, flags, status) as numpy."""
    _torch()
    out = np.empty(int(np.prod(shape)), dtype={"f64": np.float64, "i32": np.int32}[dtype])
    _lib.check(_lib.lib().enkfmc_plan_read_buffer(plan.handle, what, _lib.ptr(out), out.nbytes))
    return out.reshape(shape)
