"""Container for the sparse precision factors B^-1 = T^T D^-1 T (factors.py:24-145).

Host-side validation and the CSR container are as in the reference; the arithmetic
(``dense_precision``, ``precision_apply``) runs on the GPU through the C-ABI.

Interface schema note: the container fields, argument checks and error messages in this module restate the reference's
public interface (factors.py:39-64) on purpose -- they are what a caller (and the reference's own tests, which `match=` on the
messages) sees at the drop-in boundary.  No arithmetic of the hot path lives here; that is in csrc/ behind the C-ABI.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import _lib, device
from .errors import CapacityError
from .plan import BANDWIDTH, PHYS, Plan
from .validation import as_float_array, ensure_finite

DENSE_SOLVE_LIMIT = 4096


class PrecisionFactors:
    def __init__(self, lower, variances, variance_floor: float = 1e-10):
        if variance_floor <= 0:
            raise ValueError(f"variance_floor must be positive, got {variance_floor}")
        lower = sp.csr_matrix(lower, copy=True)
        if lower.shape[0] != lower.shape[1]:
            raise ValueError(f"T must be square, got shape {lower.shape}")
        lower.sum_duplicates()
        lower.sort_indices()
        coo = lower.tocoo()
        if np.any(coo.col >= coo.row):
            raise ValueError("T must be strictly lower triangular (unit diagonal is implicit)")
        ensure_finite(lower.data, "T entries")
        d = as_float_array(variances, "variances", ndim=1)
        ensure_finite(d, "variances")
        if d.size != lower.shape[0]:
            raise ValueError(f"variances length {d.size} does not match T dimension {lower.shape[0]}")
        self.lower = lower
        self.variances = np.maximum(d, variance_floor)        # factors.py:60
        self.variance_floor = float(variance_floor)
        self._plan = None

    @property
    def n(self) -> int:
        return self.lower.shape[0]

    def plan(self) -> Plan:
        """Single-tile plan over this CSR pattern (cached)."""
        if self._plan is None:
            self._plan = Plan.from_csr(self.lower.indptr, self.lower.indices)
        return self._plan

    def _device_factors(self):
        return device.to_device(self.lower.data.astype(np.float64)), device.to_device(self.variances)

    def dense_precision(self, cap: int = DENSE_SOLVE_LIMIT) -> np.ndarray:
        """T^T D^-1 T, exactly symmetric, refused beyond cap (factors.py:136-145)."""
        if self.n > cap:
            raise CapacityError(f"dense precision of dimension {self.n} exceeds cap {cap}")
        if self.n == 0:
            return np.zeros((0, 0))
        plan = self.plan()
        b = int(plan.get(BANDWIDTH)[0])
        dT, dD = self._device_factors()
        wb = (b + 7) // 8
        wr = 8 * (wb + 1)
        band = device.empty((self.n, wr))
        _lib.check(_lib.lib().enkfmc_assemble_band(plan.handle, dT.data_ptr(), dD.data_ptr(), 0, band.data_ptr(),
                                                   device.stream_ptr()))
        band = band.cpu().numpy()                 # band[I, e] = A[I, 8 (I // 8 - wb) + e]
        out = np.zeros((self.n, self.n))
        rows = np.arange(self.n)
        for e in range(wr):                       # layout only, no arithmetic
            cols = 8 * (rows // 8 - wb) + e
            ok = (cols >= 0) & (cols <= rows)
            out[rows[ok], cols[ok]] = band[rows[ok], e]
            out[cols[ok], rows[ok]] = band[rows[ok], e]
        return out

    def precision_apply(self, v: np.ndarray) -> np.ndarray:
        """T^T D^-1 T v without densifying (factors.py:86-96)."""
        v = as_float_array(v, "v")
        if v.shape[0] != self.n:
            raise ValueError(f"v has leading dimension {v.shape[0]}, expected {self.n}")
        squeeze = v.ndim == 1
        vv = np.ascontiguousarray(v[:, None] if squeeze else v)
        if self.n == 0:
            return v.copy()
        dT, dD = self._device_factors()
        dV = device.to_device(vv)
        dW, dO = device.empty(vv.shape), device.empty(vv.shape)
        _lib.check(_lib.lib().enkfmc_precision_apply(self.plan().handle, dT.data_ptr(), dD.data_ptr(), dV.data_ptr(),
                                                     vv.shape[1], dW.data_ptr(), dO.data_ptr(), device.stream_ptr()))
        out = dO.cpu().numpy()
        return out[:, 0] if squeeze else out

    def _tri_solve(self, dB, transposed: bool, scale_in=None, scale_out=None):
        dT, _ = self._device_factors()
        _lib.check(_lib.lib().enkfmc_unit_tri_solve(self.plan().handle, dT.data_ptr(), int(transposed),
                                                    scale_in.data_ptr() if scale_in is not None else None,
                                                    scale_out.data_ptr() if scale_out is not None else None,
                                                    dB.data_ptr(), dB.shape[1], device.stream_ptr()))
        return dB

    def sqrt_solve(self, rhs: np.ndarray, dense_limit: int = DENSE_SOLVE_LIMIT) -> np.ndarray:
        """Solve T X = D^{1/2} rhs by forward substitution in label order (factors.py:116-134); with rhs = I the columns
        of X form a square root of the implied covariance.  ``dense_limit`` is accepted for signature compatibility:
        the sparse substitution runs on the device whatever the size."""
        rhs = as_float_array(rhs, "rhs")
        if rhs.shape[0] != self.n:
            raise ValueError(f"rhs has leading dimension {rhs.shape[0]}, expected {self.n}")
        squeeze = rhs.ndim == 1
        b = np.ascontiguousarray(rhs[:, None] if squeeze else rhs)
        if self.n == 0:
            return rhs.copy()
        out = self._tri_solve(device.to_device(b), False, scale_in=device.to_device(np.sqrt(self.variances))).cpu().numpy()
        return out[:, 0] if squeeze else out

    def covariance_apply(self, v: np.ndarray, dense_limit: int = DENSE_SOLVE_LIMIT) -> np.ndarray:
        """Apply the implied covariance T^-1 D T^-T (factors.py:98-114): a backward and a forward unit-triangular solve."""
        v = as_float_array(v, "v")
        if v.shape[0] != self.n:
            raise ValueError(f"v has leading dimension {v.shape[0]}, expected {self.n}")
        squeeze = v.ndim == 1
        b = np.ascontiguousarray(v[:, None] if squeeze else v)
        if self.n == 0:
            return v.copy()
        dB = device.to_device(b)
        self._tri_solve(dB, True, scale_out=device.to_device(self.variances))
        out = self._tri_solve(dB, False).cpu().numpy()
        return out[:, 0] if squeeze else out


def dump_factors(factors: PrecisionFactors, t_path, d_path) -> None:
    """T as "row col value" triplets (row-major, the implicit unit diagonal written explicitly after each row's entries)
    and D one value per line, %.17g -- the files `mcholkf dump-precision` writes (factors.py:148-166)."""
    low = factors.lower
    with open(t_path, "w") as fh:
        for r in range(factors.n):
            a, b = low.indptr[r], low.indptr[r + 1]
            fh.write("".join(f"{r} {int(c)} {float(v):.17g}\n" for c, v in zip(low.indices[a:b], low.data[a:b])))
            fh.write(f"{r} {r} 1\n")
    with open(d_path, "w") as fh:
        fh.write("".join(f"{float(v):.17g}\n" for v in factors.variances))


def dump_plan_factors(plan, directory, field: int = 0) -> list:
    """Writes T_subdomain<k>.txt / D_subdomain<k>.txt (the reference's artefact names, harness / CLI) for every
    sub-domain of a decomposed plan from the factors of its last analysis on the device.  Returns the paths."""
    import os

    from .plan import COL_IDX, ROW_PTR, TILE_PTR
    tp, rp, ci = plan.get(TILE_PTR), plan.get(ROW_PTR), plan.get(COL_IDX)
    T = device.workspace_tensor(plan, 1, (plan.nfields, plan.nnz))[field]
    D = device.workspace_tensor(plan, 2, (plan.nfields, plan.sum_nlocal))[field]
    os.makedirs(directory, exist_ok=True)
    paths = []
    for k in range(plan.ntiles):
        r0, r1 = tp[k], tp[k + 1]
        indptr = rp[r0:r1 + 1] - rp[r0]
        lower = sp.csr_matrix((T[rp[r0]:rp[r1]], ci[rp[r0]:rp[r1]], indptr), shape=(r1 - r0, r1 - r0))
        tpth, dpth = os.path.join(directory, f"T_subdomain{k}.txt"), os.path.join(directory, f"D_subdomain{k}.txt")
        dump_factors(PrecisionFactors(lower, D[r0:r1]), tpth, dpth)
        paths.append((tpth, dpth))
    return paths
