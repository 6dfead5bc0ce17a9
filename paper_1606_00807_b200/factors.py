"""Container for the sparse precision factors B^-1 = T^T D^-1 T (factors.py:24-145).

Host-side validation and the CSR container are as in the reference; the arithmetic
(``dense_precision``, ``precision_apply``) runs on the GPU through the C-ABI.
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
