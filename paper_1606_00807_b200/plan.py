"""Python handle on an ``enkfmc_plan`` (index maps on host and device), cached per
(geometry, delta, zeta): SURVEY 7.3-4 -- the maps are cycle-invariant, only Xb/Ys change."""

from __future__ import annotations

import ctypes as C
from functools import lru_cache

import numpy as np

from . import _lib

(TILE_PTR, LOCAL_ORDER, INTERIOR_PTR, INTERIOR, INTERIOR_POS, HALO_PTR, HALO, ROW_PTR, COL_IDX, OBS_PTR, OBS_POS,
 OBS_ROW, BANDWIDTH, PHYS, REGRESSION_OF) = range(15)
_SIZE_OF = {TILE_PTR: (0, 1), LOCAL_ORDER: (1, 0), INTERIOR_PTR: (0, 1), INTERIOR: (3, 0), INTERIOR_POS: (3, 0),
            HALO_PTR: (0, 1), HALO: (4, 0), ROW_PTR: (1, 1), COL_IDX: (2, 0), OBS_POS: (6, 0), OBS_ROW: (6, 0),
            BANDWIDTH: (0, 0), PHYS: (1, 0), REGRESSION_OF: (1, 0)}


class Plan:
    """Owns one enkfmc_plan*.  Not thread-safe (one analysis at a time per plan)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        self._obs_key = None
        self._sub = None

    # -- constructors ------------------------------------------------------------------
    @classmethod
    def decomposed(cls, geometry, delta: int, zeta: int) -> "Plan":
        h = C.c_void_p()
        _lib.check(_lib.lib().enkfmc_plan_create_levels(geometry.nx, geometry.ny, int(geometry.row_major),
                                                        int(geometry.periodic), int(getattr(geometry, "nlev", 1)),
                                                        int(getattr(geometry, "zeta_v", 0)), int(geometry.nfields),
                                                        int(delta), int(zeta), C.byref(h)))
        return cls(h.value)

    @classmethod
    def local(cls, geometry, zeta: int, local_order: np.ndarray) -> "Plan":
        lo = _lib.as_i64(local_order)
        h = C.c_void_p()
        _lib.check(_lib.lib().enkfmc_plan_create_local(geometry.nx, geometry.ny, int(geometry.row_major),
                                                       int(geometry.periodic), int(zeta), lo.size, _lib.ptr(lo),
                                                       C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_csr(cls, indptr: np.ndarray, indices: np.ndarray) -> "Plan":
        ip, ii = _lib.as_i64(indptr), _lib.as_i64(indices)
        h = C.c_void_p()
        _lib.check(_lib.lib().enkfmc_plan_create_csr(ip.size - 1, _lib.ptr(ip), _lib.ptr(ii), C.byref(h)))
        return cls(h.value)

    def __del__(self):
        try:
            if self._h:
                _lib.lib().enkfmc_plan_destroy(self._h)
                self._h = None
        except Exception:
            pass

    # -- queries -----------------------------------------------------------------------
    @property
    def handle(self):
        return self._h

    def size(self, what: int) -> int:
        return int(_lib.lib().enkfmc_plan_size(self._h, what))

    ntiles = property(lambda self: self.size(0))
    sum_nlocal = property(lambda self: self.size(1))
    nnz = property(lambda self: self.size(2))
    nobs = property(lambda self: self.size(5))
    max_nlocal = property(lambda self: self.size(9))
    max_pred = property(lambda self: self.size(10))
    max_bw = property(lambda self: self.size(11))
    n_regressions = property(lambda self: self.size(14))   # distinct regressions among the owned rows
    n_owned_rows = property(lambda self: self.size(15))
    nfields = property(lambda self: self.size(12))

    def get(self, what: int) -> np.ndarray:
        if what == OBS_PTR:
            n = self.nfields * self.ntiles + 1
        else:
            sz, extra = _SIZE_OF[what]
            n = self.size(sz) + extra
        out = np.empty(n, dtype=np.int64)
        _lib.check(_lib.lib().enkfmc_plan_get(self._h, what, _lib.ptr(out), n))
        return out

    def counter(self, what: int) -> int:
        return int(_lib.lib().enkfmc_plan_counter(self._h, what))

    def set_observations(self, obs_indices: np.ndarray) -> None:
        obs = _lib.as_i64(obs_indices)
        key = (obs.size, hash(obs.tobytes()))
        if key == self._obs_key:
            return
        _lib.check(_lib.lib().enkfmc_plan_set_observations(self._h, obs.size, _lib.ptr(obs)))
        self._obs_key = key

    def set_tile_range(self, begin: int, end: int) -> None:
        """Own tiles [begin, end) only (one rank's share of the sub-domains)."""
        _lib.check(_lib.lib().enkfmc_plan_set_tile_range(self._h, int(begin), int(end)))

    def profile(self, enable: bool) -> None:
        _lib.check(_lib.lib().enkfmc_plan_profile(self._h, int(enable)))

    def stage_times(self):
        """(ncalls, [ms K0 centre, ms K2a QR, ms K2b probe/solve, ms K3 assemble+solve] summed over the profiled calls)."""
        n = C.c_int64(0)
        ms = np.zeros(4)
        _lib.check(_lib.lib().enkfmc_plan_stage_times(self._h, C.addressof(n), _lib.ptr(ms)))
        return int(n.value), ms

    def work(self, nens: int):
        """Algorithmic flops of one analysis over the owned tiles: (regressions as the reference
        runs them, local solves, regressions executed = distinct ones only)."""
        fl = np.zeros(3)
        _lib.check(_lib.lib().enkfmc_plan_work(self._h, int(nens), _lib.ptr(fl)))
        return float(fl[0]), float(fl[1]), float(fl[2])

    def subdomains(self):
        """list[Subdomain] exactly as decompose returns them (geometry.py:204-221)."""
        from .geometry import Subdomain

        if self._sub is None:
            tp, lo = self.get(TILE_PTR), self.get(LOCAL_ORDER).astype(np.intp)
            ip, it = self.get(INTERIOR_PTR), self.get(INTERIOR).astype(np.intp)
            hp, ha = self.get(HALO_PTR), self.get(HALO).astype(np.intp)
            self._sub = [
                Subdomain(id=t, interior=it[ip[t]:ip[t + 1]], halo=ha[hp[t]:hp[t + 1]], local_order=lo[tp[t]:tp[t + 1]])
                for t in range(self.ntiles)
            ]
        # fresh arrays every time: callers may modify what they get without touching the cached plan
        return [Subdomain(id=sd.id, interior=sd.interior.copy(), halo=sd.halo.copy(), local_order=sd.local_order.copy())
                for sd in self._sub]


@lru_cache(maxsize=4)      # a plan owns device workspace (tens of GB at the largest configurations): keep few alive
def get_plan(geometry, delta: int, zeta: int) -> Plan:
    return Plan.decomposed(geometry, delta, zeta)
