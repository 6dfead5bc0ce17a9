"""ctypes binding of libenkfmc.so (C-ABI declared in include/enkf_mc.h).

The library is built in-tree by ``__graft_entry__.build()`` / ``csrc/Makefile``.  Loading
fails loudly: there is no pure-Python or CPU fallback for any compute entry point.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import BackendError, CapacityError, ConfigurationError, NumericalError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libenkfmc.so")

# every symbol include/enkf_mc.h declares
SYMBOLS = (
    "enkfmc_version", "enkfmc_last_error", "enkfmc_tiling", "enkfmc_local_box", "enkfmc_predecessors",
    "enkfmc_plan_create", "enkfmc_plan_create_levels", "enkfmc_plan_create_local", "enkfmc_plan_create_csr", "enkfmc_plan_destroy",
    "enkfmc_plan_set_observations", "enkfmc_plan_size", "enkfmc_plan_get", "enkfmc_center_rows",
    "enkfmc_regress", "enkfmc_local_solve", "enkfmc_analysis_device", "enkfmc_analysis_host",
    "enkfmc_plan_counter", "enkfmc_plan_device_buffer", "enkfmc_scatter_rows", "enkfmc_assemble_band",
    "enkfmc_precision_apply", "enkfmc_plan_read_buffer", "enkfmc_plan_set_tile_range", "enkfmc_plan_profile",
    "enkfmc_plan_stage_times", "enkfmc_plan_work", "enkfmc_fp64_peak", "enkfmc_fp64_mma_peak", "enkfmc_plan_check_status", "enkfmc_unit_tri_solve", "enkfmc_advdiff_step", "enkfmc_letkf_device",
)

_lib = None
i64, f64p, i64p, i32p, vp = C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise BackendError(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a).  paper_1606_00807_b200 has no CPU fallback."
        )
    L = C.CDLL(LIB_PATH)
    L.enkfmc_version.restype = C.c_char_p
    L.enkfmc_last_error.restype = C.c_char_p
    L.enkfmc_plan_size.restype = i64
    L.enkfmc_plan_size.argtypes = [vp, C.c_int]
    L.enkfmc_plan_counter.restype = i64
    L.enkfmc_plan_counter.argtypes = [vp, C.c_int]
    L.enkfmc_plan_device_buffer.restype = C.c_void_p
    L.enkfmc_plan_device_buffer.argtypes = [vp, C.c_int]
    L.enkfmc_plan_destroy.restype = None
    L.enkfmc_plan_destroy.argtypes = [vp]
    L.enkfmc_tiling.argtypes = [i64, i64, i64, vp, vp]
    L.enkfmc_local_box.argtypes = [i64, i64, C.c_int, C.c_int, i64, i64, vp, vp]
    L.enkfmc_predecessors.argtypes = [i64, i64, C.c_int, C.c_int, i64, i64, vp, vp]
    L.enkfmc_plan_create.argtypes = [i64, i64, C.c_int, C.c_int, i64, i64, i64, vp]
    L.enkfmc_plan_create_levels.argtypes = [i64, i64, C.c_int, C.c_int, i64, i64, i64, i64, i64, vp]
    L.enkfmc_plan_create_local.argtypes = [i64, i64, C.c_int, C.c_int, i64, i64, vp, vp]
    L.enkfmc_plan_create_csr.argtypes = [i64, vp, vp, vp]
    L.enkfmc_plan_set_observations.argtypes = [vp, i64, vp]
    L.enkfmc_plan_get.argtypes = [vp, C.c_int, vp, i64]
    L.enkfmc_center_rows.argtypes = [vp, vp, i64, i64, vp]
    L.enkfmc_regress.argtypes = [vp, vp, i64, C.c_double, C.c_double, vp, vp, vp, vp]
    L.enkfmc_local_solve.argtypes = [vp, vp, vp, vp, vp, vp, i64, vp, vp, vp]
    L.enkfmc_analysis_device.argtypes = [vp, vp, vp, vp, i64, C.c_double, C.c_double, vp, vp]
    L.enkfmc_analysis_host.argtypes = [vp, vp, vp, vp, i64, C.c_double, C.c_double, vp, vp]
    L.enkfmc_scatter_rows.argtypes = [vp, vp, vp, vp, i64, i64, vp]
    L.enkfmc_assemble_band.argtypes = [vp, vp, vp, i64, vp, vp]
    L.enkfmc_precision_apply.argtypes = [vp, vp, vp, vp, i64, vp, vp, vp]
    L.enkfmc_plan_read_buffer.argtypes = [vp, C.c_int, vp, i64]
    L.enkfmc_plan_set_tile_range.argtypes = [vp, i64, i64]
    L.enkfmc_plan_profile.argtypes = [vp, C.c_int]
    L.enkfmc_plan_check_status.argtypes = [vp]
    L.enkfmc_unit_tri_solve.argtypes = [vp, vp, C.c_int, vp, vp, vp, i64, vp]
    L.enkfmc_letkf_device.argtypes = [vp, vp, vp, vp, vp, vp, vp, i64, i64, C.c_int, C.c_int, i64, i64, i64, C.c_double, vp, vp]
    L.enkfmc_advdiff_step.argtypes = [vp, vp, i64, i64, C.c_int, i64, i64, C.c_double, C.c_double, C.c_double, C.c_double, vp]
    L.enkfmc_plan_stage_times.argtypes = [vp, vp, vp]
    L.enkfmc_plan_work.argtypes = [vp, i64, vp]
    L.enkfmc_fp64_peak.argtypes = [vp, vp]
    L.enkfmc_fp64_mma_peak.argtypes = [vp, vp]
    _lib = L
    return L


_ERRORS = {-1: ConfigurationError, -2: ValueError, -3: NumericalError, -4: BackendError, -5: CapacityError}


def check(rc: int) -> None:
    """Map a negative ENKFMC_E_* code to the reference's exception type."""
    if rc == 0:
        return
    msg = lib().enkfmc_last_error().decode("utf-8", "replace")
    raise _ERRORS.get(rc, RuntimeError)(msg)


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def as_i64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.int64)
