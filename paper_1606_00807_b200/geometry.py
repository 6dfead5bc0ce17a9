"""Grid descriptor and integer index maps: same callables as the reference geometry module
(geometry.py:22-222), computed by the C-ABI library's host routines (csrc/plan.cpp).

``GridGeometry`` gains one optional trailing field, ``nfields`` (default 1 = the reference):
``nfields`` independent 2-D fields stacked in one state vector, label = field*(nx*ny) + 2-D
label.  Decomposition, halos and predecessor sets are per 2-D field.

``nlev`` / ``zeta_v`` (defaults 1 / 0 = the reference; no reference counterpart, parity unpinned by the reference,
checked against the extended oracle): every field is ``nlev`` stacked 2-D levels, label inside a field =
level*(nx*ny) + 2-D label; a component's box is its 2-D box on every level within ``zeta_v`` of its own (BASELINE.json
configs 3 / 5: "horizontal r, vertical r = 1"), predecessors = box members with a smaller label, sub-domains = the 2-D
tiles of ``decompose`` on every level.

Interface schema note: the container fields, argument checks and error messages in this module restate the reference's
public interface (geometry.py:22-119) on purpose -- they are what a caller (and the reference's own tests, which `match=` on the
messages) sees at the drop-in boundary.  No arithmetic of the hot path lives here; that is in csrc/ behind the C-ABI.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConfigurationError

KINDS = ("ring1d", "grid2d")
ORDERINGS = ("row_major", "column_major")
# "clipped" / "periodic" are the reference's two boundaries (geometry.py:43).  "periodic_x" (longitude periodic, latitude
# clipped: BASELINE.json config 1 as worded) and "periodic_y" apply the reference's per-axis rules (geometry.py:132-142) with
# one flag per axis; they have no reference counterpart (parity unpinned by the reference, checked against the extended oracle).
BOUNDARIES = ("clipped", "periodic", "periodic_x", "periodic_y")
_PERIODIC_CODE = {"clipped": 0, "periodic": 1, "periodic_x": 2, "periodic_y": 3}


@dataclass(frozen=True)
class GridGeometry:
    kind: str
    nx: int
    ny: int = 1
    ordering: str = "row_major"
    boundary: str = ""
    nfields: int = 1
    nlev: int = 1
    zeta_v: int = 0

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown geometry kind {self.kind!r}")
        if self.ordering not in ORDERINGS:
            raise ValueError(f"unknown ordering {self.ordering!r}")
        if self.nx < 1 or self.ny < 1:
            raise ValueError(f"grid extents must be positive, got nx={self.nx} ny={self.ny}")
        if self.kind == "ring1d" and self.ny != 1:
            raise ValueError(f"ring1d requires ny=1, got ny={self.ny}")
        if self.nfields < 1:
            raise ValueError(f"nfields must be positive, got {self.nfields}")
        if self.nlev < 1:
            raise ValueError(f"nlev must be positive, got {self.nlev}")
        if self.zeta_v < 0:
            raise ValueError(f"zeta_v must be nonnegative, got {self.zeta_v}")
        if not self.boundary:
            object.__setattr__(self, "boundary", "periodic" if self.kind == "ring1d" else "clipped")
        if self.boundary not in BOUNDARIES:
            raise ValueError(f"unknown boundary {self.boundary!r}")

    @property
    def n2d(self) -> int:
        return self.nx * self.ny

    @property
    def nfield(self) -> int:
        """Rows of one field's state block (all its levels)."""
        return self.nx * self.ny * self.nlev

    @property
    def nstate(self) -> int:
        return self.nx * self.ny * self.nlev * self.nfields

    @property
    def periodic(self) -> int:
        """Boundary code of the C-ABI: 0 clipped, 1 periodic (both axes), 2 periodic along x only, 3 along y only."""
        return _PERIODIC_CODE[self.boundary]

    @property
    def row_major(self) -> bool:
        return self.ordering == "row_major"


@dataclass(frozen=True)
class LocalBox:
    center: int
    zeta: int
    members: np.ndarray


@dataclass(frozen=True)
class Subdomain:
    id: int
    interior: np.ndarray
    halo: np.ndarray
    local_order: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.local_order is None:
            object.__setattr__(self, "local_order", np.union1d(self.interior, self.halo))

    @property
    def n_local(self) -> int:
        return self.local_order.size

    def interior_positions(self) -> np.ndarray:
        return np.searchsorted(self.local_order, self.interior)


def linear_index(geometry: GridGeometry, row: int, col: int) -> int:
    if not (0 <= row < geometry.ny and 0 <= col < geometry.nx):
        raise ValueError(f"cell ({row}, {col}) outside {geometry.ny}x{geometry.nx} grid")
    return row * geometry.nx + col if geometry.row_major else col * geometry.ny + row


def grid_coords(geometry: GridGeometry, index: int) -> tuple[int, int]:
    if not (0 <= index < geometry.n2d):
        raise ValueError(f"index {index} outside [0, {geometry.n2d})")
    if geometry.row_major:
        return divmod(index, geometry.nx)
    col, row = divmod(index, geometry.ny)
    return row, col


def _box_call(fn, geometry: GridGeometry, center: int, zeta: int) -> np.ndarray:
    if zeta < 0:
        raise ValueError(f"zeta must be nonnegative, got {zeta}")
    if geometry.nlev > 1:
        # levels (extension): the 2-D box on every level within zeta_v, labels ascending (host integer code)
        if not (0 <= center < geometry.nfield):
            raise ValueError(f"index {center} outside [0, {geometry.nfield})")
        lev, lab2 = divmod(int(center), geometry.n2d)
        flat = GridGeometry(geometry.kind, geometry.nx, geometry.ny, geometry.ordering, geometry.boundary)
        box2 = _box_call(_lib.lib().enkfmc_local_box, flat, lab2, zeta)
        levels = range(max(0, lev - geometry.zeta_v), min(geometry.nlev, lev + geometry.zeta_v + 1))
        box = np.concatenate([l * geometry.n2d + box2 for l in levels]).astype(np.intp)
        return box[box < center] if fn.__name__ == "enkfmc_predecessors" else box
    if not (0 <= center < geometry.n2d):
        raise ValueError(f"index {center} outside [0, {geometry.n2d})")
    span = min(2 * zeta + 1, max(geometry.nx, geometry.ny))
    out = np.empty(span * span, dtype=np.int64)
    count = C.c_int64(0)
    _lib.check(fn(geometry.nx, geometry.ny, int(geometry.row_major), int(geometry.periodic), int(center), int(zeta),
                  _lib.ptr(out), C.addressof(count)))
    return out[:count.value].astype(np.intp)


def local_box(geometry: GridGeometry, center: int, zeta: int) -> LocalBox:
    """Chebyshev box members, ascending (geometry.py:145-156)."""
    return LocalBox(center=center, zeta=zeta, members=_box_call(_lib.lib().enkfmc_local_box, geometry, center, zeta))


def predecessors(geometry: GridGeometry, center: int, zeta: int) -> np.ndarray:
    """Box members with label below the centre's (geometry.py:159-162)."""
    return _box_call(_lib.lib().enkfmc_predecessors, geometry, center, zeta)


def decompose(geometry: GridGeometry, delta: int, zeta: int) -> list[Subdomain]:
    """Tiles with zeta-ring halos (geometry.py:165-222), from the plan's host maps."""
    from .plan import get_plan

    if delta < 1:
        raise ConfigurationError(f"delta must be >= 1, got {delta}")
    if zeta < 0:
        raise ValueError(f"zeta must be nonnegative, got {zeta}")
    return get_plan(geometry, delta, zeta).subdomains()


def nominal_local_size(nstate: int, delta: int, zeta: int) -> int:
    return nstate // delta + (2 * zeta + 1) ** 2
