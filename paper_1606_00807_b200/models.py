"""Forecast hooks of the device-resident cycle loop.

Only what ``run_filter`` needs to keep the ensemble on the device between analyses: the identity model and the
periodic advection-diffusion field (models.py:53-83, 114-132).  The chaotic ring model and the rest of the
reference's model zoo are outside the hot path and are not built.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _lib, device
from .errors import ConfigurationError
from .geometry import GridGeometry

MODEL_KINDS = ("advdiff2d", "identity")


@dataclass(frozen=True)
class ModelHandle:
    kind: str
    geometry: GridGeometry
    dt: float = 0.0
    steps_per_window: int = 1
    velocity: tuple = (1.0, 0.5)
    diffusivity: float = 0.05


def identity_model(geometry: GridGeometry) -> ModelHandle:
    return ModelHandle(kind="identity", geometry=geometry, dt=1.0, steps_per_window=1)


def advdiff2d_model(geometry: GridGeometry, velocity=(1.0, 0.5), diffusivity: float = 0.05, dt: float = 0.05,
                    steps_per_window: int = 4) -> ModelHandle:
    """models.py:53-79 (same checks, same messages)."""
    if geometry.kind != "grid2d":
        raise ConfigurationError("advdiff2d requires a grid2d geometry")
    if dt <= 0 or steps_per_window < 1:
        raise ConfigurationError(f"invalid dt={dt} or steps_per_window={steps_per_window}")
    if diffusivity < 0:
        raise ConfigurationError(f"diffusivity must be nonnegative, got {diffusivity}")
    margin = diffusivity * dt * 2.0
    if margin > 0.25:
        raise ConfigurationError(f"unstable explicit diffusion: kappa*dt*(1/dx^2+1/dy^2) = {margin:.4g} > 0.25")
    return ModelHandle(kind="advdiff2d", geometry=geometry, dt=float(dt), steps_per_window=int(steps_per_window),
                       velocity=(float(velocity[0]), float(velocity[1])), diffusivity=float(diffusivity))


def window_steps(model: ModelHandle, window) -> int:
    """models.py:135-150."""
    if window is None:
        return model.steps_per_window
    if window < 0:
        raise ValueError(f"window must be nonnegative, got {window}")
    if model.kind == "identity":
        return 1 if window else 0
    ratio = window / model.dt
    steps = int(round(ratio))
    if abs(ratio - steps) > 1e-9 * max(1.0, abs(ratio)):
        raise ValueError(f"window {window} is not an integer multiple of dt {model.dt}")
    return steps


def propagate_device(model: ModelHandle, dX, dTmp, window=None):
    """Advance every member on the device; returns the tensor holding the result (dX or dTmp: they ping-pong)."""
    if model.kind not in MODEL_KINDS:
        raise ConfigurationError(f"model {model.kind!r} is outside the B200 hot path; only {MODEL_KINDS} are built")
    steps = window_steps(model, window)
    if model.kind == "identity" or steps == 0:
        return dX
    g = model.geometry
    src, dst = dX, dTmp
    for _ in range(steps):
        _lib.check(_lib.lib().enkfmc_advdiff_step(src.data_ptr(), dst.data_ptr(), g.nx, g.ny, int(g.row_major),
                                                  g.nfields * getattr(g, "nlev", 1),   # every level is advected as a 2-D field
                                                  src.shape[1], model.velocity[0], model.velocity[1], model.dt,
                                                  model.diffusivity, device.stream_ptr()))
        src, dst = dst, src
    return src
