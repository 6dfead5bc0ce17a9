"""Domain-decomposed analysis driver: the drop-in entry point (driver.py:41-253).

``assimilate_parallel`` keeps the reference signature.  One call = validate on the host,
``enkfmc_analysis_host`` (H2D -> K0 centre -> K2 regress -> K3 local solve + interior
scatter -> D2H).  Index maps are cached per (geometry, delta, zeta) and per observation
pattern, so repeated cycles only move Xb, Ys and Xa.

Interface schema note: the container fields, argument checks and error messages in this module restate the reference's
public interface (driver.py:41-125,159-192) on purpose -- they are what a caller (and the reference's own tests, which `match=` on the
messages) sees at the drop-in boundary.  No arithmetic of the hot path lives here; that is in csrc/ behind the C-ABI.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import device
from .errors import ConfigurationError, ConsistencyError, NumericalError
from .geometry import GridGeometry, Subdomain
from .kernels import EnsembleState, ObservationNetwork, perturb_observations
from .plan import get_plan

METHODS = ("enkf_mc_primal", "enkf_mc_dual", "letkf")
TIMINGS_HEADER = "cycle,method,delta,workers,t_estimation_max,t_analysis_max,t_merge,t_total"


@dataclass(frozen=True)
class AssimilationConfig:
    zeta: int = 1
    delta: int = 1
    workers: int = 1          # accepted for compatibility; results never depend on it
    method: str = "enkf_mc_primal"
    inflation: float = 1.0
    seed: int = 0
    dense_cap: int = 4096

    def __post_init__(self):
        if self.zeta < 0:
            raise ConfigurationError(f"zeta must be nonnegative, got {self.zeta}")
        if self.delta < 1:
            raise ConfigurationError(f"delta must be at least 1, got {self.delta}")
        if self.workers < 1:
            raise ConfigurationError(f"workers must be at least 1, got {self.workers}")
        if self.method not in METHODS:
            raise ConfigurationError(f"unknown method {self.method!r}; choose from {METHODS}")
        if self.inflation <= 0:
            raise ConfigurationError(f"inflation must be positive, got {self.inflation}")
        if self.dense_cap < 1:
            raise ConfigurationError(f"dense_cap must be positive, got {self.dense_cap}")


@dataclass(frozen=True)
class CycleReport:
    cycle: int
    method: str
    delta: int
    workers: int
    t_estimation: np.ndarray   # per sub-domain, seconds (device time of the fused stage / delta)
    t_analysis: np.ndarray
    t_merge: float
    t_total: float
    t_h2d: float = 0.0
    t_d2h: float = 0.0

    @property
    def t_estimation_max(self) -> float:
        return float(self.t_estimation.max()) if self.t_estimation.size else 0.0

    @property
    def t_analysis_max(self) -> float:
        return float(self.t_analysis.max()) if self.t_analysis.size else 0.0

    def csv_row(self) -> str:
        return (f"{self.cycle},{self.method},{self.delta},{self.workers},"
                f"{self.t_estimation_max:.6f},{self.t_analysis_max:.6f},{self.t_merge:.6f},{self.t_total:.6f}")


def merge_interiors(template: EnsembleState, pieces: list[tuple[Subdomain, np.ndarray]]) -> EnsembleState:
    """out[interior] = local[interior_positions] for every piece, exactly once (driver.py:99-125).

    Coverage accounting is integer host logic; the row scatter runs on the device.
    """
    counts = np.zeros(template.nstate, dtype=np.intp)
    dst_rows, src_rows, blocks, offset = [], [], [], 0
    for sd, local in pieces:
        local = np.asarray(local, dtype=np.float64)
        if local.shape != (sd.n_local, template.nens):
            raise ValueError(f"subdomain {sd.id}: local analysis has shape {local.shape}, "
                             f"expected {(sd.n_local, template.nens)}")
        dst_rows.append(sd.interior)
        src_rows.append(sd.interior_positions() + offset)
        blocks.append(local)
        offset += sd.n_local
        counts[sd.interior] += 1
    if np.any(counts != 1):
        dup, missing = np.flatnonzero(counts > 1), np.flatnonzero(counts == 0)
        raise ConsistencyError(f"interiors must cover each index exactly once: "
                               f"{dup.size} duplicated, {missing.size} missing")
    d_out = device.to_device(template.X)
    d_src = device.to_device(np.concatenate(blocks, axis=0))
    device.scatter_rows(d_out, np.concatenate(dst_rows), d_src, np.concatenate(src_rows))
    return EnsembleState(d_out.cpu().numpy(), role="analysis")


def _assimilate_dual(Xb, net, cfg, geometry, Ys, cycle, t_start):
    """method="enkf_mc_dual" (driver.py:214-229): the observation-space route sub-domain by sub-domain -- estimation and the
    covariance square root on the device, orchestration on the host.  The second route of the primal == dual self-check,
    not the timed hot path (only single-field geometries)."""
    from .estimator import fit_factors
    from .geometry import decompose
    from .kernels import analysis_dual, restrict_network
    from .validation import center_rows
    if geometry.nfields != 1 or getattr(geometry, "nlev", 1) != 1:
        raise ConfigurationError("method 'enkf_mc_dual' is built for single-field geometries only")
    subs = decompose(geometry, cfg.delta, cfg.zeta)
    out = Xb.X.copy()
    t_est, t_ana = np.zeros(len(subs)), np.zeros(len(subs))
    for k, sd in enumerate(subs):
        t0 = time.perf_counter()
        xb_loc = EnsembleState(Xb.X[sd.local_order])
        factors = fit_factors(center_rows(xb_loc.X), geometry, cfg.zeta, sd.local_order)
        t1 = time.perf_counter()
        net_loc, rows = restrict_network(net, sd.local_order)
        xa_loc = analysis_dual(xb_loc, factors, net_loc, Ys[rows])
        out[sd.interior] = xa_loc.X[sd.interior_positions()]
        t_est[k], t_ana[k] = t1 - t0, time.perf_counter() - t1
    report = CycleReport(cycle=int(cycle), method=cfg.method, delta=cfg.delta, workers=cfg.workers, t_estimation=t_est,
                         t_analysis=t_ana, t_merge=0.0, t_total=time.perf_counter() - t_start)
    return EnsembleState(out, role="analysis"), report


def assimilate_parallel(Xb: EnsembleState, net: ObservationNetwork, cfg: AssimilationConfig,
                        geometry: GridGeometry, *, Ys: np.ndarray | None = None,
                        cycle: int = 0) -> tuple[EnsembleState, CycleReport]:
    """One analysis cycle over the decomposed domain (driver.py:159-253)."""
    t_start = time.perf_counter()
    if Xb.nstate != geometry.nstate:
        raise ValueError(f"state dimension {Xb.nstate} does not match geometry {geometry.nstate}")
    if Xb.nens < 2:
        raise ConfigurationError(f"ensemble size must be at least 2, got {Xb.nens}")
    if net.nobs and net.obs_indices[-1] >= geometry.nstate:
        raise ValueError("observation indices exceed the state dimension")
    if cfg.method == "letkf":                    # the paper's comparison method (driver.py:128-156, 207-213)
        from .geometry import decompose
        from .kernels import letkf_analysis_global
        delta = len(decompose(geometry, cfg.delta, cfg.zeta))          # same decomposition errors as the reference
        xa = letkf_analysis_global(Xb, geometry, net, cfg.zeta, cfg.inflation)
        t = time.perf_counter() - t_start
        return xa, CycleReport(cycle=int(cycle), method=cfg.method, delta=cfg.delta, workers=cfg.workers,
                               t_estimation=np.zeros(delta), t_analysis=np.full(delta, t / delta), t_merge=0.0, t_total=t)
    if Ys is None:
        Ys = perturb_observations(net, Xb.nens, cfg.seed, cycle).Ys
    Ys = np.ascontiguousarray(Ys, dtype=np.float64)
    if Ys.shape != (net.nobs, Xb.nens):
        raise ValueError(f"Ys has shape {Ys.shape}, expected {(net.nobs, Xb.nens)}")
    if cfg.method == "enkf_mc_dual":
        return _assimilate_dual(Xb, net, cfg, geometry, Ys, cycle, t_start)

    plan = get_plan(geometry, cfg.delta, cfg.zeta)
    plan.set_observations(net.obs_indices)
    X = np.ascontiguousarray(Xb.X)
    Xa, tm = device.analysis_host(plan, X, np.ascontiguousarray(net.r_diag), Ys)
    delta = plan.ntiles
    report = CycleReport(
        cycle=int(cycle), method=cfg.method, delta=cfg.delta, workers=cfg.workers,
        t_estimation=np.full(delta, tm[1] * 1e-3 / delta), t_analysis=np.full(delta, tm[2] * 1e-3 / delta),
        t_merge=0.0, t_total=time.perf_counter() - t_start, t_h2d=tm[0] * 1e-3, t_d2h=tm[3] * 1e-3,
    )
    # Xa is finite by construction: K3b flags any non-finite increment per tile (status 2 -> NumericalError
    # above) and rows of tiles without observations are copies of the validated background, so the
    # O(n N) host re-scan of EnsembleState.__post_init__ is skipped.
    out = object.__new__(EnsembleState)
    object.__setattr__(out, "X", Xa)
    object.__setattr__(out, "role", "analysis")
    return out, report


@dataclass
class FilterResult:
    """Outcome of a multi-cycle run (driver.py:272-279): per-cycle analyses and reports, plus the final propagated
    background (X0 itself for an empty schedule)."""

    analyses: list
    reports: list
    final: EnsembleState


def run_filter(X0: EnsembleState, model, schedule, cfg: AssimilationConfig, *, keep_analyses: bool = True) -> FilterResult:
    """Alternate analysis and propagation over a schedule of (window, network) cycles (driver.py:282-310) with the
    ensemble resident on the device: per cycle only the perturbed observations -- generated on the host from the
    reference's (seed, cycle) stream -- and the observation error variances are uploaded; the analysis is the
    background of the next cycle after the device forecast step (models.propagate_device).  ``keep_analyses=False``
    skips the per-cycle download of the analysis ensembles (the reference returns them all)."""
    import torch

    from .models import propagate_device
    from .plan import Plan

    geometry = model.geometry
    if X0.nstate != geometry.nstate:
        raise ValueError(f"state dimension {X0.nstate} does not match geometry {geometry.nstate}")
    if X0.nens < 2:
        raise ConfigurationError(f"ensemble size must be at least 2, got {X0.nens}")
    if cfg.method != "enkf_mc_primal":
        raise ConfigurationError(f"method {cfg.method!r} is outside the B200 hot path; only 'enkf_mc_primal' is built")
    analyses, reports = [], []
    if not schedule:
        return FilterResult(analyses, reports, X0)
    plan = Plan.decomposed(geometry, cfg.delta, cfg.zeta)      # owned by this run: the cached plan of assimilate_parallel stays untouched
    dX = device.to_device(np.ascontiguousarray(X0.X))
    dXa, dTmp = torch.empty_like(dX), torch.empty_like(dX)
    for k, (window, net) in enumerate(schedule):
        t0 = time.perf_counter()
        if net.nobs and net.obs_indices[-1] >= geometry.nstate:
            raise ValueError("observation indices exceed the state dimension")
        Ys = np.ascontiguousarray(perturb_observations(net, X0.nens, cfg.seed, k).Ys)
        plan.set_observations(net.obs_indices)
        dYs = device.to_device(Ys if net.nobs else np.zeros((1, X0.nens)))
        dR = device.to_device(np.ascontiguousarray(net.r_diag) if net.nobs else np.ones(1))
        device.analysis_device(plan, dX, dR, dYs, dXa)
        device.check_status(plan)
        if keep_analyses:
            out = object.__new__(EnsembleState)
            object.__setattr__(out, "X", dXa.cpu().numpy())
            object.__setattr__(out, "role", "analysis")
            analyses.append(out)
        nxt = propagate_device(model, dXa, dTmp, window)
        if nxt is dXa:
            dX, dXa = dXa, dX
        else:                      # the forecast landed in dTmp
            dX, dTmp = dTmp, dX
        delta = plan.ntiles
        t = time.perf_counter() - t0
        reports.append(CycleReport(cycle=k, method=cfg.method, delta=cfg.delta, workers=cfg.workers,
                                   t_estimation=np.zeros(delta), t_analysis=np.zeros(delta), t_merge=0.0, t_total=t,
                                   t_h2d=0.0, t_d2h=0.0))
    torch.cuda.synchronize()
    final = EnsembleState(dX.cpu().numpy(), role="background")
    return FilterResult(analyses, reports, final)


_SHARDED: dict = {}     # (geometry, delta, zeta, rank, world) -> (plan, shard, device buffers)


def assimilate_parallel_sharded(Xb: EnsembleState | None, net: ObservationNetwork, cfg: AssimilationConfig,
                                geometry: GridGeometry, *, Ys: np.ndarray | None = None, cycle: int = 0,
                                root: int = 0, nens: int | None = None):
    """assimilate_parallel (driver.py:159-253) over the ranks of an initialised torch.distributed process group, one
    process per GPU.  The sub-domains are split by contiguous block rows (distributed.TileShard); ``root`` holds the
    background and the perturbed observations on the host (the other ranks pass ``Xb=None`` and ``nens``), uploads
    them, scatters to every rank the state rows and observation rows its tiles read, every rank analyses its tiles,
    and the interior rows are all-gathered.  Returns ``(EnsembleState, CycleReport)`` on ``root`` and ``(None, report)``
    elsewhere.  A failing sub-domain raises NumericalError on every rank."""
    import torch
    import torch.distributed as dist

    from . import distributed

    t_start = time.perf_counter()
    rank, world = dist.get_rank(), dist.get_world_size()
    if cfg.method != "enkf_mc_primal":
        raise ConfigurationError(f"method {cfg.method!r} is outside the B200 hot path; only 'enkf_mc_primal' is built")
    if rank == root:
        if Xb is None:
            raise ValueError("the root rank must pass the background ensemble")
        if Xb.nstate != geometry.nstate:
            raise ValueError(f"state dimension {Xb.nstate} does not match geometry {geometry.nstate}")
        nens = Xb.nens
        if Ys is None:
            Ys = perturb_observations(net, nens, cfg.seed, cycle).Ys
        Ys = np.ascontiguousarray(Ys, dtype=np.float64)
        if Ys.shape != (net.nobs, nens):
            raise ValueError(f"Ys has shape {Ys.shape}, expected {(net.nobs, nens)}")
    elif nens is None:
        raise ValueError("ranks other than the root must pass nens")
    if nens < 2:
        raise ConfigurationError(f"ensemble size must be at least 2, got {nens}")
    if net.nobs and net.obs_indices[-1] >= geometry.nstate:
        raise ValueError("observation indices exceed the state dimension")

    key = (geometry, cfg.delta, cfg.zeta, rank, world)
    ent = _SHARDED.get(key)
    if ent is None or ent[2]["nens"] != nens or ent[2]["nobs"] != net.nobs:
        from .plan import Plan
        plan = Plan.decomposed(geometry, cfg.delta, cfg.zeta)
        shard = distributed.TileShard(plan, geometry, rank, world)
        shard.apply()
        bufs = {"nens": nens, "nobs": net.nobs,
                "X": torch.empty((geometry.nstate, nens), dtype=torch.float64, device="cuda"),
                "Xa": torch.empty((geometry.nstate, nens), dtype=torch.float64, device="cuda"),
                "Ys": torch.empty((max(net.nobs, 1), nens), dtype=torch.float64, device="cuda")}
        ent = _SHARDED[key] = (plan, shard, bufs)
    plan, shard, bufs = ent
    plan.set_observations(net.obs_indices)
    if shard.need_obs is None or bufs.get("obs_key") != plan._obs_key:
        shard.set_observations(net.obs_indices)
        bufs["obs_key"] = plan._obs_key
        bufs["R"] = device.to_device(np.ascontiguousarray(net.r_diag))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    if rank == root:
        bufs["X"].copy_(torch.from_numpy(np.ascontiguousarray(Xb.X)), non_blocking=True)
        if net.nobs:
            bufs["Ys"][: net.nobs].copy_(torch.from_numpy(Ys), non_blocking=True)
    shard.scatter_background(bufs["X"], bufs["Ys"], root=root)
    ev[1].record()
    device.analysis_device(plan, bufs["X"], bufs["R"], bufs["Ys"], bufs["Xa"])
    ev[2].record()
    shard.gather_analysis(bufs["Xa"])
    failed = torch.zeros(1, dtype=torch.int32, device="cuda")
    err = None
    try:
        device.check_status(plan)
    except NumericalError as exc:           # raise on every rank, naming the sub-domain where one is known
        err = exc
        failed += 1
    dist.all_reduce(failed, op=dist.ReduceOp.MAX)
    if int(failed.item()):
        raise err if err is not None else NumericalError("primal analysis solve failed in a sub-domain of another rank")
    out = None
    if rank == root:
        Xa = device.pinned_empty((geometry.nstate, nens))
        torch.from_numpy(Xa).copy_(bufs["Xa"], non_blocking=True)
    ev[3].record()
    torch.cuda.synchronize()
    if rank == root:
        out = object.__new__(EnsembleState)
        object.__setattr__(out, "X", Xa)
        object.__setattr__(out, "role", "analysis")
    delta = plan.ntiles
    t_est = ev[1].elapsed_time(ev[2]) * 1e-3
    report = CycleReport(
        cycle=int(cycle), method=cfg.method, delta=cfg.delta, workers=cfg.workers,
        t_estimation=np.full(delta, t_est / delta), t_analysis=np.zeros(delta),
        t_merge=ev[2].elapsed_time(ev[3]) * 1e-3, t_total=time.perf_counter() - t_start,
        t_h2d=ev[0].elapsed_time(ev[1]) * 1e-3, t_d2h=0.0,
    )
    return out, report
