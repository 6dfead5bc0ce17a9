"""Parity of the CUDA path against the CPU oracle on the BASELINE.json configurations (GPU box).

For each configuration: index maps bit-exact, T / D / Xa errors against the oracle (all tiles for the
small configs, a sample of fields for cfg3/cfg5), regression path statistics and stage times.
Writes a Markdown table to stdout (committed under profiles/)."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import torch  # noqa: E402

import paper_1606_00807_b200 as mck  # noqa: E402
from oracle import enkf_mc_oracle as orc  # noqa: E402
from paper_1606_00807_b200 import device, synthetic  # noqa: E402
from paper_1606_00807_b200.plan import COL_IDX, LOCAL_ORDER, ROW_PTR, Plan  # noqa: E402


FLOORS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "noise_floors.json")))


def run(name, w, oracle_fields, key=None):
    geo = mck.GridGeometry("grid2d", w.nx, w.ny, boundary=w.boundary, nfields=w.nfields)
    plan = Plan.decomposed(geo, w.delta, w.zeta)
    plan.set_observations(w.obs_indices)
    dX, dR, dYs = device.to_device(w.X), device.to_device(w.r_diag), device.to_device(w.Ys)
    dXa = torch.empty_like(dX)
    device.analysis_device(plan, dX, dR, dYs, dXa)
    torch.cuda.synchronize()
    plan.profile(True)
    for _ in range(3):
        device.analysis_device(plan, dX, dR, dYs, dXa)
    n, ms = plan.stage_times()
    ms = ms / n
    Xa = dXa.cpu().numpy()
    T = device.workspace_tensor(plan, 1, (plan.nfields, plan.nnz))
    D = device.workspace_tensor(plan, 2, (plan.nfields, plan.sum_nlocal))
    flags = device.workspace_tensor(plan, 3, (plan.nfields, plan.sum_nlocal), "i32")
    fl = plan.work(w.nens)
    nrow = flags.size
    if not oracle_fields:
        sw = (flags >> 8) & 255
        tr = (flags & 1) > 0
        print(f"| {name} | {w.nstate} | {w.nens} | {w.zeta} | - | - | - | - | "
              f"{100 * ((flags & 2) > 0).sum() / nrow:.1f} | {100 * ((flags & 16) > 0).sum() / nrow:.2f} | {100 * ((flags & 8) > 0).sum() / nrow:.1f} | "
              f"{ms[1] + ms[2]:.2f} | {ms[3]:.2f} | {w.nstate / (ms.sum() * 1e-3) / 1e6:.2f} | {fl[2] / (ms[1] + ms[2]) / 1e9:.2f} | {fl[1] / ms[3] / 1e9:.2f} | "
              f"no oracle; K2a {ms[1]:.2f} K2b {ms[2]:.2f} ms; listed {100 * tr.mean():.1f} %, sweeps mean {sw[tr].mean() if tr.any() else 0:.2f} max {sw.max()}, "
              f"block/8 hist {np.bincount(((flags >> 22) & 7)[tr]).tolist() if tr.any() else []}, why hist {np.bincount(((flags >> 5) & 7)[(flags & 16) > 0]).tolist()} |", flush=True)
        return
    grid = orc.grid_for(w.nx, w.ny, w.boundary, w.nfields)
    t0 = time.perf_counter()
    ref, kept = orc.assimilate(w.X, w.obs_indices, w.r_diag, w.Ys, grid, w.delta, w.zeta, keep_tiles=True,
                               fields=oracle_fields)
    t_cpu = time.perf_counter() - t0
    maps_ok = np.array_equal(plan.get(LOCAL_ORDER), np.concatenate([r.tile.local_order for r in kept[0]]))
    maps_ok &= np.array_equal(plan.get(COL_IDX), np.concatenate([r.factors.indices for r in kept[0]]))
    terr = derr = xerr = 0.0
    for k, f in enumerate(oracle_fields):
        tref = np.concatenate([r.factors.data for r in kept[k]])
        dref = np.concatenate([r.factors.d for r in kept[k]])
        terr = max(terr, np.linalg.norm(T[f] - tref) / np.linalg.norm(tref))
        derr = max(derr, np.max(np.abs(D[f] - dref) / dref))
        sl = slice(f * w.n2d, (f + 1) * w.n2d)
        xerr = max(xerr, np.linalg.norm(Xa[sl] - ref[sl]) / np.linalg.norm(ref[sl]))
    fl_ = FLOORS.get(key or "", {})
    def fmt(v, f):
        return f"{v:.1e} ({f:.1e})" if f is not None else f"{v:.1e} (-)"
    print(f"| {name} | {w.nstate} | {w.nens} | {w.zeta} | {'yes' if maps_ok else 'NO'} | {fmt(terr, fl_.get('T'))} | {fmt(derr, fl_.get('D'))} | {fmt(xerr, fl_.get('Xa'))} | "
          f"{100 * ((flags & 2) > 0).sum() / nrow:.1f} | {100 * ((flags & 16) > 0).sum() / nrow:.2f} | {100 * ((flags & 8) > 0).sum() / nrow:.1f} | "
          f"{ms[1] + ms[2]:.2f} | {ms[3]:.2f} | {w.nstate / (ms.sum() * 1e-3) / 1e6:.2f} | {fl[2] / (ms[1] + ms[2]) / 1e9:.2f} | {fl[1] / ms[3] / 1e9:.2f} | "
          f"{len(oracle_fields)} field(s), {t_cpu:.1f} s |", flush=True)

def levels_row():
    """Config 3 as worded (vertical radius 1) on a quarter-size grid: one 7-level variable, 96 x 48, N = 80, zeta = 4, 64 tiles; the
    oracle (extended to levels) on a sample of the tiles with its own floor from the member-permutation and solver-swap probes."""
    w = synthetic.make_workload("speedy_q", nx=96, ny=48, nens=80, corr_len=5.0, zeta=4, delta=64, obs="random", obs_arg=0.5,
                                r_rel=0.1, r_abs=None, seed=23, variables=[("u", 5.0, 7)])
    geo = mck.GridGeometry("grid2d", w.nx, w.ny, nfields=1, nlev=7, zeta_v=1)
    plan = Plan.decomposed(geo, w.delta, w.zeta)
    plan.set_observations(w.obs_indices)
    dX, dR, dYs = device.to_device(w.X), device.to_device(w.r_diag), device.to_device(w.Ys)
    dXa = torch.empty_like(dX)
    device.analysis_device(plan, dX, dR, dYs, dXa)
    torch.cuda.synchronize()
    plan.profile(True)
    for _ in range(3):
        device.analysis_device(plan, dX, dR, dYs, dXa)
    n, ms = plan.stage_times()
    ms = ms / n
    device.check_status(plan)
    Xa = dXa.cpu().numpy()
    T = device.workspace_tensor(plan, 1, (plan.nfields, plan.nnz))
    D = device.workspace_tensor(plan, 2, (plan.nfields, plan.sum_nlocal))
    flags = device.workspace_tensor(plan, 3, (plan.nfields, plan.sum_nlocal), "i32")
    from paper_1606_00807_b200.plan import TILE_PTR
    tp, rp = plan.get(TILE_PTR), plan.get(ROW_PTR)
    grid = orc.grid_for(w.nx, w.ny, "clipped", 1, nlev=7, zeta_v=1)
    tiles = orc.decompose(grid, w.delta, w.zeta)
    perm = np.random.default_rng(0).permutation(w.nens)
    inv = np.argsort(perm)
    t0 = time.perf_counter()
    terr = derr = xerr = tfl = dfl = xfl = 0.0
    sample = [9, 27, 36, 63]
    for t in sample:
        tile = tiles[t]
        csr = orc.predecessor_csr(grid, w.zeta, tile.local_order)
        res = orc.analyse_tile(w.X, w.obs_indices, w.r_diag, w.Ys, grid, w.zeta, tile, csr)
        res_p = orc.analyse_tile(w.X[:, perm], w.obs_indices, w.r_diag, w.Ys[:, perm], grid, w.zeta, tile, csr)
        with orc.linear_solver("lu"):
            res_s = orc.analyse_tile(w.X, w.obs_indices, w.r_diag, w.Ys, grid, w.zeta, tile, csr)
        ipos = tile.interior_positions()
        nt = np.linalg.norm(res.factors.data)
        terr = max(terr, np.linalg.norm(T[0, rp[tp[t]]:rp[tp[t + 1]]] - res.factors.data) / nt)
        tfl = max(tfl, np.linalg.norm(res_p.factors.data - res.factors.data) / nt)
        derr = max(derr, np.max(np.abs(D[0, tp[t]:tp[t + 1]] - res.factors.d) / res.factors.d))
        dfl = max(dfl, np.max(np.abs(res_p.factors.d - res.factors.d) / res.factors.d))
        xr = res.xa_local[ipos]
        xerr = max(xerr, np.linalg.norm(Xa[tile.interior] - xr) / np.linalg.norm(xr))
        xfl = max(xfl, np.linalg.norm(res_p.xa_local[ipos][:, inv] - xr) / np.linalg.norm(xr),
                  np.linalg.norm(res_s.xa_local[ipos] - xr) / np.linalg.norm(xr))
    t_cpu = time.perf_counter() - t0
    maps_ok = np.array_equal(plan.get(LOCAL_ORDER), np.concatenate([t.local_order for t in tiles]))
    fl = plan.work(w.nens)
    nrow = flags.size
    print(f"| cfg3 as worded, quarter grid: 96x48, one 7-level variable, vertical radius 1 (121 predecessors on 80 members) | {w.nstate} | {w.nens} | 4 (+1 vertical) | "
          f"{'yes' if maps_ok else 'NO'} | {terr:.1e} ({tfl:.1e}) | {derr:.1e} ({dfl:.1e}) | {xerr:.1e} ({xfl:.1e}) | "
          f"{100 * ((flags & 2) > 0).sum() / nrow:.1f} | {100 * ((flags & 16) > 0).sum() / nrow:.2f} | {100 * ((flags & 8) > 0).sum() / nrow:.1f} | "
          f"{ms[1] + ms[2]:.2f} | {ms[3]:.2f} | {w.nstate / (ms.sum() * 1e-3) / 1e6:.2f} | {fl[2] / (ms[1] + ms[2]) / 1e9:.2f} | {fl[1] / ms[3] / 1e9:.2f} | "
          f"{len(sample)} of 64 tiles, {t_cpu:.1f} s; floor measured here (member permutation, LU for Cholesky); pinned pivots {plan.counter(5)} |", flush=True)


ap = argparse.ArgumentParser()
ap.add_argument("--which", default="cfg1,cfg1p,cfg2,cfg2n,cfg4,cfg3,cfg3n,cfg3v,cfg5")
ap.add_argument("--no-oracle", action="store_true")
ap.add_argument("--fields", type=int, default=None)
a = ap.parse_args()
print("Errors against the CPU oracle; in parentheses the oracle's own noise floor on that input (tests/golden/noise_floors.json: the larger of the dgesvd-driver "
      "swap and the member-permutation probe, oracle/noise_floor.py).  Gates of the test-suite: max(1e-9 | 1e-9 | 1e-8, 10 x floor).\n")
print("| config | n_state | N | zeta | maps bit-exact | T err norm-wise (floor) | D err max rel (floor) | Xa err norm-wise (floor) | rows truncated % | "
      "Jacobi fallback % | D at floor % | K2 ms | K3 ms | Mpts/s | K2 TF/s | K3 TF/s | oracle sample |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
_run = run
def run(name, w, fields, key=None):
    return _run(name, w, [] if a.no_oracle else fields, key)
for which in a.which.split(","):
    if which == "cfg1":
        run("cfg1 clipped", synthetic.config("cfg1"), [0], "cfg1")
    elif which == "cfg1p":
        run("cfg1 periodic", synthetic.config("cfg1", boundary="periodic"), [0], "cfg1_periodic")
        run("cfg1 longitude periodic, latitude clipped (as worded)", synthetic.config("cfg1", boundary="periodic_x"), [0], "cfg1_lon_periodic")
    elif which == "cfg2":
        run("cfg2", synthetic.config("cfg2"), [0], "cfg2")
    elif which == "cfg2n":
        run("cfg2 + 1% nugget", synthetic.config("cfg2", nugget=0.01), [0], "cfg2_nugget")
    elif which == "cfg4":
        for z in range(1, 7):
            run(f"cfg4 r={z}", synthetic.config("cfg4", zeta=z), [0], f"cfg4_r{z}")
        run("cfg4 r=5 + 1% nugget", synthetic.config("cfg4", zeta=5, nugget=0.01), [0], "cfg4_r5_nugget")
    elif which == "cfg3":
        run("cfg3 (29 fields)", synthetic.config("cfg3", fields=a.fields), [0, 14, 28] if a.fields is None else [0], "cfg3")
    elif which == "cfg3n":
        run("cfg3 + 1% nugget", synthetic.config("cfg3", nugget=0.01), [0, 28], "cfg3_nugget")
    elif which == "cfg3v":
        levels_row()
    elif which == "cfg5":
        run(f"cfg5 ({a.fields or 8} of 40 fields)", synthetic.config("cfg5", fields=a.fields or 8), [0], "cfg5")
