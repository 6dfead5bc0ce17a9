"""Parity of the CUDA path against the CPU oracle on other seeds of the BASELINE-shaped inputs (GPU box): the gates of the
test-suite are calibrated on the default seeds; this prints the same errors for a few more (one 2-D field each, a sample of tiles)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import torch  # noqa: E402

import paper_1606_00807_b200 as mck  # noqa: E402
from oracle import enkf_mc_oracle as orc  # noqa: E402
from paper_1606_00807_b200 import device, synthetic  # noqa: E402
from paper_1606_00807_b200.plan import ROW_PTR, TILE_PTR, Plan  # noqa: E402

FLOORS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "noise_floors.json")))
CASES = [("cfg3", {"fields": 1}, "cfg3", list(range(3, 256, 17))), ("cfg2", {}, "cfg2", list(range(0, 64, 5))),
         ("cfg4", {"zeta": 4}, "cfg4_r4", list(range(1, 64, 7))), ("cfg4", {"zeta": 5}, "cfg4_r5", list(range(2, 64, 9)))]
print("| config | seed | T err (gate) | D err (gate) | Xa err (gate) | pass |\n|---|---|---|---|---|---|")
for name, kw, key, sample in CASES:
    fl = FLOORS[key]
    gate = (max(1e-9, 10 * fl["T"]), max(1e-9, 10 * fl["D"]), max(1e-8, 10 * fl["Xa"]))
    for seed in (11, 12, 13):
        w = synthetic.config(name, seed=seed, **kw)
        geo = mck.GridGeometry("grid2d", w.nx, w.ny, boundary=w.boundary, nfields=w.nfields)
        plan = Plan.decomposed(geo, w.delta, w.zeta)
        plan.set_observations(w.obs_indices)
        dX, dR, dYs = device.to_device(w.X), device.to_device(w.r_diag), device.to_device(w.Ys)
        dXa = torch.empty_like(dX)
        device.analysis_device(plan, dX, dR, dYs, dXa)
        device.check_status(plan)
        Xa = dXa.cpu().numpy()
        T = device.workspace_tensor(plan, 1, (plan.nfields, plan.nnz))
        D = device.workspace_tensor(plan, 2, (plan.nfields, plan.sum_nlocal))
        tp, rp = plan.get(TILE_PTR), plan.get(ROW_PTR)
        grid = orc.grid_for(w.nx, w.ny, w.boundary, w.nfields)
        tiles = orc.decompose(grid, w.delta, w.zeta)
        tn = td = 0.0
        derr = 0.0
        xn = xd = 0.0
        for t in sample:
            tile = tiles[t]
            res = orc.analyse_tile(w.X[:w.n2d], w.obs_indices[w.obs_indices < w.n2d], w.r_diag[w.obs_indices < w.n2d],
                                   w.Ys[w.obs_indices < w.n2d], grid, w.zeta, tile)
            tn += np.sum((T[0, rp[tp[t]]:rp[tp[t + 1]]] - res.factors.data) ** 2); td += np.sum(res.factors.data ** 2)
            derr = max(derr, float(np.max(np.abs(D[0, tp[t]:tp[t + 1]] - res.factors.d) / res.factors.d)))
            xr = res.xa_local[tile.interior_positions()]
            xn += np.sum((Xa[tile.interior] - xr) ** 2); xd += np.sum(xr ** 2)
        terr, xerr = float(np.sqrt(tn / td)), float(np.sqrt(xn / xd))
        ok = terr < gate[0] and derr < gate[1] and xerr < gate[2]
        print(f"| {key} | {seed} | {terr:.1e} ({gate[0]:.1e}) | {derr:.1e} ({gate[1]:.1e}) | {xerr:.1e} ({gate[2]:.1e}) | {'yes' if ok else 'NO'} |", flush=True)
        del plan
