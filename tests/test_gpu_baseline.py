"""-m gpu: every BASELINE.json configuration against the CPU oracle, gated by the oracle's own noise floor.

The as-specified (smooth, nugget-free) inputs are ill conditioned: the reference's answer itself moves by
1e-9 (T) ... 1e-3 (Xa) when only its SVD driver or the order of the ensemble members changes
(oracle/noise_floor.py; tests/golden/noise_floors.json is written by tools/make_floors.py).  Gates are
max(north_star gate, 10 x floor): T 1e-9 norm-wise, D 1e-9 max relative, Xa 1e-8 norm-wise.  Index maps are
bit-exact.  cfg3 / cfg5 run at their full horizontal size on their first fields (fields are independent
problems); the oracle is evaluated on a sample of the tiles so that the suite stays within minutes."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

FLOORS = json.load(open(os.path.join(GOLDEN, "noise_floors.json")))


def gates(key):
    f = FLOORS[key]
    return max(1e-9, 10.0 * f["T"]), max(1e-9, 10.0 * f["D"]), max(1e-8, 10.0 * f["Xa"])


# floor key, synthetic.config name + kwargs, tile sample (None: all)
CASES = [
    ("cfg1", "cfg1", {}, None),
    ("cfg1_nugget", "cfg1", {"nugget": 0.01}, None),
    ("cfg1_periodic", "cfg1", {"boundary": "periodic"}, None),
    ("cfg1_periodic_nugget", "cfg1", {"boundary": "periodic", "nugget": 0.01}, None),
    # longitude periodic, latitude clipped (config 1 as worded): per-axis boundary, checked against the extended oracle
    # (the reference has one flag for both axes: parity unpinned by the reference)
    ("cfg1_lon_periodic", "cfg1", {"boundary": "periodic_x"}, None),
    ("cfg2", "cfg2", {}, None),
    ("cfg2_nugget", "cfg2", {"nugget": 0.01}, None),
    ("cfg3", "cfg3", {"fields": 2}, list(range(1, 256, 5))),
    ("cfg3_nugget", "cfg3", {"fields": 2, "nugget": 0.01}, list(range(2, 256, 9))),
    ("cfg4_r1", "cfg4", {"zeta": 1}, None),
    ("cfg4_r2", "cfg4", {"zeta": 2}, None),
    ("cfg4_r3", "cfg4", {"zeta": 3}, None),
    ("cfg4_r4", "cfg4", {"zeta": 4}, list(range(1, 64, 2))),
    ("cfg4_r5", "cfg4", {"zeta": 5}, list(range(1, 64, 4))),
    ("cfg4_r6", "cfg4", {"zeta": 6}, list(range(2, 64, 4))),
    ("cfg4_r5_nugget", "cfg4", {"zeta": 5, "nugget": 0.01}, list(range(3, 64, 8))),
    ("cfg5", "cfg5", {"fields": 1}, list(range(5, 1024, 37))),
]


@pytest.mark.parametrize("key,name,kw,sample", CASES, ids=[c[0] for c in CASES])
def test_baseline_config_against_oracle(key, name, kw, sample):
    import torch

    import paper_1606_00807_b200 as mck
    from oracle import enkf_mc_oracle as orc
    from paper_1606_00807_b200 import device, synthetic
    from paper_1606_00807_b200.plan import COL_IDX, LOCAL_ORDER, ROW_PTR, TILE_PTR, Plan

    w = synthetic.config(name, **kw)
    geo = mck.GridGeometry("grid2d", w.nx, w.ny, boundary=w.boundary, nfields=w.nfields)
    plan = Plan.decomposed(geo, w.delta, w.zeta)
    plan.set_observations(w.obs_indices)
    dX, dR, dYs = device.to_device(w.X), device.to_device(w.r_diag), device.to_device(w.Ys)
    dXa = torch.empty_like(dX)
    device.analysis_device(plan, dX, dR, dYs, dXa)
    torch.cuda.synchronize()
    Xa = dXa.cpu().numpy()
    T = device.workspace_tensor(plan, 1, (plan.nfields, plan.nnz))
    D = device.workspace_tensor(plan, 2, (plan.nfields, plan.sum_nlocal))
    flags = device.workspace_tensor(plan, 3, (plan.nfields, plan.sum_nlocal), "i32")
    tp, rp = plan.get(TILE_PTR), plan.get(ROW_PTR)
    lo, ci = plan.get(LOCAL_ORDER), plan.get(COL_IDX)

    grid = orc.grid_for(w.nx, w.ny, w.boundary)
    tiles = orc.decompose(grid, w.delta, w.zeta)
    ids = range(len(tiles)) if sample is None else sample
    t_num = t_den = x_num = x_den = 0.0
    d_max = 0.0
    for f in range(w.nfields):
        a, b = f * w.n2d, (f + 1) * w.n2d
        sel = np.flatnonzero((w.obs_indices >= a) & (w.obs_indices < b))
        for k in ids:
            t = tiles[k]
            res = orc.analyse_tile(w.X[a:b], w.obs_indices[sel] - a, w.r_diag[sel], w.Ys[sel], grid, w.zeta, t)
            r0, r1 = tp[k], tp[k + 1]
            if f == 0:   # index maps: bit-exact
                assert np.array_equal(lo[r0:r1], t.local_order)
                assert np.array_equal(ci[rp[r0]:rp[r1]], res.factors.indices)
                assert np.array_equal(rp[r0:r1 + 1] - rp[r0], res.factors.indptr)
            tg = T[f, rp[r0]:rp[r1]]
            t_num += np.sum((tg - res.factors.data) ** 2)
            t_den += np.sum(res.factors.data ** 2)
            d_max = max(d_max, float(np.max(np.abs(D[f, r0:r1] - res.factors.d) / res.factors.d)))
            xr = res.xa_local[t.interior_positions()]
            xg = Xa[a + t.interior]
            x_num += np.sum((xg - xr) ** 2)
            x_den += np.sum(xr ** 2)
    t_err, x_err = np.sqrt(t_num / t_den), np.sqrt(x_num / x_den)
    gt, gd, gx = gates(key)
    fb = float(((flags & 16) > 0).mean())
    print(f"{key}: T {t_err:.2e} (gate {gt:.1e})  D {d_max:.2e} (gate {gd:.1e})  Xa {x_err:.2e} (gate {gx:.1e})  "
          f"truncated {100 * ((flags & 2) > 0).mean():.1f} %  Jacobi fallback {100 * fb:.2f} %")
    assert t_err < gt, (t_err, gt)
    assert d_max < gd, (d_max, gd)
    assert x_err < gx, (x_err, gx)
    assert fb < 0.05, fb     # the general fallback stays the exception on every BASELINE configuration
    assert plan.counter(5) == 0   # no clamped Cholesky pivots
