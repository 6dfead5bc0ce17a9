"""GPU vs GPU: T, D from the full decomposed plan against per-tile fit_factors (local plans)."""
import sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/", 2)[0])
import torch
import paper_1606_00807_b200 as mck
from oracle import enkf_mc_oracle as orc
from paper_1606_00807_b200 import device, synthetic
from paper_1606_00807_b200.plan import Plan, ROW_PTR, TILE_PTR
name, nf = sys.argv[1], int(sys.argv[2])
w = synthetic.config(name, fields=nf)
geo = mck.GridGeometry("grid2d", w.nx, w.ny, nfields=w.nfields)
plan = Plan.decomposed(geo, w.delta, w.zeta)
plan.set_observations(w.obs_indices)
dX, dR, dYs = device.to_device(w.X), device.to_device(w.r_diag), device.to_device(w.Ys)
dXa = torch.empty_like(dX)
device.analysis_device(plan, dX, dR, dYs, dXa)
T = device.workspace_tensor(plan, 1, (plan.nfields, plan.nnz))
D = device.workspace_tensor(plan, 2, (plan.nfields, plan.sum_nlocal))
F = device.workspace_tensor(plan, 3, (plan.nfields, plan.sum_nlocal), "i32")
U = device.workspace_tensor(plan, 0, (w.nstate, w.nens))
print("U centred check:", np.abs(U - orc.center_rows(w.X)).max())
tp, rp = plan.get(TILE_PTR), plan.get(ROW_PTR)
geo2 = mck.GridGeometry("grid2d", w.nx, w.ny)
sds = mck.decompose(geo2, w.delta, w.zeta)
bad = 0
for f in range(w.nfields):
    for t in list(range(0, len(sds), max(1, len(sds) // 24))):
        sd = sds[t]
        Uloc = orc.center_rows(w.X[f * w.n2d + sd.local_order])
        ff, fl = mck.fit_factors(Uloc, geo2, w.zeta, local_order=sd.local_order, return_flags=True)
        a, b = rp[tp[t]], rp[tp[t + 1]]
        Tt = T[f, a:b]; Dt = D[f, tp[t]:tp[t + 1]]; Ft = F[f, tp[t]:tp[t + 1]]
        et = np.linalg.norm(Tt - ff.lower.data) / np.linalg.norm(ff.lower.data)
        ed = np.max(np.abs(Dt - ff.variances) / ff.variances)
        if et > 1e-8 or ed > 1e-8:
            bad += 1
            rows = np.flatnonzero(np.abs(Dt - ff.variances) / ff.variances > 1e-8)
            print(f"field {f} tile {t}: T {et:.2e} D {ed:.2e}; bad rows {rows[:6]} flags plan {Ft[rows[:6]]} local {fl[rows[:6]]} p {np.diff(rp[tp[t]:tp[t+1]+1])[rows[:6]]}")
print("bad tiles:", bad)
