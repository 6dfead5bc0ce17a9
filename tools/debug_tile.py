import sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/", 2)[0])
import torch
import paper_1606_00807_b200 as mck
from oracle import enkf_mc_oracle as orc
from paper_1606_00807_b200 import device, synthetic
from paper_1606_00807_b200.plan import Plan, TILE_PTR
w = synthetic.config("cfg3")
lab = w.obs_indices % w.n2d; fld = w.obs_indices // w.n2d
keep = ~((fld == 0) & (lab // w.nx < 48) & (lab % w.nx < 96))
geo = mck.GridGeometry("grid2d", w.nx, w.ny, nfields=w.nfields)
plan = Plan.decomposed(geo, w.delta, w.zeta)
plan.set_observations(w.obs_indices[keep])
dX, dR, dYs = device.to_device(w.X), device.to_device(w.r_diag[keep]), device.to_device(w.Ys[keep])
dXa = torch.empty_like(dX)
device.analysis_device(plan, dX, dR, dYs, dXa)
torch.cuda.synchronize()
st = device.workspace_tensor(plan, 4, (plan.nfields, plan.ntiles), "i32")
print("status nonzero:", np.argwhere(st != 0)[:10], st[st != 0][:10])
T = device.workspace_tensor(plan, 1, (plan.nfields, plan.nnz)); D = device.workspace_tensor(plan, 2, (plan.nfields, plan.sum_nlocal))
print("T finite", np.isfinite(T).all(), "D finite", np.isfinite(D).all(), "D min", D.min())
tp = plan.get(TILE_PTR)
for f, t in np.argwhere(st != 0)[:3]:
    geo2 = mck.GridGeometry("grid2d", w.nx, w.ny)
    sd = mck.decompose(geo2, w.delta, w.zeta)[t]
    sel = keep & (fld == f)
    net = mck.ObservationNetwork(w.obs_indices[sel] - f * w.n2d, w.r_diag[sel], w.y[sel])
    netl, rows = mck.restrict_network(net, sd.local_order)
    print("tile", t, "field", f, "n_local", sd.n_local, "nobs local", netl.nobs, "obs pos", netl.obs_indices[:8])
    Xl = w.X[f * w.n2d + sd.local_order]
    fac = mck.fit_factors(orc.center_rows(Xl), geo2, w.zeta, local_order=sd.local_order)
    try:
        xa = mck.analysis_primal(mck.EnsembleState(Xl), fac, netl, w.Ys[sel][rows])
        print("standalone analysis ok, finite:", np.isfinite(xa.X).all())
    except Exception as e:
        print("standalone failed:", e)
    ref = orc.analysis_primal(Xl, orc.fit_factors(orc.center_rows(Xl), orc.Grid(w.nx, w.ny), w.zeta, sd.local_order), netl.obs_indices, netl.r_diag, w.Ys[sel][rows])
    print("oracle finite:", np.isfinite(ref).all())
A = fac.dense_precision()
A[netl.obs_indices, netl.obs_indices] += 1.0 / netl.r_diag
print("A finite", np.isfinite(A).all(), "diag min/max", A.diagonal().min(), A.diagonal().max())
ev = np.linalg.eigvalsh(A); print("eig min/max", ev[0], ev[-1])
try:
    L = np.linalg.cholesky(A); print("numpy chol ok; min diag L", L.diagonal().min(), "max", L.diagonal().max())
    rhs = np.zeros_like(Xl); rhs[netl.obs_indices] = (w.Ys[sel][rows] - Xl[netl.obs_indices]) / netl.r_diag[:, None]
    import scipy.linalg as sl
    z = sl.solve_triangular(L, rhs, lower=True); x = sl.solve_triangular(L.T, z, lower=False)
    print("z max", np.abs(z).max(), "x max", np.abs(x).max(), "argmax row", np.unravel_index(np.abs(x).argmax(), x.shape))
except Exception as e:
    print("numpy chol failed", e)
