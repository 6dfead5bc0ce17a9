"""Diagnostics of a vertically coupled run: non-finite T / D entries, path flags, stage times (GPU box)."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import torch  # noqa: E402

import paper_1606_00807_b200 as mck  # noqa: E402
from paper_1606_00807_b200 import device, synthetic  # noqa: E402
from paper_1606_00807_b200.plan import ROW_PTR, TILE_PTR, Plan  # noqa: E402

nugget = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0
w = synthetic.make_workload("speedy_q", nx=96, ny=48, nens=80, corr_len=5.0, zeta=4, delta=64, obs="random", obs_arg=0.5,
                            r_rel=0.1, r_abs=None, seed=23, variables=[("u", 5.0, 7)], nugget=nugget)
geo = mck.GridGeometry("grid2d", w.nx, w.ny, nfields=1, nlev=7, zeta_v=1)
plan = Plan.decomposed(geo, w.delta, w.zeta)
plan.set_observations(w.obs_indices)
print("rows", plan.sum_nlocal, "nnz", plan.nnz, "max_pred", plan.max_pred, "max_bw", plan.max_bw, "distinct", plan.n_regressions)
dX, dR, dYs = device.to_device(w.X), device.to_device(w.r_diag), device.to_device(w.Ys)
dXa = torch.empty_like(dX)
plan.profile(True)
try:
    device.analysis_device(plan, dX, dR, dYs, dXa)
    torch.cuda.synchronize()
    from paper_1606_00807_b200 import _lib
    rc = _lib.lib().enkfmc_plan_check_status(plan.handle)
    print("analysis done, check_status rc", rc, _lib.lib().enkfmc_last_error().decode() if rc else "")
    xa = dXa.cpu().numpy()
    bad = np.flatnonzero(~np.isfinite(xa).all(axis=1))
    print("non-finite analysis rows", bad.size, bad[:10], "levels", np.unique(bad // (w.nx * w.ny)))
    st = device.workspace_tensor(plan, 4, (plan.nfields * plan.ntiles,), "i32") if hasattr(device, "workspace_tensor") else None
    print("status", st)
except Exception as e:  # noqa: BLE001
    print("analysis failed:", e)
n, ms = plan.stage_times()
print("stage ms", ms / max(n, 1))
T = device.workspace_tensor(plan, 1, (plan.nfields, plan.nnz))
D = device.workspace_tensor(plan, 2, (plan.nfields, plan.sum_nlocal))
flags = device.workspace_tensor(plan, 3, (plan.nfields, plan.sum_nlocal), "i32")
rp = plan.get(ROW_PTR)
p = np.diff(rp)
print("non-finite T", int((~np.isfinite(T)).sum()), "non-finite D", int((~np.isfinite(D)).sum()), "max |T|", np.nanmax(np.abs(T)))
bad_rows = np.unique(np.searchsorted(rp, np.flatnonzero(~np.isfinite(T[0])), side="right") - 1)
print("rows with non-finite T:", bad_rows[:20], "p:", p[bad_rows[:20]], "flags:", [hex(int(x)) for x in flags[0][bad_rows[:20]]])
print("D at floor %.1f %%, fallback %.2f %%, listed %.1f %%" % (100 * ((flags & 8) > 0).mean(), 100 * ((flags & 16) > 0).mean(), 100 * ((flags & 1) > 0).mean()))
fb = (flags[0] & 16) > 0
print("fallback reasons", np.bincount((flags[0][fb] >> 5) & 7, minlength=8), "p of fallback rows", np.bincount(p[fb])[-5:] if fb.any() else [])
print("pinned pivots", plan.counter(5))
