"""Diagnostics for K2 on a workload: path flags histogram and stage times (run on a GPU box)."""
import argparse
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import torch  # noqa: E402

import paper_1606_00807_b200 as mck  # noqa: E402
from paper_1606_00807_b200 import device, synthetic  # noqa: E402
from paper_1606_00807_b200.plan import ROW_PTR, get_plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg3")
ap.add_argument("--fields", type=int, default=2)
ap.add_argument("--zeta", type=int, default=None)
ap.add_argument("--nugget", type=float, default=0.0)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
w = synthetic.config(a.workload, fields=a.fields if a.workload in ("cfg3", "cfg5") else None, zeta=a.zeta, nugget=a.nugget)
geo = mck.GridGeometry("grid2d", w.nx, w.ny, boundary=w.boundary, nfields=w.nfields)
plan = get_plan(geo, w.delta, w.zeta)
plan.set_observations(w.obs_indices)
dX, dR, dYs = device.to_device(w.X), device.to_device(w.r_diag), device.to_device(w.Ys)
dXa = torch.empty_like(dX)
device.analysis_device(plan, dX, dR, dYs, dXa)
torch.cuda.synchronize()
plan.profile(True)
for _ in range(a.reps):
    device.analysis_device(plan, dX, dR, dYs, dXa)
n, ms = plan.stage_times()
print("stage ms (centre, K2a qr, K2b solve, K3):", ms / n)
flags = device.workspace_tensor(plan, 3, (plan.nfields * plan.sum_nlocal,), "i32")
p = np.tile(np.diff(plan.get(ROW_PTR)), plan.nfields)
print("rows", flags.size, "deflated(bit1&!16)", int(((flags & 2) > 0).sum() - ((flags & 16) > 0).sum()),
      "jacobi fallback", int(((flags & 16) > 0).sum()), "sweep cap", int(((flags & 4) > 0).sum()),
      "floor", int(((flags & 8) > 0).sum()))
for lo, hi in [(0, 1), (1, 16), (16, 32), (32, 41), (41, 61), (61, 200)]:
    sel = (p >= lo) & (p < hi)
    if sel.any():
        print(f"  p in [{lo},{hi}): rows {int(sel.sum())}  truncated {int(((flags[sel] & 2) > 0).sum())}  "
              f"fallback {int(((flags[sel] & 16) > 0).sum())}")
print("fallback reasons (1 zero pivot / p>N, 2 certificate inconclusive, 3 out of deflation slots, 4 refined s above threshold, 5 certificate lost to cancellation, 6 polish not converged, 7 kept direction in block):", np.bincount((flags[(flags & 16) > 0] >> 5) & 7, minlength=8))
steps = (flags >> 8) & 255
tr = (flags & 2) > 0
print("inverse-iteration steps per truncated row: mean %.2f, histogram" % steps[tr].mean(), np.bincount(steps[tr], minlength=12)[:16])
print("pinned Cholesky pivots in the last analysis:", plan.counter(5))
fb = (flags & 16) > 0
if fb.any():
    print("Jacobi sweeps per fallback row: mean %.1f, histogram" % ((flags[fb] >> 16) & 63).mean(), np.bincount((flags[fb] >> 16) & 63, minlength=31)[:31])
fl = plan.work(w.nens)
print("algorithmic GF regress/solve:", fl[2] / 1e9, fl[1] / 1e9, " -> TF/s", fl[2] / ((ms[1] + ms[2]) / n) / 1e9, fl[1] / (ms[3] / n) / 1e9)
single = ((flags & 32) > 0) & ((flags & 16) == 0) & ((flags & 1) == 0)
print("K2b-1 single-pair rows: %d, of which the s_max bound had to be sharpened by power steps: %d" % (int(single.sum()), int((single & ((flags & 64) > 0)).sum())))
