"""Per-row T error by regression path for one tile (GPU box debugging aid)."""
import argparse, sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/", 2)[0])
import paper_1606_00807_b200 as mck
from oracle import enkf_mc_oracle as orc
from paper_1606_00807_b200 import synthetic
ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg5"); ap.add_argument("--zeta", type=int, default=None)
ap.add_argument("--tile", type=int, default=None)
a = ap.parse_args()
w = synthetic.config(a.workload, fields=1 if a.workload in ("cfg3", "cfg5") else None, zeta=a.zeta)
geo = mck.GridGeometry("grid2d", w.nx, w.ny)
grid = orc.Grid(w.nx, w.ny)
sds = mck.decompose(geo, w.delta, w.zeta)
sd = sds[a.tile if a.tile is not None else len(sds) // 2 + 3]
U = orc.center_rows(w.X[sd.local_order])
f, flags = mck.fit_factors(U, geo, w.zeta, local_order=sd.local_order, return_flags=True)
ref = orc.fit_factors(U, grid, w.zeta, sd.local_order)
ip = ref.indptr
rows = []
for j in range(ref.n):
    a0, b0 = ip[j], ip[j + 1]
    if a0 == b0: continue
    s = np.linalg.svd(U[ref.indices[a0:b0]], compute_uv=False)
    m = int((s < 1e-8 * s[0]).sum())
    e = np.linalg.norm(f.lower.data[a0:b0] - ref.data[a0:b0]) / np.linalg.norm(ref.data[a0:b0])
    margin = min(abs(np.log10(s / (1e-8 * s[0]))))
    rows.append((j, b0 - a0, m, int(flags[j]), e, abs(f.variances[j] - ref.d[j]) / ref.d[j], margin, s[0] / s[-1]))
rows = np.array(rows)
print("n_local", ref.n, "rows", len(rows))
for name, sel in [("kept (flag 0/8)", (rows[:, 3].astype(int) & 19) == 0), ("deflated", ((rows[:, 3].astype(int) & 2) > 0) & ((rows[:, 3].astype(int) & 16) == 0)),
                  ("jacobi fallback", (rows[:, 3].astype(int) & 16) > 0), ("sweep cap", (rows[:, 3].astype(int) & 4) > 0)]:
    if sel.any():
        print(f"{name:16s} rows {int(sel.sum()):4d}  T err max {rows[sel, 4].max():.2e} median {np.median(rows[sel, 4]):.2e}  D err max {rows[sel, 5].max():.2e}  m hist {np.bincount(rows[sel, 2].astype(int))}")
worst = rows[np.argsort(-rows[:, 4])[:8]]
for r in worst:
    print("row %d p %d m_ref %d flag %d Terr %.2e Derr %.2e log10-margin-to-threshold %.3f cond %.1e" % tuple(r))
