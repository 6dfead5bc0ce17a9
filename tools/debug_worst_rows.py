"""Full-field per-row T/D error against the oracle, worst rows with their threshold margins."""
import multiprocessing as mp
import sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/", 2)[0])
from oracle import enkf_mc_oracle as orc
from paper_1606_00807_b200 import synthetic

G = {}
def work(t):
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=1):
        tile = G["tiles"][t]
        U = orc.center_rows(G["X"][tile.local_order])
        f = orc.fit_factors(U, G["grid"], G["zeta"], tile.local_order)
    return f.indptr, f.indices, f.data, f.d

name = sys.argv[1]; zeta = int(sys.argv[2]) if len(sys.argv) > 2 else None
w = synthetic.config(name, fields=1 if name in ("cfg3", "cfg5") else None, zeta=zeta)
grid = orc.Grid(w.nx, w.ny)
G.update(X=w.X, grid=grid, zeta=w.zeta, tiles=orc.decompose(grid, w.delta, w.zeta))
with mp.get_context("fork").Pool(16) as pool:
    res = pool.map(work, range(len(G["tiles"])), chunksize=4)
import torch
import paper_1606_00807_b200 as mck
from paper_1606_00807_b200 import device
from paper_1606_00807_b200.plan import Plan, ROW_PTR, TILE_PTR
geo = mck.GridGeometry("grid2d", w.nx, w.ny)
plan = Plan.decomposed(geo, w.delta, w.zeta)
plan.set_observations(w.obs_indices)
dX, dR, dYs = device.to_device(w.X), device.to_device(w.r_diag), device.to_device(w.Ys)
dXa = torch.empty_like(dX)
device.analysis_device(plan, dX, dR, dYs, dXa)
T = device.workspace_tensor(plan, 1, (plan.nnz,)); D = device.workspace_tensor(plan, 2, (plan.sum_nlocal,))
F = device.workspace_tensor(plan, 3, (plan.sum_nlocal,), "i32")
tp, rp = plan.get(TILE_PTR), plan.get(ROW_PTR)
Tref = np.concatenate([r[2] for r in res]); Dref = np.concatenate([r[3] for r in res])
print("norm-wise T err", np.linalg.norm(T - Tref) / np.linalg.norm(Tref), " D max rel", np.max(np.abs(D - Dref) / Dref))
rowerr = np.zeros(plan.sum_nlocal); rownorm = np.zeros(plan.sum_nlocal)
for q in range(plan.sum_nlocal):
    a, b = rp[q], rp[q + 1]
    if b > a:
        rownorm[q] = np.linalg.norm(Tref[a:b]); rowerr[q] = np.linalg.norm(T[a:b] - Tref[a:b])
print("rows with abs T err > 1e-6*|T|_total:", int((rowerr > 1e-6 * np.linalg.norm(Tref)).sum()))
order = np.argsort(-rowerr)[:10]
for q in order:
    t = int(np.searchsorted(tp, q, side="right") - 1)
    tile = G["tiles"][t]; j = q - tp[t]
    ip, ii = res[t][0], res[t][1]
    U = orc.center_rows(w.X[tile.local_order])
    s = np.linalg.svd(U[ii[ip[j]:ip[j + 1]]], compute_uv=False)
    near = s[np.argmin(np.abs(np.log10(s / (1e-8 * s[0]))))]
    print(f"row {q} tile {t} p {ip[j+1]-ip[j]} flag {F[q]} abs err {rowerr[q]:.2e} rel {rowerr[q]/rownorm[q]:.2e} |T row| {rownorm[q]:.2e} "
          f"D rel err {abs(D[q]-Dref[q])/Dref[q]:.2e} m_ref {(s < 1e-8*s[0]).sum()} nearest s/thr - 1 = {near/(1e-8*s[0]) - 1:.3e}"
          f" steps {(F[q] >> 8) & 255} smallest s/s0: {np.array2string(s[-6:][::-1] / s[0], precision=2)}")
