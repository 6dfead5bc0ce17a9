"""cProfile of assimilate_parallel on the bench workload (host-side overheads)."""
import cProfile, pstats, sys, time
sys.path.insert(0, __file__.rsplit("/", 2)[0])
import numpy as np, torch
import paper_1606_00807_b200 as mck
from paper_1606_00807_b200 import synthetic
w = synthetic.config("cfg3")
t = torch.empty(w.X.shape, dtype=torch.float64, pin_memory=True); Xh = t.numpy(); Xh[...] = w.X
t2 = torch.empty(w.Ys.shape, dtype=torch.float64, pin_memory=True); Ysh = t2.numpy(); Ysh[...] = w.Ys
geo = mck.GridGeometry("grid2d", w.nx, w.ny, nfields=w.nfields)
net = mck.ObservationNetwork(w.obs_indices, w.r_diag, w.y)
cfg = mck.AssimilationConfig(zeta=w.zeta, delta=w.delta)
xb = mck.EnsembleState(Xh)
for _ in range(3):
    xa, rep = mck.assimilate_parallel(xb, net, cfg, geo, Ys=Ysh)
pr = cProfile.Profile(); pr.enable()
for _ in range(3):
    t0 = time.perf_counter(); xa, rep = mck.assimilate_parallel(xb, net, cfg, geo, Ys=Ysh); print("call", time.perf_counter() - t0, rep.t_total, rep.t_h2d, rep.t_d2h)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
