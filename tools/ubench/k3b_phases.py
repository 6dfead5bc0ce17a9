"""Cycles per phase of K3b as seen by thread 0 of CTA 0.

Build the instrumented library and run on the GPU box (the box's copy of the repo is scratch):
    cd paper_1606_00807_b200/csrc && nvcc -O3 -std=c++17 -lineinfo -DENKFMC_K3B_TIMING -gencode arch=compute_100a,code=sm_100a \
        -Xcompiler -fPIC -Xcompiler -fvisibility=default -I../../include -I. -shared -x cu plan.cpp -x cu kernels.cu -x cu api.cu \
        -o ../../tools/ubench/libenkfmc_timing.so -lcudart_static -lpthread -ldl -lrt
    gpurun -- 'cp tools/ubench/libenkfmc_timing.so paper_1606_00807_b200/libenkfmc.so && python tools/ubench/k3b_phases.py'
"""
import ctypes as C, sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/", 3)[0])
import torch
import paper_1606_00807_b200 as mck
from paper_1606_00807_b200 import device, synthetic, _lib
from paper_1606_00807_b200.plan import get_plan
w = synthetic.config("cfg3", fields=4)
geo = mck.GridGeometry("grid2d", w.nx, w.ny, nfields=w.nfields)
plan = get_plan(geo, w.delta, w.zeta); plan.set_observations(w.obs_indices)
dX, dR, dYs = device.to_device(w.X), device.to_device(w.r_diag), device.to_device(w.Ys)
dXa = torch.empty_like(dX)
device.analysis_device(plan, dX, dR, dYs, dXa); torch.cuda.synchronize()
L = _lib.lib()
out = (C.c_ulonglong * 24)()
L.enkfmc_debug_k3b_times(out)
device.analysis_device(plan, dX, dR, dYs, dXa); torch.cuda.synchronize()
L.enkfmc_debug_k3b_times(out)
t = np.array(list(out), dtype=np.float64)
names = ["fetch item/between tiles", "tile setup (tables)", "initial window load", "first diag factor", "fwd (b) + barrier", "fwd tiles/factor/RHS", "fwd commit next row",
         "fwd barrier wait", "first panel load", "bwd S + solve + stores", "bwd commit panel", "bwd barrier wait",
         "fwd: prefetch + L store (warp 0)", "fwd: tile (0,0) (warp 0)", "fwd: factor + invert next diagonal block (warp 0)"]
tot = t.sum()
names += ["(second, hot call of the diagonal factorisation: -DENKFMC_K3B_TWICE builds only)", "bwd: global loads of z_J / background issued", "bwd: next panel fetch issued",
          "bwd: S = L_below^T x (tensor-core chain)", "bwd: S through shared memory, z_J - S (waits for z_J)", "bwd: x_J, stores"]
for n, v in zip(names, t): print(f"{n:28s} {v/1e3:10.1f} kcycles  {100*v/tot:5.1f}%")
print("total kcycles on CTA 0:", tot / 1e3)
