import os, sys, numpy as np, torch, ctypes as C
sys.path.insert(0, "/root/repo")
import paper_1606_00807_b200 as mck
from paper_1606_00807_b200 import _lib, device
G = np.load("/root/repo/tests/golden/letkf.npz")
tag = "l0"
nx, ny, zeta, periodic, infl = G[f"{tag}_meta"]
X = G[f"{tag}_X"]; obs = G[f"{tag}_obs"]; r = G[f"{tag}_r"]; y = G[f"{tag}_y"]
n, N = X.shape
m = np.full(n, -1, np.int32); m[obs] = np.arange(obs.size, dtype=np.int32)
dX = device.to_device(X); dU = torch.zeros_like(dX); dXa = torch.zeros_like(dX); dM = torch.zeros(n, dtype=torch.float64, device="cuda")
bad = C.c_int64(-5)
dMap = torch.from_numpy(m).cuda(); dR = device.to_device(r); dY = device.to_device(y)
rc = _lib.lib().enkfmc_letkf_device(dX.data_ptr(), dU.data_ptr(), dM.data_ptr(), dXa.data_ptr(), dMap.data_ptr(),
        dR.data_ptr(), dY.data_ptr(), int(nx), int(ny), 1, int(periodic), 1, N, int(zeta), float(infl), C.addressof(bad), device.stream_ptr())
print("rc", rc, "bad", bad.value, _lib.lib().enkfmc_last_error())
xa = dXa.cpu().numpy(); ref = G[f"{tag}_Xa"]
print("mean err", np.abs(dM.cpu().numpy() - X.mean(1)).max(), "U err", np.abs(dU.cpu().numpy() - (X - X.mean(1)[:, None])).max())
print("relerr", np.linalg.norm(xa - ref) / np.linalg.norm(ref), "rows wrong:", np.flatnonzero(np.abs(xa - ref).max(1) > 1e-8)[:10], "nan rows", np.isnan(xa).any(1).sum())
