"""Measures the oracle's noise floors (oracle/noise_floor.py) on the BASELINE.json configurations and writes
tests/golden/noise_floors.json (committed; the GPU parity tests gate at max(north_star gate, 10 x floor)).
CPU only; a few minutes with one process per configuration."""
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import enkf_mc_oracle as orc, noise_floor  # noqa: E402
from paper_1606_00807_b200 import synthetic  # noqa: E402

# name -> (synthetic.config kwargs, field, tile sample (None: all tiles))
CASES = {
    "cfg1": (dict(name="cfg1"), 0, None),
    "cfg1_nugget": (dict(name="cfg1", nugget=0.01), 0, None),
    "cfg1_periodic": (dict(name="cfg1", boundary="periodic"), 0, None),
    "cfg1_lon_periodic": (dict(name="cfg1", boundary="periodic_x"), 0, None),
    "cfg1_periodic_nugget": (dict(name="cfg1", boundary="periodic", nugget=0.01), 0, None),
    "cfg2": (dict(name="cfg2"), 0, None),
    "cfg2_nugget": (dict(name="cfg2", nugget=0.01), 0, None),
    "cfg3": (dict(name="cfg3", fields=1), 0, list(range(0, 256, 4))),
    "cfg3_nugget": (dict(name="cfg3", fields=1, nugget=0.01), 0, list(range(0, 256, 8))),
    "cfg4_r1": (dict(name="cfg4", zeta=1), 0, None),
    "cfg4_r2": (dict(name="cfg4", zeta=2), 0, None),
    "cfg4_r3": (dict(name="cfg4", zeta=3), 0, None),
    "cfg4_r4": (dict(name="cfg4", zeta=4), 0, list(range(0, 64, 2))),
    "cfg4_r5": (dict(name="cfg4", zeta=5), 0, list(range(0, 64, 4))),
    "cfg4_r6": (dict(name="cfg4", zeta=6), 0, list(range(0, 64, 4))),
    "cfg4_r5_nugget": (dict(name="cfg4", zeta=5, nugget=0.01), 0, list(range(0, 64, 8))),
    "cfg5": (dict(name="cfg5", fields=1), 0, list(range(0, 1024, 32))),
    # the smooth golden cases of tests/golden/make_golden.py (a2, a4, a5)
    "golden_a2": (dict(make=dict(nx=24, ny=16, nens=30, corr_len=3.0, zeta=2, delta=4, obs="lattice", obs_arg=2, r_rel=None, r_abs=0.05, seed=13)), 0, None),
    "golden_a4": (dict(make=dict(nx=32, ny=20, nens=56, corr_len=4.0, zeta=3, delta=6, obs="random", obs_arg=0.3, r_rel=None, r_abs=0.1, seed=15, boundary="periodic")), 0, None),
    "golden_a5": (dict(make=dict(nx=32, ny=20, nens=56, corr_len=8.0, zeta=3, delta=6, obs="random", obs_arg=0.3, r_rel=None, r_abs=0.1, seed=16)), 0, None),
}


def one(name):
    kw, field, tiles = CASES[name]
    kw = dict(kw)
    w = synthetic.make_workload(name, **kw["make"]) if "make" in kw else synthetic.config(kw.pop("name"), **kw)
    grid = orc.grid_for(w.nx, w.ny, w.boundary)
    lo, hi = field * w.n2d, (field + 1) * w.n2d
    sel = np.flatnonzero((w.obs_indices >= lo) & (w.obs_indices < hi))
    t0 = time.time()
    fl = noise_floor.floors(w.X[lo:hi], w.obs_indices[sel] - lo, w.r_diag[sel], w.Ys[sel], grid, w.delta, w.zeta, tiles)
    out = {"tiles": "all" if tiles is None else f"{len(tiles)} of {w.delta}", "field": field}
    for probe, (t, d, x) in fl.items():
        out[probe] = {"T": t, "D": d, "Xa": x}
    out["T"] = max(v["T"] for k, v in out.items() if isinstance(v, dict))
    out["D"] = max(v["D"] for k, v in out.items() if isinstance(v, dict))
    out["Xa"] = max(v["Xa"] for k, v in out.items() if isinstance(v, dict))
    print(f"{name}: {time.time() - t0:.0f} s  gesvd {fl['gesvd']}  perm {fl['perm']}", flush=True)
    return name, out


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    with mp.Pool(min(len(names), os.cpu_count() or 1)) as pool:
        res = dict(pool.map(one, names, chunksize=1))
    path = os.path.join(ROOT, "tests", "golden", "noise_floors.json")
    old = json.load(open(path)) if os.path.exists(path) else {}
    old.update(res)
    old["_how"] = ("tools/make_floors.py: oracle/noise_floor.py on one 2-D field of each configuration (tile sample as listed); "
                   "T norm-wise, D max relative, Xa norm-wise over tile interiors; top-level T/D/Xa = larger of the two probes")
    json.dump(old, open(path, "w"), indent=1, sort_keys=True)
    print("wrote", path)
