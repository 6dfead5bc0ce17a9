"""Generate the golden fixtures from the UNMODIFIED reference.

Run in the build container only (``/root/reference`` does not exist on the GPU box):

    cd /tmp && PYTHONDONTWRITEBYTECODE=1 python /root/repo/tests/golden/make_golden.py

It imports ``mcholkf`` from ``/root/reference/pkg/src`` (never copied), runs the
reference's own hot-path functions on small seeded inputs and stores inputs + outputs
as ``tests/golden/*.npz``.  The tests compare the oracle (CPU suite) and the CUDA path
(``-m gpu`` suite) against these files.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import mcholkf  # noqa: E402
from mcholkf.validation import center_rows  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

from paper_1606_00807_b200 import synthetic  # noqa: E402


def geometry_cases():
    """decompose / predecessors / local_box for a spread of grids (geometry.py:145-222)."""
    out = {}
    cases = [
        # nx, ny, ordering, boundary, delta, zeta
        (8, 8, "row_major", "clipped", 4, 1),
        (8, 8, "row_major", "periodic", 4, 1),
        (64, 32, "row_major", "clipped", 8, 2),
        (64, 32, "row_major", "periodic", 8, 2),
        (13, 7, "column_major", "clipped", 6, 2),
        (13, 7, "column_major", "periodic", 6, 3),
        (10, 9, "row_major", "periodic", 9, 4),
        (5, 4, "row_major", "periodic", 2, 3),      # wrap covers whole axis, de-dup
        (24, 1, "row_major", "periodic", 3, 2),     # ring1d
        (17, 11, "row_major", "clipped", 1, 2),
    ]
    for k, (nx, ny, ordering, boundary, delta, zeta) in enumerate(cases):
        kind = "ring1d" if ny == 1 else "grid2d"
        g = mcholkf.GridGeometry(kind=kind, nx=nx, ny=ny, ordering=ordering, boundary=boundary)
        sds = mcholkf.decompose(g, delta, zeta)
        out[f"g{k}_params"] = np.array([nx, ny, ordering == "row_major", boundary == "periodic", delta, zeta])
        out[f"g{k}_ids"] = np.array([sd.id for sd in sds])
        out[f"g{k}_interior"] = np.concatenate([sd.interior for sd in sds])
        out[f"g{k}_interior_ptr"] = np.cumsum([0] + [sd.interior.size for sd in sds])
        out[f"g{k}_halo"] = np.concatenate([sd.halo for sd in sds])
        out[f"g{k}_halo_ptr"] = np.cumsum([0] + [sd.halo.size for sd in sds])
        out[f"g{k}_local"] = np.concatenate([sd.local_order for sd in sds])
        out[f"g{k}_local_ptr"] = np.cumsum([0] + [sd.n_local for sd in sds])
        out[f"g{k}_intpos"] = np.concatenate([sd.interior_positions() for sd in sds])
        preds = [mcholkf.predecessors(g, c, zeta) for c in range(g.nstate)]
        out[f"g{k}_pred"] = np.concatenate(preds) if preds else np.zeros(0, np.int64)
        out[f"g{k}_pred_ptr"] = np.cumsum([0] + [p.size for p in preds])
        boxes = [mcholkf.local_box(g, c, zeta).members for c in range(g.nstate)]
        out[f"g{k}_box"] = np.concatenate(boxes)
        out[f"g{k}_box_ptr"] = np.cumsum([0] + [b.size for b in boxes])
    out["ncases"] = np.array(len(cases))
    return out


def _geometry(w):
    kind = "ring1d" if w.ny == 1 else "grid2d"
    return mcholkf.GridGeometry(kind=kind, nx=w.nx, ny=w.ny, boundary=w.boundary)


def analysis_case(w, tag):
    """Full assimilate_parallel + per-tile T, D on one 2-D workload (driver.py:159-253)."""
    g = _geometry(w)
    Xb = mcholkf.EnsembleState(w.X)
    net = mcholkf.ObservationNetwork(w.obs_indices, w.r_diag, w.y)
    cfg = mcholkf.AssimilationConfig(zeta=w.zeta, delta=w.delta, seed=w.seed)
    ys = mcholkf.perturb_observations(net, w.nens, w.seed, 0).Ys
    assert np.array_equal(ys, w.Ys)
    xa, _ = mcholkf.assimilate_parallel(Xb, net, cfg, g, Ys=w.Ys)
    out = {
        f"{tag}_params": np.array([w.nx, w.ny, w.boundary == "periodic", w.nens, w.zeta, w.delta]),
        f"{tag}_X": w.X, f"{tag}_obs": w.obs_indices, f"{tag}_r": w.r_diag, f"{tag}_y": w.y,
        f"{tag}_Ys": w.Ys, f"{tag}_Xa": xa.X,
    }
    tptr, tind, tdat, dvar, xal = [0], [], [], [], []
    rowptr = []
    for sd in mcholkf.decompose(g, w.delta, w.zeta):
        xb = w.X[sd.local_order]
        f = mcholkf.fit_factors(center_rows(xb), g, w.zeta, local_order=sd.local_order)
        net_l, rows = mcholkf.restrict_network(net, sd.local_order)
        with threadpool_limits(limits=1):      # as assimilate_parallel does (driver.py:231)
            xl = mcholkf.analysis_primal(mcholkf.EnsembleState(xb), f, net_l, w.Ys[rows])
        rowptr.append(f.lower.indptr + tptr[-1])
        tptr.append(tptr[-1] + f.lower.nnz)
        tind.append(f.lower.indices)
        tdat.append(f.lower.data)
        dvar.append(f.variances)
        xal.append(xl.X)
    out[f"{tag}_T_indptr"] = np.concatenate([rp[:-1] for rp in rowptr] + [[tptr[-1]]]).astype(np.int64)
    out[f"{tag}_T_indices"] = np.concatenate(tind).astype(np.int64)
    out[f"{tag}_T_data"] = np.concatenate(tdat)
    out[f"{tag}_D"] = np.concatenate(dvar)
    out[f"{tag}_Xa_local"] = np.concatenate(xal)
    return out


def regression_cases():
    """regression_solve known answers + random over/under-determined (estimator.py:27-61)."""
    rng = np.random.default_rng(42)
    out = {}
    k = 0
    for p, m in [(1, 4), (3, 8), (5, 12), (7, 3), (12, 20), (24, 40), (40, 80), (84, 80), (60, 128)]:
        a = rng.standard_normal((p, m))
        if p == 12:
            a[5] = a[2] * 2.0 - a[7]            # exact rank deficiency
        y = rng.standard_normal(m)
        out[f"r{k}_A"], out[f"r{k}_y"] = a, y
        out[f"r{k}_beta"] = mcholkf.regression_solve(a, y)
        k += 1
    out["ncases"] = np.array(k)
    return out


def letkf_cases():
    """LETKF baseline (kernels.py:251-335) on two small grids: clipped without inflation, periodic with inflation."""
    from mcholkf.kernels import letkf_analysis_global
    out = {}
    cases = [("l0", dict(nx=14, ny=10, nens=12, corr_len=2.5, zeta=2, delta=1, obs="random", obs_arg=0.3, r_rel=None, r_abs=0.1, seed=71), "clipped", 1.0),
             ("l1", dict(nx=12, ny=9, nens=16, corr_len=3.0, zeta=1, delta=1, obs="lattice", obs_arg=3, r_rel=None, r_abs=0.2, seed=72,
                         boundary="periodic"), "periodic", 1.1)]
    for tag, kw, boundary, infl in cases:
        w = synthetic.make_workload(tag, **kw)
        geo = mcholkf.GridGeometry("grid2d", w.nx, w.ny, boundary=boundary)
        net = mcholkf.ObservationNetwork(w.obs_indices, w.r_diag, w.y)
        ref = letkf_analysis_global(mcholkf.EnsembleState(w.X), geo, net, w.zeta, inflation=infl).X
        out.update({f"{tag}_X": w.X, f"{tag}_obs": w.obs_indices, f"{tag}_r": w.r_diag, f"{tag}_y": w.y, f"{tag}_Xa": ref,
                    f"{tag}_meta": np.array([w.nx, w.ny, w.zeta, boundary == "periodic", infl], dtype=np.float64)})
    return out


def main():
    np.savez_compressed(os.path.join(HERE, "letkf.npz"), **letkf_cases())
    np.savez_compressed(os.path.join(HERE, "geometry.npz"), **geometry_cases())
    np.savez_compressed(os.path.join(HERE, "regression.npz"), **regression_cases())
    out = {}
    # well-conditioned (1 % nugget) and as-specified smooth inputs, both boundaries
    small = dict(nx=24, ny=16, nens=30, corr_len=3.0, zeta=2, delta=4, obs="lattice", obs_arg=2,
                 r_rel=None, r_abs=0.05)
    out.update(analysis_case(synthetic.make_workload("s_clip_nug", seed=11, nugget=0.01, **small), "a0"))
    out.update(analysis_case(synthetic.make_workload("s_per_nug", seed=12, nugget=0.01, boundary="periodic", **small), "a1"))
    out.update(analysis_case(synthetic.make_workload("s_clip_smooth", seed=13, **small), "a2"))
    big = dict(nx=32, ny=20, nens=56, corr_len=4.0, zeta=3, delta=6, obs="random", obs_arg=0.3,
               r_rel=None, r_abs=0.1)
    out.update(analysis_case(synthetic.make_workload("m_clip_nug", seed=14, nugget=0.01, **big), "a3"))
    out.update(analysis_case(synthetic.make_workload("m_per_smooth", seed=15, boundary="periodic", **big), "a4"))
    trunc = dict(big, corr_len=8.0)             # rank_tol truncation active in ~40 % of rows
    out.update(analysis_case(synthetic.make_workload("m_clip_trunc", seed=16, **trunc), "a5"))
    out["ncases"] = np.array(6)
    np.savez_compressed(os.path.join(HERE, "analysis.npz"), **out)
    for f in ("geometry.npz", "regression.npz", "analysis.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")


if __name__ == "__main__":
    main()
