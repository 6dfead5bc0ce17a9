"""-m gpu: vertically coupled fields (BASELINE.json configs 3 / 5, "horizontal r, vertical r = 1") through the public entry
point against the extended oracle.  The reference has no vertical axis: parity is unpinned by the reference; the oracle
applies the reference's predecessor / decomposition rules on the extended box and the reference's arithmetic per regression
and per local analysis.  Gates: index maps bit-exact, T 1e-9 norm-wise, D 1e-9 max relative, Xa 1e-8 norm-wise on inputs
with a 1 % nugget (well-conditioned regressions); on the smooth inputs the gates of the 2-D configurations apply
(10 x the oracle's noise floor, here measured in the test itself by the member-permutation probe)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(w, nfields, nlev, zeta_v):
    import paper_1606_00807_b200 as mck
    from paper_1606_00807_b200 import device
    from paper_1606_00807_b200.plan import COL_IDX, LOCAL_ORDER, ROW_PTR, get_plan
    geo = mck.GridGeometry("grid2d", w.nx, w.ny, boundary=w.boundary, nfields=nfields, nlev=nlev, zeta_v=zeta_v)
    cfg = mck.AssimilationConfig(zeta=w.zeta, delta=w.delta, seed=w.seed)
    net = mck.ObservationNetwork(w.obs_indices, w.r_diag, w.y)
    xa, _ = mck.assimilate_parallel(mck.EnsembleState(w.X), net, cfg, geo, Ys=w.Ys)
    plan = get_plan(geo, w.delta, w.zeta)
    T = device.workspace_tensor(plan, 1, (plan.nfields, plan.nnz))
    D = device.workspace_tensor(plan, 2, (plan.nfields, plan.sum_nlocal))
    flags = device.workspace_tensor(plan, 3, (plan.nfields, plan.sum_nlocal), "i32")
    maps = (plan.get(LOCAL_ORDER), plan.get(ROW_PTR), plan.get(COL_IDX))
    return xa.X, T, D, flags, maps, plan


def _oracle(w, nfields, nlev, zeta_v, X=None, Ys=None):
    from oracle import enkf_mc_oracle as orc
    grid = orc.grid_for(w.nx, w.ny, w.boundary, nfields, nlev=nlev, zeta_v=zeta_v)
    ref, kept = orc.assimilate(w.X if X is None else X, w.obs_indices, w.r_diag, w.Ys if Ys is None else Ys, grid, w.delta,
                               w.zeta, keep_tiles=True)
    T = np.stack([np.concatenate([r.factors.data for r in k]) for k in kept])
    D = np.stack([np.concatenate([r.factors.d for r in k]) for k in kept])
    lo = np.concatenate([r.tile.local_order for r in kept[0]])
    ci = np.concatenate([r.factors.indices for r in kept[0]])
    return ref, T, D, lo, ci


def _errors(xa, T, D, ref, Tr, Dr):
    return (np.linalg.norm(T - Tr) / np.linalg.norm(Tr), np.max(np.abs(D - Dr) / Dr), np.linalg.norm(xa - ref) / np.linalg.norm(ref))


@pytest.mark.parametrize("nens,zeta,boundary", [(48, 2, "clipped"), (30, 2, "clipped"), (40, 1, "periodic_x")],
                         ids=["p<N", "p>N", "lon-periodic"])
def test_coupled_levels_against_extended_oracle(nens, zeta, boundary):
    """Two variables of three levels each, vertical radius 1: up to (2 zeta + 1)^2 + ((2 zeta + 1)^2 - 1) / 2 predecessors
    (37 at zeta = 2: more than the 30 members of the second case, where every full regression is rank deficient)."""
    from paper_1606_00807_b200 import synthetic
    w = synthetic.make_workload("lev", nx=24, ny=16, nens=nens, corr_len=3.0, zeta=zeta, delta=4, obs="random", obs_arg=0.4,
                                r_rel=0.1, r_abs=None, seed=21, nugget=0.01, boundary=boundary,
                                variables=[("a", 1.0, 3), ("b", 2.0, 3)])
    xa, T, D, flags, maps, plan = _run(w, 2, 3, 1)
    ref, Tr, Dr, lo, ci = _oracle(w, 2, 3, 1)
    assert np.array_equal(maps[0], lo) and np.array_equal(maps[2], ci)
    assert plan.max_pred == (37 if zeta == 2 else 14)    # zeta = 1, longitude periodic: 5 + 9 at the wrapped column
    terr, derr, xerr = _errors(xa, T, D, ref, Tr, Dr)
    # the oracle's own noise floor on this input (oracle/noise_floor.py: SVD driver, member order, linear solver swapped)
    from oracle import enkf_mc_oracle as orc
    from oracle import noise_floor
    grid = orc.grid_for(w.nx, w.ny, w.boundary, 2, nlev=3, zeta_v=1)
    tfl = dfl = xfl = 0.0
    for f in range(2):
        lo_, hi_ = f * grid.nfield, (f + 1) * grid.nfield
        sel = np.flatnonzero((w.obs_indices >= lo_) & (w.obs_indices < hi_))
        fl = noise_floor.floors(w.X[lo_:hi_], w.obs_indices[sel] - lo_, w.r_diag[sel], w.Ys[sel], grid, w.delta, w.zeta)
        tfl, dfl, xfl = (max(tfl, *(v[0] for v in fl.values())), max(dfl, *(v[1] for v in fl.values())),
                         max(xfl, *(v[2] for v in fl.values())))
    gate = (max(1e-9, 10 * tfl), max(1e-9, 10 * dfl), max(1e-8, 10 * xfl))
    floor_hits = float(((flags & 8) > 0).mean())
    print(f"levels nens={nens} zeta={zeta} {boundary}: p_max/N {plan.max_pred}/{nens}  T {terr:.2e} (floor {tfl:.1e})  "
          f"D {derr:.2e} (floor {dfl:.1e})  Xa {xerr:.2e} (floor {xfl:.1e})  D at floor {100 * floor_hits:.1f} %  "
          f"half-bandwidth {plan.max_bw}")
    assert terr < gate[0] and derr < gate[1] and xerr < gate[2], (terr, derr, xerr, gate)
    if nens > plan.max_pred:                 # well-conditioned regressions: the strict north_star gates
        assert terr < 1e-9 and derr < 1e-9 and xerr < 1e-8, (terr, derr, xerr)


def test_levels_without_coupling_equal_independent_fields():
    """zeta_v = 0: the same regressions as six independent 2-D fields (bitwise T and D); the local analyses are
    block-diagonal over the levels, so the analysis agrees to rounding."""
    from paper_1606_00807_b200 import synthetic
    w = synthetic.make_workload("lev0", nx=24, ny=16, nens=32, corr_len=3.0, zeta=2, delta=4, obs="random", obs_arg=0.4,
                                r_rel=0.1, r_abs=None, seed=22, nugget=0.01, variables=[("a", 1.0, 3), ("b", 2.0, 3)])
    xa3, T3, D3, _, maps3, plan3 = _run(w, 2, 3, 0)
    xa2, T2, D2, _, maps2, plan2 = _run(w, 6, 1, 0)
    # lifted tile = levels stacked inside a tile; independent fields = tiles stacked inside a field
    from paper_1606_00807_b200.plan import ROW_PTR, TILE_PTR
    tp2, rp2 = plan2.get(TILE_PTR), plan2.get(ROW_PTR)
    tp3, rp3 = plan3.get(TILE_PTR), plan3.get(ROW_PTR)
    for f in range(2):
        for t in range(plan2.ntiles):
            n2 = tp2[t + 1] - tp2[t]
            for lev in range(3):
                a = D3[f, tp3[t] + lev * n2: tp3[t] + (lev + 1) * n2]
                b = D2[3 * f + lev, tp2[t]:tp2[t + 1]]
                assert np.array_equal(a, b)
                a = T3[f, rp3[tp3[t] + lev * n2]: rp3[tp3[t] + (lev + 1) * n2]]
                b = T2[3 * f + lev, rp2[tp2[t]]:rp2[tp2[t + 1]]]
                assert np.array_equal(a, b)
    assert np.linalg.norm(xa3 - xa2) / np.linalg.norm(xa2) < 1e-12


def test_speedy_shaped_coupled_columns_smooth_inputs():
    """The shape of BASELINE.json config 3 on a quarter-size grid: 96 x 48, a 7-level variable, N = 80, horizontal radius 4,
    vertical radius 1 -> 121 predecessors > 80 members on the upper levels (every such regression is rank deficient and its
    D sits on the variance floor), smooth nugget-free inputs.  Gate: 10 x the oracle's own noise floor
    (member-permutation and solver-swap probes on this input), at least the north_star gates."""
    from oracle import enkf_mc_oracle as orc
    from paper_1606_00807_b200 import synthetic
    w = synthetic.make_workload("speedy_q", nx=96, ny=48, nens=80, corr_len=5.0, zeta=4, delta=64, obs="random", obs_arg=0.5,
                                r_rel=0.1, r_abs=None, seed=23, variables=[("u", 5.0, 7)])
    xa, T, D, flags, maps, plan = _run(w, 1, 7, 1)
    assert plan.max_pred == 121
    grid = orc.grid_for(w.nx, w.ny, "clipped", 1, nlev=7, zeta_v=1)
    tiles = orc.decompose(grid, w.delta, w.zeta)
    sample = [9, 27, 36, 63]
    perm = np.random.default_rng(0).permutation(w.nens)
    from paper_1606_00807_b200.plan import ROW_PTR, TILE_PTR
    tp, rp = plan.get(TILE_PTR), plan.get(ROW_PTR)
    terr = derr = xerr = tfl = dfl = xfl = 0.0
    for t in sample:
        tile = tiles[t]
        csr = orc.predecessor_csr(grid, w.zeta, tile.local_order)
        res = orc.analyse_tile(w.X, w.obs_indices, w.r_diag, w.Ys, grid, w.zeta, tile, csr)
        res_p = orc.analyse_tile(w.X[:, perm], w.obs_indices, w.r_diag, w.Ys[:, perm], grid, w.zeta, tile, csr)
        with orc.linear_solver("lu"):
            res_s = orc.analyse_tile(w.X, w.obs_indices, w.r_diag, w.Ys, grid, w.zeta, tile, csr)
        ipos = tile.interior_positions()
        Tg, Dg = T[0, rp[tp[t]]:rp[tp[t + 1]]], D[0, tp[t]:tp[t + 1]]
        nt = np.linalg.norm(res.factors.data)
        terr = max(terr, np.linalg.norm(Tg - res.factors.data) / nt)
        tfl = max(tfl, np.linalg.norm(res_p.factors.data - res.factors.data) / nt)
        derr = max(derr, np.max(np.abs(Dg - res.factors.d) / res.factors.d))
        dfl = max(dfl, np.max(np.abs(res_p.factors.d - res.factors.d) / res.factors.d))
        xr = res.xa_local[ipos]
        xerr = max(xerr, np.linalg.norm(xa[tile.interior] - xr) / np.linalg.norm(xr))
        inv = np.argsort(perm)
        xfl = max(xfl, np.linalg.norm(res_p.xa_local[ipos][:, inv] - xr) / np.linalg.norm(xr),
                  np.linalg.norm(res_s.xa_local[ipos] - xr) / np.linalg.norm(xr))
    gate = (max(1e-9, 10 * tfl), max(1e-9, 10 * dfl), max(1e-8, 10 * xfl))
    print(f"speedy-shaped coupled columns: p_max/N 121/80  T {terr:.2e} (floor {tfl:.1e})  D {derr:.2e} (floor {dfl:.1e})  "
          f"Xa {xerr:.2e} (floor {xfl:.1e})  D at floor {100 * float(((flags & 8) > 0).mean()):.1f} %  "
          f"Jacobi fallback {100 * float(((flags & 16) > 0).mean()):.2f} %  half-bandwidth {plan.max_bw}")
    assert terr < gate[0] and derr < gate[1] and xerr < gate[2], (terr, derr, xerr, gate)


def test_run_filter_with_coupled_levels():
    """The device-resident cycle loop on a vertically coupled geometry: bit-equal to assimilate_parallel cycle by cycle with the
    forecast on the host (every level is advected as a 2-D field)."""
    import paper_1606_00807_b200 as mck
    from paper_1606_00807_b200 import synthetic
    w = synthetic.make_workload("levcyc", nx=20, ny=12, nens=24, corr_len=3.0, zeta=1, delta=4, obs="random", obs_arg=0.3,
                                r_rel=0.1, r_abs=None, seed=31, nugget=0.02, variables=[("a", 1.0, 3)])
    geo = mck.GridGeometry("grid2d", w.nx, w.ny, nlev=3, zeta_v=1)
    cfg = mck.AssimilationConfig(zeta=w.zeta, delta=w.delta, seed=7)
    net = mck.ObservationNetwork(w.obs_indices, w.r_diag, w.y)
    model = mck.advdiff2d_model(geo, velocity=(0.8, -0.4), diffusivity=0.03, dt=0.05, steps_per_window=2)

    def advdiff_host(X, steps):
        out = X.copy()
        ux, uy = model.velocity
        for lev in range(3):
            sl = slice(lev * w.n2d, (lev + 1) * w.n2d)
            for j in range(X.shape[1]):
                u = out[sl, j].reshape(w.ny, w.nx)
                for _ in range(steps):
                    ddx = u - np.roll(u, 1, axis=1) if ux >= 0 else np.roll(u, -1, axis=1) - u
                    ddy = u - np.roll(u, 1, axis=0) if uy >= 0 else np.roll(u, -1, axis=0) - u
                    lap = np.roll(u, 1, axis=0) + np.roll(u, -1, axis=0) + np.roll(u, 1, axis=1) + np.roll(u, -1, axis=1) - 4.0 * u
                    u = u + model.dt * (-ux * ddx - uy * ddy + model.diffusivity * lap)
                out[sl, j] = u.reshape(-1)
        return out

    schedule = [(None, net), (None, net)]
    res = mck.run_filter(mck.EnsembleState(w.X), model, schedule, cfg)
    x = mck.EnsembleState(w.X)
    for k, (_, nk) in enumerate(schedule):
        xa, _ = mck.assimilate_parallel(x, nk, cfg, geo, cycle=k)
        assert np.array_equal(res.analyses[k].X, xa.X), k
        x = mck.EnsembleState(advdiff_host(xa.X, model.steps_per_window), role="background")
    assert np.array_equal(res.final.X, x.X)
    assert not np.array_equal(res.analyses[0].X, w.X)


def test_too_many_coupled_predecessors_are_refused():
    """Config 5 as worded (horizontal radius 5, vertical radius 1) has 60 + 121 = 181 predecessors: beyond the 128 the regression
    kernels hold; the analysis is refused with CapacityError instead of running something else."""
    import paper_1606_00807_b200 as mck
    from paper_1606_00807_b200 import synthetic
    w = synthetic.make_workload("cap", nx=40, ny=24, nens=24, corr_len=3.0, zeta=5, delta=4, obs="random", obs_arg=0.3,
                                r_rel=0.1, r_abs=None, seed=33, nugget=0.02, variables=[("a", 1.0, 2)])
    geo = mck.GridGeometry("grid2d", w.nx, w.ny, nlev=2, zeta_v=1)
    net = mck.ObservationNetwork(w.obs_indices, w.r_diag, w.y)
    with pytest.raises(mck.CapacityError, match="predecessor"):
        mck.assimilate_parallel(mck.EnsembleState(w.X), net, mck.AssimilationConfig(zeta=w.zeta, delta=w.delta), geo, Ys=w.Ys)
