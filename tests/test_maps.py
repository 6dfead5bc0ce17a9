"""CPU: the C-ABI library's host index maps (csrc/plan.cpp) -- bit-exact against the golden
fixtures and the oracle; no GPU needed (no compute entry point is called)."""

import numpy as np
import pytest

import paper_1606_00807_b200 as mck
from oracle import enkf_mc_oracle as orc
from paper_1606_00807_b200 import plan as P
from paper_1606_00807_b200.plan import Plan, get_plan


def _geo(nx, ny, rm=True, per=False, nfields=1):
    return mck.GridGeometry("ring1d" if ny == 1 else "grid2d", nx, ny, "row_major" if rm else "column_major",
                            "periodic" if per else "clipped", nfields)


def test_decompose_predecessors_golden(golden_geometry):
    G = golden_geometry
    for k in range(int(G["ncases"])):
        nx, ny, rm, per, delta, zeta = [int(v) for v in G[f"g{k}_params"]]
        g = _geo(nx, ny, bool(rm), bool(per))
        sds = mck.decompose(g, delta, zeta)
        assert [s.id for s in sds] == list(G[f"g{k}_ids"])
        assert np.array_equal(np.concatenate([s.interior for s in sds]), G[f"g{k}_interior"])
        assert np.array_equal(np.concatenate([s.halo for s in sds]), G[f"g{k}_halo"])
        assert np.array_equal(np.concatenate([s.local_order for s in sds]), G[f"g{k}_local"])
        assert np.array_equal(np.concatenate([s.interior_positions() for s in sds]), G[f"g{k}_intpos"])
        assert all(s.interior.dtype == np.intp for s in sds)
        pp, pr = G[f"g{k}_pred_ptr"], G[f"g{k}_pred"]
        bp, bx = G[f"g{k}_box_ptr"], G[f"g{k}_box"]
        for c in range(0, g.n2d, max(1, g.n2d // 97)):
            assert np.array_equal(mck.predecessors(g, c, zeta), pr[pp[c]:pp[c + 1]])
            assert np.array_equal(mck.local_box(g, c, zeta).members, bx[bp[c]:bp[c + 1]])
        # the single-tile plan over the whole grid reproduces every predecessor list
        pl = Plan.local(g, zeta, np.arange(g.n2d))
        assert np.array_equal(pl.get(P.ROW_PTR), pp) and np.array_equal(pl.get(P.COL_IDX), pr)


@pytest.mark.parametrize("cfg", [(64, 32, False, 8, 2), (64, 32, True, 8, 2), (192, 96, False, 64, 3), (48, 24, True, 6, 5)])
def test_tile_csr_matches_oracle(cfg):
    nx, ny, per, delta, zeta = cfg
    g = _geo(nx, ny, True, per)
    grid = orc.Grid(nx, ny, True, per)
    pl = get_plan(g, delta, zeta)
    tp, rp, ci = pl.get(P.TILE_PTR), pl.get(P.ROW_PTR), pl.get(P.COL_IDX)
    bw, ph = pl.get(P.BANDWIDTH), pl.get(P.PHYS)
    for t, tile in enumerate(orc.decompose(grid, delta, zeta)):
        ip, ii = orc.predecessor_csr(grid, zeta, tile.local_order)
        lo, hi = tp[t], tp[t + 1]
        assert np.array_equal(rp[lo:hi + 1] - rp[lo], ip)
        assert np.array_equal(ci[rp[lo]:rp[hi]], ii)
        phys = ph[lo:hi]
        assert np.array_equal(np.sort(phys), np.arange(hi - lo))          # a permutation
        if not per:
            assert np.array_equal(phys, np.arange(hi - lo))               # clipped: physical == label order
        rows = np.repeat(np.arange(hi - lo), np.diff(ip))
        span = max((max(phys[r], phys[ii[ip[r]:ip[r + 1]]].max(initial=0)) - min(phys[r], phys[ii[ip[r]:ip[r + 1]]].min(initial=10**9))
                    for r in range(hi - lo)), default=0)
        assert bw[t] == span and rows.size == ii.size
    if not per and zeta == 3:
        assert pl.max_bw == 93 and pl.sum_nlocal == 32292 and pl.nnz == 654624


def test_restrict_observations_per_field_tile():
    g = _geo(24, 16, True, True, nfields=3)
    grid = orc.Grid(24, 16, True, True, 3)
    rng = np.random.default_rng(4)
    obs = np.sort(rng.choice(g.nstate, 300, replace=False))
    pl = Plan.decomposed(g, 6, 2)
    pl.set_observations(obs)
    optr, opos, orow = pl.get(P.OBS_PTR), pl.get(P.OBS_POS), pl.get(P.OBS_ROW)
    tiles = orc.decompose(grid, 6, 2)
    for f in range(3):
        sel = np.flatnonzero((obs >= f * g.n2d) & (obs < (f + 1) * g.n2d))
        for t, tile in enumerate(tiles):
            pos, rows = orc.restrict_observations(obs[sel] - f * g.n2d, tile.local_order)
            a, b = optr[f * 6 + t], optr[f * 6 + t + 1]
            assert np.array_equal(opos[a:b], pos) and np.array_equal(orow[a:b], sel[rows])
    net = mck.ObservationNetwork(obs[obs < g.n2d], np.ones((obs < g.n2d).sum()), np.zeros((obs < g.n2d).sum()))
    loc, rows = mck.restrict_network(net, tiles[2].local_order)
    pos, rows_ref = orc.restrict_observations(net.obs_indices, tiles[2].local_order)
    assert np.array_equal(loc.obs_indices, pos) and np.array_equal(rows, rows_ref)


def test_work_counts_match_survey_and_tile_ranges():
    g = _geo(192, 96, nfields=29)
    pl = Plan.decomposed(g, 256, 4)
    reg, sol, reg_distinct = pl.work(80)
    assert reg == pytest.approx(2.86e11, rel=0.01) and sol == pytest.approx(6.48e10, rel=0.01)
    assert 0.6 * reg < reg_distinct < 0.7 * reg          # halo rows shared between tiles are regressed once
    pl.set_tile_range(0, 128)
    r0, _, d0 = pl.work(80)
    pl.set_tile_range(128, 256)
    r1, _, d1 = pl.work(80)
    assert r0 + r1 == pytest.approx(reg, rel=1e-12)
    assert d0 + d1 > reg_distinct                        # rows straddling the cut are regressed by both ranks
    with pytest.raises(ValueError):
        pl.set_tile_range(10, 300)


def test_errors_follow_the_reference():
    with pytest.raises(mck.ConfigurationError, match="7"):
        mck.decompose(_geo(3, 2), 7, 1)                                    # test_geometry.py:189-191
    with pytest.raises(mck.ConfigurationError):
        mck.decompose(_geo(3, 2), 0, 1)
    with pytest.raises(ValueError):
        mck.decompose(_geo(3, 2), 2, -1)
    with pytest.raises(ValueError):
        mck.predecessors(_geo(3, 2), 99, 1)
    with pytest.raises(ValueError, match="strictly increasing"):
        Plan.local(_geo(4, 4), 1, np.array([3, 2, 5]))
    with pytest.raises(ValueError, match="strictly lower"):
        Plan.from_csr(np.array([0, 1]), np.array([0]))
    pl = Plan.decomposed(_geo(4, 4), 4, 1)
    with pytest.raises(ValueError, match="exceed"):
        pl.set_observations(np.array([3, 16]))
    with pytest.raises(ValueError):
        mck.GridGeometry("grid3d", 4, 4)
    with pytest.raises(mck.ConfigurationError):
        mck.AssimilationConfig(method="bogus")
    with pytest.raises(ValueError, match="lengths"):
        mck.ObservationNetwork(np.array([1, 2]), np.array([1.0]), np.array([0.0, 0.0]))
    with pytest.raises(ValueError, match="positive"):
        mck.ObservationNetwork(np.array([1]), np.array([0.0]), np.array([0.0]))
    with pytest.raises(ValueError, match="finite"):
        mck.EnsembleState(np.array([[np.nan, 1.0]]))
    assert mck.linear_index(_geo(5, 3, rm=False), 2, 4) == 14 and mck.grid_coords(_geo(5, 3, rm=False), 14) == (2, 4)


def test_perturb_observations_is_the_reference_stream(golden_analysis):
    A = golden_analysis
    net = mck.ObservationNetwork(A["a0_obs"], A["a0_r"], A["a0_y"])
    assert np.array_equal(mck.perturb_observations(net, int(A["a0_params"][3]), 11, 0).Ys, A["a0_Ys"])


def test_shared_regressions_are_identical_problems():
    """Halo rows regressed by several tiles: rows mapped onto one regression must have the same state
    row and the same predecessor list (estimator.py:123-131), and every distinct problem is kept once."""
    from paper_1606_00807_b200 import plan as planmod
    geo = mck.GridGeometry("grid2d", 24, 18)
    for periodic in (False, True):
        geo = mck.GridGeometry("grid2d", 24, 18, boundary="periodic" if periodic else "clipped")
        plan = planmod.Plan.decomposed(geo, 12, 2)
        tile_ptr, local_order = plan.get(planmod.TILE_PTR), plan.get(planmod.LOCAL_ORDER)
        row_ptr, col_idx = plan.get(planmod.ROW_PTR), plan.get(planmod.COL_IDX)
        rep = plan.get(planmod.REGRESSION_OF)
        tile_of = np.repeat(np.arange(plan.ntiles), np.diff(tile_ptr))

        def problem(q):
            base = tile_ptr[tile_of[q]]
            return (int(local_order[q]), tuple(local_order[base + col_idx[row_ptr[q]:row_ptr[q + 1]]].tolist()))

        problems = [problem(q) for q in range(len(rep))]
        assert all(problems[q] == problems[rep[q]] for q in range(len(rep)))
        assert all(rep[rep[q]] == rep[q] for q in range(len(rep)))
        assert plan.n_regressions == len(set(problems)) == len(set(rep.tolist()))
        assert plan.n_regressions < plan.n_owned_rows == len(rep)
        # one rank's share: only owned rows are mapped, and only onto owned rows
        plan.set_tile_range(2, 5)
        rep = plan.get(planmod.REGRESSION_OF)
        owned = (tile_of >= 2) & (tile_of < 5)
        assert np.all(rep[~owned] == -1) and np.all(owned[rep[owned]])
        assert plan.n_owned_rows == int(owned.sum())


def test_per_axis_boundary_against_extended_oracle():
    """Longitude periodic / latitude clipped (BASELINE.json config 1 as worded) and the transposed case: the plan's index
    maps against the extended oracle (the reference's per-axis rules, geometry.py:132-142, with one flag per axis).  The
    reference has a single boundary flag: parity for the mixed cases is unpinned by the reference; the two reference
    boundaries keep their bit-exact golden tests above."""
    import paper_1606_00807_b200 as mck
    from oracle import enkf_mc_oracle as orc
    from paper_1606_00807_b200.plan import COL_IDX, LOCAL_ORDER, Plan
    for boundary in ("periodic_x", "periodic_y"):
        for ordering in ("row_major", "column_major"):
            geo = mck.GridGeometry("grid2d", 20, 12, ordering=ordering, boundary=boundary)
            grid = orc.grid_for(20, 12, boundary, row_major=ordering == "row_major")
            assert grid.px == (boundary == "periodic_x") and grid.py == (boundary == "periodic_y")
            plan = Plan.decomposed(geo, 6, 2)
            tiles = orc.decompose(grid, 6, 2)
            assert np.array_equal(plan.get(LOCAL_ORDER), np.concatenate([t.local_order for t in tiles]))
            assert np.array_equal(plan.get(COL_IDX),
                                  np.concatenate([orc.predecessor_csr(grid, 2, t.local_order)[1] for t in tiles]))
            for sd, t in zip(mck.decompose(geo, 6, 2), tiles):
                assert np.array_equal(sd.interior, t.interior) and np.array_equal(sd.halo, t.halo)
            for c in (0, 19, 20 * 11, 239, 125):
                assert np.array_equal(mck.predecessors(geo, c, 2), orc.predecessors(grid, c, 2))
                assert np.array_equal(mck.local_box(geo, c, 2).members, orc.local_box(grid, c, 2))
    # the seam: the last column sees the first two through the wrap (row-major labels, zeta = 2)
    lon = mck.GridGeometry("grid2d", 20, 12, boundary="periodic_x")
    assert mck.predecessors(lon, 19 + 20 * 5, 2).size == 14 and mck.predecessors(mck.GridGeometry("grid2d", 20, 12), 19 + 20 * 5, 2).size == 8
    # brute-force definition of the box for one cell
    r0, c0 = 5, 19
    want = sorted(r * 20 + (c % 20) for r in range(max(0, r0 - 2), min(12, r0 + 3)) for c in range(c0 - 2, c0 + 3))
    assert mck.local_box(lon, c0 + 20 * r0, 2).members.tolist() == sorted(set(want))


# ---- vertically coupled levels (extension; BASELINE.json configs 3 / 5 "vertical r = 1"; parity unpinned by the reference:
# the integer maps are checked against the extended oracle, which applies the reference's rules on the extended box) ----
@pytest.mark.parametrize("nx,ny,nlev,zeta_v,delta,zeta,boundary", [
    (12, 8, 3, 1, 4, 2, "clipped"), (10, 9, 4, 2, 6, 1, "periodic_x"), (16, 6, 2, 0, 4, 3, "periodic"),
    (7, 5, 3, 1, 1, 2, "clipped"), (9, 9, 5, 1, 9, 0, "clipped"),
])
def test_level_maps_match_extended_oracle(nx, ny, nlev, zeta_v, delta, zeta, boundary):
    import paper_1606_00807_b200 as mck
    from oracle import enkf_mc_oracle as orc
    from paper_1606_00807_b200.plan import COL_IDX, HALO, INTERIOR, INTERIOR_POS, LOCAL_ORDER, ROW_PTR, Plan
    g = mck.GridGeometry("grid2d", nx, ny, boundary=boundary, nlev=nlev, zeta_v=zeta_v)
    og = orc.grid_for(nx, ny, boundary, nlev=nlev, zeta_v=zeta_v)
    assert g.nstate == og.nstate == nx * ny * nlev
    plan = Plan.decomposed(g, delta, zeta)
    tiles = orc.decompose(og, delta, zeta)
    assert np.array_equal(plan.get(LOCAL_ORDER), np.concatenate([t.local_order for t in tiles]))
    assert np.array_equal(plan.get(INTERIOR), np.concatenate([t.interior for t in tiles]))
    assert np.array_equal(plan.get(HALO), np.concatenate([t.halo for t in tiles]))
    assert np.array_equal(plan.get(INTERIOR_POS), np.concatenate([t.interior_positions() for t in tiles]))
    assert np.array_equal(np.sort(plan.get(INTERIOR)), np.arange(g.nstate))          # interiors partition the field
    csr = [orc.predecessor_csr(og, zeta, t.local_order) for t in tiles]
    assert np.array_equal(plan.get(COL_IDX), np.concatenate([c[1] for c in csr]))
    assert np.array_equal(plan.get(ROW_PTR), np.concatenate([[0]] + [np.diff(c[0]) for c in csr]).cumsum())
    for c in (0, nx + 1, g.nstate - 1, (nlev - 1) * nx * ny + 2 * nx + 3):
        assert np.array_equal(mck.geometry.local_box(g, c, zeta).members, orc.local_box(og, c, zeta))
        assert np.array_equal(mck.geometry.predecessors(g, c, zeta), orc.predecessors(og, c, zeta))


def test_levels_without_vertical_coupling_are_stacked_fields():
    """zeta_v = 0: the predecessor lists of a lifted tile are those of the 2-D tile on every level."""
    import paper_1606_00807_b200 as mck
    from paper_1606_00807_b200.plan import COL_IDX, ROW_PTR, TILE_PTR, Plan
    p3 = Plan.decomposed(mck.GridGeometry("grid2d", 14, 10, nlev=3, zeta_v=0), 4, 2)
    p2 = Plan.decomposed(mck.GridGeometry("grid2d", 14, 10), 4, 2)
    assert p3.max_pred == p2.max_pred and p3.nnz == 3 * p2.nnz
    tp3, tp2, rp3, rp2, ci3, ci2 = (p3.get(TILE_PTR), p2.get(TILE_PTR), p3.get(ROW_PTR), p2.get(ROW_PTR), p3.get(COL_IDX),
                                    p2.get(COL_IDX))
    for t in range(4):
        n2 = tp2[t + 1] - tp2[t]
        for lev in range(3):
            for j in (0, n2 // 2, n2 - 1):
                a = ci3[rp3[tp3[t] + lev * n2 + j]:rp3[tp3[t] + lev * n2 + j + 1]]
                b = ci2[rp2[tp2[t] + j]:rp2[tp2[t] + j + 1]]
                assert np.array_equal(a, b + lev * n2)


def test_level_geometry_validation():
    import paper_1606_00807_b200 as mck
    with pytest.raises(ValueError, match="nlev must be positive"):
        mck.GridGeometry("grid2d", 4, 4, nlev=0)
    with pytest.raises(ValueError, match="zeta_v must be nonnegative"):
        mck.GridGeometry("grid2d", 4, 4, nlev=2, zeta_v=-1)
