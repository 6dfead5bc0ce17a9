"""CPU, world_size 2 over gloo: the sub-domain sharding (tile ranges per rank, owned interior rows,
analysis all-gather) reproduces the single-process analysis.  The per-tile compute is stood in by the
oracle (checker role only) -- the host-side partition/exchange logic is what is under test."""

import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, nfields, out, nlev=1):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1606_00807_b200 as mck
    from oracle import enkf_mc_oracle as orc
    from paper_1606_00807_b200 import distributed, synthetic
    from paper_1606_00807_b200.plan import Plan

    w = synthetic.make_workload("d", nx=20, ny=12, nens=16, corr_len=2.0, zeta=1, delta=6, obs="random", obs_arg=0.4,
                                r_rel=0.1, r_abs=None, seed=5, nugget=0.01,
                                variables=[("u", 1.0, nfields * nlev)])
    # nlev > 1: the same state read as nfields vertically coupled fields of nlev levels (extension)
    geo = mck.GridGeometry("grid2d", w.nx, w.ny, nfields=nfields, nlev=nlev, zeta_v=1 if nlev > 1 else 0)
    plan = Plan.decomposed(geo, w.delta, w.zeta)
    shard = distributed.TileShard(plan, geo, rank, world)
    shard.apply()
    assert sum(b - a for a, b in shard.tile_ranges) == plan.ntiles
    # slab scatter: every rank receives exactly the rows its tiles read (interiors + halos, all fields) and the rows of
    # the perturbed observations inside them; everything else stays untouched
    from paper_1606_00807_b200.plan import LOCAL_ORDER, TILE_PTR
    shard.set_observations(w.obs_indices)
    X = torch.from_numpy(w.X.copy()) if rank == 0 else torch.full(w.X.shape, float("nan"), dtype=torch.float64)
    Ys = torch.from_numpy(w.Ys.copy()) if rank == 0 else torch.full(w.Ys.shape, float("nan"), dtype=torch.float64)
    shard.scatter_background(X, Ys)
    tp, lo = plan.get(TILE_PTR), plan.get(LOCAL_ORDER)
    t0, t1 = shard.tile_ranges[rank]
    read2d = np.unique(lo[tp[t0]:tp[t1]])
    read = (np.arange(nfields)[:, None] * geo.nfield + read2d[None, :]).ravel()
    assert np.array_equal(shard.need[rank], read)
    assert np.array_equal(X.numpy()[read], w.X[read])
    obs_read = np.flatnonzero(np.isin(w.obs_indices, read))
    assert np.array_equal(shard.need_obs[rank], obs_read)
    assert np.array_equal(Ys.numpy()[obs_read], w.Ys[obs_read])
    if rank != 0:
        untouched = np.setdiff1d(np.arange(geo.nstate), read)
        assert np.all(np.isnan(X.numpy()[untouched]))
        assert read.size < geo.nstate                      # a slab, not the whole ensemble
    for _ in range(2):                                     # buffers are reused: a second exchange gives the same result
        shard.scatter_background(X, Ys)
    assert np.array_equal(X.numpy()[read], w.X[read])
    assert 0.0 < shard.memory_fraction() < 1.0
    # owned tiles analysed by the oracle, everything else poisoned
    grid = orc.Grid(w.nx, w.ny, nfields=nfields, nlev=nlev, zeta_v=1 if nlev > 1 else 0)
    full = orc.assimilate(w.X, w.obs_indices, w.r_diag, w.Ys, grid, w.delta, w.zeta)
    Xa = torch.full(w.X.shape, float("nan"), dtype=torch.float64)
    rows = shard.rows[rank]
    Xa[torch.from_numpy(rows)] = torch.from_numpy(full[rows])
    shard.gather_analysis(Xa)
    ok = np.array_equal(Xa.numpy(), full)
    covered = np.sort(np.concatenate(shard.rows))
    ok = ok and np.array_equal(covered, np.arange(geo.nstate))
    flag = torch.tensor([int(ok)])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        out.put(int(flag.item()))
    dist.destroy_process_group()


@pytest.mark.parametrize("nfields,nlev", [(1, 1), (3, 1), (2, 3)])
def test_two_rank_shard_and_gather(nfields, nlev):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = 29500 + (os.getpid() + nfields + 7 * nlev) % 400
    procs = [ctx.Process(target=_worker, args=(r, 2, port, nfields, out, nlev)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    assert out.get(timeout=5) == 1


def test_block_row_cuts_balance():
    from paper_1606_00807_b200.distributed import block_row_cuts
    assert block_row_cuts(16, 8) == [0, 2, 4, 6, 8, 10, 12, 14, 16]
    assert block_row_cuts(2, 8)[-1] == 2 and len(block_row_cuts(2, 8)) == 9
    assert block_row_cuts(8, 3) == [0, 2, 5, 8]
