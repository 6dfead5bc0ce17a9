"""-m gpu: the sharded public entry point over NCCL, one process per GPU.  World size 1 runs everywhere (the same call path:
process group, shard, scatter, analysis, gather, status exchange); world size 2 needs two GPUs and is skipped otherwise.  The
result on the root must equal the single-process assimilate_parallel bit for bit: tiles are independent units and every
rank runs the same kernels on its block rows."""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out_path):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    import paper_1606_00807_b200 as mck
    from paper_1606_00807_b200 import synthetic
    w = synthetic.make_workload("multi", nx=40, ny=24, nens=24, corr_len=3.0, zeta=2, delta=8, obs="random", obs_arg=0.3,
                                r_rel=0.1, r_abs=None, seed=41, nugget=0.01, variables=[("u", 1.0, 2), ("q", 1e-2, 1)])
    geo = mck.GridGeometry("grid2d", w.nx, w.ny, nfields=w.nfields)
    cfg = mck.AssimilationConfig(zeta=w.zeta, delta=w.delta, seed=w.seed)
    net = mck.ObservationNetwork(w.obs_indices, w.r_diag, w.y)
    for _ in range(2):                                   # the second call reuses the cached shard and buffers
        xa, rep = mck.assimilate_parallel_sharded(mck.EnsembleState(w.X) if rank == 0 else None, net, cfg, geo,
                                                  Ys=w.Ys if rank == 0 else None, nens=w.nens)
    if rank == 0:
        np.save(out_path, xa.X)
    else:
        assert xa is None
    dist.barrier()
    dist.destroy_process_group()


def _run(world, tmp_path):
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs, found {torch.cuda.device_count()}")
    out_path = str(tmp_path / "xa.npy")
    port = 29900 + (os.getpid() + 13 * world) % 90
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, out_path)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    import paper_1606_00807_b200 as mck
    from paper_1606_00807_b200 import synthetic
    w = synthetic.make_workload("multi", nx=40, ny=24, nens=24, corr_len=3.0, zeta=2, delta=8, obs="random", obs_arg=0.3,
                                r_rel=0.1, r_abs=None, seed=41, nugget=0.01, variables=[("u", 1.0, 2), ("q", 1e-2, 1)])
    geo = mck.GridGeometry("grid2d", w.nx, w.ny, nfields=w.nfields)
    cfg = mck.AssimilationConfig(zeta=w.zeta, delta=w.delta, seed=w.seed)
    net = mck.ObservationNetwork(w.obs_indices, w.r_diag, w.y)
    ref, _ = mck.assimilate_parallel(mck.EnsembleState(w.X), net, cfg, geo, Ys=w.Ys)
    got = np.load(out_path)
    assert np.array_equal(got, ref.X)
    assert not np.array_equal(got, w.X)


def test_sharded_entry_point_one_rank_nccl(tmp_path):
    _run(1, tmp_path)


def test_sharded_entry_point_two_ranks_nccl(tmp_path):
    _run(2, tmp_path)
