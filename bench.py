#!/usr/bin/env python
"""Benchmark of the EnKF-MC analysis step (BASELINE.json metric: analysis grid-points/sec).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg3] [--impl b200|reference]

A "step" is one full analysis (K0 centre -> K2 regress -> K3 local solve + interior scatter) of the
synthetic workload.  `value` = state components / device time with inputs resident in HBM;
`e2e` = the same through `assimilate_parallel` with pinned HOST buffers (H2D + D2H inside the timed
region).  `roofline` is for the dominant stage (K2 regress = K2a + K2b): algorithmic flops (SURVEY 8d:
Householder-QR least squares, SVD extras not credited) / its CUDA-event time, against the FP64 peak
measured live (`enkfmc_fp64_peak` / `enkfmc_fp64_mma_peak`, the larger; MEASURED_PEAKS.json has no FP64
figure); `roofline_k2a` and `roofline_solve` give K2a alone and K3.
`--impl reference` times the CPU oracle port (the reference is pure Python and cannot travel to the
GPU box) on a bounded sample with all host cores.

N > 1 (torchrun): sub-domains are sharded by contiguous block rows across ranks; per step rank 0's
background is broadcast (NCCL), every rank analyses its tiles, the interiors are all-gathered.
Total work is fixed as N grows ("strong").
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NCU_TRAFFIC_K2 = 15.15e9         # dram bytes read + written per bench launch: K2a 3.59 + 5.55 GB, K2b 5.65 + 0.35 GB (ncu --set full)
NCU_TRAFFIC_SOURCE = "profiles/r1_ncu_full_k2_bench_launch.csv"
METRIC = "EnKF-MC analysis grid-points/sec (B^-1 est + local solve)"
UNIT = "grid-points/s"

# ------------------------------------------------------------------------------------------
# CPU arm: oracle port, one process per core over the tiles of a bounded sample of fields
# ------------------------------------------------------------------------------------------
_G = {}


def _cpu_tile(t):
    from threadpoolctl import threadpool_limits

    from oracle import enkf_mc_oracle as orc
    with threadpool_limits(limits=1):                  # as the reference does (driver.py:231)
        res = orc.analyse_tile(_G["X"], _G["obs"], _G["r"], _G["Ys"], _G["grid"], _G["zeta"], _G["tiles"][t],
                               _G["csr"][t])
    return res.tile.interior, res.xa_local[res.tile.interior_positions()]


def cpu_sample_setup(w, field=0):
    from oracle import enkf_mc_oracle as orc
    grid = orc.Grid(w.nx, w.ny, True, w.boundary == "periodic")
    lo, hi = field * w.n2d, (field + 1) * w.n2d
    sel = np.flatnonzero((w.obs_indices >= lo) & (w.obs_indices < hi))
    tiles = orc.decompose(grid, w.delta, w.zeta)
    _G.update(X=w.X[lo:hi], obs=w.obs_indices[sel] - lo, r=w.r_diag[sel], Ys=w.Ys[sel], grid=grid, zeta=w.zeta,
              tiles=tiles, csr=[orc.predecessor_csr(grid, w.zeta, t.local_order) for t in tiles])
    return len(tiles)


def cpu_sample_run(pool, ntiles):
    """One pass of the CPU path over the sample (one 2-D field); returns seconds."""
    t0 = time.perf_counter()
    out = _G["X"].copy()
    for interior, rows in pool.imap_unordered(_cpu_tile, range(ntiles), chunksize=1):
        out[interior] = rows
    return time.perf_counter() - t0, out


# ------------------------------------------------------------------------------------------
def clocks_sampler(gpu_index, stop, samples):
    q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    try:
        proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", os.environ.get("ENKFMC_BENCH_SMI_MS", "100"),
                                 "-i", str(gpu_index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    except OSError:
        return
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    try:
        while not stop.is_set():
            line = proc.stdout.readline()
            if not line:
                break
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                samples.append((float(parts[0]), float(parts[1]), float(parts[2]),
                                [n for n, v in zip(names, parts[3:7]) if v.lower().startswith("active")]))
            except ValueError:
                continue
    finally:
        proc.terminate()


def summarize_clocks(samples):
    if not samples:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
    sm = sorted(s[0] for s in samples)
    reasons = sorted({r for s in samples for r in s[3]})
    return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": samples[0][1], "reasons": reasons, "samples": len(samples),
            "power_w_max": max(s[2] for s in samples)}


def pinned(a):
    import torch
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    out = t.numpy()
    out[...] = a
    return out, t


def run_reference(args, rank, world):
    """CPU arm: rank 0 only; each step = one 2-D field of the workload on all host cores."""
    if rank != 0:
        return
    from paper_1606_00807_b200 import synthetic
    full_fields = {"cfg3": 29, "cfg5": 40}.get(args.workload)
    w = synthetic.config(args.workload, fields=1 if full_fields else None)
    cores = os.cpu_count() or 1
    ntiles = cpu_sample_setup(w, 0)
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        for _ in range(args.warmup):
            cpu_sample_run(pool, ntiles)
        times = [cpu_sample_run(pool, ntiles)[0] for _ in range(args.steps)]
    t = float(np.mean(times))
    val = w.n2d / t
    sample = f"1 of the workload's 2-D fields ({w.ny}x{w.nx}, N={w.nens}, zeta={w.zeta}, {ntiles} tiles) per step"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.workload, w, full_fields=full_fields),
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def workload_config(name, w, full_fields):
    """Both arms report the full workload; the CPU arm builds one of its fields only (full_fields set)."""
    nf = full_fields if full_fields else w.nfields
    nbytes = w.X.nbytes * nf // w.nfields
    return {"workload": name, "grid": f"{w.ny}x{w.nx}", "fields": nf, "nstate": w.n2d * nf, "nens": w.nens, "zeta": w.zeta,
            "delta": w.delta, "boundary": w.boundary, "nugget": w.nugget,
            "nobs": int(w.obs_indices.size) * nf // w.nfields,
            "cache": "inputs larger than L2 (ensemble + T factors >> 126 MB)" if nbytes > 2.5e8 else
                     "L2 flushed between steps (256 MB write)"}


def run_b200(args, rank, world, local_rank):
    from paper_1606_00807_b200 import synthetic

    # ---- workload + CPU baseline first (fork before CUDA is initialised) -----------------------
    w = synthetic.config(args.workload, nugget=args.nugget, fields=args.fields)
    cpu_baseline = None
    if world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        ntiles = cpu_sample_setup(w, 0)
        with mp.get_context("fork").Pool(cores) as pool:
            cpu_sample_run(pool, min(ntiles, cores))            # touch the pool / page in LAPACK
            t_cpu, cpu_field0 = cpu_sample_run(pool, ntiles)
        cpu_baseline = {"value": w.n2d / t_cpu, "unit": UNIT, "cores": cores, "kind": "port",
                        "sample": f"field 0 of {w.nfields} ({w.ny}x{w.nx}, N={w.nens}, {ntiles} tiles), "
                                  f"{t_cpu:.2f} s, oracle port, one process per core"}
    else:
        cpu_field0 = None

    import torch
    import torch.distributed as dist

    import paper_1606_00807_b200 as mck
    from paper_1606_00807_b200 import _lib, device, distributed
    from paper_1606_00807_b200.plan import get_plan

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    geo = mck.GridGeometry("ring1d" if w.ny == 1 else "grid2d", w.nx, w.ny, boundary=w.boundary, nfields=w.nfields)
    plan = get_plan(geo, w.delta, w.zeta)
    plan.set_observations(w.obs_indices)
    shard = distributed.TileShard(plan, geo, rank, world)
    shard.apply()

    dX = device.to_device(w.X)
    dR = device.to_device(w.r_diag)
    dYs = device.to_device(w.Ys)
    dXa = torch.empty_like(dX)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda") if w.X.nbytes <= 2.5e8 else None

    def step():
        if flush is not None:
            flush.zero_()
        if world > 1:
            shard.broadcast_background(dX)
        device.analysis_device(plan, dX, dR, dYs, dXa)
        if world > 1:
            shard.gather_analysis(dXa)

    peak = np.zeros(1)
    _lib.check(_lib.lib().enkfmc_fp64_peak(_lib.ptr(peak), device.stream_ptr()))
    peak_mma = np.zeros(1)
    _lib.check(_lib.lib().enkfmc_fp64_mma_peak(_lib.ptr(peak_mma), device.stream_ptr()))

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # ---- timed region -------------------------------------------------------------------------
    stop, samples = threading.Event(), []
    sampler = None
    if rank == 0:
        sampler = threading.Thread(target=clocks_sampler, args=(torch.cuda.current_device(), stop, samples), daemon=True)
        sampler.start()
        time.sleep(0.3)
    launches0 = plan.counter(0)
    plan.profile(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    ncalls, stage_ms = plan.stage_times()
    plan.profile(False)
    launches = (plan.counter(0) - launches0) // args.steps
    if world > 1:
        tmax = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        ms = float(tmax.item())

    # ---- parity spot check of the timed output against the CPU sample (field 0) ----------------
    parity = None
    if cpu_field0 is not None:
        got = dXa[: w.n2d].cpu().numpy()
        parity = float(np.linalg.norm(got - cpu_field0) / np.linalg.norm(cpu_field0))

    # ---- end to end through the public API with pinned host buffers ------------------------
    Xh, _keep1 = pinned(w.X)
    Ysh, _keep2 = pinned(w.Ys)
    net = mck.ObservationNetwork(w.obs_indices, w.r_diag, w.y)
    cfg = mck.AssimilationConfig(zeta=w.zeta, delta=w.delta)
    xb = mck.EnsembleState(Xh)
    for _ in range(max(args.warmup, 3)):   # same ownership pattern as the timed loop: the pinned result pool reaches its
        xa, rep = mck.assimilate_parallel(xb, net, cfg, geo, Ys=Ysh)   # steady state (two buffers) before timing starts
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        xa, rep = mck.assimilate_parallel(xb, net, cfg, geo, Ys=Ysh)
    torch.cuda.synchronize()
    t_e2e = (time.perf_counter() - t0) / args.steps
    if world > 1:
        tmax = torch.tensor([t_e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        t_e2e = float(tmax.item())
    stop.set()
    if sampler is not None:
        sampler.join(timeout=2.0)

    if rank == 0:
        # fl_reg: the regressions the kernels execute (distinct ones); fl_reg_ref: one per local row as the reference runs them
        fl_reg_ref, fl_sol, fl_reg = plan.work(w.nens)
        nc = max(ncalls, 1)
        t_qr, t_prb, t_sol = stage_ms[1] / nc * 1e-3, stage_ms[2] / nc * 1e-3, stage_ms[3] / nc * 1e-3
        t_reg = t_qr + t_prb
        # FP64 peak of this device, measured in this run: the larger of the DFMA chain kernel and the mma.m8n8k4.f64
        # (tensor-core) kernel -- K2a and K3b run their block products on the latter
        pk_fma, pk_mma = float(peak[0]), float(peak_mma[0])
        pk = max(pk_fma, pk_mma)
        peak_note = (f"FP64, measured in this run: DFMA chain {pk_fma:.1f}, mma.m8n8k4.f64 (DMMA, tensor cores) {pk_mma:.1f} TFLOP/s; "
                     "the larger is the denominator (MEASURED_PEAKS.json holds HBM and bf16 figures only)")
        ach_qr = fl_reg / t_qr * 1e-12 if t_qr > 0 else 0.0
        ach = fl_reg / t_reg * 1e-12 if t_reg > 0 else 0.0
        ach_sol = fl_sol / t_sol * 1e-12 if t_sol > 0 else 0.0
        nstate = w.nstate
        out = {
            "metric": METRIC, "value": nstate / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.workload, w, None),
            # the regression stage is one unit of work split over two kernels: K2a executes the credited flops
            # (Householder-QR least squares), K2b (the longer of the two) turns the QR into the reference's
            # truncated-SVD answer and is uncredited -- `roofline` therefore charges both kernels' time to the QR flops
            "roofline": {"kernel": "regress_qr_mma_kernel + regress_solve_kernel (K2a + K2b: one regression stage)",
                         "bound": "tensor", "achieved": ach, "peak": pk,
                         "unit": "TFLOP/s", "frac": ach / pk if pk > 0 else None,
                         "traffic": NCU_TRAFFIC_K2 if args.workload == "cfg3" and world == 1 else None,
                         "traffic_source": NCU_TRAFFIC_SOURCE,
                         "peak_source": peak_note,
                         "ms_per_launch": t_reg * 1e3, "algorithmic_flops_per_launch": fl_reg,
                         "distinct_regressions_per_launch": plan.n_regressions * w.nfields,
                         "reference_regressions_per_launch": plan.n_owned_rows * w.nfields,
                         "reference_equivalent_flops": fl_reg_ref},
            "roofline_k2a": {"kernel": "regress_qr_mma_kernel (K2a alone)", "bound": "tensor", "achieved": ach_qr, "peak": pk,
                             "unit": "TFLOP/s", "frac": ach_qr / pk if pk > 0 else None, "ms_per_launch": t_qr * 1e3,
                             "algorithmic_flops_per_launch": fl_reg},
            "roofline_solve": {"kernel": "assemble_band_tile_kernel + local_solve_kernel (K3)", "bound": "tensor", "achieved": ach_sol,
                               "peak": pk, "unit": "TFLOP/s", "frac": ach_sol / pk if pk > 0 else None,
                               "ms_per_launch": t_sol * 1e3, "algorithmic_flops_per_launch": fl_sol},
            "stage_ms": {"center": stage_ms[0] / nc, "regress_qr": t_qr * 1e3, "regress_solve": t_prb * 1e3,
                         "local_solve": t_sol * 1e3},
            "cpu_baseline": cpu_baseline,
            "e2e": {"value": nstate / t_e2e, "unit": UNIT, "ms_per_step": t_e2e * 1e3,
                    # busy time of each stage summed over the field groups; the copies of one group run on a copy
                    # stream under the compute of its neighbours, so the sum exceeds the wall time of the call
                    "breakdown_ms": {"h2d": rep.t_h2d * 1e3, "estimation": float(rep.t_estimation.sum()) * 1e3,
                                     "analysis": float(rep.t_analysis.sum()) * 1e3, "d2h": rep.t_d2h * 1e3,
                                     "call_wall": rep.t_total * 1e3},
                    "pipelined": "5 groups of fields: H2D of group g+1 and D2H of group g-1 overlap the kernels of group g",
                    "h2d_bytes_per_step": int(w.X.nbytes + w.Ys.nbytes + w.r_diag.nbytes),
                    "d2h_bytes_per_step": int(w.X.nbytes),
                    "api": "assimilate_parallel(EnsembleState, ObservationNetwork, AssimilationConfig, GridGeometry, Ys=)"},
            "gpu_launches": int(launches),
            "clocks": summarize_clocks(samples),
            "parity_vs_cpu_sample": parity,
        }
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--fields", type=int, default=None, help="truncate a multi-field workload (debug only)")
    ap.add_argument("--nugget", type=float, default=0.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_b200(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
