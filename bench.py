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

N > 1: `python bench.py --gpus N` re-executes itself under torch.distributed.run with N ranks (one per GPU); under
torchrun WORLD_SIZE must equal --gpus.  Sub-domains are sharded by contiguous block rows across ranks; per step rank 0
scatters to every rank the background rows and perturbed-observation rows its tiles read (NCCL point-to-point), every
rank analyses its tiles, the interiors are all-gathered.  Total work is fixed as N grows ("strong").  `e2e` at N > 1 is
`assimilate_parallel_sharded` (host buffers on rank 0 -> upload -> scatter -> compute -> gather -> download).
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

NCU_TRAFFIC_SOURCE = "profiles/r2_ncu_full_bench_launch.csv"   # written by tools/make_profiles.py from one ncu --set full capture


def ncu_traffic():
    """{kernel name prefix: dram bytes read + written per launch} from the committed ncu summary (None if absent)."""
    path = os.path.join(ROOT, NCU_TRAFFIC_SOURCE)
    if not os.path.exists(path):
        return None
    import csv
    out = {}
    with open(path) as fh:
        for row in csv.DictReader(fh):
            try:
                out[row["kernel"]] = float(row["dram_bytes_read"]) + float(row["dram_bytes_write"])
            except (KeyError, ValueError):
                continue
    return out or None


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
    grid = orc.grid_for(w.nx, w.ny, w.boundary)
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
    from paper_1606_00807_b200.plan import Plan, get_plan

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    geo = mck.GridGeometry("ring1d" if w.ny == 1 else "grid2d", w.nx, w.ny, boundary=w.boundary, nfields=w.nfields)
    plan = get_plan(geo, w.delta, w.zeta) if world == 1 else Plan.decomposed(geo, w.delta, w.zeta)
    plan.set_observations(w.obs_indices)
    shard = distributed.TileShard(plan, geo, rank, world, w.obs_indices)
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
            shard.scatter_background(dX, dYs)
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

    # ---- outcome of the timed analyses: per-tile status (a failed tile must not be timed as a success) and a parity
    #      spot check of the timed output against the CPU sample (field 0), gated by the oracle's measured noise floor ---
    clamped = device.check_status(plan)          # raises NumericalError naming the sub-domain
    parity, parity_gate = None, None
    if cpu_field0 is not None:
        got = dXa[: w.n2d].cpu().numpy()
        parity = float(np.linalg.norm(got - cpu_field0) / np.linalg.norm(cpu_field0))
        floors_path = os.path.join(ROOT, "tests", "golden", "noise_floors.json")
        key = args.workload + ("_nugget" if args.nugget > 0 else "")
        floor = json.load(open(floors_path)).get(key, {}).get("Xa") if os.path.exists(floors_path) else None
        parity_gate = max(1e-8, 10.0 * floor) if floor is not None else None
        if parity_gate is not None and not parity < parity_gate:
            raise SystemExit(f"bench: analysis differs from the CPU oracle by {parity:.3e} (gate {parity_gate:.1e}): number not reported")

    # ---- end to end through the public API: host buffers in, host analysis out -----------------------
    net = mck.ObservationNetwork(w.obs_indices, w.r_diag, w.y)
    cfg = mck.AssimilationConfig(zeta=w.zeta, delta=w.delta)

    def e2e_loop(xb, ys):
        if world == 1:
            call = lambda: mck.assimilate_parallel(xb, net, cfg, geo, Ys=ys)
        else:
            call = lambda: mck.assimilate_parallel_sharded(xb if rank == 0 else None, net, cfg, geo,
                                                            Ys=ys if rank == 0 else None, nens=w.nens)
        for _ in range(max(args.warmup, 3)):   # same ownership pattern as the timed loop: the pinned result pool reaches its
            xa, rep = call()                   # steady state (two buffers) before timing starts
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            xa, rep = call()
        torch.cuda.synchronize()
        t = (time.perf_counter() - t0) / args.steps
        if world > 1:
            tmax = torch.tensor([t], dtype=torch.float64, device="cuda")
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
            t = float(tmax.item())
        return t, rep

    Xh, _keep1 = pinned(w.X)
    Ysh, _keep2 = pinned(w.Ys)
    t_e2e, rep = e2e_loop(mck.EnsembleState(Xh), Ysh)                    # page-locked inputs: asynchronous, pipelined copies
    t_e2e_pageable, _ = e2e_loop(mck.EnsembleState(w.X), w.Ys)           # ordinary numpy arrays: staged copies
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
        tr = ncu_traffic()

        def traffic_of(*prefixes):
            if not tr:
                return None
            tot = sum(v for k, v in tr.items() if any(k.startswith(px) for px in prefixes))
            return tot or None

        peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
        hbm_measured = os.path.exists(peaks_path)
        hbm_peak = float(json.load(open(peaks_path)).get("hbm_gbs", 6551.0)) if hbm_measured else 6551.0
        out = {
            "metric": METRIC, "value": nstate / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.workload, w, None),
            # the regression stage is one unit of work split over two kernels: K2a executes the credited flops
            # (Householder-QR least squares), K2b (the longer of the two) turns the QR into the reference's
            # truncated-SVD answer and is uncredited -- `roofline` therefore charges both kernels' time to the QR flops
            "roofline": {"kernel": "regress_qr_mma_kernel + regress_clean_kernel + regress_trunc_kernel (K2a + K2b: one regression stage)",
                         "bound": "tensor", "achieved": ach, "peak": pk,
                         "unit": "TFLOP/s", "frac": ach / pk if pk > 0 else None,
                         "traffic": traffic_of("regress_") if args.workload == "cfg3" and world == 1 else None,
                         "traffic_source": NCU_TRAFFIC_SOURCE,
                         "peak_source": peak_note,
                         "ms_per_launch": t_reg * 1e3, "algorithmic_flops_per_launch": fl_reg,
                         "distinct_regressions_per_launch": plan.n_regressions * w.nfields,
                         "reference_regressions_per_launch": plan.n_owned_rows * w.nfields,
                         "reference_equivalent_flops": fl_reg_ref},
            "roofline_k2a": {"kernel": "regress_qr_mma_kernel (K2a alone)", "bound": "tensor", "achieved": ach_qr, "peak": pk,
                             "unit": "TFLOP/s", "frac": ach_qr / pk if pk > 0 else None, "ms_per_launch": t_qr * 1e3,
                             "algorithmic_flops_per_launch": fl_reg,
                             "traffic": traffic_of("regress_qr") if args.workload == "cfg3" and world == 1 else None},
            "roofline_solve": {"kernel": "assemble_band_tile_kernel + local_solve_kernel (K3)", "bound": "tensor", "achieved": ach_sol,
                               "peak": pk, "unit": "TFLOP/s", "frac": ach_sol / pk if pk > 0 else None,
                               "ms_per_launch": t_sol * 1e3, "algorithmic_flops_per_launch": fl_sol,
                               "traffic": traffic_of("assemble_band", "local_solve") if args.workload == "cfg3" and world == 1 else None},
            "roofline_center": {"kernel": "center_rows_kernel (K0)", "bound": "hbm",
                                "achieved": 16.0 * w.nstate * w.nens / (stage_ms[0] / nc * 1e-3) * 1e-9 if stage_ms[0] > 0 else None,
                                "peak": hbm_peak, "unit": "GB/s",
                                "frac": (16.0 * w.nstate * w.nens / (stage_ms[0] / nc * 1e-3) * 1e-9 / hbm_peak) if stage_ms[0] > 0 and hbm_peak else None,
                                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if hbm_measured else "fallback 6551 GB/s (MEASURED_PEAKS.json absent)"},
            "stage_ms": {"center": stage_ms[0] / nc, "regress_qr": t_qr * 1e3, "regress_solve": t_prb * 1e3,
                         "local_solve": t_sol * 1e3},
            "cpu_baseline": cpu_baseline,
            "e2e": {"value": nstate / t_e2e, "unit": UNIT, "ms_per_step": t_e2e * 1e3,
                    # busy time of each stage summed over the field groups; the copies of one group run on a copy
                    # stream under the compute of its neighbours, so the sum exceeds the wall time of the call
                    "breakdown_ms": {"h2d": rep.t_h2d * 1e3, "estimation": float(rep.t_estimation.sum()) * 1e3,
                                     "analysis": float(rep.t_analysis.sum()) * 1e3, "d2h": rep.t_d2h * 1e3,
                                     "call_wall": rep.t_total * 1e3},
                    "pipelined": ("5 groups of fields: H2D of group g+1 and D2H of group g-1 overlap the kernels of group g" if world == 1
                                  else "rank 0 uploads, scatters the slabs, all ranks compute, all-gather, rank 0 downloads"),
                    "h2d_bytes_per_step": int(w.X.nbytes + w.Ys.nbytes + w.r_diag.nbytes),
                    "d2h_bytes_per_step": int(w.X.nbytes),
                    "api": ("assimilate_parallel" if world == 1 else "assimilate_parallel_sharded") +
                           "(EnsembleState, ObservationNetwork, AssimilationConfig, GridGeometry, Ys=)",
                    "inputs": "page-locked host arrays"},
            "e2e_pageable": {"value": nstate / t_e2e_pageable, "unit": UNIT, "ms_per_step": t_e2e_pageable * 1e3,
                             "inputs": "ordinary (pageable) numpy arrays: a staged copy blocks the host, so the fields go in 12 groups and the upload of group g + 1 is issued right after the kernels of group g and is staged while they run"},
            "gpu_launches": int(launches),
            "clocks": summarize_clocks(samples),
            "parity_vs_cpu_sample": parity, "parity_gate": parity_gate, "clamped_pivots": int(clamped),
            "rank_memory_fraction": shard.memory_fraction(),
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
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-execute under torch.distributed.run (what the driver does itself for N > 1)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.execv(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
                                  "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:])
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}: launch with --nproc-per-node {args.gpus}")
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")          # the communicator / transport log goes to stderr
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_b200(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
