"""Regenerates the committed summaries under profiles/ from one gpurun pass:
gpurun_out/b_plain.json (bench without ncu), launches.csv (ncu launch list of the same command) and
r1_bench_full.ncu-rep (ncu --set full of the bench launch of the four main kernels)."""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
plain = json.load(open(os.path.join(G, "b_plain.json")))
st, step = plain["stage_ms"], plain["ms_per_step"]

# ---- launch list -> shares -----------------------------------------------------------------
rows = list(csv.reader(open(os.path.join(G, "launches.csv"))))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h, data = rows[hi], rows[hi + 1:]
kn, mv, mn = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
agg = collections.OrderedDict()
for r in data:
    if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
        continue
    agg.setdefault(r[kn].split("(")[0].replace("void ", ""), []).append(float(r[mv].replace(",", "")) / 1e6)
full = {k: v[:5] for k, v in agg.items() if k != "fp64_peak_kernel"}
tot = sum(sum(v) / len(v) for v in full.values())
ev = {"center_rows_kernel": st["center"], "regress_qr_mma_kernel<10>": st["regress_qr"], "regress_solve_kernel<2>": st["regress_solve"]}
out = ["ncu --metrics gpu__time_duration.sum --clock-control none -c 400, `python bench.py --steps 2 --warmup 3 --no-cpu-baseline` (cfg3, 29 fields).", "",
       "The command launches every kernel 25 times: 5 device-resident steps (3 warm-up + 2 timed) with all 29 fields per launch, then 5 calls of the "
       "host path, each split into 4 groups of fields (20 smaller launches).  The table uses the 5 full-size launches; per-launch times under ncu are "
       "serialised and cold-cache, so only the shares are compared with the CUDA-event shares of the same command run without ncu "
       f"({step:.2f} ms/step; K2a {st['regress_qr']:.2f}, K2b {st['regress_solve']:.2f}, K3 {st['local_solve']:.2f}, K0 {st['center']:.2f} ms).", "",
       "| kernel | full-size launches | avg ms (ncu) | share of step (ncu) | share of step (CUDA events, no ncu) |", "|---|---|---|---|---|"]
k3 = sum(sum(v) / len(v) for k, v in full.items() if k in ("assemble_band_tile_kernel", "local_solve_kernel"))
for k, v in full.items():
    a = sum(v) / len(v)
    if k in ev:
        es = f"{100 * ev[k] / step:.1f}%"
    elif k in ("assemble_band_tile_kernel", "local_solve_kernel"):
        es = f"K3a+K3b: {100 * st['local_solve'] / step:.1f}%"
    else:
        es = "(inside K2's event bracket)"
    out.append(f"| {k} | {len(v)} | {a:.3f} | {100 * a / tot:.1f}% | {es} |")
out += ["", f"ncu sum of the step: {tot:.2f} ms; K3a + K3b under ncu: {k3:.2f} ms ({100 * k3 / tot:.1f}%)."]
open(os.path.join(P, "r1_launch_shares_bench_cfg3.md"), "w").write("\n".join(out) + "\n")
subprocess.run(["cp", os.path.join(G, "launches.csv"), os.path.join(P, "r1_ncu_launch_list_bench_cfg3.csv")], check=True)

# ---- full capture -> metric table ---------------------------------------------------------------
M = ("gpu__time_duration.sum,launch__registers_per_thread,launch__block_size,launch__grid_size,launch__shared_mem_per_block_dynamic,"
     "sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__inst_executed.avg.per_cycle_elapsed,"
     "smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,"
     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,"
     "dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,"
     + ",".join(f"smsp__average_warps_issue_stalled_{x}_per_issue_active.ratio" for x in
                ("wait", "short_scoreboard", "long_scoreboard", "barrier", "math_pipe_throttle", "no_instruction")))
rep = os.path.join(G, "r1_bench_full.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", M], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
keep = [i for i, c in enumerate(rr[0]) if c == "Kernel Name" or "__" in c]
with open(os.path.join(P, "r1_ncu_full_k2_bench_launch.csv"), "w") as f:
    f.write("# ncu --set full --clock-control none -k regex:regress_solve|regress_qr|assemble_band|local_solve -s 12 -c 4, "
            "python bench.py --steps 1 --warmup 3 --no-cpu-baseline (cfg3, all 29 fields: the bench launch)\n")
    w = csv.writer(f)
    for r in rr:
        w.writerow([r[i] for i in keep])
hh = [rr[0][i] for i in keep]
for r in rr[2:]:
    d = dict(zip(hh, [r[i] for i in keep]))
    print(d["Kernel Name"][:34], "ms", d["gpu__time_duration.sum"], "dram GB r/w", d["dram__bytes_read.sum"], d["dram__bytes_write.sum"],
          "issue %", d["smsp__issue_active.avg.pct_of_peak_sustained_active"][:5])

# ---- hot lines ------------------------------------------------------------------------------------
out = ["Source lines with the most stall samples (ncu --set full --import-source on, the bench launch of each kernel, cfg3 29 fields;",
       "`tools/ncu_lines.py` joins the SASS-level counters with nvdisasm line info; code inlined from CUDA headers keeps the header's name).", ""]
for k in ("regress_qr_mma", "regress_solve", "local_solve", "assemble_band_tile"):
    txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, k, "400"], capture_output=True, text=True).stdout
    lines, head = [], None
    for ln in txt.split("\n"):
        if head is None:
            head = ln.strip()
        m = re.match(r"\s*([\d.]+)% inst\s+([\d.]+)% samp\s+L(\d+): (.*)", ln)
        if m:
            lines.append((float(m.group(2)), float(m.group(1)), int(m.group(3)), m.group(4).strip()[:120]))
    lines.sort(reverse=True)
    out += ["## " + head, "", "| stall samples | instructions | line | source |", "|---|---|---|---|"]
    out += [f"| {a:.1f}% | {b:.1f}% | {c or ''} | `{d.replace('|', chr(92) + '|')}` |" for a, b, c, d in lines[:14]]
    out.append("")
open(os.path.join(P, "r1_hot_lines_bench_cfg3.md"), "w").write("\n".join(out))
