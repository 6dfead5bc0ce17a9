"""Attribute an ncu report's per-instruction counters to CUDA source lines (needs -lineinfo).

usage: ncu_lines.py <report.ncu-rep> <kernel-regex> [top]
Joins `ncu --page source --csv` (SASS rows, in address order) with `nvdisasm -g` line info of the
same kernel extracted from libenkfmc.so.
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
kname = rows[0][1]
hdr = rows[1]
ci, si, ai = hdr.index("Instructions Executed"), hdr.index("# Samples"), hdr.index("Address")
mangled = None
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_1606_00807_b200", "libenkfmc.so")], cwd=td,
                   capture_output=True)
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(td, "kernels.sm_100a.cubin")], capture_output=True, text=True).stdout
base_name = re.sub(r"^void ", "", kname).split("(")[0].split("<")[0]
targs = re.findall(r"\(int\)(\d+)", kname)
sections = re.split(r"\n\t\.section\t\.text\.", dis)
sec = None
for s in sections[1:]:
    name = s.split(",")[0]
    if base_name in name and all(f"Li{t}E" in name for t in targs) and name.count("Li") == len(targs):
        sec = s
        break
assert sec is not None, kname
addr2line, addr2fn, cur, fn = {}, {}, None, "(kernel body)"
CSRC = os.path.join(ROOT, "paper_1606_00807_b200", "csrc")
for ln in sec.split("\n"):
    m = re.search(r'//## File "(.*?)", line (\d+)', ln)
    if m:   # own sources: (file, line); inlined CUDA header code (shuffles, math) keeps its header name
        own = os.path.dirname(m.group(1)) == CSRC
        cur = (os.path.basename(m.group(1)), int(m.group(2))) if own else os.path.basename(m.group(1)) + ":" + m.group(2)
        continue
    m = re.match(r"\s*(_Z\w+|\$\w+\$\w+):\s*$", ln)
    if m and not m.group(1).startswith(".L"):
        fn = m.group(1)
        continue
    m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+\S", ln)
    if m:
        addr2line[int(m.group(1), 16)] = cur
        addr2fn[int(m.group(1), 16)] = fn
base = int(rows[2][ai], 16)
agg, fagg = {}, {}
for r in rows[2:]:
    try:
        off, n, s = int(r[ai], 16) - base, int(r[ci]), int(r[si])
    except (ValueError, IndexError):
        continue
    a = agg.setdefault(addr2line.get(off), [0, 0])
    a[0] += n
    a[1] += s
    a = fagg.setdefault(addr2fn.get(off), [0, 0])
    a[0] += n
    a[1] += s
srcs = {}
def text_of(l):
    if isinstance(l, tuple):
        if l[0] not in srcs:
            srcs[l[0]] = open(os.path.join(CSRC, l[0])).read().split("\n")
        return f"{l[0]}:{l[1]}: " + srcs[l[0]][l[1] - 1].strip()[:100]
    return "(CUDA header) " + l if l else "?"
tot, ts = sum(a[0] for a in agg.values()), sum(a[1] for a in agg.values())
print(f"{kname}: {tot:.4g} warp instructions, {ts} samples")
print("by function:")
for f, a in sorted(fagg.items(), key=lambda kv: -kv[1][0]):
    try:
        dem = subprocess.run(["cu++filt", f], capture_output=True, text=True).stdout.strip()
        dem = re.sub(r"\[clone |\]$", "", dem)
        dem = re.sub(r"void regress_\w+<\(int\)\d+>\(RegressParams\)::", "", dem)[:110]
    except OSError:
        dem = f
    print("%5.1f%% inst %5.1f%% samp  %s" % (100 * a[0] / tot, 100 * a[1] / max(ts, 1), dem))
print("by line:")
for l, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print("%5.1f%% inst %5.1f%% samp  %s" % (100 * a[0] / tot, 100 * a[1] / max(ts, 1), text_of(l)))
