"""Per-CUDA-line totals of an ncu SASS source page: stall samples and executed
instructions, mapped through nvdisasm line info of the same cubin.

    python scripts/ncu_lines.py report.ncu-rep kernel.cubin <mangled-substring> [top] [source.cu]
    NCU_LINES_INLINE=1: key lines by "line@call-site line" (nvdisasm -gi)
"""
import csv
import io
import os
import re
import subprocess
import sys
from collections import defaultdict

rep, cubin, fsub = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
INLINE = bool(os.environ.get("NCU_LINES_INLINE"))
SRC_NAME = os.path.basename(sys.argv[5]) if len(sys.argv) > 5 else ".cu"
dis = subprocess.run(["nvdisasm", "-gi" if INLINE else "-g", "-c", cubin], capture_output=True, text=True).stdout
line_of = {}
cur = None
infn = False
for ln in dis.splitlines():
    if ln.startswith("\t.section\t.text.") or ln.startswith(".section .text.") or ".text." in ln and "section" in ln:
        infn = fsub in ln
        continue
    if not infn:
        continue
    m = re.search(r'line (\d+)', ln)
    if "//##" in ln and m:
        cur = int(m.group(1))
        # with -gi: "line N inlined at "<file>", line M" -> key "N@M" (call site in this file)
        mi = re.search(r'line (\d+) inlined at "([^"]+)", line (\d+)', ln)
        if mi and INLINE:
            cur = f"{mi.group(1)}@{mi.group(3)}" if mi.group(2).endswith(SRC_NAME) else f"{mi.group(1)}@ext"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m and cur is not None:
        line_of[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# one section per profiled kernel ("Kernel Name" row, header row, SASS rows): the first
sec_end = next((x for x in range(2, len(rows)) if rows[x] and rows[x][0] == "Kernel Name"), len(rows))
h = rows[1]
ia, iss, iex = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = [r for r in rows[2:sec_end] if len(r) == len(h)]
base = min(int(r[ia], 16) for r in data)
agg = defaultdict(lambda: [0, 0])
tot_s = tot_i = 0
for r in data:
    off = int(r[ia], 16) - base
    L = line_of.get(off, -1)
    s, i = int(r[iss] or 0), int(r[iex] or 0)
    agg[L][0] += s
    agg[L][1] += i
    tot_s += s
    tot_i += i
src = open(sys.argv[5]).read().splitlines() if len(sys.argv) > 5 else None
print(f"mapped {len(line_of)} SASS offsets; total samples {tot_s}, warp instructions {tot_i}")
for L, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    ln = int(str(L).split("@")[0])
    txt = src[ln - 1].strip()[:80] if src and 0 < ln <= len(src) else ""
    print(f"{str(L):>9} {100 * s / tot_s:6.2f}% samp {100 * i / max(tot_i, 1):6.2f}% inst  {txt}")
