"""Per-CUDA-line totals of an ncu SASS source page: stall samples and executed
instructions, mapped through nvdisasm line info of the same cubin.

    python scripts/ncu_lines.py report.ncu-rep kernel.cubin <mangled-substring> [top]
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, cubin, fsub = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
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
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m and cur is not None:
        line_of[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, iss, iex = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = [r for r in rows[2:] if len(r) == len(h)]
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
    txt = src[L - 1].strip()[:90] if src and 0 < L <= len(src) else ""
    print(f"{L:5d} {100 * s / tot_s:6.2f}% samp {100 * i / max(tot_i, 1):6.2f}% inst  {txt}")
