"""Warp-stall samples of an ncu --set full capture aggregated per source line
(file:line via nvdisasm -g of the kernel's cubin).  Tools only.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL.cubin [top]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys

rep, cubin = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
ia, iss = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
base = int(data[0][ia], 16)
cur = None
off2line = {}
for ln in subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1), int(m.group(2)))
        continue
    m2 = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m2 and cur is not None:
        off2line[int(m2.group(1), 16)] = cur
agg, ex = collections.Counter(), collections.Counter()
for r in data:
    key = off2line.get(int(r[ia], 16) - base, ("?", 0))
    agg[key] += int(r[iss])
    ex[key] += int(r[iex])
files = {}
tot = sum(agg.values())
print(f"total stall samples {tot}")
for (f, l), c in agg.most_common(top):
    if f not in files and os.path.exists(f):
        files[f] = open(f).read().split("\n")
    src = files.get(f, [])
    text = src[l - 1].strip()[:80] if 0 < l <= len(src) else "?"
    print(f"{c:6d} {100 * c / tot:5.1f}% {os.path.basename(f)}:{l:<4d} ex={ex[(f, l)]:9d}  {text}")
