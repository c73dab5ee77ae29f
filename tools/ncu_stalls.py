#!/usr/bin/env python
"""Top warp-stall SASS sites of one kernel in an ncu report.
  python tools/ncu_stalls.py <rep> <kernel-name-substring> [top=20]"""
import csv
import io
import subprocess
import sys

rep, sub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
blocks, cur = [], None
for x in r:
    if x and x[0] == "Kernel Name":
        cur = {"name": x[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(x)
b = next(b for b in blocks if sub in b["name"])
h = b["rows"][0]
si, ni, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
rows = [x for x in b["rows"][1:] if len(x) == len(h)]
tot = sum(int(x[si]) for x in rows if x[si].isdigit()) or 1
print(b["name"][:100], "| samples", tot, "| warp instructions", sum(int(x[ei]) for x in rows if x[ei].isdigit()))
for x in sorted(rows, key=lambda x: -int(x[si] or 0))[:top]:
    print(f"{100 * int(x[si] or 0) / tot:5.1f}%  {x[ni].strip()[:100]}")
