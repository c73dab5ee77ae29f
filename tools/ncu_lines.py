#!/usr/bin/env python
"""Per-CUDA-source-line stall samples and executed warp instructions of one kernel.
  python tools/ncu_lines.py <rep> [top=40] [kernel-substring]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
start = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[start]
si, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")


def iv(x):
    try:
        return int(x)
    except ValueError:
        return 0


agg = collections.defaultdict(lambda: [0, 0])
line = None
for r in rows[start + 1:]:
    if len(r) < len(h) or r[0] == "Line No":
        continue
    if r[0].strip():
        line = (int(r[0]), r[1])
    a = agg[line]
    a[0] += iv(r[si])
    a[1] += iv(r[ei])
tot = sum(a[0] for a in agg.values()) or 1
tins = sum(a[1] for a in agg.values())
print("samples", tot, "warp instructions", tins)
for k, a in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100 * a[0] / tot:5.1f}% ex={a[1]:>10} L{k[0]:>4} {k[1].strip()[:100]}")
