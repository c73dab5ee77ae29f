#!/usr/bin/env python
"""Stall-reason breakdown per CUDA source line in a line range of one file.
  python tools/ncu_range.py <rep> <file-substring> <lo> <hi>"""
import csv
import io
import subprocess
import sys

rep, fsub, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file = None
h = None
agg = {}
line = None
for r in rows:
    if r and r[0] in ("File Name", "File Path"):
        cur_file = r[1]
        continue
    if r and r[0] == "Line No":
        h = r
        continue
    if h is None or len(r) < len(h):
        continue
    if r[0].strip():
        line = int(r[0])
        src = r[1]
    if cur_file is None or fsub not in cur_file or not (lo <= line <= hi):
        continue
    a = agg.setdefault(line, {"src": src})
    for i, name in enumerate(h):
        if name.startswith("stall_") and "Not Issued" not in name or name in ("Instructions Executed",
                                                                             "Warp Stall Sampling (All Samples)"):
            try:
                a[name] = a.get(name, 0) + int(r[i])
            except ValueError:
                pass
for ln in sorted(agg):
    a = agg[ln]
    st = sorted(((v, k) for k, v in a.items() if k.startswith("stall_") and v), reverse=True)[:4]
    print(f"L{ln:4d} samp={a.get('Warp Stall Sampling (All Samples)', 0):6d} ex={a.get('Instructions Executed', 0):9d} "
          f"{' '.join(f'{k[6:]}={v}' for v, k in st):60s} {a['src'].strip()[:60]}")
