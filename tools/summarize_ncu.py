#!/usr/bin/env python
"""Summarise gpurun_out/ ncu artefacts into profiles/ (tracked).

  python tools/summarize_ncu.py launches <launches.csv> <out.txt> [--step-kernels N]
  python tools/summarize_ncu.py full <report.ncu-rep> <out.txt>

`launches`: per-kernel launch counts and summed gpu__time_duration from an
`ncu --metrics gpu__time_duration.sum` launch list (cold-cache, serialised:
compare shares, not absolutes).  `full`: the key counters of one
`ncu --set full` capture (duration, DRAM bytes, pipe utilisations, occupancy,
top SASS stall sites).
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys


def launches(path, out, window=None):
    """window = (kernel, first, last): keep launches from the `first`-th launch
    of `kernel` up to (excluding) its `last`-th launch (1-based), e.g. the
    timed steps of a bench run."""
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    if window:
        kn, a, b = window
        idx = [i for i, x in enumerate(data) if kn in x["Kernel Name"]]
        lo = idx[a - 1]
        hi = idx[b - 1] if b - 1 < len(idx) else len(data)
        data = data[lo:hi]
    agg = collections.OrderedDict()
    for x in data:
        name = x["Kernel Name"].split("(")[0].replace("void ", "").replace("sivf::<unnamed>::", "")
        unit = x["Metric Unit"]
        v = float(x["Metric Value"]) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                                        "msecond": 1e3}[unit]
        a = agg.setdefault(name, [0, 0.0, []])
        a[0] += 1
        a[1] += v
        a[2].append(v)
    tot = sum(a[1] for a in agg.values())
    lines = [f"# ncu launch list: {path}" + (f" window {window}" if window else ""), f"# {len(data)} launches, {tot:.1f} us total (cold-cache, serialised)",
             f"{'launches':>8} {'total_us':>10} {'mean_us':>9} {'share':>6}  kernel"]
    for n, (c, t, _) in sorted(agg.items(), key=lambda z: -z[1][1]):
        lines.append(f"{c:8d} {t:10.1f} {t / c:9.2f} {100 * t / tot:5.1f}%  {n}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:20]))


KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tc.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size",
    "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum",
]


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, units = r[0], r[1]
    lines = [f"# ncu --set full: {rep}"]
    for row in r[2:]:
        if len(row) != len(hdr):
            continue
        name = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines.append(f"## kernel: {name[:120]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"{k:90s} {row[i]:>16s} {units[i]}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    s = list(csv.reader(io.StringIO(src)))
    if len(s) > 2 and "Warp Stall Sampling (All Samples)" in s[1]:
        h = s[1]
        i, j = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
        rows = [(int(x[i]), x[j].strip()) for x in s[2:] if len(x) == len(h) and x[i].isdigit()]
        tot = sum(a for a, _ in rows) or 1
        lines.append(f"## top SASS stall sites (all samples, total {tot})")
        for a, b in sorted(rows, reverse=True)[:25]:
            lines.append(f"{100 * a / tot:5.1f}%  {b}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    if mode == "launches":
        w = None
        if len(sys.argv) > 4:  # kernel:first:last
            kn, a, b = sys.argv[4].split(":")
            w = (kn, int(a), int(b))
        launches(src, dst, w)
    else:
        full(src, dst)
