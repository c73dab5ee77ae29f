"""Per-kernel Blackwell opcode summary of the built libsivf.so (cuobjdump -sass):
counts of the tcgen05 / TMA / bulk-copy / mbarrier instructions that prove the
kernels use the 5th-generation tensor cores, TMEM and the async copy engines.
  python tools/sass_summary.py [lib] > profiles/<round>_sass_opcodes.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2601_11808_b200/lib/libsivf.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "UTMACCTL",
        "SYNCS.EXCH", "SYNCS.ARRIVE", "SYNCS.PHASECHK", "FFMA", "FMNMX", "HMMA", "IMMA", "LDGSTS"]
cur, counts = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if m:
        op = m.group(1)
        for k in KEYS:
            if op.startswith(k):
                counts[cur][k] += 1
demangle = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.split("\n")
print(f"# cuobjdump -sass {lib}: per-kernel counts of selected opcodes (static instructions)")
print("# UTCHMMA = tcgen05.mma, LDTM/STTM = tcgen05.ld/st (TMEM), UTMALDG/UTMASTG = TMA tensor load/store,")
print("# UBLKCP = cp.async.bulk, SYNCS.* = mbarrier ops, UTCBAR = tcgen05.commit")
for (name, c), dn in zip(counts.items(), demangle):
    if not c:
        continue
    short = re.sub(r"\(.*", "", dn.replace("sivf::(anonymous namespace)::", "")).strip()
    print(f"{short:48s} " + " ".join(f"{k}={v}" for k, v in c.items() if k not in ("FFMA", "FMNMX") or v))
