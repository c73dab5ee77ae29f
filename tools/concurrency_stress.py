"""SPEC publication suite repeated: 8 writer views x 10k unique ids with id-derived
payloads, 4 reader views at nprobe = nlist, 12 streams; every run checks no torn payload,
live = 80k, every id retrievable, no invariant violation (tests/test_gpu_concurrent.py).
  python tools/concurrency_stress.py [runs] [writers] [per_writer]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.test_gpu_concurrent import _publication_run  # noqa: E402

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 100
nw = int(sys.argv[2]) if len(sys.argv) > 2 else 8
pw = int(sys.argv[3]) if len(sys.argv) > 3 else 10_000
t0 = time.time()
hits = 0
for r in range(runs):
    hits += _publication_run(1000 + r, n_writers=nw, per_writer=pw)
print(f"{runs} runs x ({nw} writers x {pw} ids, 4 readers): all checks passed; {hits} concurrent search hits "
      f"verified against their payloads; {time.time() - t0:.1f} s")
