"""Run only the H leg of bench.py (for development): python tools/h_only.py N"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2601_11808_b200 as S
log = lambda m: print(f"[h] {m}", file=sys.stderr, flush=True)
t0 = time.time()
r = bench.leg_h(S, torch.device("cuda", 0), log, 1, 0, None, int(sys.argv[1]))
print(json.dumps(r), flush=True)
print("wall", time.time() - t0, file=sys.stderr)
