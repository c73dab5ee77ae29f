"""Scan-kernel experiment: 1M SIFT-shaped index, time search phases (used with SIVF_LIB_PATH variants)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_11808_b200 as S
from datagen import Generator, sift_shape
N, D, NL, NQ = 1_000_000, 128, 1024, 10_000
gen = Generator(sift_shape(seed=0x51F7))
ix = S.Index(D, NL, N, S.num_slabs_for(N, NL), max_batch=65536, max_queries=NQ, max_k=32, max_nprobe=128, max_train=262144, seed=1)
ix.train(torch.from_numpy(gen.train(262144)).cuda(), niter=10)
X = torch.from_numpy(gen.range(0, N)).cuda()
ids = torch.arange(N, device="cuda")
for b in range(0, N, 65536):
    ix.insert(ids[b:b+65536], X[b:b+65536])
Q = torch.from_numpy(gen.queries(0, NQ)).cuda()
two = int(os.environ.get("TWO_PHASE", "0"))
ix.set_option(2, two)
ix.set_option(99, int(os.environ.get("DBG", "0")))
ix.set_option(5, int(os.environ.get("SPLIT", "1")))
seeds = [int(v) for v in os.environ.get("SEEDS", "8").split(",")]
for seed, npb in [(sd, npb) for sd in seeds for npb in (8, 32)]:
    ix.set_option(4, seed)
    ix.search(Q, 10, npb); torch.cuda.synchronize()
    ix.profile(True); ix.profile_read()
    for _ in range(5): ix.search(Q, 10, npb)
    torch.cuda.synchronize()
    p = ix.profile_read(); ix.profile(False)
    tot = {k: v[0] / 5 for k, v in p.items() if v[1]}
    print(os.path.basename(S.LIB_PATH), "two" if two else "one", "nprobe", npb, "seed", seed, {k: round(v, 4) for k, v in tot.items()}, flush=True)
