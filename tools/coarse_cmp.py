"""Coarse-step paths on the SIFT1M-shaped index (timing only): the stored-matrix +
per-row selection path (SIVF_OPT_COARSE_SELECT 1) against the fused two-pass epilogue
(0, N-tiles split over CTAs for small row counts): assign phase of 10k / 64k insert
batches, coarse phase of 10k / 1k query batches at nprobe 8 and 32."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_11808_b200 as S
from datagen import Generator, sift_shape

N, D, NL = 1_000_000, 128, int(os.environ.get("NL", "1024"))
gen = Generator(sift_shape(seed=0x51F7))
ix = S.Index(D, NL, N + 200_000, S.num_slabs_for(N + 200_000, NL), max_batch=65536, max_queries=10_000, max_k=32,
             max_nprobe=128, max_train=262144, seed=1)
ix.train(torch.from_numpy(gen.train(262144)).cuda(), niter=10)
X = torch.from_numpy(gen.range(0, N)).cuda()
ids = torch.arange(N, device="cuda")
for b in range(0, N, 65536):
    ix.insert(ids[b:b + 65536], X[b:b + 65536])
Q = torch.from_numpy(gen.queries(0, 10_000)).cuda()
Xn = torch.from_numpy(gen.range(N, 65536)).cuda()
nid = torch.arange(N, N + 65536, device="cuda")
for sel in (1, 0):
    ix.set_option(S.OPT_COARSE_SELECT, sel)
    res = {}
    for nb in (10_000, 65536):
        ts = []
        for r in range(4):
            ix.profile(True)
            ix.profile_read()
            ix.insert(nid[:nb], Xn[:nb])
            torch.cuda.synchronize()
            p = ix.profile_read()
            ix.profile(False)
            ix.delete(nid[:nb])
            ix.reclaim()
            if r:
                ts.append(p["assign"][0])
        res[f"assign{nb}"] = round(statistics.median(ts), 4)
    for nq in (10_000, 1000):
        for npb in (8, 32):
            ix.search(Q[:nq], 10, npb)
            ix.profile(True)
            ix.profile_read()
            for _ in range(3):
                ix.search(Q[:nq], 10, npb)
            torch.cuda.synchronize()
            p = ix.profile_read()
            ix.profile(False)
            res[f"coarse{nq}_np{npb}"] = round(p["coarse"][0] / 3, 4)
    print("COARSE_SELECT", sel, res, flush=True)
