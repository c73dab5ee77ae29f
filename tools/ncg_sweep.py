"""KP=0 coarse GEMM: N-tile split factor sweep (SIVF_OPT_DEBUG bits 16-18), timing only:
assign phase of a 10k insert batch and coarse phase of 10k queries on the SIFT1M index."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_11808_b200 as S
from datagen import Generator, sift_shape

N, D, NL = 1_000_000, 128, 1024
gen = Generator(sift_shape(seed=0x51F7))
ix = S.Index(D, NL, N + 200_000, S.num_slabs_for(N + 200_000, NL), max_batch=65536, max_queries=10_000, max_k=32,
             max_nprobe=128, max_train=262144, seed=1)
ix.train(torch.from_numpy(gen.train(262144)).cuda(), niter=10)
X = torch.from_numpy(gen.range(0, N)).cuda()
ids = torch.arange(N, device="cuda")
for b in range(0, N, 65536):
    ix.insert(ids[b:b + 65536], X[b:b + 65536])
Q = torch.from_numpy(gen.queries(0, 10_000)).cuda()
Xn = torch.from_numpy(gen.range(N, 10_000)).cuda()
nid = torch.arange(N, N + 10_000, device="cuda")
for ncg in (0, 1, 2, 3, 4):
    ix.set_option(99, ncg << 16)
    a = []
    for r in range(5):
        ix.profile(True)
        ix.profile_read()
        ix.insert(nid, Xn)
        torch.cuda.synchronize()
        p = ix.profile_read()
        ix.profile(False)
        ix.delete(nid)
        ix.reclaim()
        if r:
            a.append(p["assign"][0])
    ix.search(Q, 10, 32)
    ix.profile(True)
    ix.profile_read()
    for _ in range(5):
        ix.search(Q, 10, 32)
    torch.cuda.synchronize()
    p = ix.profile_read()
    ix.profile(False)
    print(f"ncg {ncg or 'auto'}: assign10k {statistics.median(a):.4f} ms  coarse10k {p['coarse'][0] / 5:.4f} ms", flush=True)
