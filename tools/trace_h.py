"""(prof builds: per-role clock totals of k_scan_tc blocks 0-1 are printed by the kernel)
Config H shard on one GPU (timing only): shard 0 of a G-way id sharding of the 100M x 128
SIFT-shaped set (n/G vectors, nlist 16384 trained on a 1M sample), 10k queries, k = 10,
nprobe 32: search phases (coarse, invmap, scan, merge), and the probe-slice coarse of the
query-sharded path.  G from env (default 8)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_11808_b200 as S
from datagen import TRAIN_BASE, QUERY_BASE, DeviceGenerator, sift_shape

G = int(os.environ.get("G", "8"))
N_TOTAL, NLH, DIM, NQ = 100_000_000, 16384, 128, 10_000
gen = DeviceGenerator(sift_shape(seed=0x100A))
local_n = (N_TOTAL + G - 1) // G
ix = S.Index(DIM, NLH, N_TOTAL + 64, S.num_slabs_for(local_n + 1, NLH), max_batch=1 << 20, max_queries=NQ,
             max_k=10, max_nprobe=128, max_train=1 << 20, shard_rank=0, shard_count=G, seed=0x100A)
Xt = torch.empty(1 << 20, DIM, device="cuda")
gen.range_into(Xt, TRAIN_BASE, 1)
ix.train(Xt, niter=int(os.environ.get("NITER", "10")))
del Xt
B = 1 << 20
Xb = torch.empty(B, DIM, device="cuda")
for j0 in range(0, local_n, B):
    nb = min(B, local_n - j0)
    gen.range_into(Xb[:nb], j0 * G, G)
    ix.insert(G * torch.arange(j0, j0 + nb, device="cuda", dtype=torch.int64), Xb[:nb])
del Xb
Q = torch.empty(NQ, DIM, device="cuda")
gen.range_into(Q, QUERY_BASE, 1)
for npb in (32,):
    for _ in range(2):
        ix.search(Q, 10, npb)
    ix.profile(True)
    ix.profile_read()
    for _ in range(3):
        ix.search(Q, 10, npb)
    torch.cuda.synchronize()
    p = ix.profile_read()
    ix.profile(False)
    print(f"G={G} local_n={local_n} nprobe {npb}:", {k: round(v[0] / 3, 4) for k, v in p.items() if v[1]}, flush=True)
