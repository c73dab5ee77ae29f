"""Scan-kernel ablation on the SIFT1M-shaped index (BASELINE configs[1]): search 10k
queries (k=10) and time the scan phase under the SIVF_OPT_DEBUG switches of k_scan_tc
(bit0 skip slow path, bit1 skip fast path, bit2 skip MMAs, bit3 skip B copies, bit4 skip
A loads, bit5 skip TMEM loads, bit6 keep the previous search's per-query bounds) and the
work-order options.  Results are NOT correct under the switches: timing only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_11808_b200 as S
from datagen import Generator, sift_shape

N, D, NL, NQ = 1_000_000, 128, 1024, 10_000
gen = Generator(sift_shape(seed=0x51F7))
ix = S.Index(D, NL, N, S.num_slabs_for(N, NL), max_batch=65536, max_queries=NQ, max_k=32, max_nprobe=128,
             max_train=262144, seed=1)
ix.train(torch.from_numpy(gen.train(262144)).cuda(), niter=10)
X = torch.from_numpy(gen.range(0, N)).cuda()
ids = torch.arange(N, device="cuda")
for b in range(0, N, 65536):
    ix.insert(ids[b:b + 65536], X[b:b + 65536])
del X
Q = torch.from_numpy(gen.queries(0, NQ)).cuda()
configs = os.environ.get("CONFIGS", "0,1,3,35,39,43,47,63,64,16").split(",")
ix.set_option(9, int(os.environ.get("SEEDLIST", "0")))  # SIVF_OPT_SEED_LIST (library default 0)
splits = [int(v) for v in os.environ.get("SPLITS", "1").split(",")]
stages = [int(v) for v in os.environ.get("STAGES", "0").split(",")]
seeds = [int(v) for v in os.environ.get("SEEDS", "0").split(",")]
for npb in [int(v) for v in os.environ.get("NPROBES", "32,16").split(",")]:
    for split in splits:
      for nstg in stages:
       ix.set_option(98, nstg)
       for sd in seeds:
        ix.set_option(S.OPT_SEED_SLABS, sd)
        for c in configs:
            dbg = int(c)
            ix.set_option(S.OPT_RANK_SPLIT, split)
            ix.set_option(99, 0)
            ix.search(Q, 10, npb)  # bounds of an ordinary search (bit 6 keeps them)
            ix.set_option(99, dbg)
            ix.search(Q, 10, npb)
            torch.cuda.synchronize()
            ix.profile(True)
            ix.profile_read()
            for _ in range(5):
                ix.search(Q, 10, npb)
            torch.cuda.synchronize()
            p = ix.profile_read()
            ix.profile(False)
            t = {k: v[0] / v[1] for k, v in p.items() if v[1]}
            print(f"nprobe {npb} split {split} stages {nstg} seed {sd} dbg {dbg:3d}: scan {t['scan']:.4f} ms  "
                  f"coarse {t['coarse']:.4f} invmap {t['invmap']:.4f} merge {t['merge']:.4f}", flush=True)
