#!/usr/bin/env python
"""Microbenchmark of the coarse step (assignment of a 10k batch, probe selection
of 10k queries) on SIFT-/GIST-shaped data: tensor-core path vs exact CUDA-core
path, CUDA-event timed on the library's phase timers.

  python tools/prof_coarse.py [--dim 128] [--nlist 1024] [--nprobe 32] [--reps 10]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_11808_b200 as S  # noqa: E402
from datagen import Generator, gist_shape, sift_shape  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dim", type=int, default=128)
ap.add_argument("--nlist", type=int, default=1024)
ap.add_argument("--nprobe", type=int, default=32)
ap.add_argument("--n", type=int, default=10000)
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()

shape = sift_shape() if args.dim == 128 else gist_shape(dim=args.dim)
gen = Generator(shape)
X = torch.from_numpy(gen.range(0, args.n * 4)).cuda()
Q = torch.from_numpy(gen.queries(0, args.n)).cuda()
rng = np.random.default_rng(0)
C = X[torch.from_numpy(rng.choice(args.n * 4, args.nlist, replace=False)).cuda()].contiguous()
for tc in (1, 0):
    ix = S.Index(args.dim, args.nlist, args.n * (args.reps + 2), S.num_slabs_for(args.n * (args.reps + 2), args.nlist),
                 max_batch=args.n, max_queries=args.n, max_k=10, max_nprobe=args.nprobe)
    ix.set_option(S.OPT_TC_COARSE, tc)
    ix.set_centroids(C)
    ids = torch.arange(args.n * (args.reps + 2), device="cuda")
    ix.insert(ids[: args.n], X[: args.n])
    ix.search(Q, 10, args.nprobe)
    torch.cuda.synchronize()
    ix.profile(True)
    ix.profile_read()
    for r in range(args.reps):
        ix.insert(ids[(r + 1) * args.n:(r + 2) * args.n], X[(r % 4) * args.n:((r % 4) + 1) * args.n])
        ix.search(Q, 10, args.nprobe)
    torch.cuda.synchronize()
    p = ix.profile_read()
    print(f"tc_coarse={tc} dim={args.dim} nlist={args.nlist} nprobe={args.nprobe}: "
          f"assign {p['assign'][0] / p['assign'][1] * 1e3:.1f} us, coarse {p['coarse'][0] / p['coarse'][1] * 1e3:.1f} us, "
          f"scan {p['scan'][0] / p['scan'][1] * 1e3:.1f} us")
