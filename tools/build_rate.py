"""Bulk-build rate of the SIFT1M-shaped index (bench.py's build): 1M inserts in 64k batches,
device-timed, with the per-phase split (assign vs the rest of the insert)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_11808_b200 as S
from datagen import Generator, sift_shape
N, D, NL = 1_000_000, 128, 1024
B = int(os.environ.get("BATCH", "65536"))
gen = Generator(sift_shape(seed=0x51F7))
X = torch.from_numpy(gen.range(0, N)).cuda()
ids = torch.arange(N, device="cuda")
for rep in range(2):
    ix = S.Index(D, NL, N, S.num_slabs_for(N, NL), max_batch=max(B, 65536), max_queries=16, max_k=16,
                 max_train=262144, seed=1)
    ix.train(torch.from_numpy(gen.train(262144)).cuda(), niter=4)
    ix.set_option(S.OPT_COARSE_SELECT, int(os.environ.get("COARSE_SELECT", "1")))
    torch.cuda.synchronize()
    ix.profile(rep == 1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for b0 in range(0, N, B):
        ix.insert(ids[b0:b0 + B], X[b0:b0 + B])
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    if rep == 1:
        p = ix.profile_read()
        print(f"batch {B}: {N / (ms / 1e3) / 1e6:.1f} M vec/s (profiled run: per-batch "
              + ", ".join(f"{k} {v[0] / v[1]:.4f} ms" for k, v in p.items() if v[1]) + ")")
    else:
        print(f"batch {B}: {N / (ms / 1e3) / 1e6:.1f} M vec/s ({ms:.2f} ms)")
    del ix
