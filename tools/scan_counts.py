"""Survivor statistics of k_scan_tc (prof build): per search of 10k queries at nprobe 32."""
import ctypes, os, sys
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
c = np.zeros(4, np.uint64)
for split, seed in ((1, 0), (1, 1), (1, 4)):
    for npb in (8, 32):
        ix.set_option(5, split)
        ix.set_option(4, seed)
        ix.search(Q, 10, npb); torch.cuda.synchronize()
        S.lib().sivf_debug_scnt(c.ctypes.data_as(ctypes.c_void_p), 1)
        ix.search(Q, 10, npb); torch.cuda.synchronize()
        S.lib().sivf_debug_scnt(c.ctypes.data_as(ctypes.c_void_p), 1)
        print(f"seed {seed} split {split} nprobe {npb}: slow entries/query {c[0]/NQ:.1f} survivors/query {c[1]/NQ:.1f} insertions/query {c[2]/NQ:.1f} (with the row bound still +inf: {c[3]/NQ:.1f})")
