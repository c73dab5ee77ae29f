"""Coarse quantisation in isolation (nlist=1024, d=128, 10k queries / 10k inserts): phase
times, and one search + one insert bracketed by cudaProfilerStart/Stop for
`ncu --profile-from-start off`."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_11808_b200 as S
from datagen import Generator, sift_shape
N, D, NL, NQ = 200_000, 128, 1024, 10_000
gen = Generator(sift_shape(seed=0x51F7))
ix = S.Index(D, NL, N, S.num_slabs_for(N, NL), max_batch=10000, max_queries=NQ, max_k=32, max_nprobe=128,
             max_train=65536, seed=1)
ix.set_option(6, int(os.environ.get("SEL", "1")))
ix.train(torch.from_numpy(gen.train(65536)).cuda(), niter=4)
X = torch.from_numpy(gen.range(0, 10000)).cuda()
Q = torch.from_numpy(gen.queries(0, NQ)).cuda()
ids = torch.arange(10000, device="cuda")
npb = int(os.environ.get("NPROBE", "32"))
for _ in range(3):
    ix.search(Q, 10, npb)
torch.cuda.synchronize()
ix.profile(True); ix.profile_read()
for _ in range(5):
    ix.search(Q, 10, npb)
    ix.insert(ids, X); ix.delete(ids)
torch.cuda.synchronize()
p = ix.profile_read(); ix.profile(False)
print("SEL", os.environ.get("SEL", "1"), {k: round(v[0] / v[1], 4) for k, v in p.items() if v[1]})
torch.cuda.profiler.start()
ix.search(Q, 10, npb)
ix.insert(ids, X)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
if os.environ.get("HIST"):
    import ctypes, numpy as np
    h = np.zeros((2, 64), np.uint32)
    S.lib().sivf_debug_selhist(h.ctypes.data_as(ctypes.c_void_p))
    for mode in (0, 1):
        nz = {i: int(v) for i, v in enumerate(h[mode]) if v}
        print("mode", mode, "nc histogram", nz)
    c = np.zeros((2, 8), np.uint64)
    S.lib().sivf_debug_selclk(c.ctypes.data_as(ctypes.c_void_p))
    print("clk mode1 [loads, U', superset+U, candidates, approx-sort path, exact<=64 path]:", c[1][:6].tolist())
    print("clk mode0:", c[0][:6].tolist())
