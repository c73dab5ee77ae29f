"""GIST1M-shaped search in isolation (1M x 960, nlist=1024, 10k queries, k=100, nprobe=32):
phase times; the last search is bracketed by cudaProfilerStart/Stop for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_11808_b200 as S
from datagen import DeviceGenerator, gist_shape, TRAIN_BASE, QUERY_BASE
N, D, NL, NQ, K = 1_000_000, 960, 1024, 10_000, 100
gen = DeviceGenerator(gist_shape())
ix = S.Index(D, NL, N, S.num_slabs_for(N, NL), max_batch=65536, max_queries=NQ, max_k=K, max_nprobe=64,
             max_train=262144, seed=1)
Xt = torch.empty(262144, D, device="cuda"); gen.range_into(Xt, TRAIN_BASE)
ix.train(Xt, niter=10); del Xt
X = torch.empty(65536, D, device="cuda")
for b in range(0, N, 65536):
    n = min(65536, N - b)
    gen.range_into(X[:n], b)
    ix.insert(torch.arange(b, b + n, device="cuda"), X[:n])
Q = torch.empty(NQ, D, device="cuda"); gen.range_into(Q, QUERY_BASE)
npb = int(os.environ.get("NPROBE", "32"))
ix.search(Q, K, npb); torch.cuda.synchronize()
ix.profile(True); ix.profile_read()
for _ in range(2):
    ix.search(Q, K, npb)
torch.cuda.synchronize()
p = ix.profile_read(); ix.profile(False)
print("gist", {k: round(v[0] / v[1], 3) for k, v in p.items() if v[1]}, flush=True)
torch.cuda.profiler.start()
ix.search(Q, K, npb)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
