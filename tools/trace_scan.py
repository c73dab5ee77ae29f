"""Dump the k_scan_tc block-0 event trace (prof build: SIVF_LIB_PATH=build/libsivf_prof.so)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_11808_b200 as S
from datagen import Generator, sift_shape
N, D, NL, NQ = 1_000_000, 128, 1024, 10_000
npb = int(os.environ.get("NPROBE", "32"))
gen = Generator(sift_shape(seed=0x51F7))
ix = S.Index(D, NL, N, S.num_slabs_for(N, NL), max_batch=65536, max_queries=NQ, max_k=32, max_nprobe=128, max_train=262144, seed=1)
ix.train(torch.from_numpy(gen.train(262144)).cuda(), niter=10)
X = torch.from_numpy(gen.range(0, N)).cuda()
ids = torch.arange(N, device="cuda")
for b in range(0, N, 65536):
    ix.insert(ids[b:b+65536], X[b:b+65536])
Q = torch.from_numpy(gen.queries(0, NQ)).cuda()
ix.set_option(4, 0)
ix.set_option(5, int(os.environ.get("SPLIT", "1")))
ix.set_option(99, int(os.environ.get("DBG", "0")))
for _ in range(3):
    ix.search(Q, 10, npb)
torch.cuda.synchronize()
buf = np.zeros((6, 1024), np.int64)
rc = S.lib().sivf_debug_trace(buf.ctypes.data_as(ctypes.c_void_p))
t0 = buf[0][0]
print("rc", rc, "cols: g prod_issue full_seen mma_issue epi_start epi_end epi2_start (cycles rel. to first issue)")
for g in range(0, 60):
    print(g, *[int(buf[r][g] - t0) if buf[r][g] else -1 for r in range(6)])
# summary over the traced groups of block 0
g = [i for i in range(1, 1024) if all(buf[r][i] for r in range(5))]
if g:
    a = np.array([[buf[r][i] for r in range(6)] for i in g], np.float64)
    span = (a[-1, 2] - a[0, 2]) / max(1, len(g) - 1)
    print(f"groups {len(g)}  mma_issue interval {span:.0f} cyc/group")
    print(f"  issue->full   {np.median(a[:,1]-a[:,0]):.0f} (median)  p90 {np.percentile(a[:,1]-a[:,0],90):.0f}")
    print(f"  full->mma     {np.median(a[:,2]-a[:,1]):.0f}  (grp_free wait)")
    print(f"  mma->epi      {np.median(a[:,3]-a[:,2]):.0f}")
    print(f"  epi duration  {np.median(a[:,4]-a[:,3]):.0f}  p90 {np.percentile(a[:,4]-a[:,3],90):.0f}")
