"""Work statistics of the scan at the SIFT1M-shaped search (items, groups, row fill)."""
import os, sys
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
_, lpl, _ = ix.dump_state()
live = lpl.cpu().numpy()
slabs = (live + 31) // 32
print("lists: live mean %.0f max %d min %d; slabs mean %.1f max %d" % (live.mean(), live.max(), live.min(), slabs.mean(), slabs.max()))
for npb in (8, 16, 32):
    _, _, pr = ix.search(Q, 10, npb, return_probes=True)
    pr = pr.cpu().numpy()
    for split in (0, 1):
        if split:
            r0 = npb // 2
            cs = [np.bincount(pr[:, :r0].ravel(), minlength=NL), np.bincount(pr[:, r0:].ravel(), minlength=NL)]
        else:
            cs = [np.bincount(pr.ravel(), minlength=NL)]
        items = sum(int(np.sum((c + 127) // 128)) for c in cs)
        groups = sum(int(np.sum(((c + 127) // 128) * ((slabs + 3) // 4))) for c in cs)
        rows = sum(int(np.sum(np.minimum(c, 128 * ((c + 127) // 128)))) for c in cs)
        warps = sum(int(np.sum(((c + 31) // 32) * ((slabs + 3) // 4))) for c in cs)  # active epilogue row-warps x groups
        cand = int(np.sum(np.bincount(pr.ravel(), minlength=NL) * live))
        print(f"nprobe {npb} split {split}: items {items} groups {groups} ({groups/148:.0f}/SM) "
              f"row fill {rows/(items*128):.2f} active row-warps/group {warps/groups:.2f} "
              f"cand {cand/1e6:.0f}M useful/issued {cand/(groups*128*128):.2f} B bytes {groups*65536/1e9:.2f} GB")
