"""§4.3 search cell with the split-fp16 copy (SIVF_CFG_SPLIT_COPY), timing only: uniform
d = 128, N = 100K (env N), nlist 1024, 10k queries, k = 10, nprobe 32: QPS and
the search phases (coarse, invmap, scan, merge = k_gs_select)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_11808_b200 as S
from tools.param_grids import build

n = int(os.environ.get("N", "100000"))
nl = int(os.environ.get("NL", "1024"))
for flags in (S.CFG_SPLIT_COPY, 0):
    ix, gen, _ = build(n, nl, flags=flags)
    Q = torch.empty(10_000, 128, device="cuda")
    gen.range_into(Q, 1 << 40)
    for _ in range(2):
        ix.search(Q, 10, 32)
    ix.profile(True)
    ix.profile_read()
    for _ in range(5):
        ix.search(Q, 10, 32)
    torch.cuda.synchronize()
    p = ix.profile_read()
    ix.profile(False)
    ph = {k: round(v[0] / 5, 4) for k, v in p.items() if v[1]}
    print("split" if flags else "fp16", n, nl, ph, "sum", round(sum(ph.values()), 4), flush=True)
    del ix
    torch.cuda.empty_cache()
