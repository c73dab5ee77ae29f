"""Memory efficiency and reclamation (paper §4.8).

Part 1 — footprint vs N (100K..1M, d = 128 SIFT-shaped and d = 960 GIST-shaped):
allocated arena, slabs in use, the paper's per-slab header accounting
(`overhead_paper` = 128 / (32 (4d + 8))) and this build's own metadata
(`overhead_actual`) and fp16 scan copy (`overhead_scan_copy`) against the live
payload, beside a compact static array (N x (4d + 8) B: payload + id).

Part 2 — "deletion of 50 % of the dataset followed by immediate re-insertion"
 on GIST-shaped 200K x 960, twice over:
  fifo:   delete the oldest half (ids 0 .. N/2-1), reclaim, re-insert them;
  strided: delete every other id, reclaim, re-insert them.
Per 100K delete batch: device time (CUDA events on the library stream).  The
arena is pre-allocated and never changes size; the pool's slabs in use are
reported before/after, with the search result of 100 queries before the cycle
and after it (same vectors, same ids -> identical top-10 ids and distances).
Slots are not reused in place (reading C16): a fully dead slab returns to the
pool at the reclaim, a partially dead one keeps its holes until it dies.

  python tools/mem_experiment.py [--out profiles/r01s5_memory.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2601_11808_b200 as S
from datagen import DeviceGenerator, gist_shape, sift_shape

NL = 1024


def build(dim, shape, n, flags=0, max_batch=100_000, pool_n=None):
    ix = S.Index(dim, NL, n, S.num_slabs_for(pool_n or n, NL), max_batch=max_batch, max_queries=100, max_k=10,
                 max_nprobe=64, flags=flags)
    gen = DeviceGenerator(shape)
    cent = torch.empty(NL, dim, device="cuda")
    gen.range_into(cent, 1 << 41)  # centroids = sampled points (footprint does not depend on training)
    ix.set_centroids(cent)
    buf = torch.empty(max_batch, dim, device="cuda")
    for b in range(0, n, max_batch):
        m = min(max_batch, n - b)
        gen.range_into(buf[:m], b)
        ix.insert(torch.arange(b, b + m, device="cuda"), buf[:m])
    torch.cuda.synchronize()
    return ix, gen


def footprint():
    rows = []
    for dim, shape, flags in ((128, sift_shape(), 0), (128, sift_shape(), S.CFG_NO_SCAN_COPY), (960, gist_shape(), 0)):
        for n in (100_000, 250_000, 500_000, 1_000_000):
            ix, _ = build(dim, shape, n, flags)
            st = ix.stats()
            compact = n * (4 * dim + 8)
            rows.append({"dim": dim, "n": n, "scan_copy": bool(dim <= 128 and not flags),
                         "arena_bytes": ix.arena_bytes, "compact_bytes": compact,
                         "slabs_in_use": st["slabs_in_use"], "live": st["live"],
                         "overhead_paper": st["overhead_paper"], "overhead_actual": st["overhead_actual"],
                         "overhead_scan_copy": st["overhead_scan_copy"],
                         "slab_bytes_in_use_over_compact": st["slabs_in_use"] * 32 * (4 * dim + 4) / compact})
            print(json.dumps(rows[-1]), flush=True)
            del ix
            torch.cuda.empty_cache()
    return rows


def cycle(order, n=200_000, rounds=2):
    dim = 960
    ix, gen = build(dim, gist_shape(), n, pool_n=int(1.5 * n))
    Q = torch.empty(100, dim, device="cuda")
    gen.range_into(Q, 1 << 40)
    d0, i0 = ix.search(Q, 10, 32)
    s = torch.cuda.current_stream()
    out = {"order": order, "n": n, "dim": dim, "arena_bytes": ix.arena_bytes, "num_slabs": ix.cfg.num_slabs,
           "rounds": []}
    half = torch.arange(0, n // 2, device="cuda") if order == "fifo" else torch.arange(0, n, 2, device="cuda")
    buf = torch.empty(100_000, dim, device="cuda")
    for r in range(rounds):
        before = ix.stats()
        ms = []
        for b in range(0, half.numel(), 100_000):
            ids = half[b:b + 100_000]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            ix.delete(ids)
            e1.record(s)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        reclaimed = ix.reclaim()
        torch.cuda.synchronize()
        mid = ix.stats()
        for b in range(0, half.numel(), 100_000):
            ids = half[b:b + 100_000]
            if order == "fifo":
                gen.range_into(buf[:ids.numel()], int(ids[0]))
            else:
                gen.range_into(buf[:ids.numel()], int(ids[0]), 2)
            st, _ = ix.insert(ids, buf[:ids.numel()])
            assert int((st != 0).sum()) == 0, "re-insert failed"
        torch.cuda.synchronize()
        after = ix.stats()
        d1, i1 = ix.search(Q, 10, 32)
        out["rounds"].append({"delete_100k_ms": ms, "live_before": before["live"], "slabs_before": before["slabs_in_use"],
                              "slabs_after_delete_reclaim": mid["slabs_in_use"], "slabs_after_reinsert": after["slabs_in_use"],
                              "live_after": after["live"], "pool_exhausted": after["pool_exhausted_items"],
                              "reclaimed_total": after["reclaimed_slabs"],
                              "search_ids_identical": bool(torch.equal(i0, i1)),
                              "search_dist_identical": bool(torch.equal(d0, d1))})
        print(json.dumps(out["rounds"][-1]), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/memory.json")
    a = ap.parse_args()
    res = {"footprint": footprint(), "cycle_fifo": cycle("fifo"), "cycle_strided": cycle("strided")}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
