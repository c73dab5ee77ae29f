"""The paper's parameter and scale grids, on one B200.

  §4.2 ingestion: N in {1M, 2M, 4M} x nlist in {1024, 4096, 16384}:
       inserts/s over 100K-vector batches (device time, CUDA events around the whole build).
  §4.3 search: N in {100K, 300K, 500K} x nlist in {1024, 4096, 16384}:
       QPS of 10K queries, k = 10, nprobe = 32 (the paper does not state k / nprobe).
  §4.6 sensitivity: maxvec_factor x slab_factor in {1.0, 1.1, 1.2, 1.3}^2 at
       N = 1M, nlist = 4096: inserts/s, and delete latency of batches {100, 1K, 10K}.

Data: the paper's microbenchmarks use uniform random vectors of an unstated
dimension (reading C27): here uniform d = 128 (datagen kind UNIFORM, seed 0x0E1F),
centroids = sampled points (throughput does not depend on training).

  python tools/param_grids.py [--out gpurun_out/grids.json] [--quick]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_11808_b200 as S
from datagen import DeviceGenerator, uniform_shape

D = 128
BATCH = 100_000


def timed(fn, s):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    fn()
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1)


def build(n, nlist, mf=1.2, sf=1.2, max_queries=10_000, flags=0):
    gen = DeviceGenerator(uniform_shape(0x0E1F, D))
    ix = S.Index(D, nlist, n, S.num_slabs_for(n, nlist, mf, sf), max_batch=BATCH, max_queries=max_queries, max_k=10,
                 max_nprobe=min(64, nlist), flags=flags)
    cent = torch.empty(nlist, D, device="cuda")
    gen.range_into(cent, 1 << 41)
    ix.set_centroids(cent)
    xs = torch.empty(n, D, device="cuda")
    gen.range_into(xs, 0)
    ids = torch.arange(n, device="cuda")
    s = torch.cuda.current_stream()
    ix.insert(ids[:BATCH], xs[:BATCH])  # warm-up batch (then deleted and reclaimed)
    ix.delete(ids[:BATCH])
    ix.reclaim()
    torch.cuda.synchronize()

    def all_batches():
        for b in range(0, n, BATCH):
            ix.insert(ids[b:b + BATCH], xs[b:b + BATCH])

    ms = timed(all_batches, s)
    st = ix.stats()
    assert st["live"] == n and st["pool_exhausted_items"] == 0, st
    return ix, gen, n / (ms / 1e3)


def ingestion(ns, nls):
    out = []
    for n in ns:
        for nl in nls:
            ix, _, ips = build(n, nl)
            out.append({"n": n, "nlist": nl, "inserts_per_s": ips})
            print(json.dumps(out[-1]), flush=True)
            del ix
            torch.cuda.empty_cache()
    return out


def search(ns, nls, flags=0):
    # flags = S.CFG_SPLIT_COPY: the split-fp16 copy + GEMM scan for this float data
    out = []
    for n in ns:
        for nl in nls:
            ix, gen, _ = build(n, nl, flags=flags)
            Q = torch.empty(10_000, D, device="cuda")
            gen.range_into(Q, 1 << 40)
            s = torch.cuda.current_stream()
            npb = min(32, nl)
            ix.search(Q, 10, npb)
            ms = min(timed(lambda: ix.search(Q, 10, npb), s) for _ in range(5))
            out.append({"n": n, "nlist": nl, "nprobe": npb, "k": 10, "qps": 10_000 / (ms / 1e3), "ms_10k": ms,
                        "scan_copy": "split-fp16 (SIVF_CFG_SPLIT_COPY)" if flags else "fp16"})
            print(json.dumps(out[-1]), flush=True)
            del ix
            torch.cuda.empty_cache()
    return out


def sensitivity(fs):
    out = []
    for mf in fs:
        for sf in fs:
            ix, _, ips = build(1_000_000, 4096, mf, sf)
            s = torch.cuda.current_stream()
            lat = {}
            base = 0
            for bs in (100, 1000, 10_000):
                ms = []
                for r in range(5):
                    ids = torch.arange(base, base + bs, device="cuda")
                    base += bs
                    ms.append(timed(lambda: ix.delete(ids), s))
                lat[str(bs)] = sorted(ms)[len(ms) // 2]
            out.append({"maxvec_factor": mf, "slab_factor": sf, "num_slabs": ix.cfg.num_slabs, "inserts_per_s": ips,
                        "delete_ms_median": lat, "deletes_per_s_10k": 10_000 / (lat["10000"] / 1e3)})
            print(json.dumps(out[-1]), flush=True)
            del ix
            torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/grids.json")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--search-only", action="store_true")
    a = ap.parse_args()
    q = a.quick
    if a.search_only:
        ns = [100_000] if q else [100_000, 300_000, 500_000]
        res = {"search": search(ns, [1024, 4096, 16384]),
               "search_split_copy": search(ns, [1024, 4096, 16384], S.CFG_SPLIT_COPY)}
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        json.dump(res, open(a.out, "w"), indent=1)
        return
    res = {"data": "uniform d=128 (P:485; dimension unstated, reading C27), centroids = sampled points",
           "ingestion": ingestion([1_000_000] if q else [1_000_000, 2_000_000, 4_000_000], [1024, 4096, 16384]),
           "search": search([100_000] if q else [100_000, 300_000, 500_000], [1024, 4096, 16384]),
           "sensitivity": sensitivity([1.0, 1.3] if q else [1.0, 1.1, 1.2, 1.3])}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
