"""GPU parity for the configurations round 1 left untested (VERDICT r01 "Next round" 1):
large-nlist coarse quantisation (the fused k_coarse_gemm<1|32> + k_coarse_rerank path,
config H's nlist 16384), the id-sharded index on one GPU, the sivf_search graph cache,
nprobe = max_nprobe = 1024, and a drifting stream that forces directory compaction."""
from __future__ import annotations

import os

import numpy as np
import pytest
import torch

import oracle as O
import paper_2601_11808_b200 as S
from paper_2601_11808_b200 import shard
from datagen import Generator, sift_shape
from tests.checkers import check_state
from tests.test_gpu_parity import T, dele, ins, make_pair, srch

pytestmark = pytest.mark.gpu


# ------------------------------------------------------------------ a3/a7 at nlist > 1024
@pytest.mark.parametrize("NL", [4096, 16384])
def test_coarse_large_nlist_sift_shaped(NL):
    # SIFT-shaped rows, quantizer = sampled points + small integer jitter (distinct
    # centroids, integer data: dist32 exact); every assignment of a 20k insert and the
    # probe sets of 1k queries at nprobe 1/8/32 (tensor-core fused path) and 64 (CUDA
    # cores) bit-exact with the oracle
    O.set_threads(os.cpu_count() or 1)
    gen = Generator(sift_shape(seed=0x100A))
    rng = np.random.default_rng(NL)
    C = (gen.range(1 << 41, NL) + rng.integers(-2, 3, (NL, 128))).astype(np.float32)
    N = 20000
    g, o = make_pair(128, NL, N, C, max_batch=19000, max_queries=1000, max_k=32, max_nprobe=64)
    X = gen.range(0, N)
    # 149 row tiles, then 8 (one CTA per row tile for the assignment); the 8-tile query
    # batches below split their N-tiles over CTAs (per-range bounds, shared counters)
    ins(g, o, np.arange(19000), X[:19000])  # ins() asserts statuses and assigned lists equal
    ins(g, o, np.arange(19000, N), X[19000:])
    check_state(g, o, f"nlist {NL}")
    Q = gen.queries(0, 1000)
    for npb in (1, 8, 32, 64):
        srch(g, o, Q, 10, npb)


def test_coarse_large_nlist_band_overflow():
    # nlist 16384 centroids all at exactly the same distance from the zero vector (signed
    # permutations of one integer vector): every list is in the certified band, the
    # candidate buffers overflow and the full exact re-rank must pick the lowest indices
    rng = np.random.default_rng(14)
    v = rng.integers(1, 20, 32).astype(np.float32)
    NL = 16384
    C = np.stack([rng.permutation(v) * rng.choice([-1.0, 1.0], 32) for _ in range(NL)]).astype(np.float32)
    g, o = make_pair(32, NL, 100, C, max_batch=64, max_queries=8, max_nprobe=64)
    Z = np.zeros((8, 32), np.float32)
    st, ls = g.insert(T(np.arange(8), torch.int64), T(Z))
    assert (ls.cpu().numpy() == 0).all()
    for npb in (1, 8, 32):
        _, _, p = g.search(T(Z), 1, npb, return_probes=True)
        assert (np.sort(p.cpu().numpy(), axis=1) == np.arange(npb)).all()


# ------------------------------------------------------------------ §8(e) on one GPU
@pytest.mark.parametrize("G", [2, 4])
def test_sharded_index_on_one_gpu(G):
    # G shard indexes (owner(id) = id mod G, ATT index id / G) on cuda:0 against G oracle
    # shards and one unsharded oracle: statuses (WRONG_SHARD for foreign ids of a full
    # batch), foreign-id deletes as no-ops, per-shard state bit-exact, and the per-shard
    # searches merged with sivf_merge_topk == the unsharded oracle, bitwise (integer data)
    gen = Generator(sift_shape(seed=0x7111))
    N, NL = 12000, 64
    X = gen.range(0, N)
    C = O.kmeans(X[:6000], NL, 8, 0x7111)
    ref = O.Index(128, NL, N)
    ref.set_centroids(C)
    shards = [make_pair(128, NL, N, C, max_batch=N, max_queries=200, shard_rank=r, shard_count=G) for r in range(G)]
    # full batch to every rank: non-owned ids -> WRONG_SHARD
    ids = np.arange(6000)
    ref.insert(ids, X[ids])
    for r, (g, o) in enumerate(shards):
        st = ins(g, o, ids, X[ids])
        assert (st[ids % G != r] == S.ST_WRONG_SHARD).all() and (st[ids % G == r] == S.ST_OK).all()
    # routed batches: each rank gets only its own ids
    ids = np.arange(6000, N)
    ref.insert(ids, X[ids])
    for r, (g, o) in enumerate(shards):
        mine = ids[ids % G == r]
        st = ins(g, o, mine, X[mine])
        assert (st == S.ST_OK).all()
    # full delete batch to every rank: foreign ids are no-ops
    dels = np.random.default_rng(1).choice(N, 3000, replace=False)
    total = sum(dele(g, o, dels) for g, o in shards)
    assert total == ref.delete(dels) == 3000
    for r, (g, o) in enumerate(shards):
        check_state(g, o, f"shard {r}/{G}")
    Q = gen.queries(0, 200)
    for k, npb in ((10, 8), (32, 64)):
        outs = []
        for g, o in shards:
            srch(g, o, Q, k, npb)  # per shard vs its oracle shard
            outs.append(g.search(T(Q), k, npb))
        dg = torch.stack([d for d, _ in outs])
        ig = torch.stack([i for _, i in outs])
        md, mi = S.merge_topk(dg, ig)
        od, oi, op = ref.search(Q, k, npb)
        assert np.array_equal(mi.cpu().numpy(), oi) and np.array_equal(md.cpu().numpy(), od)
        # NEXT-3 query-sharded coarse step: rank r computes the probe sets of its query
        # slice (sivf_probe), the slices are concatenated (the all-gather), and every
        # shard scans with the full probe sets (sivf_search_probed): the merged result is
        # the unsharded oracle's, bitwise, and each shard's equals its own sivf_search
        Qt = T(Q)
        parts = []
        for r, (g, _) in enumerate(shards):
            lo, hi = shard.query_slice(len(Q), G, r)
            parts.append(g.probe(Qt[lo:hi], npb))
        probes = torch.cat(parts, 0)
        assert np.array_equal(np.sort(probes.cpu().numpy(), 1), np.sort(np.asarray(op), 1))
        outs2 = [g.search_probed(Qt, probes, k) for g, _ in shards]
        for (d1, i1), (d2, i2) in zip(outs, outs2):
            assert torch.equal(i1, i2) and torch.equal(d1, d2)
        md2, mi2 = S.merge_topk(torch.stack([d for d, _ in outs2]), torch.stack([i for _, i in outs2]))
        assert torch.equal(md2, md) and torch.equal(mi2, mi)


# ------------------------------------------------------------------ sivf_search graph cache
def test_search_graph_cache_replay():
    # the second identical sivf_search call is captured as a CUDA graph and later calls
    # replay it: each replay must read the current queries and index state
    gen = Generator(sift_shape(seed=0x51F7))
    C = O.kmeans(gen.train(4000), 64, 8, 9)
    g, o = make_pair(128, 64, 40000, C, max_batch=20000, max_queries=256)
    ins(g, o, np.arange(20000), gen.range(0, 20000))
    q_d = torch.empty(256, 128, device="cuda")
    out = (torch.empty(256, 10, device="cuda"), torch.empty(256, 10, dtype=torch.int64, device="cuda"))
    launches = []
    for t in range(8):
        if t % 2 == 1:
            new = np.arange(20000 + t * 1000, 21000 + t * 1000)
            ins(g, o, new, gen.range(new[0], 1000))
            dele(g, o, np.arange(t * 1000, t * 1000 + 700))
        Q = gen.queries(t * 256, 256)
        q_d.copy_(T(Q))
        l0 = g.launch_count()
        d, i = g.search(q_d, 10, 16, out=out)
        launches.append(g.launch_count() - l0)
        od, oi, _ = o.search(Q, 10, 16)
        assert np.array_equal(i.cpu().numpy(), oi) and np.array_equal(d.cpu().numpy(), od), f"call {t}"
    assert len(set(launches)) == 1 and launches[0] > 0


# ------------------------------------------------------------------ sivf_probe / sivf_search_probed
def test_probe_and_probed_search_edges():
    # host-detectable argument errors enqueue nothing; empty batches are no-ops; probe
    # sets in any order give the same result (the order only steers the work)
    gen = Generator(sift_shape(seed=0x7E57))
    X = gen.range(0, 8000)
    C = O.kmeans(X[:4000], 32, 5, 3)
    g, o = make_pair(128, 32, 8000, C, max_batch=8000, max_queries=64, max_nprobe=16)
    ins(g, o, np.arange(8000), X)
    Q = T(gen.queries(0, 64))
    with pytest.raises(S.SivfError):
        g.probe(Q, 17)  # nprobe > max_nprobe
    with pytest.raises(S.SivfError):
        g.probe(T(gen.queries(0, 65)), 8)  # nq > max_queries
    assert g.probe(Q[:0], 8).shape == (0, 8)
    p = g.probe(Q, 8)
    d0, i0 = g.search(Q, 10, 8)
    d1, i1 = g.search_probed(Q, p, 10)
    d2, i2 = g.search_probed(Q, p.flip(1).contiguous(), 10)  # reversed probe order
    assert torch.equal(i0, i1) and torch.equal(d0, d1) and torch.equal(i0, i2) and torch.equal(d0, d2)
    with pytest.raises(S.SivfError):
        g.search_probed(Q, p, 0)  # k = 0
    d3, i3 = g.search_probed(Q[:0], p[:0], 10)
    assert d3.shape == (0, 10)


# ------------------------------------------------------------------ per-list seed of the bounds
@pytest.mark.parametrize("kind", ["sift", "float"])
def test_seed_list_changes_nothing(kind):
    # SIVF_OPT_SEED_LIST (default on with >= 4 queries per list): the k-th distance bounds
    # seeded from each query's nearest list prune work only.  The same index and queries
    # with and without it: identical results, and equal to the oracle (integer data) or
    # within the float tolerance (float data)
    gen = Generator(sift_shape(seed=0x5EED))
    if kind == "sift":
        X, Q = gen.range(0, 30000), gen.queries(0, 2000)
    else:
        rng = np.random.default_rng(5)
        X = rng.random((30000, 128), dtype=np.float32)
        Q = rng.random((2000, 128), dtype=np.float32)
    C = O.kmeans(X[:8000], 64, 6, 12)
    g, o = make_pair(128, 64, 30000, C, max_batch=30000, max_queries=2000)
    ins(g, o, np.arange(30000), X)
    dele(g, o, np.arange(0, 30000, 9))
    for k, npb in ((10, 16), (32, 8), (1, 4)):
        g.set_option(S.OPT_SEED_LIST, 1)
        d1, i1 = g.search(T(Q), k, npb)
        g.set_option(S.OPT_SEED_LIST, 0)
        d2, i2 = g.search(T(Q), k, npb)
        assert torch.equal(i1, i2) and torch.equal(d1, d2), (kind, k, npb)
        if kind == "sift":
            od, oi, _ = o.search(Q, k, npb)
            assert np.array_equal(i1.cpu().numpy(), oi) and np.array_equal(d1.cpu().numpy(), od)
        else:
            assert srch(g, o, Q, k, npb, exact=False) <= 3


# ------------------------------------------------------------------ nprobe = max_nprobe = 1024
def test_nprobe_1024_full_probe():
    # k_select_probes needs 64 nprobe B of shared memory (64 KB at 1024);
    # nprobe = nlist = 1024 is exactly brute force
    gen = Generator(sift_shape(seed=0x51F7))
    X = gen.range(0, 30000)
    rng = np.random.default_rng(15)
    C = (X[rng.choice(30000, 1024, replace=False)] + rng.integers(-3, 4, (1024, 128))).astype(np.float32)
    g, o = make_pair(128, 1024, 30000, C, max_batch=30000, max_queries=100, max_nprobe=1024)
    ins(g, o, np.arange(30000), X)
    Q = gen.queries(0, 100)
    srch(g, o, Q, 10, 1024)
    bd, bi = o.bruteforce(Q, 10)
    d, i = g.search(T(Q), 10, 1024)
    assert np.array_equal(i.cpu().numpy(), bi) and np.array_equal(d.cpu().numpy(), bd)
    # and the shard merge at k > 768 (64 k B of shared memory)
    G, nq, k = 2, 8, 1000
    dd = np.sort(rng.integers(0, 10**6, (G, nq, k)).astype(np.float32), axis=2)
    ii = rng.permutation(G * nq * k).reshape(G, nq, k).astype(np.int64)
    gd, gi = S.merge_topk(T(dd), T(ii))
    od, oi = O.merge_topk(dd, ii, k)
    assert np.array_equal(gi.cpu().numpy(), oi) and np.array_equal(gd.cpu().numpy(), od)


# ------------------------------------------------------------------ drifting stream
def test_drifting_stream_directory_compaction():
    # a hot set of 2 lists moving one list per step through 64 lists: every list's
    # directory peaks in turn, so bump-allocated directory space would exceed the arena
    # many times over; k_reserve must compact the directories (into the idle half) and
    # the state must stay exact, with no device error and no invariant violation
    NL, D, B, WB = 64, 8, 320, 4
    C = np.zeros((NL, D), np.float32)
    C[:, 0] = np.arange(NL) * 1000.0
    rng = np.random.default_rng(16)
    steps = 160
    cap = B * (steps + 1)
    ns = S.num_slabs_for(B * (WB + 1), NL) + 32
    g, o = make_pair(D, NL, cap, C, num_slabs=ns, max_batch=B, max_queries=64, max_nprobe=NL)
    batches = []
    for t in range(steps):
        ids = np.arange(t * B, (t + 1) * B)
        hot = np.where(np.arange(B) < B // 2, t % NL, (t + 1) % NL)
        X = (C[hot] + rng.integers(-50, 51, (B, D))).astype(np.float32)
        st = ins(g, o, ids, X)
        assert (st == S.ST_OK).all(), f"step {t}"
        batches.append(ids)
        if len(batches) > WB:
            dele(g, o, batches.pop(0))
        assert int(g.reclaim().item()) == o.reclaim()
        if t % 20 == 19:
            check_state(g, o, f"step {t}")
            srch(g, o, (C[rng.integers(0, NL, 64)] + rng.integers(-50, 51, (64, D))).astype(np.float32), 10, NL)
    s = g.stats()
    assert s["device_errors"] == 0 and s["dir_compactions"] >= 2, s
