"""GPU parity tests: the CUDA path (through the C ABI) against the CPU oracle,
element by element on the same seeded inputs (SURVEY §8(c) parity matrix)."""
from __future__ import annotations

import os

import numpy as np
import pytest
import torch

import oracle as O
import paper_2601_11808_b200 as S
from datagen import Generator, gist_shape, sift_shape
from tests.checkers import check_assign, check_search, check_state

pytestmark = pytest.mark.gpu

DEV = "cuda"


def T(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(DEV)


def make_pair(dim, nlist, cap, C, num_slabs=None, max_batch=4096, max_queries=1024, max_k=128, max_nprobe=None,
              shard_rank=0, shard_count=1, max_train=0, tc=True, coarse=True, flags=0):
    if num_slabs is None:
        num_slabs = S.num_slabs_for(cap, nlist)
    g = S.Index(dim, nlist, cap, num_slabs, max_batch=max_batch, max_queries=max_queries, max_k=max_k,
                max_nprobe=max_nprobe, shard_rank=shard_rank, shard_count=shard_count, max_train=max_train,
                flags=flags)
    g.set_option(S.OPT_TC_SCAN, 1 if tc else 0)
    g.set_option(S.OPT_TC_COARSE, 1 if coarse else 0)
    o = O.Index(dim, nlist, cap, num_slabs=num_slabs, shard_rank=shard_rank, shard_count=shard_count)
    g.set_centroids(T(C))
    o.set_centroids(C)
    return g, o


def ins(g, o, ids, X):
    st, ls = g.insert(T(ids, torch.int64), T(X))
    ost, ols = o.insert(ids, X)
    st, ls = st.cpu().numpy(), ls.cpu().numpy()
    assert np.array_equal(st, ost), f"insert statuses differ: {np.nonzero(st != ost)[0][:10]}"
    assert np.array_equal(ls, ols), f"assigned lists differ: {np.nonzero(ls != ols)[0][:10]}"
    return st


def dele(g, o, ids):
    n = int(g.delete(T(ids, torch.int64)).item())
    assert n == o.delete(ids)
    return n


def srch(g, o, Q, k, nprobe, exact=True):
    gd, gi, gp = g.search(T(Q), k, nprobe, return_probes=True)
    od, oi, op = o.search(Q, k, nprobe)
    return check_search((gd.cpu().numpy(), gi.cpu().numpy(), gp.cpu().numpy()), (od, oi, op), exact=exact,
                        ref=o, Q=np.asarray(Q, np.float32))


# ------------------------------------------------------------------ SPEC examples
def test_spec_worked_example():
    g, o = make_pair(2, 1, 16, np.zeros((1, 2), np.float32))
    ins(g, o, np.array([0, 1, 2]), np.array([[0, 0], [3, 4], [1, 1]], np.float32))
    d, i = g.search(T(np.zeros((1, 2), np.float32)), 2, 1)
    assert i.cpu().tolist() == [[0, 2]] and d.cpu().tolist() == [[0.0, 2.0]]
    check_state(g, o)


def test_spec_equivalence_suite_full_probe_is_bruteforce():
    # N=2000, d=16, nlist=64, 100 queries, k=10, nprobe=64 -> exactly brute force
    rng = np.random.default_rng(0)
    X = rng.integers(0, 32, (2000, 16)).astype(np.float32)
    C = X[rng.choice(2000, 64, replace=False)] + 0.5
    g, o = make_pair(16, 64, 2000, C)
    ins(g, o, np.arange(2000), X)
    Q = rng.integers(0, 32, (100, 16)).astype(np.float32)
    srch(g, o, Q, 10, 64)
    bd, bi = o.bruteforce(Q, 10)
    d, i = g.search(T(Q), 10, 64)
    assert np.array_equal(i.cpu().numpy(), bi) and np.array_equal(d.cpu().numpy(), bd)
    check_state(g, o)


# ------------------------------------------------------------------ tiny config (BJ configs[0])
@pytest.mark.parametrize("tc", [True, False], ids=["tcgen05-scan", "simt-scan"])
def test_tiny_config_rounds(tc):
    gen = Generator(sift_shape(seed=0x7111))
    X = gen.range(0, 10000)
    C = O.kmeans(X, 64, 20, 0x7111)
    g, o = make_pair(128, 64, 10000, C, max_batch=1000, max_queries=100, tc=tc)
    Q = gen.queries(0, 100)
    live = []
    rng = np.random.default_rng(0x7111)
    for r in range(10):
        ids = np.arange(r * 1000, (r + 1) * 1000)
        ins(g, o, ids, X[ids])
        live.extend(ids.tolist())
        check_state(g, o, f"round {r} insert")
        if r >= 1:
            dels = rng.choice(np.array(live), 1000, replace=False)
            dele(g, o, dels)
            live = sorted(set(live) - set(dels.tolist()))
            check_state(g, o, f"round {r} delete")
        srch(g, o, Q, 10, 8)
        srch(g, o, Q, 10, 64)  # nprobe = nlist: exactly brute force
        bd, bi = o.bruteforce(Q, 10)
        d, i = g.search(T(Q), 10, 64)
        assert np.array_equal(i.cpu().numpy(), bi)


# ------------------------------------------------------------------ structure cases
def test_first_insert_and_33rd_insert():
    g, o = make_pair(4, 1, 100, np.zeros((1, 4), np.float32), num_slabs=8)
    X = np.arange(400, dtype=np.float32).reshape(100, 4)
    ins(g, o, np.array([0]), X[:1])
    assert g.stats()["slabs_in_use"] == 1
    ins(g, o, np.arange(1, 33), X[1:33])
    assert g.stats()["slabs_in_use"] == 2
    check_state(g, o)


def test_skew_single_list_10k():
    gen = Generator(sift_shape(seed=5))
    X = gen.range(0, 10000)
    C = np.stack([X.mean(0), X.mean(0) + 1e4]).astype(np.float32)
    g, o = make_pair(128, 2, 10000, C, max_batch=10000)
    ins(g, o, np.arange(10000), X)
    loi, lpl, viol = g.dump_state()
    assert lpl.cpu().tolist() == [10000, 0] and viol.item() == 0
    assert g.stats()["slabs_in_use"] == 313  # ceil(10000/32)
    check_state(g, o)
    srch(g, o, gen.queries(0, 50), 10, 2)


def test_duplicates_oor_shard_and_reinsert():
    rng = np.random.default_rng(3)
    X = rng.standard_normal((64, 8)).astype(np.float32)
    C = rng.standard_normal((4, 8)).astype(np.float32)
    g, o = make_pair(8, 4, 50, C)
    st = ins(g, o, np.array([0, 1, 1, 49, 50, -3, 7, 0]), X[:8])
    assert st.tolist() == [0, 0, 2, 0, 3, 3, 0, 2]
    st = ins(g, o, np.array([1, 2]), X[8:10])  # live duplicate
    assert st.tolist() == [2, 0]
    assert dele(g, o, np.array([1, 1, 2, 99, -1, 30])) == 2
    assert dele(g, o, np.array([1, 2])) == 0  # idempotent
    st = ins(g, o, np.array([1, 2]), X[10:12])  # re-insert after delete
    assert st.tolist() == [0, 0]
    check_state(g, o)


def test_delete_everything_then_search_and_k_gt_live():
    rng = np.random.default_rng(4)
    X = rng.integers(0, 100, (300, 16)).astype(np.float32)
    C = X[:8] + 0.5
    g, o = make_pair(16, 8, 300, C)
    ins(g, o, np.arange(300), X)
    dele(g, o, np.arange(295))
    Q = X[:20]
    srch(g, o, Q, 10, 8)  # k > live (5): all live, sorted, padded
    dele(g, o, np.arange(295, 300))
    d, i = g.search(T(Q), 10, 8)
    assert (i.cpu().numpy() == -1).all() and torch.isinf(d).all()
    check_state(g, o)


def test_equidistant_centroid_tie():
    C = np.array([[0, 2, 0, 0], [2, 0, 0, 0], [0, -2, 0, 0], [-2, 0, 0, 0], [9, 9, 9, 9]], np.float32)
    g, o = make_pair(4, 5, 10, C)
    st = ins(g, o, np.array([0, 1]), np.array([[0, 0, 0, 0], [1, 1, 0, 0]], np.float32))
    _, ls = o.insert(np.array([5]), np.zeros((1, 4), np.float32))
    loi, _, _ = g.dump_state()
    assert loi.cpu().tolist()[0] == 0  # ties -> lowest list
    d, i, p = g.search(T(np.zeros((1, 4), np.float32)), 2, 4, return_probes=True)
    assert p.cpu().tolist()[0] == [0, 1, 2, 3]


def test_near_tie_centroids_ulp():
    # centroids 1 ulp apart around a query: exact dist32 decides (zero exemptions)
    q = np.full(16, 100.0, np.float32)
    c0 = q.copy()
    c0[0] = np.nextafter(np.float32(101.0), np.float32(200.0))
    c1 = q.copy()
    c1[0] = np.float32(101.0)
    c2 = q.copy()
    c2[1] = np.float32(101.0)
    C = np.stack([c0, c1, c2]).astype(np.float32)
    g, o = make_pair(16, 3, 10, C)
    ins(g, o, np.array([0, 1]), np.stack([q, q]))
    d, i, p = g.search(T(q[None]), 2, 2, return_probes=True)
    assert set(p.cpu().tolist()[0]) == set(O.probe(C, q, 2).tolist())


def test_pool_exhaustion_then_reclaim():
    C = np.array([[0, 0], [100, 100]], np.float32)
    g, o = make_pair(2, 2, 1000, C, num_slabs=3)
    X = np.zeros((200, 2), np.float32)
    st = ins(g, o, np.arange(100), X[:100])
    assert (st[96:] == S.ST_POOL_EXHAUSTED).all()
    check_state(g, o, "exhausted")
    dele(g, o, np.arange(32, 64))
    assert int(g.reclaim().item()) == o.reclaim() == 1
    check_state(g, o, "after reclaim")
    st = ins(g, o, np.arange(100, 140), X[:40])
    check_state(g, o, "re-insert")
    X2 = np.array([[100, 100]] * 40 + [[0, 0]] * 40, np.float32)
    st = ins(g, o, np.arange(200, 280), X2)  # lists served in ascending order
    check_state(g, o, "two lists")


@pytest.mark.parametrize("tc", [True, False], ids=["tcgen05-scan", "simt-scan"])
def test_ragged_and_empty_batches(tc):
    rng = np.random.default_rng(6)
    X = rng.integers(0, 50, (3001, 20)).astype(np.float32)  # D=20 -> padded to 24
    C = X[:37] + 0.25
    g, o = make_pair(20, 37, 3001, C, max_batch=3001, max_queries=333, tc=tc)
    ins(g, o, np.arange(0), X[:0])
    ins(g, o, np.arange(3001), X)
    assert dele(g, o, np.arange(0)) == 0
    dele(g, o, np.arange(0, 3001, 7))
    check_state(g, o)
    Q = rng.integers(0, 50, (333, 20)).astype(np.float32)
    srch(g, o, Q, 7, 5)
    srch(g, o, Q, 33, 37)
    srch(g, o, Q, 128, 11)


def test_gist_shaped_float_data():
    gen = Generator(gist_shape(seed=0x6157))
    X = gen.range(0, 4000)
    C = O.kmeans(X, 32, 5, 1)
    g, o = make_pair(960, 32, 4000, C, max_queries=64)
    ins(g, o, np.arange(4000), X)
    dele(g, o, np.arange(0, 4000, 3))
    check_state(g, o)
    Q = gen.queries(0, 64)
    ex = srch(g, o, Q, 100, 8, exact=False)
    assert ex <= 2
    ex = srch(g, o, Q, 10, 32, exact=False)
    assert ex <= 2


@pytest.mark.parametrize("tc", [True, False], ids=["tcgen05-scan", "simt-scan"])
def test_float_data_d128_rerank_path(tc):
    # GIST-like non-integer data at d=128: the tensor-core distance only filters;
    # survivors are re-ranked exactly (certified band)
    gen = Generator(gist_shape(seed=0x6157, dim=128))
    X = gen.range(0, 6000)
    C = O.kmeans(X, 48, 6, 2)
    g, o = make_pair(128, 48, 6000, C, max_batch=6000, max_queries=300, tc=tc)
    ins(g, o, np.arange(6000), X)
    dele(g, o, np.arange(1, 6000, 5))
    Q = gen.queries(0, 300)
    for k, npb in ((10, 8), (1, 1), (32, 48), (17, 3)):
        assert srch(g, o, Q, k, npb, exact=False) <= 3
    # scaled inputs: large norms (||q||^2 + ||x||^2 >= 2^24 forces the re-rank even on integers)
    Xi = np.rint(X * 1000).astype(np.float32)
    g2, o2 = make_pair(128, 48, 6000, np.rint(C * 1000).astype(np.float32), max_batch=6000, max_queries=300, tc=tc)
    ins(g2, o2, np.arange(6000), Xi)
    assert srch(g2, o2, np.rint(Q * 1000).astype(np.float32), 10, 8, exact=False) <= 3


def test_no_scan_copy_flag():
    # SIVF_CFG_NO_SCAN_COPY: the paper's footprint (no fp16 copy), search on CUDA cores, same results
    gen = Generator(sift_shape(seed=0x51F7))
    X = gen.range(0, 5000)
    C = O.kmeans(X, 32, 6, 4)
    g, o = make_pair(128, 32, 5000, C, max_batch=5000, max_queries=200, flags=S.CFG_NO_SCAN_COPY)
    g2, o2 = make_pair(128, 32, 5000, C, max_batch=5000, max_queries=200)
    ins(g, o, np.arange(5000), X)
    ins(g2, o2, np.arange(5000), X)
    dele(g, o, np.arange(0, 5000, 3))
    dele(g2, o2, np.arange(0, 5000, 3))
    Q = gen.queries(0, 200)
    assert srch(g, o, Q, 10, 8) == 0 and srch(g2, o2, Q, 10, 8) == 0
    s, s2 = g.stats(), g2.stats()
    # per slab in use: the fp16 copy (2 Dh B per slot) + the record's norm and id copies (8 B per slot)
    want = (2.0 * 128 + 8.0) * 32 * s2["slabs_in_use"] / (s2["live"] * (4.0 * 128 + 4.0))
    assert s["overhead_scan_copy"] == 0.0 and abs(s2["overhead_scan_copy"] - want) < 1e-12
    assert s["overhead_actual"] == s2["overhead_actual"] and g2.arena_bytes > g.arena_bytes


@pytest.mark.parametrize("tc", [True, False], ids=["tcgen05-scan", "simt-scan"])
def test_values_beyond_fp16_range(tc):
    # the tensor-core scan filters with an fp16 copy of the slabs and queries;
    # values with |v| > 65504 have none: those slabs (flag) and queries re-rank
    # every valid slot exactly, so results match the oracle as for any data
    gen = Generator(gist_shape(seed=0x6158, dim=128))
    X = gen.range(0, 4000) * 1000.0
    X[::7] *= 100.0  # some vectors (hence some slabs) beyond the fp16 range
    X = X.astype(np.float32)
    C = O.kmeans(X, 32, 6, 3)
    g, o = make_pair(128, 32, 4000, C, max_batch=4000, max_queries=200, tc=tc)
    ins(g, o, np.arange(4000), X)
    dele(g, o, np.arange(2, 4000, 9))
    Q = gen.queries(0, 200) * 1000.0
    Q[::5] *= 100.0  # and some queries
    Q = Q.astype(np.float32)
    for k, npb in ((10, 8), (5, 32)):
        assert srch(g, o, Q, k, npb, exact=False) <= 3


def test_sliding_window_scaled():
    gen = Generator(sift_shape(seed=0x51F7))
    W, B, steps = 20000, 1000, 25
    C = O.kmeans(gen.train(4000), 64, 10, 9)
    cap = W + B * (steps + 1)
    g, o = make_pair(128, 64, cap, C, num_slabs=S.num_slabs_for(W, 64) + 2 * (B // 32 + 64), max_batch=W,
                     max_queries=100)
    ins(g, o, np.arange(W), gen.range(0, W))
    for t in range(steps):
        new = np.arange(W + t * B, W + (t + 1) * B)
        old = np.arange(t * B, (t + 1) * B)
        Q = gen.queries(t * 100, 100)
        dist, ids, status, ndel = g.sliding_window_step(T(new, torch.int64), T(gen.range(new[0], B)),
                                                        T(old, torch.int64), T(Q), 10, 16)
        ost, _ = o.insert(new, gen.range(new[0], B))
        assert np.array_equal(status.cpu().numpy()[:B], ost)
        assert int(ndel.item()) == o.delete(old) == B
        od, oi, _ = o.search(Q, 10, 16)
        assert np.array_equal(ids.cpu().numpy(), oi) and np.array_equal(dist.cpu().numpy(), od)
        o.reclaim()
        check_state(g, o, f"step {t}")
        assert g.stats()["live"] == W


def test_full_size_sift1m_step_sampled():
    # BASELINE configs[1] at full size, in the launch configuration bench.py times:
    # 1M x 128 SIFT-shaped, nlist 1024, one sliding step (insert 10k + delete the 10k
    # oldest + search 10k queries at k = 10, nprobe = 32 through sivf_sliding_window_step).
    # Every one of the 1M + 10k assignments and the whole mutation state are compared
    # bit-exact with the oracle; the search on a sample of 500 queries (integer data:
    # ids and distances exact).
    N, NL, B, NQ = 1_000_000, 1024, 10_000, 10_000
    O.set_threads(os.cpu_count() or 1)
    gen = Generator(sift_shape(seed=0x51F7))
    C = gen.range(1 << 41, NL)  # quantizer: sampled points (parity does not depend on training)
    g, o = make_pair(128, NL, N + B, C, num_slabs=S.num_slabs_for(N, NL), max_batch=100_000, max_queries=NQ,
                     max_k=32, max_nprobe=128)
    for b0 in range(0, N, 100_000):
        ins(g, o, np.arange(b0, b0 + 100_000), gen.range(b0, 100_000))
    check_state(g, o, "built")
    new, old = np.arange(N, N + B), np.arange(0, B)
    Xn, Q = gen.range(N, B), gen.queries(0, NQ)
    dist, ids, status, ndel = g.sliding_window_step(T(new, torch.int64), T(Xn), T(old, torch.int64), T(Q), 10, 32)
    ost, _ = o.insert(new, Xn)
    assert np.array_equal(status.cpu().numpy()[:B], ost)
    assert int(ndel.item()) == o.delete(old) == B
    o.reclaim()
    check_state(g, o, "after the step")
    sample = np.random.default_rng(11).choice(NQ, 500, replace=False)
    od, oi, _ = o.search(Q[sample], 10, 32)
    assert np.array_equal(ids.cpu().numpy()[sample], oi)
    assert np.array_equal(dist.cpu().numpy()[sample], od)


def test_full_size_gist1m_mutations_sampled():
    # BASELINE configs[2] at full size: 1M x 960 GIST-shaped float data, nlist 1024; a
    # 10k delete batch and a 10k insert batch; 1M + 10k assignments and the mutation
    # state bit-exact; k = 100, nprobe = 32 search on 100 sampled queries (float data:
    # distances within 1e-4 relative, id differences only at near-ties)
    N, NL, B = 1_000_000, 1024, 10_000
    O.set_threads(os.cpu_count() or 1)
    gen = Generator(gist_shape(seed=0x6157, dim=960))
    C = gen.range(1 << 41, NL)
    g, o = make_pair(960, NL, N + B, C, num_slabs=S.num_slabs_for(N + B, NL), max_batch=100_000, max_queries=100,
                     max_k=128, max_nprobe=128)
    for b0 in range(0, N, 100_000):
        ins(g, o, np.arange(b0, b0 + 100_000), gen.range(b0, 100_000))
    dele(g, o, np.arange(0, N, 100)[:B])
    ins(g, o, np.arange(N, N + B), gen.range(N, B))
    o.reclaim()
    g.reclaim()
    check_state(g, o, "gist 1M")
    Q = gen.queries(0, 100)
    assert srch(g, o, Q, 100, 32, exact=False) <= 3


def test_sliding_window_step_graph_replay():
    # SIVF_OPT_STEP_GRAPH: repeat calls with the same buffers replay one captured CUDA
    # graph; each replay must read the current inputs and index state (bit-exact vs the
    # oracle every step), a new signature (k, nprobe) or an option change recaptures
    gen = Generator(sift_shape(seed=0x51F7))
    W, B = 20000, 1000
    C = O.kmeans(gen.train(4000), 64, 10, 9)
    cap = W + B * 14
    g, o = make_pair(128, 64, cap, C, num_slabs=S.num_slabs_for(W, 64) + 2 * (B // 32 + 64), max_batch=W,
                     max_queries=100)
    ins(g, o, np.arange(W), gen.range(0, W))
    new_d = torch.empty(B, dtype=torch.int64, device="cuda")
    x_d = torch.empty(B, 128, device="cuda")
    old_d = torch.empty(B, dtype=torch.int64, device="cuda")
    q_d = torch.empty(100, 128, device="cuda")
    st_d = torch.empty(B, dtype=torch.int32, device="cuda")
    nd_d = torch.empty(1, dtype=torch.int64, device="cuda")
    outs = {kk: (torch.empty(100, kk, device="cuda"), torch.empty(100, kk, dtype=torch.int64, device="cuda"))
            for kk in (10, 16)}
    launches = []
    for t in range(13):
        k, npb = (10, 16) if t < 6 else (16, 8)
        if t == 9:
            g.set_option(S.OPT_RANK_SPLIT, 0)  # options epoch: recapture
        new, old = np.arange(W + t * B, W + (t + 1) * B), np.arange(t * B, (t + 1) * B)
        new_d.copy_(T(new, torch.int64))
        x_d.copy_(T(gen.range(new[0], B)))
        old_d.copy_(T(old, torch.int64))
        q_d.copy_(T(gen.queries(t * 100, 100)))
        l0 = g.launch_count()
        dist, ids, status, ndel = g.sliding_window_step(new_d, x_d, old_d, q_d, k, npb,
                                                        out=(outs[k][0], outs[k][1], st_d, nd_d))
        launches.append(g.launch_count() - l0)
        ost, _ = o.insert(new, gen.range(new[0], B))
        assert np.array_equal(status.cpu().numpy()[:B], ost)
        assert int(ndel.item()) == o.delete(old) == B
        od, oi, _ = o.search(gen.queries(t * 100, 100), k, npb)
        assert np.array_equal(ids.cpu().numpy(), oi) and np.array_equal(dist.cpu().numpy(), od), f"step {t}"
        o.reclaim()
        check_state(g, o, f"step {t}")
    assert min(launches) > 0 and len(set(launches[1:6])) == 1  # replays count the captured kernels


def test_merge_topk_matches_oracle():
    rng = np.random.default_rng(8)
    G, nq, k = 4, 50, 10
    d = np.sort(rng.integers(0, 1000, (G, nq, k)).astype(np.float32), axis=2)
    ids = rng.permutation(G * nq * k).reshape(G, nq, k).astype(np.int64)
    ids[1, :, 7:] = -1
    d[1, :, 7:] = np.inf
    gd, gi = S.merge_topk(T(d), T(ids))
    od, oi = O.merge_topk(d, ids, k)
    assert np.array_equal(gi.cpu().numpy(), oi) and np.array_equal(gd.cpu().numpy(), od)


def test_att_encoding_and_slot_uniqueness():
    rng = np.random.default_rng(9)
    X = rng.standard_normal((500, 8)).astype(np.float32)
    C = rng.standard_normal((5, 8)).astype(np.float32)
    g, o = make_pair(8, 5, 500, C)
    ins(g, o, np.arange(500), X)
    att = g.dump_att().cpu().numpy().view(np.uint64)
    slab, slot = att >> np.uint64(32), att & np.uint64(0xFFFFFFFF)
    assert (slot < 32).all() and (slab < g.cfg.num_slabs).all()  # Eq. att_encoding
    coords = set(zip(slab.tolist(), slot.tolist()))
    assert len(coords) == 500  # slot exclusivity
    dele(g, o, np.arange(100))
    att = g.dump_att().cpu().numpy().view(np.uint64)
    assert (att[:100] == np.uint64(0xFFFFFFFFFFFFFFFF)).all()  # INVALID sentinel


# ------------------------------------------------------------------ tensor-core coarse quantisation (a3, a7)
@pytest.mark.parametrize("coarse", [True, False], ids=["tcgen05-coarse", "simt-coarse"])
def test_coarse_sift_shaped_nlist1024(coarse):
    # BJ configs[1] geometry: nlist=1024, nprobe=32; assignments and probe sets bit-exact
    gen = Generator(sift_shape(seed=0x51F7))
    X = gen.range(0, 20000)
    rng = np.random.default_rng(11)
    C = (X[rng.choice(20000, 1024, replace=False)] + rng.integers(-3, 4, (1024, 128))).astype(np.float32)
    g, o = make_pair(128, 1024, 20000, C, max_batch=10000, max_queries=1000, max_nprobe=128, coarse=coarse)
    ins(g, o, np.arange(10000), X[:10000])  # 10k batch: assignment parity
    ins(g, o, np.arange(10000, 20000), X[10000:])
    Q = gen.queries(0, 1000)
    for npb in (1, 8, 32, 33, 128):  # 33/128 exercise the CUDA-core fallback of the probe selection
        srch(g, o, Q, 10, npb)
    check_state(g, o)


def test_coarse_gist_shaped_d960_float():
    gen = Generator(gist_shape(seed=0x6157))
    X = gen.range(0, 3000)
    rng = np.random.default_rng(12)
    C = X[rng.choice(3000, 300, replace=False)] * np.float32(1.001)
    g, o = make_pair(960, 300, 3000, C, max_batch=3000, max_queries=200)
    ins(g, o, np.arange(3000), X)
    Q = gen.queries(0, 200)
    for npb in (1, 7, 32):
        gd, gi, gp = g.search(T(Q), 10, npb, return_probes=True)
        op = np.stack([np.sort(O.probe(C, q, npb)) for q in Q])
        assert np.array_equal(np.sort(gp.cpu().numpy(), axis=1), op)
    check_state(g, o)


def test_coarse_exact_ties_and_band_overflow():
    # every centroid at exactly the same distance from the query (sign flips /
    # permutations of one integer vector): the whole nlist is inside the band,
    # the candidate buffer overflows, and the full exact re-rank must return the
    # lowest list indices (reading C2/C3)
    rng = np.random.default_rng(13)
    v = rng.integers(1, 20, 32).astype(np.float32)
    C = np.stack([rng.permutation(v) * rng.choice([-1.0, 1.0], 32) for _ in range(1024)]).astype(np.float32)
    g, o = make_pair(32, 1024, 100, C, max_batch=64, max_queries=8, max_nprobe=64)
    Z = np.zeros((8, 32), np.float32)
    st, ls = g.insert(T(np.arange(8), torch.int64), T(Z))
    assert (ls.cpu().numpy() == 0).all()
    _, _, p = g.search(T(Z), 1, 32, return_probes=True)
    assert (np.sort(p.cpu().numpy(), axis=1) == np.arange(32)).all()
    # near-ties 1 ulp apart inside the band (integer data, exact distances)
    q = rng.integers(0, 100, (4, 32)).astype(np.float32)
    C2 = np.repeat(q[:1], 300, axis=0)
    C2[:, 0] += np.arange(300, dtype=np.float32) % 3  # distances 0, 1, 4 repeating
    g2, o2 = make_pair(32, 300, 100, C2.astype(np.float32), max_batch=64, max_queries=8, max_nprobe=64)
    ins(g2, o2, np.arange(4), q)
    srch(g2, o2, q, 5, 32)


# ------------------------------------------------------------------ k-means (a1)
def test_train_centroids_bitexact():
    gen = Generator(sift_shape(seed=0x7111))
    Xt = gen.train(6000)
    for nlist, it, seed in ((1, 3, 1), (64, 10, 0x7111), (100, 4, 5)):
        g = S.Index(128, nlist, 10, 64, max_batch=16, max_queries=16, max_train=6000, seed=seed)
        g.train(T(Xt), niter=it)
        Cg = g.get_centroids().cpu().numpy()
        Co = O.kmeans(Xt, nlist, it, seed)
        assert np.array_equal(Cg, Co), f"k-means differs (nlist={nlist}): max |d| {np.abs(Cg - Co).max()}"


def test_train_spec_4_points_and_empty_clusters():
    P = np.array([[0, 0], [0, 1], [10, 10], [10, 11]], np.float32)
    g = S.Index(2, 2, 10, 8, max_batch=4, max_queries=4, max_train=4, seed=3)
    g.train(T(P), niter=5)
    got = sorted(map(tuple, g.get_centroids().cpu().numpy().tolist()))
    assert got == [(0.0, 0.5), (10.0, 10.5)]
    X = np.array([[0, 0]] * 6 + [[50, 50], [51, 50]], np.float32)
    g = S.Index(2, 4, 10, 8, max_batch=8, max_queries=8, max_train=8, seed=3)
    g.train(T(X), niter=4)
    assert np.array_equal(g.get_centroids().cpu().numpy(), O.kmeans(X, 4, 4, 3))
