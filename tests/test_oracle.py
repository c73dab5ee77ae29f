"""Pins for the CPU oracle (no GPU).  Each test ties an oracle function to
something other than itself: a value printed in PAPER.md/SPEC.md, a closed
form, an invariant, or brute force in exact arithmetic on tiny inputs.
"""
from __future__ import annotations

import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
from datagen import Generator, sift_shape, gist_shape

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _read_golden(name):
    rows = []
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


def exact_sqdist(a, b) -> Fraction:
    return sum((Fraction(float(x)) - Fraction(float(y))) ** 2 for x, y in zip(a, b))


# ---------------------------------------------------------------- dist32 (Eq. l2)
def test_dist32_integer_data_is_exact():
    # SIFT-shaped integer data: every partial sum is an integer < 2^24, so the
    # fp32 sum equals the exact integer.
    rng = np.random.default_rng(1)
    for _ in range(50):
        a = rng.integers(0, 256, 128).astype(np.float32)
        b = rng.integers(0, 256, 128).astype(np.float32)
        exact = int(((a.astype(np.int64) - b.astype(np.int64)) ** 2).sum())
        assert O.dist32(a, b) == float(exact)
        assert O.dist64(a, b) == float(exact)


def test_dist32_error_bound_on_float_data():
    # Higham: a sum of D non-negative rounded terms has relative error <= gamma_{D+1}
    rng = np.random.default_rng(2)
    u = 2.0**-24
    for d in (2, 16, 128, 960):
        gamma = (d + 1) * u / (1 - (d + 1) * u)
        for _ in range(5):
            a = rng.standard_normal(d).astype(np.float32)
            b = rng.standard_normal(d).astype(np.float32)
            ex = exact_sqdist(a, b)
            got = Fraction(O.dist32(a, b))
            assert abs(got - ex) <= Fraction(gamma) * ex


def test_dist32_is_unfused_sequential():
    # Not a pin (same formula): guards against FMA contraction sneaking into the build.
    rng = np.random.default_rng(3)
    a = rng.standard_normal(64).astype(np.float32)
    b = rng.standard_normal(64).astype(np.float32)
    s = np.float32(0)
    for x, y in zip(a, b):
        t = np.float32(x - y)
        s = np.float32(s + np.float32(t * t))
    assert O.dist32(a, b) == s


# ---------------------------------------------------------------- assign / probe
def test_assign_spec_examples():
    C = np.array([[0, 0], [10, 10]], np.float32)
    assert O.assign(C, [[1, 1]])[0] == 0
    # equidistant from lists 2 and 5 -> 2 (tie to lowest index)
    C6 = np.array([[100, 100], [50, -50], [1, 0], [70, 70], [-40, 40], [-1, 0]], np.float32)
    assert O.assign(C6, [[0, 0]])[0] == 2


def test_assign_matches_exact_argmin():
    rng = np.random.default_rng(4)
    C = rng.standard_normal((64, 16)).astype(np.float32)
    X = rng.standard_normal((500, 16)).astype(np.float32)
    got = O.assign(C, X)
    D = ((X[:, None, :].astype(np.float64) - C[None, :, :]) ** 2).sum(-1)
    srt = np.sort(D, axis=1)
    sep = srt[:, 1] - srt[:, 0] > 1e-4 * srt[:, 0]  # well separated: rounding cannot flip
    assert sep.sum() > 450
    assert np.array_equal(got[sep], D.argmin(1)[sep])


def test_probe_properties():
    rng = np.random.default_rng(5)
    C = rng.standard_normal((32, 8)).astype(np.float32)
    for _ in range(20):
        q = rng.standard_normal(8).astype(np.float32)
        full = O.probe(C, q, 32)
        assert sorted(full.tolist()) == list(range(32))  # S:205 permutation
        assert O.probe(C, q, 1)[0] == O.assign(C, q[None])[0]
        d = ((C.astype(np.float64) - q) ** 2).sum(1)
        order = np.argsort(d, kind="stable")
        gaps = np.diff(np.sort(d))
        if np.all(gaps[:5] > 1e-4 * np.sort(d)[1:6]):
            assert full[:5].tolist() == order[:5].tolist()


def test_probe_tie_order_by_index():
    # four centroids equidistant from the origin: order must be by index (C3)
    C = np.array([[0, 2], [2, 0], [0, -2], [-2, 0], [5, 5]], np.float32)
    assert O.probe(C, np.zeros(2, np.float32), 5).tolist() == [0, 1, 2, 3, 4]


# ---------------------------------------------------------------- search
def test_search_spec_worked_example():
    rows = _read_golden("spec_search_example.txt")
    dim = int(rows[0][1])
    vecs = [(int(r[1]), [float(x) for x in r[2:]]) for r in rows if r[0] == "vector"]
    q = [float(x) for x in next(r for r in rows if r[0] == "query")[1:]]
    k = int(next(r for r in rows if r[0] == "k")[1])
    expect = [(int(r[1]), float(r[2])) for r in rows if r[0] == "expect"]
    ix = O.Index(dim, 1, 16)
    ix.set_centroids(np.zeros((1, dim), np.float32))
    st, _ = ix.insert([v[0] for v in vecs], np.array([v[1] for v in vecs], np.float32))
    assert (st == O.ST_OK).all()
    d, i, _ = ix.search(np.array([q], np.float32), k, 1)
    assert [(int(a), float(b)) for a, b in zip(i[0], d[0])] == expect


def _int_index(seed=0, n=2000, d=16, nlist=64):
    rng = np.random.default_rng(seed)
    X = rng.integers(0, 32, (n, d)).astype(np.float32)
    C = X[rng.choice(n, nlist, replace=False)] + 0.5
    ix = O.Index(d, nlist, n)
    ix.set_centroids(C)
    ids = np.arange(n)
    st, _ = ix.insert(ids, X)
    assert (st == 0).all()
    return ix, X, C, rng


def _exact_topk(Q, X, ids, k):
    D = ((Q[:, None, :].astype(np.int64) - X[None].astype(np.int64)) ** 2).sum(-1)
    out_d, out_i = [], []
    for r in range(Q.shape[0]):
        order = np.lexsort((ids, D[r]))[:k]
        out_d.append(D[r][order].astype(np.float32))
        out_i.append(ids[order])
    return np.array(out_d), np.array(out_i)


def test_full_probe_equals_bruteforce_exactly():
    # S:557 oracle-equivalence suite: N=2000, d=16, nlist=64, 100 queries, k=10, nprobe=64
    ix, X, C, rng = _int_index()
    Q = rng.integers(0, 32, (100, 16)).astype(np.float32)
    d, i, P = ix.search(Q, 10, 64)
    ed, ei = _exact_topk(Q, X, np.arange(2000), 10)
    assert np.array_equal(i, ei) and np.array_equal(d, ed)
    bd, bi = ix.bruteforce(Q, 10)
    assert np.array_equal(bi, ei) and np.array_equal(bd, ed)


def test_search_partial_probe_is_subset_topk():
    ix, X, C, rng = _int_index(seed=7)
    Q = rng.integers(0, 32, (50, 16)).astype(np.float32)
    d, i, P = ix.search(Q, 10, 4)
    lists = O.assign(C, X)
    for r in range(50):
        mask = np.isin(lists, P[r])
        ed, ei = _exact_topk(Q[r:r + 1], X[mask], np.arange(2000)[mask], 10)
        assert np.array_equal(i[r], ei[0]) and np.array_equal(d[r], ed[0])


def test_search_all_deleted_and_k_gt_live():
    ix, X, C, rng = _int_index(seed=8, n=100, nlist=4)
    q = X[:1]
    assert ix.delete(np.arange(97)) == 97
    d, i, _ = ix.search(q, 5, 4)
    live = np.arange(97, 100)
    ed, ei = _exact_topk(q, X[live], live, 3)
    assert i[0, :3].tolist() == ei[0].tolist() and (i[0, 3:] == -1).all() and np.isinf(d[0, 3:]).all()
    assert ix.delete(live) == 3
    d, i, _ = ix.search(q, 5, 4)
    assert (i == -1).all() and np.isinf(d).all()


# ---------------------------------------------------------------- insert / delete state
def test_insert_delete_semantics_spec():
    ix = O.Index(2, 1, 10)
    ix.set_centroids(np.zeros((1, 2), np.float32))
    X = np.arange(20, dtype=np.float32).reshape(10, 2)
    st, _ = ix.insert([0, 1, 1, 11, -1], X[:5])  # in-batch dup, out of range
    assert st.tolist() == [O.ST_OK, O.ST_OK, O.ST_DUPLICATE, O.ST_ID_OUT_OF_RANGE, O.ST_ID_OUT_OF_RANGE]
    st, _ = ix.insert([1], X[:1])  # live duplicate
    assert st.tolist() == [O.ST_DUPLICATE]
    assert ix.delete([1, 1, 5, 99]) == 1  # duplicates counted once, absent/OOR no-ops
    assert ix.delete([1]) == 0  # idempotent
    st, _ = ix.insert([1], X[:1])  # re-insert after delete
    assert st.tolist() == [O.ST_OK]
    s = ix.stats()
    assert s["live"] == s["inserted"] - s["deleted"] == 2


def test_state_invariants_random_ops():
    rng = np.random.default_rng(9)
    n, d, nlist = 3000, 8, 16
    ix = O.Index(d, nlist, n)
    C = rng.standard_normal((nlist, d)).astype(np.float32)
    ix.set_centroids(C)
    live = set()
    X = rng.standard_normal((n, d)).astype(np.float32)
    ok_total, del_total = 0, 0
    for _ in range(20):
        ids = rng.integers(0, n, 200)
        st, ls = ix.insert(ids, X[ids])
        seen = set()
        for a, s in zip(ids, st):
            exp = O.ST_DUPLICATE if (a in live or a in seen) else O.ST_OK
            assert s == exp
            seen.add(a)
            if s == O.ST_OK:
                live.add(int(a))
                ok_total += 1
        dels = rng.integers(0, n, 150)
        c = ix.delete(dels)
        assert c == len(set(dels.tolist()) & live)
        live -= set(dels.tolist())
        del_total += c
        loi, lpl = ix.dump_state()
        assert set(np.nonzero(loi >= 0)[0].tolist()) == live  # every live id reachable exactly once
        assert lpl.sum() == len(live)
        lists = O.assign(C, X[sorted(live)])
        assert np.array_equal(loi[sorted(live)], lists)
        assert np.bincount(lists, minlength=nlist).tolist() == lpl.tolist()
        s = ix.stats()
        assert s["live"] == len(live) == ok_total - del_total


def test_slab_count_model_spec():
    ix = O.Index(2, 1, 100, num_slabs=10)
    ix.set_centroids(np.zeros((1, 2), np.float32))
    X = np.zeros((40, 2), np.float32)
    ix.insert([0], X[:1])
    assert ix.stats()["slabs_in_use"] == 1  # S:253 first insert -> one slab
    ix.insert(np.arange(1, 33), X[:32])
    assert ix.stats()["slabs_in_use"] == 2  # S:254 the 33rd insert opens a second slab


def test_pool_exhaustion_and_reclaim():
    # slab_factor 1.0 + single-list skew -> POOL_EXHAUSTED, then reclaim restores.
    ix = O.Index(2, 2, 1000, num_slabs=3)
    ix.set_centroids(np.array([[0, 0], [100, 100]], np.float32))
    X = np.zeros((200, 2), np.float32)
    st, _ = ix.insert(np.arange(100), X[:100])
    assert (st[:96] == O.ST_OK).all() and (st[96:] == O.ST_POOL_EXHAUSTED).all()
    assert ix.stats()["slabs_free"] == 0 and ix.stats()["pool_exhausted_items"] == 4
    assert ix.delete(np.arange(32, 64)) == 32  # the middle slab is full and dead
    assert ix.reclaim() == 1
    assert ix.stats()["slabs_free"] == 1
    st, _ = ix.insert(np.arange(100, 110), X[:10])
    assert (st == O.ST_OK).all()
    loi, lpl = ix.dump_state()
    assert lpl[0] == 64 + 10


def test_exhaustion_serves_lists_in_ascending_order():
    ix = O.Index(1, 2, 1000, num_slabs=3)
    ix.set_centroids(np.array([[0], [100]], np.float32))
    X = np.array([[100]] * 40 + [[0]] * 40, np.float32)
    st, ls = ix.insert(np.arange(80), X)
    # list 0 (items 40..79) is served first and takes 2 slabs; list 1 gets the
    # last slab: its first 32 items (batch order) succeed, the rest fail.
    assert (st[40:80] == 0).all()
    assert (st[:32] == 0).all() and (st[32:40] == O.ST_POOL_EXHAUSTED).all()


def test_memory_overhead_matches_paper():
    for row in _read_golden("paper_numbers.txt"):
        if row[0] == "overhead":
            d, pct = int(row[1]), float(row[2])
            ix = O.Index(d, 1, 1)
            assert round(100 * ix.stats()["overhead_paper"], 2) == pct
            assert ix.stats()["overhead_paper"] < 0.008  # BASELINE "<0.8%"


# ---------------------------------------------------------------- sharding (§8(e))
@pytest.mark.parametrize("G", [2, 4, 8])
def test_sharded_oracles_merge_equals_single(G):
    rng = np.random.default_rng(10 + G)
    n, d, nlist = 1500, 16, 32
    X = rng.integers(0, 64, (n, d)).astype(np.float32)
    C = X[:nlist] + 0.25
    one = O.Index(d, nlist, n)
    one.set_centroids(C)
    one.insert(np.arange(n), X)
    dels = rng.choice(n, 300, replace=False)
    one.delete(dels)
    shards = []
    for r in range(G):
        s = O.Index(d, nlist, n, shard_rank=r, shard_count=G)
        s.set_centroids(C)
        st, _ = s.insert(np.arange(n), X)
        assert ((st == O.ST_OK) == (np.arange(n) % G == r)).all()
        assert ((st == O.ST_WRONG_SHARD) == (np.arange(n) % G != r)).all()
        s.delete(dels)
        shards.append(s)
    Q = rng.integers(0, 64, (40, d)).astype(np.float32)
    d1, i1, _ = one.search(Q, 10, 8)
    parts = [s.search(Q, 10, 8) for s in shards]
    dm, im = O.merge_topk(np.stack([p[0] for p in parts]), np.stack([p[1] for p in parts]), 10)
    assert np.array_equal(im, i1) and np.array_equal(dm, d1)


# ---------------------------------------------------------------- recall
def test_recall_monotone_and_full_at_nlist():
    g = Generator(sift_shape(seed=0x7111))
    X = g.range(0, 3000)
    C = O.kmeans(X, 32, 5, 0x7111)
    ix = O.Index(128, 32, 3000)
    ix.set_centroids(C)
    ix.insert(np.arange(3000), X)
    Q = g.queries(0, 40)
    _, truth = ix.bruteforce(Q, 10)
    prev = -1.0
    for npb in (1, 2, 4, 8, 16, 32):
        _, i, _ = ix.search(Q, 10, npb)
        rec = np.mean([len(set(a) & set(b)) / 10 for a, b in zip(i, truth)])
        assert rec >= prev
        prev = rec
    assert prev == 1.0


# ---------------------------------------------------------------- k-means (a1)
def test_kmeans_nlist1_is_mean():
    rng = np.random.default_rng(11)
    X = rng.integers(0, 1000, (777, 5)).astype(np.float32)
    C = O.kmeans(X, 1, 3, 1)
    exact = [Fraction(int(X[:, k].astype(np.int64).sum()), 777) for k in range(5)]
    assert np.array_equal(C[0], np.array([float(e) for e in exact], np.float32))


def test_kmeans_spec_4_points():
    rows = _read_golden("spec_kmeans_4pt.txt")
    P = np.array([[float(x) for x in r[1:]] for r in rows if r[0] == "point"], np.float32)
    nlist = int(next(r for r in rows if r[0] == "nlist")[1])
    iters = int(next(r for r in rows if r[0] == "iters")[1])
    exp = sorted(tuple(float(x) for x in r[1:]) for r in rows if r[0] == "centroid")
    for seed in range(8):
        C = O.kmeans(P, nlist, iters, seed)
        assert sorted(tuple(map(float, c)) for c in C) == exp


def test_kmeans_deterministic_and_objective_nonincreasing():
    g = Generator(gist_shape(dim=32))
    X = g.range(0, 4000)
    C1, J = O.kmeans(X, 16, 8, 0xABC, with_objective=True)
    C2 = O.kmeans(X, 16, 8, 0xABC)
    assert np.array_equal(C1, C2)
    assert all(J[i + 1] <= J[i] * (1 + 1e-6) for i in range(len(J) - 1))


def test_kmeans_empty_cluster_reseed():
    # 6 identical points + 2 far points, nlist 4: duplicates force empty clusters;
    # every cluster must end non-empty and centroids stay finite.
    X = np.array([[0, 0]] * 6 + [[50, 50], [51, 50]], np.float32)
    C = O.kmeans(X, 4, 4, 3)
    assert np.isfinite(C).all()
    a = O.assign(C, X)
    assert len(set(a.tolist())) >= 3


def test_kmeans_init_hash_pinned():
    # init uses splitmix64: H(seed, i) = mix64(seed ^ mix64(i)); mix64(0) is the
    # first splitmix64 output for state 0 (tests/golden/paper_numbers.txt)
    row = next(r for r in _read_golden("paper_numbers.txt") if r[0] == "mix64")
    m0 = int(row[2])
    assert O.kmeans_hash(0, 0) != 0
    # mix64(0 ^ mix64(0)) computed from the pinned constant with Python ints:
    def mix(z):
        z = (z + 0x9E3779B97F4A7C15) & (2**64 - 1)
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
        return z ^ (z >> 31)
    assert mix(0) == m0
    assert O.kmeans_hash(0, 0) == mix(mix(0))


def _mix64(z):
    z = (z + 0x9E3779B97F4A7C15) & (2**64 - 1)
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
    return z ^ (z >> 31)


def _init_perm(n, nlist, seed):
    # reading C31 / SURVEY §8(c) step 9: partial Fisher-Yates, j = i + H(seed, i) mod (n - i),
    # H(s, i) = mix64(s ^ mix64(i)) (mix64 pinned by test_kmeans_init_hash_pinned)
    perm = list(range(n))
    for i in range(nlist):
        j = i + _mix64(seed ^ _mix64(i)) % (n - i)
        perm[i], perm[j] = perm[j], perm[i]
    return perm


def _empty_cluster_case(nlist, seed):
    """Hand-built 1-D data (2nd coordinate 0) with known initial centroids:
    X[perm[0]] = 0, X[perm[1..nlist)] = 100 (duplicates: clusters 2.. start empty),
    the other four points, in ascending index order, = 1, 90, 96, 104."""
    n = nlist + 4
    perm = _init_perm(n, nlist, seed)
    X = np.zeros((n, 2), np.float32)
    X[perm[0], 0] = 0.0
    for l in range(1, nlist):
        X[perm[l], 0] = 100.0
    rest = sorted(perm[nlist:])
    for i, v in zip(rest, (1.0, 90.0, 96.0, 104.0)):
        X[i, 0] = v
    return X


@pytest.mark.parametrize("seed", [3, 17, 0x51F7])
def test_kmeans_empty_cluster_rule_hand_derived(seed):
    # S:184 / reading C31: an empty cluster e (ascending) takes, from the LARGEST cluster
    # (ties: lowest list), its point FARTHEST from that cluster's centroid (ties: lowest
    # point index).  One iteration by hand, nlist = 3: c = (0, 100, 100); assignment
    # (ties to the lower list): cluster 0 = {0, 1}, cluster 1 = {100, 100, 90, 96, 104},
    # cluster 2 empty; the farthest member of cluster 1 from 100 is 90 (distance 100)
    # -> c = (0.5, (100+100+96+104)/4, 90) = (0.5, 100, 90).  Wrong readings give:
    # nearest point -> (0.5, 97.5, 100); smallest/first cluster -> (0, 100, 1).
    X = _empty_cluster_case(3, seed)
    C = O.kmeans(X, 3, 1, seed)
    assert C[:, 0].tolist() == [0.5, 100.0, 90.0] and (C[:, 1] == 0).all()
    # nlist = 4: c = (0, 100, 100, 100), clusters 2 and 3 empty, cluster 1 = {100 x3, 90,
    # 96, 104}.  e = 2: L = 1 (6 members) gives 90; e = 3: L = 1 again (5 vs 2), farthest
    # of {100 x3, 96, 104} from 100 is a tie 96 / 104 (distance 16) -> the lower point
    # index, which holds 96 (values placed in ascending index order)
    # -> c = (0.5, (100+100+100+104)/4, 90, 96) = (0.5, 101, 90, 96)
    # (the highest index instead would give (0.5, 99, 90, 104)).
    X4 = _empty_cluster_case(4, seed)
    C4 = O.kmeans(X4, 4, 1, seed)
    assert C4[:, 0].tolist() == [0.5, 101.0, 90.0, 96.0]


def test_topk_candidates_equals_search_on_probed_members():
    # the restricted scan used by the sampled H check: over exactly the live members of
    # the probed lists it must reproduce or_search (and pad with (+inf, -1))
    g = Generator(sift_shape(seed=0x100A, dim=16))
    X = g.range(0, 2000)
    C = O.kmeans(X, 32, 3, 5)
    o = O.Index(16, 32, 2000)
    o.set_centroids(C)
    o.insert(np.arange(2000), X)
    o.delete(np.arange(0, 2000, 3))
    loi, _ = o.dump_state()
    Q = g.queries(0, 10)
    d, i, p = o.search(Q, 10, 4)
    for q in range(10):
        mem = np.nonzero(np.isin(loi, p[q]))[0]
        dd, ii = O.topk_candidates(Q[q], X[mem], mem, 10)
        assert np.array_equal(dd, d[q]) and np.array_equal(ii, i[q])
    dd, ii = O.topk_candidates(Q[0], X[:3], np.array([5, 6, 7]), 5)
    assert ii[3:].tolist() == [-1, -1] and np.isinf(dd[3:]).all()
