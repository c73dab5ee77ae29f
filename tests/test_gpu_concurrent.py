"""NEXT-2: concurrent mutation + search across streams with the paper's
lock-free protocol (Alg. 2; publish protocol P:263-266).

* single stream: sivf_insert_concurrent's (list, live) state equals the oracle's
  (placement and slot order are nondeterministic, the state is not), duplicates /
  out-of-range / pool exhaustion / full directories give their statuses, the
  invariants hold, a quiescent reclaim returns leaked slabs;
* the SPEC publication suite: 8 writer views x 10k unique ids with
  id-derived integer payloads and 4 reader views searching at nprobe = nlist on
  12 streams at once: every hit's distance equals the exact distance to the
  payload f(hit id) (no torn payload), and afterwards live = 80k, every id is
  retrievable at distance 0 and the ATT is injective (no invariant violation);
* search overlapping delete: a hit for a deleted id is allowed only if the id was
  live when the search started (lazy eviction), never a garbage id.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle as O
import paper_2601_11808_b200 as S
from tests.test_gpu_parity import T, make_pair

pytestmark = pytest.mark.gpu

D = 32


def payload(ids: np.ndarray) -> np.ndarray:
    """Id-derived integer payload f(id): 6-bit values of a 64-bit mix of (id, d) (uniform;
    exact distances: every value < 64)."""
    ids = np.asarray(ids, np.int64).astype(np.uint64)[:, None]
    d = np.arange(D, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        z = ids * np.uint64(0x9E3779B97F4A7C15) + d * np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(31)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(29)
    return (z >> np.uint64(58)).astype(np.float32)


def exact_d(q: np.ndarray, x: np.ndarray) -> np.ndarray:
    return ((q.astype(np.float64) - x.astype(np.float64)) ** 2).sum(-1)


def centroids(nlist: int, seed: int = 5) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return payload(rng.choice(1 << 30, nlist, replace=False)) + 0.25


def test_insert_concurrent_single_stream_state_equals_oracle():
    nl, N = 16, 6000
    C = centroids(nl)
    g, o = make_pair(D, nl, N + 100, C, num_slabs=3 * S.num_slabs_for(N, nl), max_batch=4096, max_queries=256,
                     flags=S.CFG_CONCURRENT)
    X = payload(np.arange(N))
    # an ordinary batched insert first, then the concurrent phase on top of it
    st, _ = g.insert(T(np.arange(1000), torch.int64), T(X[:1000]))
    o.insert(np.arange(1000), X[:1000])
    with pytest.raises(S.SivfError):  # directories not prepared since the last quiescent mutation
        g.insert_concurrent(T(np.arange(1000, 1010), torch.int64), T(X[1000:1010]))
    g.reserve_directories(64)
    ids = np.concatenate([np.arange(1000, 4000), [5, 7, 1500, 1500, N + 1000, -3]])
    Xi = np.concatenate([X[1000:4000], X[[5, 7, 1500, 1500]], np.zeros((2, D), np.float32)])
    st, ls = g.insert_concurrent(T(ids, torch.int64), T(Xi))
    st, ls = st.cpu().numpy(), ls.cpu().numpy()
    assert (st[:3000] == S.ST_OK).all() or (st[:3000] != S.ST_OK).sum() == 1  # 1500 may lose to its duplicate
    assert st[3000] == S.ST_DUPLICATE and st[3001] == S.ST_DUPLICATE  # live since the batched insert
    assert sorted(st[[500, 3002, 3003]].tolist()).count(S.ST_OK) == 1  # three claims of id 1500: one wins
    assert st[3004] == S.ST_ID_OUT_OF_RANGE and st[3005] == S.ST_ID_OUT_OF_RANGE
    o.insert(np.arange(1000, 4000), X[1000:4000])
    want = O.assign(C, Xi[:3000])
    ok = st[:3000] == S.ST_OK
    assert np.array_equal(ls[:3000][ok], want[ok])
    loi, lpl, viol = g.dump_state()
    oloi, olpl = o.dump_state()
    assert int(viol.item()) == 0
    assert np.array_equal(loi.cpu().numpy(), oloi) and np.array_equal(lpl.cpu().numpy(), olpl)
    s = g.stats()
    assert s["live"] == 4000 and s["device_errors"] == 0
    print("leaked slabs", s["leaked_slabs"])
    # concurrent inserts interleave with deletes and searches on the same stream too
    g.delete(T(np.arange(0, 4000, 3), torch.int64))
    o.delete(np.arange(0, 4000, 3))
    Q = X[:64]
    gd, gi = g.search(T(Q), 10, nl)
    od, oi, _ = o.search(Q, 10, nl)
    assert np.array_equal(gi.cpu().numpy(), oi) and np.array_equal(gd.cpu().numpy(), od)


def test_insert_concurrent_pool_exhaustion_dir_full_and_leak_reclaim():
    nl = 4
    C = centroids(nl, 9)
    num_slabs = 40
    g, o = make_pair(D, nl, 5000, C, num_slabs=num_slabs, max_batch=4096, flags=S.CFG_CONCURRENT)
    g.reserve_directories(6)  # at most 6 new slabs per list while concurrent
    X = payload(np.arange(4000))
    st, ls = g.insert_concurrent(T(np.arange(4000), torch.int64), T(X))
    st = st.cpu().numpy()
    ok = st == S.ST_OK
    assert set(np.unique(st).tolist()) <= {S.ST_OK, S.ST_POOL_EXHAUSTED, S.ST_DIR_FULL}
    assert (~ok).any() and ok.sum() <= 4 * 8 * 32  # directories of cap max(8, len + 6) = 8 entries
    loi, lpl, viol = g.dump_state()
    assert int(viol.item()) == 0
    loi = loi.cpu().numpy()
    want = O.assign(C, X)
    assert np.array_equal(loi[:4000][ok], want[ok]) and (loi[:4000][~ok] == -1).all()
    s = g.stats()
    assert s["live"] == ok.sum()
    g.reclaim()  # quiescent: leaked slabs (if any) go back to the pool
    s2 = g.stats()
    assert s2["leaked_recycled"] == s["leaked_slabs"]
    assert int(g.dump_state()[2].item()) == 0


def _publication_run(seed: int, n_writers: int = 8, per_writer: int = 10_000, n_readers: int = 4,
                     batches: int = 10, searches: int = 12):
    nl = 128
    N = n_writers * per_writer
    # k-means centroids (balanced lists: random data points as centroids give hub lists in 32 dims)
    C = O.kmeans(payload(np.random.default_rng(seed).choice(N, 8192, replace=False)), nl, 8, seed)
    g = S.Index(D, nl, N + 16, S.num_slabs_for(N, nl, 1.3, 1.3), max_batch=per_writer // batches,
                max_queries=256, max_k=10, max_nprobe=nl, flags=S.CFG_CONCURRENT)
    g.set_centroids(T(C))
    g.reserve_directories(256)  # ~20 slabs per list get added while concurrent
    writers = [g.view() for _ in range(n_writers)]
    readers = [g.view() for _ in range(n_readers)]
    ws = [torch.cuda.Stream() for _ in range(n_writers)]
    rs = [torch.cuda.Stream() for _ in range(n_readers)]
    rng = np.random.default_rng(seed)
    order = rng.permutation(N)  # writer w owns ids order[w::n_writers]
    Xall = T(payload(np.arange(N)))
    idx_all = T(np.arange(N), torch.int64)
    torch.cuda.synchronize()
    statuses = []
    outs = []
    per = per_writer // batches
    qsets = [rng.integers(0, N, 256) for _ in range(n_readers * searches)]
    qts = [T(payload(q)) for q in qsets]
    for b in range(batches):
        for w in range(n_writers):
            with torch.cuda.stream(ws[w]):  # the ids' H2D copy must be ordered before the insert on ws[w]
                mine = T(order[w::n_writers][b * per:(b + 1) * per], torch.int64)
                st, _ = writers[w].insert_concurrent(mine, Xall[mine], stream=ws[w])
                statuses.append(st)
        for r in range(n_readers):
            if b < searches:
                with torch.cuda.stream(rs[r]):
                    dd, ii = readers[r].search(qts[r * searches + b], 10, nl, stream=rs[r])
                    outs.append((r * searches + b, dd, ii))
    torch.cuda.synchronize()
    # 1) no torn payload: every hit's distance is the exact distance to f(hit id)
    hits = 0
    for qi, dd, ii in outs:
        dd, ii = dd.cpu().numpy(), ii.cpu().numpy()
        Q = payload(qsets[qi])
        m = ii >= 0
        assert (ii[m] < N).all()
        want = exact_d(Q[:, None, :].repeat(10, 1)[m], payload(ii[m]))
        if not np.array_equal(dd[m].astype(np.float64), want):
            bad = np.nonzero(dd[m].astype(np.float64) != want)[0]
            qq = np.nonzero(m)[0][bad[:5]]
            info = []
            for j in bad[:5]:
                r_, c_ = np.argwhere(m)[j]
                info.append((int(qsets[qi][r_]), int(ii[r_, c_]), float(dd[r_, c_]), float(want[j]),
                             dd[r_].tolist(), ii[r_].tolist()))
            raise AssertionError(f"a hit's distance does not match its payload ({len(bad)} of {m.sum()} hits, "
                                 f"search {qi}): {info}")
        hits += int(m.sum())
    st = torch.cat(statuses).cpu().numpy()
    assert (st == S.ST_OK).all(), np.unique(st, return_counts=True)
    # 2) final state: live = N, every id retrievable at distance 0, ATT injective
    s = g.stats()
    assert s["live"] == N and s["device_errors"] == 0
    print(f"publication run {seed}: hits {hits}, leaked slabs {s['leaked_slabs']}")
    loi, lpl, viol = g.dump_state()
    loi = loi.cpu().numpy()
    if int(viol.item()) != 0:
        att = g.dump_att().cpu().numpy().view(np.uint64)
        live = att != np.uint64(0xFFFFFFFFFFFFFFFF)
        coords, counts = np.unique(att[live], return_counts=True)
        import ctypes
        vt = np.zeros(7, np.int64)
        S.lib().sivf_debug_violations(g._h, vt.ctypes.data_as(ctypes.c_void_p))
        raise AssertionError(f"{int(viol.item())} invariant violations (by type {vt.tolist()}); live ATT entries {int(live.sum())}, "
                             f"coordinates shared by 2+ ids: {int((counts > 1).sum())}, list_of_id == assign: "
                             f"{np.array_equal(loi[:N], O.assign(C, payload(np.arange(N))))}, stats {g.stats()}")
    assert np.array_equal(loi[:N], O.assign(C, payload(np.arange(N)))) and (loi[N:] == -1).all()
    for q0 in range(0, N, 256):
        q = np.arange(q0, min(N, q0 + 256))
        dd, ii = g.search(T(payload(q)), 1, nl)
        dd, ii = dd.cpu().numpy(), ii.cpu().numpy()
        assert (dd[:, 0] == 0).all()
        # the nearest is f(id) itself or an id with an identical payload (then equal distance 0)
        assert np.array_equal(exact_d(payload(q), payload(ii[:, 0])), np.zeros(len(q)))
    del writers, readers
    return hits


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_spec_publication_suite(seed):
    hits = _publication_run(seed)
    assert hits > 0


def test_search_overlapping_delete_is_lazy():
    nl, N = 32, 20000
    C = centroids(nl, 11)
    g = S.Index(D, nl, N, S.num_slabs_for(N, nl), max_batch=N, max_queries=512, max_k=10, max_nprobe=nl,
                flags=S.CFG_CONCURRENT)
    g.set_centroids(T(C))
    X = payload(np.arange(N))
    g.insert(T(np.arange(N), torch.int64), T(X))
    g.reserve_directories(8)
    dv, rv = g.view(), g.view()
    sd, sr = torch.cuda.Stream(), torch.cuda.Stream()
    gone = np.arange(0, N, 2)
    Q = X[np.arange(1, 512 * 2, 2)]  # queries equal to odd ids' payloads
    torch.cuda.synchronize()
    Qd, gone_d = T(Q), T(gone, torch.int64)
    torch.cuda.synchronize()
    with torch.cuda.stream(sr):
        dd, ii = rv.search(Qd, 10, nl, stream=sr)
    with torch.cuda.stream(sd):
        dv.delete(gone_d, stream=sd)
    torch.cuda.synchronize()
    ii = ii.cpu().numpy()
    dd = dd.cpu().numpy()
    assert ((ii >= 0) & (ii < N)).all()  # every hit was live when the search started
    assert np.array_equal(dd.astype(np.float64),
                          exact_d(Q[:, None, :].repeat(10, 1), payload(ii.ravel()).reshape(ii.shape + (D,))))
    s = g.stats()
    assert s["live"] == N - len(gone)
    d2, i2 = g.search(T(Q), 10, nl)
    assert not np.isin(i2.cpu().numpy(), gone).any()  # after the delete, no even id is returned
