"""GPU-vs-oracle checkers (SURVEY §8(c) "Checkers"), used by the -m gpu tests."""
from __future__ import annotations

import numpy as np

import oracle as O


def gpu_state(ix):
    loi, lpl, viol = ix.dump_state()
    return loi.cpu().numpy(), lpl.cpu().numpy(), int(viol.item())


def check_state(ix, ref: "O.Index", what: str = ""):
    """Mutation state, bit-exact: list_of_id, live_per_list, counters, invariants."""
    g_loi, g_lpl, viol = gpu_state(ix)
    o_loi, o_lpl = ref.dump_state()
    assert viol == 0, f"{what}: {viol} invariant violations (K10)"
    if not np.array_equal(g_loi, o_loi):
        bad = np.nonzero(g_loi != o_loi)[0][:10]
        raise AssertionError(f"{what}: list_of_id differs at {bad.tolist()}: gpu {g_loi[bad].tolist()} "
                             f"oracle {o_loi[bad].tolist()}")
    assert np.array_equal(g_lpl, o_lpl), f"{what}: live_per_list differs"
    gs, os_ = ix.stats(), ref.stats()
    for key in ("live", "inserted", "deleted", "slabs_in_use", "pool_exhausted_items"):
        assert gs[key] == os_[key], f"{what}: stats[{key}] gpu {gs[key]} oracle {os_[key]}"
    assert gs["device_errors"] == 0


def check_search(g, o, exact: bool, ref=None, Q=None, rel: float = 1e-4, what: str = ""):
    """g, o = (dist [nq,k], ids [nq,k], probes [nq,nprobe]) numpy (GPU, oracle).
    SURVEY §8(c) "Search, per query":
      - probe sets equal;
      - exact=True (integer-valued data): ids and distances identical;
      - otherwise: sorted distance lists agree within rel; every GPU id is live,
        lies in a probed list and is unique, and its reported distance is within
        rel of dist64(q, x_id) (needs ref = the oracle Index holding the same
        state, and Q); every id in R xor O is a near-tie of the k-th distance."""
    gd, gi, gp = g
    od, oi, op = o
    nq, k = od.shape
    for q in range(nq):
        assert set(gp[q].tolist()) == set(op[q].tolist()), f"{what}: probe set differs for query {q}"
    if exact:
        assert np.array_equal(gi, oi), f"{what}: ids differ: first rows {np.nonzero((gi != oi).any(1))[0][:5]}"
        assert np.array_equal(gd, od), f"{what}: distances differ"
        return 0
    loi = ref.dump_state()[0] if ref is not None else None
    exemptions = 0
    for q in range(nq):
        live_o = oi[q] >= 0
        assert ((gi[q] >= 0) == live_o).all(), f"{what}: padding differs for query {q}"
        m = live_o
        assert np.all(np.abs(gd[q][m] - od[q][m]) <= rel * np.maximum(od[q][m], 1e-30)), \
            f"{what}: distances out of tolerance for query {q}: {gd[q][m]} vs {od[q][m]}"
        assert len(set(gi[q][m].tolist())) == m.sum(), f"{what}: duplicate ids for query {q}"
        if ref is not None:
            probed = set(op[q].tolist())
            for j in np.nonzero(m)[0]:
                i = int(gi[q][j])
                lid = i // ref.shard_count
                assert i % ref.shard_count == ref.shard_rank and 0 <= lid < len(loi) and loi[lid] >= 0, \
                    f"{what}: query {q} returned id {i}, which is not live"
                assert int(loi[lid]) in probed, f"{what}: query {q} id {i} is in list {loi[lid]}, not probed"
                d64 = O.dist64(Q[q], ref.get_vector(i))
                assert abs(float(gd[q][j]) - d64) <= rel * max(d64, 1e-30), \
                    f"{what}: query {q} id {i}: reported {gd[q][j]} vs dist64 {d64}"
        diff = set(gi[q][m].tolist()) ^ set(oi[q][m].tolist())
        if diff:
            kth = od[q][m][-1]
            for i in diff:
                # the id's reported distance (either side) must be a near-tie with the k-th distance
                dd = gd[q][gi[q] == i] if (gi[q] == i).any() else od[q][oi[q] == i]
                assert abs(float(dd[0]) - kth) <= rel * max(kth, 1e-30), \
                    f"{what}: query {q} id {i} differs and is not a near-tie"
            exemptions += 1
    return exemptions


def check_assign(g_list, ref_C, X, ok_mask):
    """Assignments bit-exact (tie exemption only within 1e-5 relative, BJ)."""
    o_list = O.assign(ref_C, X)
    mism = np.nonzero((g_list != o_list) & ok_mask)[0]
    for i in mism:
        dg = O.dist32(X[i], ref_C[g_list[i]])
        do = O.dist32(X[i], ref_C[o_list[i]])
        assert dg - do <= 1e-5 * max(do, 1.1754944e-38), f"assignment of row {i} differs beyond the tie tolerance"
    return len(mism)
