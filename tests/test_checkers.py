"""The GPU-vs-oracle checker itself (tests/checkers.py), on oracle data only: a
result that is wrong in the ways §8(c) lists must be rejected even on float data
where the id comparison allows near-ties."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from datagen import Generator, gist_shape
from tests.checkers import check_search


def _setup():
    gen = Generator(gist_shape(seed=0x6157, dim=32))
    X = gen.range(0, 3000)
    C = O.kmeans(X, 16, 4, 1)
    o = O.Index(32, 16, 3000)
    o.set_centroids(C)
    o.insert(np.arange(3000), X)
    o.delete(np.arange(0, 3000, 4))
    Q = gen.queries(0, 20)
    return o, Q, X


def test_checker_accepts_the_oracle_itself():
    o, Q, _ = _setup()
    r = o.search(Q, 10, 4)
    assert check_search(r, r, exact=False, ref=o, Q=Q) == 0


def test_checker_rejects_dead_id_with_plausible_distance():
    o, Q, X = _setup()
    d, i, p = o.search(Q, 10, 4)
    gi = i.copy()
    # replace the last id of query 0 by a deleted id (multiple of 4) from a probed list
    # with the same reported distance: the distance comparison alone cannot see it
    loi_all = O.assign(O.kmeans(X, 16, 4, 1), X)
    dead = next(int(j) for j in range(0, 3000, 4) if loi_all[j] in set(p[0].tolist()) and j not in gi[0])
    gi[0, -1] = dead
    with pytest.raises(AssertionError, match="not live"):
        check_search((d, gi, p), (d, i, p), exact=False, ref=o, Q=Q)


def test_checker_rejects_unprobed_id_and_wrong_distance():
    o, Q, X = _setup()
    d, i, p = o.search(Q, 10, 4)
    loi, _ = o.dump_state()
    probed = set(p[0].tolist())
    other = next(int(j) for j in range(3000) if loi[j] >= 0 and loi[j] not in probed)
    gi = i.copy()
    gi[0, -1] = other
    with pytest.raises(AssertionError, match="not probed"):
        check_search((d, gi, p), (d, i, p), exact=False, ref=o, Q=Q)
    gd = d.copy()
    gd[1, 0] = np.nextafter(gd[1, 0], np.float32(np.inf)) * np.float32(1.001)  # beyond 1e-4
    with pytest.raises(AssertionError):
        check_search((gd, i, p), (d, i, p), exact=False, ref=o, Q=Q)
    gi = i.copy()
    gi[2, 1] = gi[2, 0]
    with pytest.raises(AssertionError, match="duplicate"):
        check_search((d, gi, p), (d, i, p), exact=False, ref=o, Q=Q)
