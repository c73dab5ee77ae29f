"""GPU parity of the D > 128 GEMM scan (k_scan_gs.cu: split-fp16 tcgen05 scan, dense
distance rows, per-query selection; SIMT fallback for items beyond the dense buffer).
Float data: distances within 1e-4 relative of dist64 and id differences only at near-ties
(BASELINE.json north_star), every returned id live, in a probed list and unique
(tests/checkers.py::check_search)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle as O
import paper_2601_11808_b200 as S
from datagen import Generator, gist_shape
from tests.test_gpu_parity import T, dele, ins, make_pair, srch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dim", [200, 960])
def test_gs_scan_float_data(dim):
    # D = 200 pads the copy to 256 dims (4 chunks), D = 960 is GIST's 15 chunks;
    # lists of 5-6 slabs (ragged last group), k from 1 to 128
    gen = Generator(gist_shape(seed=0x6157, dim=dim))
    X = gen.range(0, 6000)
    C = O.kmeans(X[:3000], 32, 5, 2)
    g, o = make_pair(dim, 32, 6000, C, max_queries=300, max_nprobe=32, max_batch=6000)
    ins(g, o, np.arange(6000), X)
    dele(g, o, np.arange(0, 6000, 7))
    Q = gen.queries(0, 300)
    for k, npb in ((1, 1), (10, 4), (100, 8), (128, 32)):
        assert srch(g, o, Q, k, npb, exact=False) <= 3


@pytest.mark.parametrize("dim", [16, 100, 128])
def test_split_copy_flag_dim_le_128_float(dim):
    # SIVF_CFG_SPLIT_COPY: the split-fp16 copy and the GEMM scan at dim <= 128 (float
    # data: uniform [0, 1) as the paper's grids); the default fp16 copy is absent
    # (its tensor-core scan is not used)
    rng = np.random.default_rng(dim)
    X = rng.random((6000, dim), dtype=np.float32)
    C = O.kmeans(X[:3000], 32, 5, 4)
    g, o = make_pair(dim, 32, 6000, C, max_queries=300, max_nprobe=32, max_batch=6000, flags=S.CFG_SPLIT_COPY)
    ins(g, o, np.arange(6000), X)
    dele(g, o, np.arange(0, 6000, 5))
    Q = rng.random((300, dim), dtype=np.float32)
    for k, npb in ((1, 1), (10, 8), (32, 32), (100, 4)):
        assert srch(g, o, Q, k, npb, exact=False) <= 3
    d1, i1 = g.search(T(Q), 10, 8)
    g.set_option(S.OPT_TC_SCAN, 0)  # the CUDA-core scan of the same index
    d2, i2 = g.search(T(Q), 10, 8)
    assert np.allclose(d1.cpu().numpy(), d2.cpu().numpy(), rtol=1e-4, atol=1e-6)
    assert (i1 == i2).float().mean().item() > 0.99


def test_gs_scan_matches_simt_scan():
    # the same index searched by the GEMM scan and by the CUDA-core scan (OPT_TC_SCAN 0):
    # ids equal up to near-ties, distances within 1e-4 relative
    gen = Generator(gist_shape(seed=0x6159, dim=960))
    X = gen.range(0, 8000)
    C = O.kmeans(X[:4000], 16, 5, 3)
    g, o = make_pair(960, 16, 8000, C, max_queries=200, max_nprobe=16, max_batch=8000)
    ins(g, o, np.arange(8000), X)
    Q = T(gen.queries(0, 200))
    d1, i1 = g.search(Q, 50, 4)
    g.set_option(S.OPT_TC_SCAN, 0)
    d2, i2 = g.search(Q, 50, 4)
    d1, d2 = d1.cpu().numpy(), d2.cpu().numpy()
    assert np.allclose(d1, d2, rtol=1e-4, atol=0)
    same = (i1 == i2).float().mean().item()
    assert same > 0.99, same


def test_gs_fallback_long_list():
    # 3/4 of the vectors in list 1: its items exceed the dense buffer (sized for lists
    # up to twice the average) and take the CUDA-core fallback, the small lists stay
    # dense; with nprobe 2 a query can have one pair of each kind, merged per query
    rng = np.random.default_rng(21)
    D, NL, N = 160, 32, 20000
    C = np.zeros((NL, D), np.float32)
    C[:, 0] = np.arange(NL) * 1e4
    lst = np.where(np.arange(N) < 15000, 1, rng.integers(2, NL, N))
    X = (rng.random((N, D)) * 3).astype(np.float32)
    X[:, 0] += lst * 1e4
    g, o = make_pair(D, NL, N, C, max_queries=64, max_nprobe=2, max_batch=N)
    ins(g, o, np.arange(N), X)
    Q = (rng.random((64, D)) * 3).astype(np.float32)
    Q[:, 0] += np.where(np.arange(64) < 32, 1, rng.integers(2, NL, 64)) * 1e4 + 4e3
    for k, npb in ((10, 1), (100, 2)):
        assert srch(g, o, Q, k, npb, exact=False) <= 3


def test_gs_sliding_and_empty():
    # empty index, then a window that slides (dead slabs skipped, reclaim) on D = 256
    gen = Generator(gist_shape(seed=0x615A, dim=256))
    X = gen.range(0, 9000)
    C = O.kmeans(X[:3000], 16, 5, 4)
    g, o = make_pair(256, 16, 9000, C, max_queries=100, max_nprobe=16)
    Q = gen.queries(0, 100)
    d, i = g.search(T(Q), 10, 4)
    assert (i.cpu().numpy() == -1).all() and np.isinf(d.cpu().numpy()).all()
    for t in range(6):
        ins(g, o, np.arange(t * 1500, (t + 1) * 1500), X[t * 1500:(t + 1) * 1500])
        if t >= 2:
            dele(g, o, np.arange((t - 2) * 1500, (t - 1) * 1500))
        assert int(g.reclaim().item()) == o.reclaim()
        assert srch(g, o, Q, 20, 4, exact=False) <= 3
