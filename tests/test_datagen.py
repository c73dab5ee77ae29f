"""Pins for the seeded input generator (harness module shared by both sides)."""
import os

import numpy as np
import pytest

import datagen as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_mix64_reference_vector():
    rows = [l.split() for l in open(os.path.join(GOLD, "paper_numbers.txt")) if l.startswith("mix64")]
    assert G.mix64(int(rows[0][1])) == int(rows[0][2])


def test_n01_moments():
    v = np.array([G.N01(123, 7, j) for j in range(20000)])
    assert abs(v.mean()) < 0.03 and abs(v.var() - 1.0) < 0.05
    assert v.min() >= -2 * 1.7320508 - 1e-6 and v.max() < 2 * 1.7320508


def test_shapes_deterministic_and_ranged():
    s = G.Generator(G.sift_shape(seed=0x7111))
    a = s.range(0, 500)
    b = s.range(0, 500)
    assert np.array_equal(a, b)
    assert np.array_equal(s.take(np.arange(100, 200)), a[100:200])
    assert (a == np.rint(a)).all() and a.min() >= 0 and a.max() <= 255  # integer-valued
    g = G.Generator(G.gist_shape(dim=64))
    x = g.range(5, 300)
    assert (x >= 0).all() and np.isfinite(x).all() and (x == 0).mean() > 0.05
    u = G.Generator(G.uniform_shape(9, 16)).range(0, 200)
    assert (u >= 0).all() and (u < 1).all()


def test_threading_invariant():
    s = G.Generator(G.gist_shape(dim=96))
    a = s.range(0, 2000, nthreads=1)
    b = s.range(0, 2000, nthreads=7)
    assert np.array_equal(a, b)


def test_delete_order_is_permutation():
    live = np.arange(1000, 1100)
    p = G.delete_order(1, 3, live)
    assert sorted(p.tolist()) == live.tolist() and not np.array_equal(p, live)


@pytest.mark.gpu
def test_device_generator_bit_identical():
    import torch

    for shape in (G.sift_shape(seed=0x100A), G.gist_shape(dim=960)):
        host = G.Generator(shape)
        dev = G.DeviceGenerator(shape)
        out = torch.empty(300, shape.dim, dtype=torch.float32, device="cuda")
        dev.range_into(out, 12345, 3)  # ids 12345 + 3 i (rank-local ids of an id-sharded index)
        ref = host.take(12345 + 3 * np.arange(300))
        assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))
        gs = np.random.default_rng(1).integers(0, 10**8, 257).astype(np.int64)
        out2 = torch.empty(257, shape.dim, dtype=torch.float32, device="cuda")
        dev.take_into(out2, torch.from_numpy(gs).cuda())  # arbitrary id lists (sampled H checks)
        assert np.array_equal(out2.cpu().numpy().view(np.uint32), host.take(gs).view(np.uint32))
