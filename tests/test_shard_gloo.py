"""World-size-2 (gloo, CPU) tests of the id-sharded path's host logic
(paper_2601_11808_b200/shard.py, the code bench.py uses): routing by id mod G
covers every id exactly once, and all-gathering the per-shard top-k then merging
reproduces the unsharded search exactly.  The per-shard searches are the CPU
oracle's (test infrastructure); the GPU merge kernel has its own GPU test."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from datagen import Generator, sift_shape
from paper_2601_11808_b200 import shard

N, D, NL, NQ, K, NPROBE = 3000, 32, 16, 40, 10, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data():
    gen = Generator(sift_shape(seed=0x5A5A, dim=D))
    X = gen.range(0, N)
    Q = gen.queries(0, NQ)
    C = O.kmeans(X[:1024], NL, 5, 11)
    return X, Q, C


def _worker(rank, G, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=G)
    X, Q, C = _data()
    ids = np.arange(N, dtype=np.int64)
    mine, Xm = shard.route(ids, G, rank, X)
    assert len(mine) == shard.local_count(N, G, rank)
    ix = O.Index(D, NL, N, shard_rank=rank, shard_count=G)
    ix.set_centroids(C)
    st, _ = ix.insert(mine, Xm)
    assert (st == O.ST_OK).all()
    # a delete batch routed by id: every rank receives only its own ids
    dels, = shard.route(np.arange(0, N, 7, dtype=np.int64), G, rank)
    ix.delete(dels)
    d, i, P = ix.search(Q, K, NPROBE)
    # query-sharded coarse step (NEXT-3): this rank's slice of the probe sets, all-gathered
    lo, hi = shard.query_slice(NQ, G, rank)
    Pg = shard.allgather_probes(dist, torch.from_numpy(np.ascontiguousarray(np.asarray(P, np.int32)[lo:hi])), NQ)
    assert np.array_equal(Pg.numpy(), np.asarray(P, np.int32))
    gd, gi = shard.allgather_topk(dist, torch.from_numpy(np.ascontiguousarray(d)),
                                  torch.from_numpy(np.ascontiguousarray(i)))
    if rank == 0:
        md, mi = O.merge_topk(gd.numpy(), gi.numpy(), K)
        np.save(out + ".d.npy", md)
        np.save(out + ".i.npy", mi)
        np.save(out + ".n.npy", np.array([gd.shape[0]]))
    dist.barrier()
    dist.destroy_process_group()


def test_query_slices_partition_batch():
    for nq, G in ((10, 3), (2, 4), (10000, 8), (0, 2)):
        sl = [shard.query_slice(nq, G, r) for r in range(G)]
        assert sl[0][0] == 0 and sl[-1][1] == nq
        assert all(sl[r][1] == sl[r + 1][0] for r in range(G - 1))
        assert max(h - l for l, h in sl) - min(h - l for l, h in sl) <= 1


def test_route_partitions_ids():
    ids = np.arange(1000, dtype=np.int64)
    parts = [shard.route(ids, 3, r)[0] for r in range(3)]
    allp = np.concatenate(parts)
    assert np.array_equal(np.sort(allp), ids)
    assert all((p % 3 == r).all() for r, p in enumerate(parts))
    assert sum(shard.local_count(1000, 3, r) for r in range(3)) == 1000


def test_gloo_world2_sharded_search_equals_single(tmp_path):
    G = 2
    out = str(tmp_path / "res")
    mp.spawn(_worker, args=(G, _free_port(), out), nprocs=G, join=True)
    X, Q, C = _data()
    ref = O.Index(D, NL, N)
    ref.set_centroids(C)
    ref.insert(np.arange(N, dtype=np.int64), X)
    ref.delete(np.arange(0, N, 7, dtype=np.int64))
    od, oi, _ = ref.search(Q, K, NPROBE)
    assert int(np.load(out + ".n.npy")[0]) == G
    assert np.array_equal(np.load(out + ".i.npy"), oi)
    assert np.array_equal(np.load(out + ".d.npy").view(np.uint32), od.view(np.uint32))
