"""Host-side plumbing of the id-sharded index.

owner(id) = id mod G.  Mutations are routed by id with no collective; a search
broadcasts the queries, every rank searches its shard, and the per-shard top-k
lists are all-gathered ([G][nq][k]) for the exact merge (sivf_merge_topk on the
GPU: the top-k of the union of per-shard top-ks is the top-k of the union).
This module is marshalling only: the merge itself runs in libsivf.so.
"""
from __future__ import annotations

import numpy as np


def owner(ids, G: int):
    """Rank owning each id (owner(id) = id mod G)."""
    return ids % G


def route(ids, G: int, rank: int, *arrays):
    """The sub-batch of `ids` (and of row-aligned `arrays`) owned by `rank`, order kept."""
    m = owner(ids, G) == rank
    return (ids[m],) + tuple(a[m] for a in arrays)


def local_count(n_total: int, G: int, rank: int) -> int:
    """Number of ids in [0, n_total) owned by `rank`."""
    return len(range(rank, n_total, G))


def allgather_topk(pg, d, i):
    """All-gather per-shard results d [nq][k] (float32) and i [nq][k] (int64) into
    [G][nq][k] tensors on every rank (NCCL: one all_gather_into_tensor each; other
    backends: the list form)."""
    import torch

    G = pg.get_world_size()
    if G == 1:
        return d[None], i[None]
    gd = torch.empty((G,) + tuple(d.shape), dtype=d.dtype, device=d.device)
    gi = torch.empty((G,) + tuple(i.shape), dtype=i.dtype, device=i.device)
    if pg.get_backend() == "nccl":
        pg.all_gather_into_tensor(gd.view(-1), d.reshape(-1).contiguous())
        pg.all_gather_into_tensor(gi.view(-1), i.reshape(-1).contiguous())
    else:
        pg.all_gather(list(gd.unbind(0)), d.contiguous())
        pg.all_gather(list(gi.unbind(0)), i.contiguous())
    return gd, gi


def query_slice(nq: int, G: int, rank: int):
    """The rank's contiguous slice [lo, hi) of a batch of nq queries (query-sharded coarse
    step, NEXT-3): sizes differ by at most one."""
    lo = rank * nq // G
    return lo, (rank + 1) * nq // G


def allgather_probes(pg, probes_local, nq: int):
    """All-gather the per-rank probe sets [hi - lo][nprobe] (int32) of the query slices
    into the full [nq][nprobe] on every rank (one all_gather_into_tensor of equal-size
    padded blocks under NCCL; the list form otherwise)."""
    import torch

    G = pg.get_world_size()
    if G == 1:
        return probes_local
    nprobe = probes_local.shape[1]
    blk = -(-nq // G)  # ceil: every rank contributes a padded block of blk rows
    pad = torch.zeros((blk, nprobe), dtype=probes_local.dtype, device=probes_local.device)
    pad[: probes_local.shape[0]] = probes_local
    g = torch.empty((G, blk, nprobe), dtype=probes_local.dtype, device=probes_local.device)
    if pg.get_backend() == "nccl":
        pg.all_gather_into_tensor(g.view(-1), pad.view(-1))
    else:
        pg.all_gather(list(g.unbind(0)), pad)
    parts = []
    for r in range(G):
        lo, hi = query_slice(nq, G, r)
        parts.append(g[r, : hi - lo])
    return torch.cat(parts, 0)


def sharded_search(pg, ix, Q, k: int, nprobe: int):
    """Id-sharded search with the coarse step sharded over queries (§8(e), NEXT-3):
    rank r computes the probe sets of its query slice (sivf_probe), the slices are
    all-gathered, every rank scans its shard with the full probe sets
    (sivf_search_probed), and the per-shard top-k lists are all-gathered and merged
    (sivf_merge_topk).  Bit-identical to the replicated-coarse search: the probe
    sets do not depend on the shard."""
    from . import merge_topk

    G, rank = pg.get_world_size(), pg.get_rank()
    nq = Q.shape[0]
    lo, hi = query_slice(nq, G, rank)
    probes = allgather_probes(pg, ix.probe(Q[lo:hi], nprobe), nq)
    d, i = ix.search_probed(Q, probes, k)
    gd, gi = allgather_topk(pg, d, i)
    return merge_topk(gd, gi)


__all__ = ["owner", "route", "local_count", "allgather_topk", "query_slice", "allgather_probes", "sharded_search"]
_ = np  # numpy arrays and torch tensors both route (ids % G works on either)
