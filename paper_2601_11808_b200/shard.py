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


__all__ = ["owner", "route", "local_count", "allgather_topk"]
_ = np  # numpy arrays and torch tensors both route (ids % G works on either)
