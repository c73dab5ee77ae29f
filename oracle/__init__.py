"""CPU oracle for the SIVF hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(paper_2601_11808_b200) never imports it; the two share no code.

ctypes wrapper over oracle/libsivf_oracle.so (sivf_oracle.cpp).  Every
function cites the PAPER.md passage it follows in sivf_oracle.cpp.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsivf_oracle.so")

ST_OK, ST_POOL_EXHAUSTED, ST_DUPLICATE, ST_ID_OUT_OF_RANGE, ST_WRONG_SHARD = 0, 1, 2, 3, 4

_P = ctypes.c_void_p
_i32, _i64, _u64, _cf32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float


class Stats(ctypes.Structure):
    _fields_ = [
        ("live", _i64),
        ("inserted", _i64),
        ("deleted", _i64),
        ("slabs_in_use", _i64),
        ("slabs_free", _i64),
        ("pool_exhausted_items", _i64),
        ("overhead_paper", ctypes.c_double),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `make oracle`")
        L = ctypes.CDLL(_LIB_PATH)
        sig = {
            "or_create": (_P, [_i32, _i32, _i64, _i64, _i32, _i32]),
            "or_destroy": (None, [_P]),
            "or_set_centroids": (None, [_P, _P]),
            "or_set_threads": (None, [_i32]),
            "or_dist32": (_cf32, [_P, _P, _i32]),
            "or_dist64": (ctypes.c_double, [_P, _P, _i32]),
            "or_assign": (_i32, [_P, _i32, _i32, _P]),
            "or_assign_batch": (None, [_P, _i32, _i32, _P, _i64, _P]),
            "or_probe": (None, [_P, _i32, _i32, _P, _i32, _P]),
            "or_insert": (None, [_P, _P, _P, _i64, _P, _P]),
            "or_delete": (_i64, [_P, _P, _i64]),
            "or_search": (None, [_P, _P, _i64, _i32, _i32, _P, _P, _P]),
            "or_bruteforce": (None, [_P, _P, _i64, _i32, _P, _P]),
            "or_topk_candidates": (None, [_P, _i32, _P, _P, _i64, _i32, _P, _P]),
            "or_reclaim": (_i64, [_P]),
            "or_dump_state": (None, [_P, _P, _P]),
            "or_stats": (None, [_P, ctypes.POINTER(Stats)]),
            "or_local_capacity": (_i64, [_P]),
            "or_adopt_list": (_i32, [_P, _i64, _i32]),
            "or_get_vector": (_i32, [_P, _i64, _P]),
            "or_merge_topk": (None, [_P, _P, _i32, _i64, _i32, _P, _P]),
            "or_kmeans": (None, [_P, _i64, _i32, _i32, _i32, _u64, _P, _P]),
            "or_kmeans_hash": (_u64, [_u64, _u64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().or_set_threads(int(n))


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _p(a: np.ndarray):
    return a.ctypes.data


def dist32(a, b) -> float:
    a, b = _f32(a), _f32(b)
    return float(lib().or_dist32(_p(a), _p(b), a.shape[-1]))


def dist64(a, b) -> float:
    a, b = _f32(a), _f32(b)
    return float(lib().or_dist64(_p(a), _p(b), a.shape[-1]))


def assign(C, X) -> np.ndarray:
    C, X = _f32(C), _f32(np.atleast_2d(X))
    out = np.empty(X.shape[0], dtype=np.int32)
    lib().or_assign_batch(_p(C), C.shape[0], C.shape[1], _p(X), X.shape[0], _p(out))
    return out


def probe(C, q, m: int) -> np.ndarray:
    C, q = _f32(C), _f32(q)
    out = np.empty(m, dtype=np.int32)
    lib().or_probe(_p(C), C.shape[0], C.shape[1], _p(q), m, _p(out))
    return out


def topk_candidates(q, X, ids, k: int):
    """Top-k by (dist32, id) of query q over the candidates X[n][d] with ids[n]."""
    q = _f32(q).reshape(-1)
    X = _f32(X).reshape(-1, q.shape[0])
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    d = np.empty(k, np.float32)
    i = np.empty(k, np.int64)
    lib().or_topk_candidates(_p(q), q.shape[0], _p(X), _p(ids), ids.shape[0], k, _p(d), _p(i))
    return d, i


def merge_topk(dist_g, ids_g, k: int):
    dist_g = _f32(dist_g)
    ids_g = np.ascontiguousarray(ids_g, dtype=np.int64)
    G, nq = dist_g.shape[0], dist_g.shape[1]
    d = np.empty((nq, k), np.float32)
    i = np.empty((nq, k), np.int64)
    lib().or_merge_topk(_p(dist_g), _p(ids_g), G, nq, k, _p(d), _p(i))
    return d, i


def kmeans(X, nlist: int, niter: int, seed: int, with_objective: bool = False):
    X = _f32(X)
    out = np.empty((nlist, X.shape[1]), np.float32)
    obj = np.empty(max(niter, 1), np.float64)
    lib().or_kmeans(_p(X), X.shape[0], X.shape[1], nlist, niter, seed, _p(out), _p(obj) if with_objective else None)
    return (out, obj[:niter]) if with_objective else out


def kmeans_hash(seed: int, i: int) -> int:
    return int(lib().or_kmeans_hash(seed, i))


class Index:
    """Plain IVF-Flat with per-list arrays (sivf_oracle.cpp)."""

    def __init__(self, dim: int, nlist: int, id_capacity: int, num_slabs: int = 0, shard_rank: int = 0,
                 shard_count: int = 1):
        self.dim, self.nlist = dim, nlist
        self.shard_rank, self.shard_count = shard_rank, shard_count
        self._h = lib().or_create(dim, nlist, id_capacity, num_slabs, shard_rank, shard_count)
        if not self._h:
            raise ValueError("or_create: invalid arguments")
        self.local_capacity = int(lib().or_local_capacity(self._h))

    def __del__(self):
        try:
            if self._h:
                lib().or_destroy(self._h)
        except Exception:
            pass

    def set_centroids(self, C):
        C = _f32(C)
        assert C.shape == (self.nlist, self.dim)
        lib().or_set_centroids(self._h, _p(C))

    def insert(self, ids, X):
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        X = _f32(X).reshape(ids.shape[0], self.dim)
        st = np.empty(ids.shape[0], np.int32)
        ls = np.empty(ids.shape[0], np.int32)
        lib().or_insert(self._h, _p(ids), _p(X), ids.shape[0], _p(st), _p(ls))
        return st, ls

    def delete(self, ids) -> int:
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        return int(lib().or_delete(self._h, _p(ids), ids.shape[0]))

    def search(self, Q, k: int, nprobe: int):
        Q = _f32(Q).reshape(-1, self.dim)
        nq = Q.shape[0]
        d = np.empty((nq, k), np.float32)
        i = np.empty((nq, k), np.int64)
        P = np.empty((nq, nprobe), np.int32)
        lib().or_search(self._h, _p(Q), nq, k, nprobe, _p(d), _p(i), _p(P))
        return d, i, P

    def bruteforce(self, Q, k: int):
        Q = _f32(Q).reshape(-1, self.dim)
        nq = Q.shape[0]
        d = np.empty((nq, k), np.float32)
        i = np.empty((nq, k), np.int64)
        lib().or_bruteforce(self._h, _p(Q), nq, k, _p(d), _p(i))
        return d, i

    def reclaim(self) -> int:
        return int(lib().or_reclaim(self._h))

    def dump_state(self):
        loi = np.empty(self.local_capacity, np.int32)
        lpl = np.empty(self.nlist, np.int64)
        lib().or_dump_state(self._h, _p(loi), _p(lpl))
        return loi, lpl

    def stats(self) -> dict:
        s = Stats()
        lib().or_stats(self._h, ctypes.byref(s))
        return {f: getattr(s, f) for f, _ in Stats._fields_}

    def adopt_list(self, id_: int, list_: int) -> bool:
        return bool(lib().or_adopt_list(self._h, id_, list_))

    def get_vector(self, id_: int):
        out = np.empty(self.dim, np.float32)
        ok = lib().or_get_vector(self._h, id_, _p(out))
        return out if ok else None
