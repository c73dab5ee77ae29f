"""paper_2601_11808_b200 — B200-native SIVF hot path (arXiv 2601.11808).

Thin Python binding over the C ABI of ``lib/libsivf.so`` (include/sivf.h).
Argument marshalling only: every step of insert / delete / search / sliding
window / k-means runs in the library's sm_100a kernels.  PyTorch provides
device memory (the arena and I/O tensors) and the CUDA stream.  There is no
CPU fallback: if the library or a GPU is missing, construction raises.
"""
from __future__ import annotations

import ctypes
import math
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_DEFAULT_LIB = os.path.join(_HERE, "lib", "libsivf.so")
LIB_PATH = os.environ.get("SIVF_LIB_PATH") or _DEFAULT_LIB  # override: experiments

ST_OK, ST_POOL_EXHAUSTED, ST_DUPLICATE, ST_ID_OUT_OF_RANGE, ST_WRONG_SHARD = 0, 1, 2, 3, 4
ST_DIR_FULL, ST_RETRY_LIMIT = 5, 6  # sivf_insert_concurrent only

_i32, _i64, _u64, _P = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p


class Config(ctypes.Structure):
    _fields_ = [
        ("dim", _i32),
        ("nlist", _i32),
        ("id_capacity", _i64),
        ("num_slabs", _i64),
        ("max_batch", _i32),
        ("max_queries", _i32),
        ("max_k", _i32),
        ("max_nprobe", _i32),
        ("max_train", _i32),
        ("shard_rank", _i32),
        ("shard_count", _i32),
        ("flags", _i32),
        ("seed", _u64),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("live", _i64),
        ("inserted", _i64),
        ("deleted", _i64),
        ("slabs_in_use", _i64),
        ("slabs_free", _i64),
        ("pool_exhausted_items", _i64),
        ("reclaimed_slabs", _i64),
        ("device_errors", _i64),
        ("overhead_paper", ctypes.c_double),
        ("overhead_actual", ctypes.c_double),
        ("overhead_scan_copy", ctypes.c_double),
        ("dir_compactions", _i64),
        ("leaked_slabs", _i64),
        ("leaked_recycled", _i64),
    ]


EXPORTS = {
    "sivf_arena_bytes": (_i32, [ctypes.POINTER(Config), ctypes.POINTER(ctypes.c_size_t)]),
    "sivf_create": (_i32, [ctypes.POINTER(Config), _P, ctypes.c_size_t, _P, ctypes.POINTER(_P)]),
    "sivf_destroy": (_i32, [_P]),
    "sivf_set_centroids": (_i32, [_P, _P, _P]),
    "sivf_get_centroids": (_i32, [_P, _P, _P]),
    "sivf_train_centroids": (_i32, [_P, _P, _i64, _i32, _P]),
    "sivf_insert": (_i32, [_P, _P, _P, _i64, _P, _P, _P]),
    "sivf_delete": (_i32, [_P, _P, _i64, _P, _P]),
    "sivf_search": (_i32, [_P, _P, _i64, _i32, _i32, _P, _P, _P, _P]),
    "sivf_probe": (_i32, [_P, _P, _i64, _i32, _P, _P]),
    "sivf_search_probed": (_i32, [_P, _P, _i64, _i32, _i32, _P, _P, _P, _P]),
    "sivf_sliding_window_step": (_i32, [_P, _P, _P, _i64, _P, _i64, _P, _i64, _i32, _i32, _P, _P, _P, _P, _P]),
    "sivf_merge_topk": (_i32, [_P, _P, _i32, _i64, _i32, _P, _P, _P]),
    "sivf_reclaim": (_i32, [_P, _P, _P]),
    "sivf_dump_state": (_i32, [_P, _P, _P, _P, _P]),
    "sivf_dump_att": (_i32, [_P, _P, _P]),
    "sivf_stats": (_i32, [_P, ctypes.POINTER(Stats), _P]),
    "sivf_local_capacity": (_i64, [_P]),
    "sivf_launch_count": (_i64, [_P]),
    "sivf_probe_launch": (_i32, [ctypes.c_int32, _P]),
    "sivf_view_arena_bytes": (_i32, [ctypes.POINTER(Config), ctypes.POINTER(ctypes.c_size_t)]),
    "sivf_create_view": (_i32, [_P, _P, ctypes.c_size_t, _P, ctypes.POINTER(_P)]),
    "sivf_insert_concurrent": (_i32, [_P, _P, _P, ctypes.c_int64, _P, _P, _P]),
    "sivf_reserve_directories": (_i32, [_P, ctypes.c_int32, _P]),
    "sivf_probe_chase": (_i32, [_P, ctypes.c_int64, ctypes.c_int32, _P, _P]),
    "sivf_rc_string": (ctypes.c_char_p, [_i32]),
    "sivf_profile_enable": (_i32, [_P, _i32]),
    "sivf_profile_read": (_i32, [_P, _P, _P]),
    "sivf_set_option": (_i32, [_P, _i32, _i64]),
}

CFG_NO_SCAN_COPY = 1  # sivf_config.flags: no fp16 scan copy (paper footprint, CUDA-core scan)
CFG_CONCURRENT = 2  # sivf_config.flags: directory room for sivf_reserve_directories (NEXT-2)
CFG_SPLIT_COPY = 4  # sivf_config.flags: split-fp16 copy + GEMM scan at dim <= 128 (float-valued data)
OPT_TC_SCAN = 1
OPT_TC_TWO_PHASE = 2
OPT_TC_COARSE = 3
OPT_SEED_SLABS = 4
OPT_RANK_SPLIT = 5
OPT_COARSE_SELECT = 6
OPT_STEP_GRAPH = 7
OPT_CONCURRENT = 8
OPT_SEED_LIST = 9

PHASES = ("assign", "append", "delete", "coarse", "invmap", "scan", "merge", "reclaim")

_lib = None


def lib():
    """Load libsivf.so (raises if it has not been built: no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing; build it with `make sivf` (nvcc, sm_100a)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            if LIB_PATH != _DEFAULT_LIB and not hasattr(L, name):
                continue  # experiments (SIVF_LIB_PATH): an older build may lack newer entry points
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class SivfError(RuntimeError):
    pass


def _check(rc: int, what: str):
    if rc != 0:
        raise SivfError(f"{what}: {lib().sivf_rc_string(rc).decode()} ({rc})")


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _dev(t: torch.Tensor, dtype, name: str) -> torch.Tensor:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (use the host e2e helpers for host buffers)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    return t.contiguous()


def num_slabs_for(expected_n: int, nlist: int, maxvec_factor: float = 1.2, slab_factor: float = 1.2,
                  extra: int = 0) -> int:
    """Pool size: ceil(slab_factor * ceil(maxvec_factor * n / 32))
    plus one partially filled tail slab per list (reading C33)."""
    return int(math.ceil(slab_factor * math.ceil(maxvec_factor * expected_n / 32))) + nlist + extra


class Index:
    """GPU-resident SIVF index on the current CUDA device (one arena tensor)."""

    def __init__(self, dim: int, nlist: int, id_capacity: int, num_slabs: int, max_batch: int = 10000,
                 max_queries: int = 10000, max_k: int = 128, max_nprobe: int | None = None, max_train: int = 0,
                 shard_rank: int = 0, shard_count: int = 1, seed: int = 0, flags: int = 0, device=None,
                 stream=None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2601_11808_b200 needs a CUDA device (no CPU fallback)")
        L = lib()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        c = Config()
        c.dim, c.nlist, c.id_capacity, c.num_slabs = dim, nlist, id_capacity, num_slabs
        c.max_batch, c.max_queries, c.max_k = max_batch, max_queries, max_k
        c.max_nprobe = min(nlist, 1024) if max_nprobe is None else max_nprobe
        c.max_train, c.shard_rank, c.shard_count, c.seed, c.flags = max_train, shard_rank, shard_count, seed, flags
        self.cfg = c
        nbytes = ctypes.c_size_t(0)
        _check(L.sivf_arena_bytes(ctypes.byref(c), ctypes.byref(nbytes)), "sivf_arena_bytes")
        self.arena_bytes = nbytes.value
        with torch.cuda.device(self.device):
            self.arena = torch.empty(self.arena_bytes, dtype=torch.uint8, device=self.device)
            h = ctypes.c_void_p()
            _check(L.sivf_create(ctypes.byref(c), _ptr(self.arena), self.arena_bytes, _stream(stream),
                                 ctypes.byref(h)), "sivf_create")
        self._h = h
        self.dim, self.nlist = dim, nlist
        self.local_capacity = int(L.sivf_local_capacity(h))

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().sivf_destroy(self._h)
                self._h = None
        except Exception:
            pass

    # ---------------------------------------------------------------- NEXT-2: views, concurrent insert
    def view(self, stream=None) -> "IndexView":
        """A view sharing this index's state with its own scratch (sivf_create_view): views on
        different streams may run search / delete / insert_concurrent at the same time."""
        return IndexView(self, stream)

    def reserve_directories(self, spare: int, stream=None):
        """Quiescent: every list gets >= spare free directory entries (sivf_reserve_directories;
        synchronises the stream)."""
        _check(lib().sivf_reserve_directories(self._h, int(spare), _stream(stream)), "sivf_reserve_directories")

    def insert_concurrent(self, ids: torch.Tensor, X: torch.Tensor, status: torch.Tensor | None = None,
                          lists: torch.Tensor | None = None, stream=None):
        """sivf_insert_concurrent: the paper's lock-free protocol (Alg. 2) per vector."""
        ids = _dev(ids, torch.int64, "ids")
        X = _dev(X, torch.float32, "x")
        n = ids.shape[0]
        assert X.shape == (n, self.dim)
        if status is None:
            status = torch.empty(n, dtype=torch.int32, device=self.device)
        if lists is None:
            lists = torch.empty(n, dtype=torch.int32, device=self.device)
        _check(lib().sivf_insert_concurrent(self._h, _ptr(ids), _ptr(X), n, _ptr(status), _ptr(lists),
                                            _stream(stream)), "sivf_insert_concurrent")
        return status, lists

    # ---------------------------------------------------------------- quantizer
    def set_centroids(self, C: torch.Tensor, stream=None):
        C = _dev(C, torch.float32, "centroids")
        assert C.shape == (self.nlist, self.dim)
        _check(lib().sivf_set_centroids(self._h, _ptr(C), _stream(stream)), "sivf_set_centroids")
        self._keep = C  # keep alive until the copy has run

    def get_centroids(self, stream=None) -> torch.Tensor:
        out = torch.empty(self.nlist, self.dim, dtype=torch.float32, device=self.device)
        _check(lib().sivf_get_centroids(self._h, _ptr(out), _stream(stream)), "sivf_get_centroids")
        return out

    def train(self, X: torch.Tensor, niter: int = 20, stream=None):
        X = _dev(X, torch.float32, "x")
        _check(lib().sivf_train_centroids(self._h, _ptr(X), X.shape[0], niter, _stream(stream)),
               "sivf_train_centroids")
        self._keep = X

    # ---------------------------------------------------------------- mutation
    def insert(self, ids: torch.Tensor, X: torch.Tensor, status: torch.Tensor | None = None,
               lists: torch.Tensor | None = None, stream=None):
        ids = _dev(ids, torch.int64, "ids")
        X = _dev(X, torch.float32, "x")
        n = ids.shape[0]
        assert X.shape == (n, self.dim)
        if status is None:
            status = torch.empty(n, dtype=torch.int32, device=self.device)
        if lists is None:
            lists = torch.empty(n, dtype=torch.int32, device=self.device)
        _check(lib().sivf_insert(self._h, _ptr(ids), _ptr(X), n, _ptr(status), _ptr(lists), _stream(stream)),
               "sivf_insert")
        return status, lists

    def delete(self, ids: torch.Tensor, ndeleted: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        ids = _dev(ids, torch.int64, "ids")
        if ndeleted is None:
            ndeleted = torch.empty(1, dtype=torch.int64, device=self.device)
        _check(lib().sivf_delete(self._h, _ptr(ids), ids.shape[0], _ptr(ndeleted), _stream(stream)), "sivf_delete")
        return ndeleted

    def reclaim(self, stream=None) -> torch.Tensor:
        out = torch.empty(1, dtype=torch.int64, device=self.device)
        _check(lib().sivf_reclaim(self._h, _ptr(out), _stream(stream)), "sivf_reclaim")
        return out

    # ---------------------------------------------------------------- search
    def search(self, Q: torch.Tensor, k: int, nprobe: int, return_probes: bool = False, out=None, stream=None):
        Q = _dev(Q, torch.float32, "queries")
        nq = Q.shape[0]
        if out is None:
            dist = torch.empty(nq, k, dtype=torch.float32, device=self.device)
            ids = torch.empty(nq, k, dtype=torch.int64, device=self.device)
        else:
            dist, ids = out
        probes = torch.empty(nq, nprobe, dtype=torch.int32, device=self.device) if return_probes else None
        _check(lib().sivf_search(self._h, _ptr(Q), nq, k, nprobe, _ptr(dist), _ptr(ids), _ptr(probes),
                                 _stream(stream)), "sivf_search")
        return (dist, ids, probes) if return_probes else (dist, ids)

    def probe(self, Q: torch.Tensor, nprobe: int, out=None, stream=None) -> torch.Tensor:
        """Coarse step only (sivf_probe): the exact probe set [nq][nprobe] of each query."""
        Q = _dev(Q, torch.float32, "queries")
        nq = Q.shape[0]
        probes = torch.empty(nq, nprobe, dtype=torch.int32, device=self.device) if out is None else out
        _check(lib().sivf_probe(self._h, _ptr(Q), nq, nprobe, _ptr(probes), _stream(stream)), "sivf_probe")
        return probes

    def search_probed(self, Q: torch.Tensor, probes: torch.Tensor, k: int, out=None, stream=None):
        """Scan + merge with given probe sets (sivf_search_probed); probes [nq][nprobe] int32."""
        Q = _dev(Q, torch.float32, "queries")
        probes = _dev(probes, torch.int32, "probes")
        nq, nprobe = probes.shape
        if out is None:
            dist = torch.empty(nq, k, dtype=torch.float32, device=self.device)
            ids = torch.empty(nq, k, dtype=torch.int64, device=self.device)
        else:
            dist, ids = out
        _check(lib().sivf_search_probed(self._h, _ptr(Q), nq, k, nprobe, _ptr(probes), _ptr(dist), _ptr(ids),
                                        _stream(stream)), "sivf_search_probed")
        return dist, ids

    def sliding_window_step(self, new_ids, new_x, old_ids, Q, k: int, nprobe: int, out=None, stream=None):
        new_ids = _dev(new_ids, torch.int64, "new_ids")
        new_x = _dev(new_x, torch.float32, "new_x")
        old_ids = _dev(old_ids, torch.int64, "old_ids")
        nq = 0 if Q is None else Q.shape[0]
        if out is None:
            dist = torch.empty(max(nq, 1), k, dtype=torch.float32, device=self.device)
            ids = torch.empty(max(nq, 1), k, dtype=torch.int64, device=self.device)
            status = torch.empty(max(new_ids.shape[0], 1), dtype=torch.int32, device=self.device)
            ndel = torch.empty(1, dtype=torch.int64, device=self.device)
        else:
            dist, ids, status, ndel = out
        _check(lib().sivf_sliding_window_step(self._h, _ptr(new_ids), _ptr(new_x), new_ids.shape[0], _ptr(old_ids),
                                              old_ids.shape[0], _ptr(Q) if nq else None, nq, k, nprobe, _ptr(dist),
                                              _ptr(ids), _ptr(status), _ptr(ndel), _stream(stream)),
               "sivf_sliding_window_step")
        return dist, ids, status, ndel

    # ---------------------------------------------------------------- introspection
    def dump_state(self, stream=None):
        loi = torch.empty(max(self.local_capacity, 1), dtype=torch.int32, device=self.device)
        lpl = torch.empty(self.nlist, dtype=torch.int64, device=self.device)
        viol = torch.empty(1, dtype=torch.int64, device=self.device)
        _check(lib().sivf_dump_state(self._h, _ptr(loi), _ptr(lpl), _ptr(viol), _stream(stream)), "sivf_dump_state")
        return loi[: self.local_capacity], lpl, viol

    def dump_att(self, stream=None) -> torch.Tensor:
        att = torch.empty(max(self.local_capacity, 1), dtype=torch.int64, device=self.device)
        _check(lib().sivf_dump_att(self._h, _ptr(att), _stream(stream)), "sivf_dump_att")
        return att[: self.local_capacity]

    def stats(self, stream=None) -> dict:
        s = Stats()
        _check(lib().sivf_stats(self._h, ctypes.byref(s), _stream(stream)), "sivf_stats")
        return {f: getattr(s, f) for f, _ in Stats._fields_}

    def launch_count(self) -> int:
        return int(lib().sivf_launch_count(self._h))

    def set_option(self, option: int, value: int):
        _check(lib().sivf_set_option(self._h, option, value), "sivf_set_option")

    def profile(self, on: bool = True):
        _check(lib().sivf_profile_enable(self._h, 1 if on else 0), "sivf_profile_enable")

    def profile_read(self) -> dict:
        ms = (ctypes.c_double * len(PHASES))()
        cnt = (ctypes.c_int64 * len(PHASES))()
        _check(lib().sivf_profile_read(self._h, ms, cnt), "sivf_profile_read")
        return {p: (ms[i], cnt[i]) for i, p in enumerate(PHASES)}


def merge_topk(dist_g: torch.Tensor, ids_g: torch.Tensor, stream=None):
    """Per query, the k smallest (distance, id) over G shard lists [G][nq][k]."""
    dist_g = _dev(dist_g, torch.float32, "dist_g")
    ids_g = _dev(ids_g, torch.int64, "ids_g")
    G, nq, k = dist_g.shape
    dist = torch.empty(nq, k, dtype=torch.float32, device=dist_g.device)
    ids = torch.empty(nq, k, dtype=torch.int64, device=dist_g.device)
    _check(lib().sivf_merge_topk(_ptr(dist_g), _ptr(ids_g), G, nq, k, _ptr(dist), _ptr(ids), _stream(stream)),
           "sivf_merge_topk")
    return dist, ids


def probe_launch(n: int, stream=None):
    """Enqueue n empty-kernel launches (latency floor measurement; sivf_probe_launch)."""
    _check(lib().sivf_probe_launch(int(n), _stream(stream)), "sivf_probe_launch")


def probe_chase(next_idx: torch.Tensor, hops: int, out: torch.Tensor, stream=None):
    """One thread follows `hops` dependent loads through next_idx (int32, device); the final
    index lands in out[0] (sivf_probe_chase)."""
    next_idx = _dev(next_idx, torch.int32, "next_idx")
    out = _dev(out, torch.int32, "out")
    _check(lib().sivf_probe_chase(_ptr(next_idx), next_idx.numel(), int(hops), _ptr(out), _stream(stream)),
           "sivf_probe_chase")


class IndexView(Index):
    """A view of an Index (sivf_create_view): shares the owner's index state, owns its scratch.
    search / delete / insert_concurrent only; the owner must outlive it."""

    def __init__(self, owner: Index, stream=None):  # noqa: super().__init__ is not called (no new index)
        L = lib()
        self.owner = owner
        self.device = owner.device
        self.cfg = owner.cfg
        nbytes = ctypes.c_size_t(0)
        _check(L.sivf_view_arena_bytes(ctypes.byref(owner.cfg), ctypes.byref(nbytes)), "sivf_view_arena_bytes")
        self.arena_bytes = nbytes.value
        with torch.cuda.device(self.device):
            self.arena = torch.empty(max(self.arena_bytes, 256), dtype=torch.uint8, device=self.device)
            h = ctypes.c_void_p()
            _check(L.sivf_create_view(owner._h, _ptr(self.arena), self.arena_bytes, _stream(stream), ctypes.byref(h)),
                   "sivf_create_view")
        self._h = h
        self.dim, self.nlist = owner.dim, owner.nlist
        self.local_capacity = owner.local_capacity
