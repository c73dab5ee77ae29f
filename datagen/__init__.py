"""Seeded synthetic workload generator (harness code, shared by tests/bench).

Thin ctypes wrapper over ``libsivfgen.so`` (datagen_host.c + sivf_datagen.h).
It contains none of the method's arithmetic: it maps (seed, g) to vectors.
Recipe and parameters: SURVEY.md §8(d); DESIGN.md "Input recipe".
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsivfgen.so")

SIFT, GIST, UNIFORM = 0, 1, 2
QUERY_BASE = 1 << 40
TRAIN_BASE = 1 << 41


class _Params(ctypes.Structure):
    _fields_ = [
        ("seed", ctypes.c_uint64),
        ("dim", ctypes.c_int32),
        ("M", ctypes.c_int32),
        ("r", ctypes.c_int32),
        ("kind", ctypes.c_int32),
        ("a", ctypes.c_float),
        ("b_over_sqrt_r", ctypes.c_float),
        ("sigma", ctypes.c_float),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `make -C {os.path.dirname(_HERE)} datagen`")
        L = ctypes.CDLL(_LIB_PATH)
        L.sivfgen_model_new.restype = ctypes.c_void_p
        L.sivfgen_model_new.argtypes = [ctypes.POINTER(_Params)]
        L.sivfgen_model_free.argtypes = [ctypes.c_void_p]
        L.sivfgen_range.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int]
        L.sivfgen_list.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int]
        L.sivfgen_mix64_x.restype = ctypes.c_uint64
        L.sivfgen_mix64_x.argtypes = [ctypes.c_uint64]
        L.sivfgen_H_x.restype = ctypes.c_uint64
        L.sivfgen_H_x.argtypes = [ctypes.c_uint64] * 3
        L.sivfgen_N01_x.restype = ctypes.c_float
        L.sivfgen_N01_x.argtypes = [ctypes.c_uint64] * 3
        _lib = L
    return _lib


@dataclass(frozen=True)
class Shape:
    """Generator parameters (M, r, a, b, sigma) for one data family."""

    seed: int
    dim: int
    kind: int = SIFT
    M: int = 50
    r: int = 24
    a: float = 60.0
    b: float = 50.0
    sigma: float = 15.0

    def _params(self) -> _Params:
        p = _Params()
        p.seed = self.seed
        p.dim = self.dim
        p.M = self.M
        p.r = self.r
        p.kind = self.kind
        p.a = float(np.float32(self.a))
        p.b_over_sqrt_r = float(np.float32(self.b / np.sqrt(self.r))) if self.r > 0 else 0.0
        p.sigma = float(np.float32(self.sigma))
        return p


# Frozen families (SURVEY §8(d) pre-calibration; DESIGN.md records the calibration).
def sift_shape(seed: int = 0x51F7, dim: int = 128) -> Shape:
    return Shape(seed=seed, dim=dim, kind=SIFT, M=50, r=24, a=60.0, b=50.0, sigma=15.0)


def gist_shape(seed: int = 0x6157, dim: int = 960) -> Shape:
    return Shape(seed=seed, dim=dim, kind=GIST, M=50, r=48, a=0.12, b=0.15, sigma=0.015)


def uniform_shape(seed: int, dim: int) -> Shape:
    return Shape(seed=seed, dim=dim, kind=UNIFORM, M=1, r=0, a=0.0, b=0.0, sigma=0.0)


class Generator:
    def __init__(self, shape: Shape):
        self.shape = shape
        self._p = shape._params()
        self._m = lib().sivfgen_model_new(ctypes.byref(self._p))

    def __del__(self):
        try:
            if self._m:
                lib().sivfgen_model_free(self._m)
        except Exception:
            pass

    def range(self, g0: int, n: int, out: np.ndarray | None = None, nthreads: int = 0) -> np.ndarray:
        if out is None:
            out = np.empty((n, self.shape.dim), dtype=np.float32)
        assert out.dtype == np.float32 and out.flags.c_contiguous and out.shape == (n, self.shape.dim)
        lib().sivfgen_range(self._m, g0, n, out.ctypes.data, nthreads)
        return out

    def take(self, gs, nthreads: int = 0) -> np.ndarray:
        gs = np.ascontiguousarray(np.asarray(gs, dtype=np.uint64))
        out = np.empty((gs.shape[0], self.shape.dim), dtype=np.float32)
        lib().sivfgen_list(self._m, gs.ctypes.data, gs.shape[0], out.ctypes.data, nthreads)
        return out

    def base(self, ids) -> np.ndarray:
        return self.take(np.asarray(ids, dtype=np.uint64))

    def queries(self, q0: int, n: int) -> np.ndarray:
        return self.range(QUERY_BASE + q0, n)

    def train(self, n: int) -> np.ndarray:
        return self.range(TRAIN_BASE, n)


class DeviceGenerator:
    """The same (seed, g) -> vector map evaluated on the GPU (libsivfgen_cuda.so;
    harness code).  Outputs are bit-identical to Generator (tests/test_datagen.py)."""

    def __init__(self, shape: Shape):
        path = os.path.join(_HERE, "libsivfgen_cuda.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C {os.path.dirname(_HERE)} datagen_cuda`")
        self._L = ctypes.CDLL(path)
        self._L.sivfgen_cuda_model_new.restype = ctypes.c_void_p
        self._L.sivfgen_cuda_model_new.argtypes = [ctypes.POINTER(_Params)]
        self._L.sivfgen_cuda_model_free.argtypes = [ctypes.c_void_p]
        self._L.sivfgen_cuda_range.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64,
                                               ctypes.c_void_p, ctypes.c_void_p]
        self._L.sivfgen_cuda_list.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                              ctypes.c_void_p]
        self.shape = shape
        self._p = shape._params()
        self._m = self._L.sivfgen_cuda_model_new(ctypes.byref(self._p))
        if not self._m:
            raise RuntimeError("sivfgen_cuda_model_new failed")

    def __del__(self):
        try:
            if self._m:
                self._L.sivfgen_cuda_model_free(self._m)
        except Exception:
            pass

    def range_into(self, out, g0: int, gstride: int = 1, stream=None):
        """out: a CUDA float32 tensor [n][dim]; row i = vector(g0 + i * gstride)."""
        import torch

        assert out.is_cuda and out.dtype == torch.float32 and out.is_contiguous() and out.shape[1] == self.shape.dim
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        rc = self._L.sivfgen_cuda_range(self._m, g0, gstride, out.shape[0], out.data_ptr(), st)
        if rc != 0:
            raise RuntimeError(f"sivfgen_cuda_range: CUDA error {rc}")
        return out


    def take_into(self, out, gs, stream=None):
        """out: CUDA float32 [n][dim]; gs: CUDA int64 [n] indices; row i = vector(gs[i])."""
        import torch

        assert out.is_cuda and out.dtype == torch.float32 and out.is_contiguous() and out.shape[1] == self.shape.dim
        assert gs.is_cuda and gs.dtype == torch.int64 and gs.is_contiguous() and gs.shape[0] == out.shape[0]
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        rc = self._L.sivfgen_cuda_list(self._m, gs.data_ptr(), gs.shape[0], out.data_ptr(), st)
        if rc != 0:
            raise RuntimeError(f"sivfgen_cuda_list: CUDA error {rc}")
        return out


def mix64(z: int) -> int:
    return int(lib().sivfgen_mix64_x(z))


def H(s: int, a: int, b: int) -> int:
    return int(lib().sivfgen_H_x(s, a, b))


def N01(s: int, a: int, b: int) -> float:
    return float(lib().sivfgen_N01_x(s, a, b))


def delete_order(seed: int, batch: int, live_ids: np.ndarray) -> np.ndarray:
    """Seeded Fisher-Yates over the live set with H(seed ^ 0xDE1, batch, i)
    (SURVEY §8(d) "Delete selection"); returns a permutation of live_ids."""
    a = np.array(live_ids, dtype=np.int64, copy=True)
    n = a.shape[0]
    s = (seed ^ 0xDE1) & 0xFFFFFFFFFFFFFFFF
    L = lib()
    for i in range(n - 1):
        j = i + int(L.sivfgen_H_x(s, batch, i)) % (n - i)
        a[i], a[j] = a[j], a[i]
    return a
