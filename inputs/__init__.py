"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO triangle-counting arithmetic: it only produces raw edge
samples (which may contain self-loops, duplicates and both orientations) and
the hard-coded Zachary karate fixture.  Both sides canonicalise independently.

Configs follow BASELINE.json ``configs`` and SURVEY.md §8(d) "Synthetic inputs":
  C1 karate        34 vertices, 78 edges
  C2 rmat16        Graph500 R-MAT scale 16, ef 16, (a,b,c) = (.57,.19,.19)
  C3 orkut         Chung-Lu, n=3,072,441, m=117,185,083, dmax=33,313, gamma=2.3314
  C4 rmat24        Graph500 R-MAT scale 24, ef 16
  C5 friendster    Chung-Lu, n=65,608,366, m=1,806,067,135, dmax=5,214, gamma=2.0
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libbbtcgen.so")
_lib = None

_u32p = ctypes.POINTER(ctypes.c_uint32)


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run __graft_entry__.build() (make)")
        lib = ctypes.CDLL(_LIB_PATH)
        lib.bbtcgen_u64.restype = ctypes.c_uint64
        lib.bbtcgen_u64.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        lib.bbtcgen_rmat.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_uint64, _u32p, _u32p, ctypes.c_int]
        lib.bbtcgen_chunglu.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_uint64, _u32p, _u32p, ctypes.POINTER(ctypes.c_double),
                                        ctypes.c_int]
        lib.bbtcgen_gnp.argtypes = [ctypes.c_uint32, ctypes.c_double, ctypes.c_uint64, _u32p, _u32p,
                                    ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
        lib.bbtcgen_uniform_pairs.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, _u32p, _u32p]
        lib.bbtcgen_rmat_range.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                           _u32p, _u32p, ctypes.c_int]
        lib.bbtcgen_chunglu_range.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                                              ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _u32p, _u32p,
                                              ctypes.POINTER(ctypes.c_double), ctypes.c_int]
        lib.bbtcgen_last_error.restype = ctypes.c_char_p
        _lib = lib
    return _lib


def _check(rc):
    if rc != 0:
        raise ValueError(_load().bbtcgen_last_error().decode())


def _ptr(a: np.ndarray):
    assert a.dtype == np.uint32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_u32p)


def _out(n, out):
    if out is None:
        return np.empty(n, np.uint32), np.empty(n, np.uint32)
    s, d = out
    assert len(s) >= n and len(d) >= n
    return s[:n], d[:n]


def u64(seed: int, counter: int) -> int:
    return int(_load().bbtcgen_u64(seed, counter))


def rmat(scale: int, edgefactor: int = 16, seed: int = 1, a=0.57, b=0.19, c=0.19, out=None, threads=0):
    """Graph500 R-MAT raw samples: (src, dst) uint32 arrays of length edgefactor<<scale."""
    n = edgefactor << scale
    s, d = _out(n, out)
    _check(_load().bbtcgen_rmat(scale, edgefactor, a, b, c, seed, _ptr(s), _ptr(d), threads))
    return s, d


def chunglu(n: int, m: int, gamma: float, dmax: float, seed: int = 1, out=None, threads=0):
    """Chung-Lu truncated power-law raw samples: (src, dst) of length m, plus the solved dmin."""
    s, d = _out(m, out)
    dmin = ctypes.c_double()
    _check(_load().bbtcgen_chunglu(n, m, gamma, dmax, seed, _ptr(s), _ptr(d), ctypes.byref(dmin), threads))
    return s, d, dmin.value


def gnp(n: int, q: float, seed: int = 1):
    """Erdős–Rényi G(n,q): every unordered pair u<v kept with probability q."""
    cnt = ctypes.c_uint64()
    _check(_load().bbtcgen_gnp(n, q, seed, None, None, 0, ctypes.byref(cnt)))
    s = np.empty(cnt.value, np.uint32)
    d = np.empty(cnt.value, np.uint32)
    _check(_load().bbtcgen_gnp(n, q, seed, _ptr(s), _ptr(d), cnt.value, ctypes.byref(cnt)))
    return s, d


def uniform_pairs(n: int, count: int, seed: int = 1):
    s = np.empty(count, np.uint32)
    d = np.empty(count, np.uint32)
    _check(_load().bbtcgen_uniform_pairs(n, count, seed, _ptr(s), _ptr(d)))
    return s, d


# Zachary karate club, 0-based ids as in networkx (public data).
KARATE_EDGES = [
    (0, 1), (0, 2), (0, 3), (0, 4), (0, 5), (0, 6), (0, 7), (0, 8), (0, 10), (0, 11), (0, 12), (0, 13),
    (0, 17), (0, 19), (0, 21), (0, 31), (1, 2), (1, 3), (1, 7), (1, 13), (1, 17), (1, 19), (1, 21), (1, 30),
    (2, 3), (2, 7), (2, 8), (2, 9), (2, 13), (2, 27), (2, 28), (2, 32), (3, 7), (3, 12), (3, 13), (4, 6),
    (4, 10), (5, 6), (5, 10), (5, 16), (6, 16), (8, 30), (8, 32), (8, 33), (9, 33), (13, 33), (14, 32),
    (14, 33), (15, 32), (15, 33), (18, 32), (18, 33), (19, 33), (20, 32), (20, 33), (22, 32), (22, 33),
    (23, 25), (23, 27), (23, 29), (23, 32), (23, 33), (24, 25), (24, 27), (24, 31), (25, 31), (26, 29),
    (26, 33), (27, 33), (28, 31), (28, 33), (29, 32), (29, 33), (30, 32), (30, 33), (31, 32), (31, 33),
    (32, 33),
]


def karate():
    e = np.asarray(KARATE_EDGES, dtype=np.uint32)
    return np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1])


@dataclass(frozen=True)
class Config:
    name: str
    kind: str          # karate | rmat | chunglu
    p: int
    scale: int = 0
    n: int = 0
    m: int = 0
    gamma: float = 0.0
    dmax: float = 0.0
    desc: str = ""

    @property
    def n_samples(self) -> int:
        if self.kind == "karate":
            return len(KARATE_EDGES)
        if self.kind == "rmat":
            return 16 << self.scale
        return self.m

    def shard(self, rank: int, world: int) -> tuple:
        """[start, end) of rank's contiguous share of the raw samples."""
        E = self.n_samples
        return E * rank // world, E * (rank + 1) // world

    def generate_range(self, start: int, count: int, seed: int = 1, out=None, threads=0):
        """Raw samples [start, start+count) of this config (a rank's shard)."""
        if self.kind == "karate":
            s, d = karate()
            s, d = s[start:start + count].copy(), d[start:start + count].copy()
            if out is not None:
                out[0][:count] = s
                out[1][:count] = d
                return out[0][:count], out[1][:count]
            return s, d
        s, d = _out(count, out)
        L = _load()
        if self.kind == "rmat":
            _check(L.bbtcgen_rmat_range(self.scale, 16, 0.57, 0.19, 0.19, seed, start, count, _ptr(s), _ptr(d),
                                        threads))
        else:
            dmin = ctypes.c_double()
            _check(L.bbtcgen_chunglu_range(self.n, self.m, self.gamma, self.dmax, seed, start, count, _ptr(s),
                                           _ptr(d), ctypes.byref(dmin), threads))
        return s, d

    def generate(self, seed: int = 1, out=None, threads=0):
        """Raw (src, dst) uint32 samples for this config."""
        if self.kind == "karate":
            s, d = karate()
            if out is not None:
                out[0][: len(s)] = s
                out[1][: len(d)] = d
                return out[0][: len(s)], out[1][: len(d)]
            return s, d
        if self.kind == "rmat":
            return rmat(self.scale, 16, seed, out=out, threads=threads)
        s, d, _ = chunglu(self.n, self.m, self.gamma, self.dmax, seed, out=out, threads=threads)
        return s, d

    @property
    def n_hint(self) -> int:
        if self.kind == "karate":
            return 34
        if self.kind == "rmat":
            return 1 << self.scale
        return self.n


CONFIGS = {
    "karate": Config("karate", "karate", p=2, desc="Zachary karate club, 2x2 blocks"),
    "rmat16": Config("rmat16", "rmat", p=4, scale=16, desc="R-MAT scale 16 ef 16, 4x4 blocks"),
    "orkut": Config("orkut", "chunglu", p=8, n=3_072_441, m=117_185_083, gamma=2.3314, dmax=33_313,
                    desc="com-Orkut-shaped Chung-Lu, 8x8 blocks"),
    # p = 10: the measured best step in round 2 (profiles/r02/ab1: p = 8 / 10 / 12: 92.7 / 92.2 /
    # 95.7 ms; round 1's sweep picked 12 of 12 / 14 / 16); SURVEY §8(d) proposed 16, the paper 28.
    "rmat24": Config("rmat24", "rmat", p=10, scale=24, desc="R-MAT scale 24 ef 16, 10x10 blocks"),
    "friendster": Config("friendster", "chunglu", p=4, n=65_608_366, m=1_806_067_135, gamma=2.0,
                         dmax=5_214, desc="Friendster-shaped Chung-Lu, 4x4 blocks"),
}
