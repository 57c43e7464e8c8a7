"""CPU oracle for BBTC triangle counts (ctypes binding to oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  The product
path (paper_2009_12457_b200) never imports it, and it shares no code with it.

Every function follows a passage of PAPER.md (see oracle.cpp for the per-step
citations).  Pins (tests/test_oracle.py): brute force on tiny graphs, K_n closed
forms, textbook graph families, karate = 45 with its per-task golden values,
Σ per-vertex = 3T, Σ per-task = T for every p and random cuts, invariance under
relabelling / duplicates / self-loops, and an independent scipy cross-check.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_vp = ctypes.c_void_p


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run __graft_entry__.build() (make)")
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_build.restype = _vp
        L.oracle_build.argtypes = [_u32p, _u32p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int]
        L.oracle_free.argtypes = [_vp]
        L.oracle_n.restype = ctypes.c_uint32
        L.oracle_n.argtypes = [_vp]
        L.oracle_m.restype = ctypes.c_uint64
        L.oracle_m.argtypes = [_vp]
        L.oracle_rank.argtypes = [_vp, _u32p]
        L.oracle_degrees.argtypes = [_vp, _u32p]
        L.oracle_csr.argtypes = [_vp, _u64p, _u32p]
        L.oracle_effective_p.restype = ctypes.c_uint32
        L.oracle_effective_p.argtypes = [_vp, ctypes.c_uint32]
        L.oracle_default_cuts.restype = ctypes.c_uint32
        L.oracle_default_cuts.argtypes = [_vp, ctypes.c_uint32, _u32p]
        L.oracle_count.argtypes = [_vp, ctypes.c_uint32, _u32p, ctypes.c_int, _u64p, _u64p, _u64p]
        L.oracle_count_task.argtypes = [_vp, ctypes.c_uint32, _u32p, ctypes.c_uint32, ctypes.c_uint32,
                                        ctypes.c_uint32, ctypes.c_int, _u64p]
        L.oracle_task_list.argtypes = [ctypes.c_uint32, _u32p, _u32p, _u32p]
        L.oracle_count_rows.argtypes = [_vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int, _u64p, _u64p]
        L.oracle_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _p32(a):
    return a.ctypes.data_as(_u32p)


def _p64(a):
    return a.ctypes.data_as(_u64p)


def n_tasks(p: int) -> int:
    return p * (p + 1) * (p + 2) // 6


class OracleGraph:
    """Canonicalised, degree-ranked, oriented graph (oracle steps 1-4)."""

    def __init__(self, src, dst, n_hint: int = 0, threads: int = 0):
        src = np.ascontiguousarray(src, dtype=np.uint32)
        dst = np.ascontiguousarray(dst, dtype=np.uint32)
        assert src.shape == dst.shape
        self._h = _load().oracle_build(_p32(src), _p32(dst), len(src), n_hint, threads)
        self.threads = threads

    def __del__(self):
        if getattr(self, "_h", None):
            _load().oracle_free(self._h)
            self._h = None

    @property
    def n(self) -> int:
        return int(_load().oracle_n(self._h))

    @property
    def m(self) -> int:
        return int(_load().oracle_m(self._h))

    def rank(self):
        r = np.empty(self.n, np.uint32)
        _load().oracle_rank(self._h, _p32(r))
        return r

    def degrees(self):
        d = np.empty(self.n, np.uint32)
        _load().oracle_degrees(self._h, _p32(d))
        return d

    def csr(self):
        row = np.empty(self.n + 1, np.uint64)
        col = np.empty(self.m, np.uint32)
        _load().oracle_csr(self._h, _p64(row), _p32(col))
        return row, col

    def effective_p(self, p: int) -> int:
        return int(_load().oracle_effective_p(self._h, p))

    def default_cuts(self, p: int):
        pe = self.effective_p(p)
        if pe == 0:
            raise ValueError("p must be >= 1")
        cuts = np.empty(pe + 1, np.uint32)
        _load().oracle_default_cuts(self._h, p, _p32(cuts))
        return cuts

    def count(self, p: int = 1, cuts=None, per_vertex: bool = False):
        """Returns (total, per_task[Alg. 4 order], per_vertex or None, cuts)."""
        if cuts is None:
            cuts = self.default_cuts(p)
        cuts = np.ascontiguousarray(cuts, dtype=np.uint32)
        p = len(cuts) - 1
        tot = ctypes.c_uint64()
        pt = np.zeros(n_tasks(p), np.uint64)
        pv = np.zeros(self.n, np.uint64) if per_vertex else None
        rc = _load().oracle_count(self._h, p, _p32(cuts), self.threads, ctypes.byref(tot), _p64(pt),
                                  _p64(pv) if per_vertex else None)
        if rc != 0:
            raise ValueError(_load().oracle_last_error().decode())
        return int(tot.value), pt, pv, cuts

    def count_task(self, cuts, i: int, j: int, k: int) -> int:
        cuts = np.ascontiguousarray(cuts, dtype=np.uint32)
        c = ctypes.c_uint64()
        rc = _load().oracle_count_task(self._h, len(cuts) - 1, _p32(cuts), i, j, k, self.threads, ctypes.byref(c))
        if rc != 0:
            raise ValueError(_load().oracle_last_error().decode())
        return int(c.value)

    def count_rows(self, u0: int, u1: int, stride: int = 1):
        """Unblocked node iterator over rows u0, u0+stride, ... < u1: (triangles, edges visited)."""
        t = ctypes.c_uint64()
        e = ctypes.c_uint64()
        _load().oracle_count_rows(self._h, u0, u1, stride, self.threads, ctypes.byref(t), ctypes.byref(e))
        return int(t.value), int(e.value)


def task_list(p: int):
    """Alg. 4 enumeration order as an (n_tasks, 3) array."""
    nt = n_tasks(p)
    a, b, c = (np.empty(nt, np.uint32) for _ in range(3))
    _load().oracle_task_list(p, _p32(a), _p32(b), _p32(c))
    return np.stack([a, b, c], axis=1)


def count(src, dst, n_hint: int = 0, p: int = 1, cuts=None, per_vertex: bool = False, threads: int = 0):
    """One-shot oracle: returns dict(total, per_task, per_vertex, cuts, n, m)."""
    g = OracleGraph(src, dst, n_hint, threads)
    tot, pt, pv, cuts = g.count(p, cuts, per_vertex)
    return dict(total=tot, per_task=pt, per_vertex=pv, cuts=cuts, n=g.n, m=g.m)
