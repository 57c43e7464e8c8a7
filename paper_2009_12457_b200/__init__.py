"""bbtc-b200: B200-native block-based triangle counting (BBTC, arXiv 2009.12457).

Thin Python layer over libbbtc.so (include/bbtc.h).  The classes only marshal
arguments and own handles; every step of the path (canonicalise, degree order,
partition, BCSR, count) runs in the library's sm_100a kernels.

    ctx   = Context(device=0)
    g     = Graph.from_edges(ctx, src, dst, n_hint)   # numpy (host) or torch CUDA tensors
    plan  = Plan(ctx, g, p=16)                       # cuts, blocks, tasks (Alg. 4)
    total, per_task = plan.count()                   # uint64 total + per-task (Alg. 4 order)
"""
from __future__ import annotations

import atexit
import ctypes
import weakref

import numpy as np

from . import _lib as L
from ._lib import BBTCError, MEM_DEVICE, MEM_HOST, PLAN_STATS

__all__ = ["Context", "Graph", "Plan", "BBTCError", "n_tasks", "task_index", "task_ijk", "count_triangles",
           "read_edges", "EdgeMap", "FORMATS", "auto_p"]

FORMATS = {"text": L.FMT_TEXT, "mm": L.FMT_MM, "bin": L.FMT_BIN}


def read_edges(path, fmt: str = "text"):
    """bbtc_edges_read: (src, dst, n_hint) of an edge-list file (host only, no device)."""
    e = L.bbtc_edge_list()
    L.check(L.bbtc_edges_read(str(path).encode(), FORMATS[fmt], ctypes.byref(e)))
    try:
        n = e.n_edges
        src = np.ctypeslib.as_array(e.src, shape=(n,)).copy() if n else np.empty(0, np.uint32)
        dst = np.ctypeslib.as_array(e.dst, shape=(n,)).copy() if n else np.empty(0, np.uint32)
        return src, dst, int(e.n_hint)
    finally:
        L.bbtc_edges_free(ctypes.byref(e))


class EdgeMap:
    """bbtc_edges_map: a binary edge file (interleaved uint32 pairs) memory-mapped
    read-only; `pairs` is an (n_edges, 2) numpy view of the mapping (valid until close)."""

    def __init__(self, path):
        self._m = L.bbtc_edge_map()
        L.check(L.bbtc_edges_map(str(path).encode(), ctypes.byref(self._m)))
        n = int(self._m.n_edges)
        self.n_edges = n
        self.pairs = (np.ctypeslib.as_array(self._m.pairs, shape=(n, 2)) if n
                      else np.empty((0, 2), np.uint32))
        self.pairs.flags.writeable = False   # a PROT_READ mapping: writes would fault

    def close(self):
        if getattr(self, "_m", None) is not None and L is not None and L.lib is not None:
            self.pairs = None
            L.bbtc_edges_unmap(ctypes.byref(self._m))
        self._m = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        self.close()


def _ptr(x, want_dtype):
    """(pointer, length, mem) of a host numpy array or a CUDA tensor."""
    if hasattr(x, "data_ptr") and hasattr(x, "is_cuda"):
        import torch
        assert x.is_contiguous(), "tensor must be contiguous"
        assert x.dtype in (torch.int32, torch.uint32), "edge arrays must be 32-bit"
        return ctypes.c_void_p(x.data_ptr()), x.numel(), (MEM_DEVICE if x.is_cuda else MEM_HOST)
    a = np.asarray(x)
    if a.dtype != want_dtype:
        # Vertex ids are u32 with 0xFFFFFFFF reserved (bbtc.h); refuse values a cast would wrap.
        if a.size and (a.dtype.kind not in "iu" or int(a.min()) < 0 or int(a.max()) > 0xFFFFFFFE):
            raise OverflowError("vertex ids must be integers in [0, 2^32-2]")
    a = np.ascontiguousarray(a, dtype=want_dtype)
    return ctypes.c_void_p(a.ctypes.data), len(a), MEM_HOST, a


def n_tasks(p: int) -> int:
    return int(L.bbtc_n_tasks(p))


def task_index(p: int, i: int, j: int, k: int) -> int:
    out = ctypes.c_uint64()
    L.check(L.bbtc_task_index(p, i, j, k, ctypes.byref(out)))
    return int(out.value)


def task_ijk(p: int, idx: int):
    i, j, k = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
    L.check(L.bbtc_task_ijk(p, idx, ctypes.byref(i), ctypes.byref(j), ctypes.byref(k)))
    return int(i.value), int(j.value), int(k.value)


_LIVE = weakref.WeakSet()   # live contexts


@atexit.register
def _close_all():
    """Free every live context (and its graphs and plans) while the interpreter and the
    CUDA runtime are intact — not in arbitrary order during module teardown."""
    for c in list(_LIVE):
        try:
            c.close()
        except Exception:  # noqa: BLE001
            pass


class Context:
    """A CUDA device + the stream the library enqueues on (bbtc_ctx)."""

    def __init__(self, device: int = 0, stream: int | None = None, copy_streams: int = 0):
        """stream: a cudaStream_t handle (e.g. torch.cuda.Stream().cuda_stream) to enqueue on, or None
        for a library-created stream.  0 (the legacy default stream) is rejected: the library's own
        streams are non-blocking and would not be ordered with it."""
        if stream == 0:
            raise ValueError("pass a non-default stream handle (torch.cuda.Stream().cuda_stream) or None")
        o = L.bbtc_ctx_opts(device, ctypes.c_void_p(stream) if stream else None, copy_streams, 0)
        h = ctypes.c_void_p()
        L.check(L.bbtc_ctx_create(ctypes.byref(o), ctypes.byref(h)))
        self._h = h
        self.device = device
        self._children = weakref.WeakSet()   # graphs / plans: freed before the context
        _LIVE.add(self)

    @property
    def handle(self):
        return self._h

    def sync(self):
        L.check(L.bbtc_ctx_sync(self._h))

    @property
    def stream(self) -> int:
        """The cudaStream_t handle this context enqueues on (bbtc_ctx_stream)."""
        s = ctypes.c_void_p()
        L.check(L.bbtc_ctx_stream(self._h, ctypes.byref(s)))
        return int(s.value or 0)

    @property
    def launches(self) -> int:
        return int(L.bbtc_ctx_launches(self._h))

    def close(self):
        if getattr(self, "_h", None) and L is not None and L.lib is not None:
            for c in list(getattr(self, "_children", ())):
                c.close()
            L.bbtc_ctx_free(self._h)
        self._h = None

    def __del__(self):
        self.close()


class Graph:
    """Canonical, degree-ranked, oriented graph on the device (bbtc_graph)."""

    def __init__(self, ctx: Context, h):
        self.ctx = ctx
        self._h = h
        ctx._children.add(self)

    @classmethod
    def from_edges(cls, ctx: Context, src, dst, n_hint: int = 0) -> "Graph":
        ps = _ptr(src, np.uint32)
        pd = _ptr(dst, np.uint32)
        assert ps[1] == pd[1], "src and dst differ in length"
        assert ps[2] == pd[2], "src and dst must both be host or both device"
        h = ctypes.c_void_p()
        L.check(L.bbtc_graph_from_edges(ctx.handle, ps[0], pd[0], ps[1], n_hint, ps[2], ctypes.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_pairs(cls, ctx: Context, pairs, n_hint: int = 0) -> "Graph":
        """bbtc_graph_from_pairs: interleaved (n, 2) uint32 pairs, host (numpy, incl. an
        EdgeMap's mapping) or device (CUDA tensor)."""
        if hasattr(pairs, "data_ptr"):
            assert pairs.dim() == 2 and pairs.shape[1] == 2, "pairs must be (n, 2)"
            ptr, n, mem = _ptr(pairs.reshape(-1), np.uint32)[:3]
            n //= 2
        else:
            a = np.asarray(pairs)
            assert a.ndim == 2 and a.shape[1] == 2, "pairs must be (n, 2)"
            if not (a.dtype == np.uint32 and a.flags["C_CONTIGUOUS"]):
                a = _ptr(a.reshape(-1), np.uint32)[3].reshape(-1, 2)
            ptr, n, mem = ctypes.c_void_p(a.ctypes.data), a.shape[0], MEM_HOST
        h = ctypes.c_void_p()
        L.check(L.bbtc_graph_from_pairs(ctx.handle, ptr, n, n_hint, mem, ctypes.byref(h)))
        return cls(ctx, h)

    @classmethod
    def load_mapped(cls, ctx: Context, path, n_hint: int = 0) -> "Graph":
        """bbtc_graph_load_mapped: a binary edge file, memory-mapped (never read whole
        into RAM), built into the graph (a1-a2)."""
        h = ctypes.c_void_p()
        L.check(L.bbtc_graph_load_mapped(ctx.handle, str(path).encode(), n_hint, ctypes.byref(h)))
        return cls(ctx, h)

    @classmethod
    def load(cls, ctx: Context, path, fmt: str = "text", n_hint: int = 0) -> "Graph":
        """bbtc_graph_load: read an edge-list file and build the graph (a1-a2)."""
        h = ctypes.c_void_p()
        L.check(L.bbtc_graph_load(ctx.handle, str(path).encode(), FORMATS[fmt], n_hint, ctypes.byref(h)))
        return cls(ctx, h)

    def stats(self) -> dict:
        s = L.bbtc_graph_stats()
        L.check(L.bbtc_graph_stats_get(self._h, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in s._fields_ if f != "reserved"}

    def size(self):
        """(n, m) without device work (bbtc_graph_size)."""
        n, m = ctypes.c_uint32(), ctypes.c_uint64()
        L.check(L.bbtc_graph_size(self._h, ctypes.byref(n), ctypes.byref(m)))
        return int(n.value), int(m.value)

    @property
    def n(self) -> int:
        return self.size()[0]

    @property
    def m(self) -> int:
        return self.size()[1]

    def rank(self) -> np.ndarray:
        r = np.empty(self.n, np.uint32)
        L.check(L.bbtc_graph_rank(self.ctx.handle, self._h, r.ctypes.data_as(L._u32p)))
        return r

    def csr(self):
        st = self.stats()
        row = np.empty(st["n"] + 1, np.uint64)
        col = np.empty(st["m"], np.uint32)
        L.check(L.bbtc_graph_csr(self.ctx.handle, self._h, row.ctypes.data_as(L._u64p), col.ctypes.data_as(L._u32p)))
        return row, col

    def close(self):
        if getattr(self, "_h", None) and L is not None and L.lib is not None:
            L.bbtc_graph_free(self._h)
        self._h = None

    def __del__(self):
        self.close()


def refine_cuts(ctx: "Context", graph: "Graph", p: int, cuts=None, max_evals: int = 200):
    """bbtc_cuts_refine (§8(f)#4): PBD-like cuts minimising m_max; returns (cuts, m_max)."""
    out = np.empty(p + 1, np.uint32)
    mm = ctypes.c_uint64()
    cin = None if cuts is None else np.ascontiguousarray(cuts, dtype=np.uint32)
    L.check(L.bbtc_cuts_refine(ctx.handle, graph._h, p, None if cin is None else cin.ctypes.data_as(L._u32p),
                               max_evals, out.ctypes.data_as(L._u32p), ctypes.byref(mm)))
    n = graph.n
    pe = p if cin is not None else (min(p, n) if n else 1)   # the default rule clamps p to n
    return out[:pe + 1].copy(), int(mm.value)


def auto_p(ctx: "Context", graph: "Graph", budget_bytes: int, depth: int = 2, row_major: bool = False) -> int:
    """bbtc_plan_auto_p: the smallest p whose largest task footprint x depth fits the budget."""
    p = ctypes.c_uint32()
    L.check(L.bbtc_plan_auto_p(ctx.handle, graph._h, int(budget_bytes), depth,
                               L.PLAN_ROWMAJOR if row_major else 0, ctypes.byref(p)))
    return int(p.value)


class Plan:
    """Cut vector + BCSR blocks + task list (bbtc_plan)."""

    def __init__(self, ctx: Context, graph: Graph, p: int = 1, cuts=None, stats: bool = False,
                 row_major: bool = False, sparse: bool = False):
        """row_major: walk each G_ij row by row (stage N(G_ik,u), gather N(G_jk,v)) instead of the
        default column order (stage N(G_jk,v), gather N(G_ik,u)).  sparse: no dense (bit-row)
        tasks, every task through the list kernel.  Same counts either way."""
        self.ctx = ctx
        h = ctypes.c_void_p()
        cptr = None
        if cuts is not None:
            self._cuts_in = np.ascontiguousarray(cuts, dtype=np.uint32)
            p = len(self._cuts_in) - 1
            cptr = self._cuts_in.ctypes.data_as(L._u32p)
        flags = ((L.PLAN_STATS if stats else 0) | (L.PLAN_ROWMAJOR if row_major else 0)
                 | (L.PLAN_SPARSE if sparse else 0))
        L.check(L.bbtc_plan_create(ctx.handle, graph._h, p, cptr, flags, ctypes.byref(h)))
        self._h = h
        ctx._children.add(self)

    def info(self) -> dict:
        i = L.bbtc_plan_info()
        L.check(L.bbtc_plan_info_get(self._h, ctypes.byref(i)))
        d = {f: getattr(i, f) for f, _ in i._fields_}
        d["lambda"] = d.pop("lambda_")
        return d

    @property
    def p(self) -> int:
        return self.info()["p"]

    @property
    def n_tasks(self) -> int:
        return self.info()["n_tasks"]

    def cuts(self) -> np.ndarray:
        c = np.empty(self.p + 1, np.uint32)
        L.check(L.bbtc_plan_cuts(self._h, c.ctypes.data_as(L._u32p)))
        return c

    def block(self, i: int, j: int):
        """(row_ptr, col, row) of block G_ij with block-local ids."""
        nnz = ctypes.c_uint64()
        L.check(L.bbtc_plan_block(self.ctx.handle, self._h, i, j, None, None, None, ctypes.byref(nnz)))
        c = self.cuts()
        rp = np.empty(int(c[i + 1] - c[i]) + 1, np.uint32)
        col = np.empty(nnz.value, np.uint32)
        row = np.empty(nnz.value, np.uint32)
        L.check(L.bbtc_plan_block(self.ctx.handle, self._h, i, j, rp.ctypes.data_as(L._u32p),
                                  col.ctypes.data_as(L._u32p), row.ctypes.data_as(L._u32p), None))
        return rp, col, row

    def to_host(self):
        L.check(L.bbtc_plan_to_host(self.ctx.handle, self._h))

    def set_budget(self, nbytes: int):
        """Out-of-core: keep at most nbytes of blocks on the device when counting a host plan."""
        L.check(L.bbtc_plan_set_budget(self._h, nbytes))

    def stage(self):
        L.check(L.bbtc_stage(self.ctx.handle, self._h))

    def stage_blocks(self, ids, resident: bool = False):
        """bbtc_stage_blocks: copy these blocks of a host plan to the device (§8(e) owner copy)."""
        a = np.ascontiguousarray(ids, dtype=np.uint32)
        L.check(L.bbtc_stage_blocks(self.ctx.handle, self._h, a.ctypes.data_as(L._u32p), len(a), 1 if resident else 0))

    def unstage(self):
        L.check(L.bbtc_unstage(self.ctx.handle, self._h))

    def count(self, rank: int = 0, world: int = 1, timing: bool = False):
        """Synchronous count: (total, per_task uint64[n_tasks] in Alg. 4 order[, timing dict])."""
        tot = ctypes.c_uint64()
        pt = np.zeros(self.n_tasks, np.uint64)
        tm = L.bbtc_timing()
        L.check(L.bbtc_count(self.ctx.handle, self._h, rank, world, 0, ctypes.byref(tot),
                             pt.ctypes.data_as(L._u64p), ctypes.byref(tm)))
        if timing:
            return int(tot.value), pt, {f: getattr(tm, f) for f, _ in tm._fields_}
        return int(tot.value), pt

    def block_nnz(self) -> np.ndarray:
        """nnz of every block, block order b = j(j+1)/2 + i (bbtc_plan_block_nnz)."""
        p = self.p
        out = np.empty(p * (p + 1) // 2, np.uint64)
        L.check(L.bbtc_plan_block_nnz(self._h, out.ctypes.data_as(L._u64p)))
        return out

    def task_times(self) -> np.ndarray:
        """Device ms of every task alone, canonical order (bbtc_task_times; a study tool)."""
        out = np.empty(self.n_tasks, np.float64)
        L.check(L.bbtc_task_times(self.ctx.handle, self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def count_hybrid(self, cpu_threads: int = 0, cutoff: float = 0.5, gpu_chunk: int = 0):
        """bbtc_count_hybrid (§8(f)#3): GPU from the heavy end of the ExecTime queue, CPU threads
        from the light end up to the cut-off.  Needs to_host() + stage().  Returns
        (total, per_task, stats dict)."""
        tot = ctypes.c_uint64()
        pt = np.zeros(self.n_tasks, np.uint64)
        o = L.bbtc_hybrid_opts(cpu_threads, gpu_chunk, cutoff)
        tm = L.bbtc_timing()
        hs = L.bbtc_hybrid_stats()
        L.check(L.bbtc_count_hybrid(self.ctx.handle, self._h, ctypes.byref(o), ctypes.byref(tot),
                                    pt.ctypes.data_as(L._u64p), ctypes.byref(tm), ctypes.byref(hs)))
        st = {f: getattr(hs, f) for f, _ in hs._fields_}
        st["t_total_ms"] = tm.t_total_ms
        return int(tot.value), pt, st

    def count_async(self, d_counts, rank: int = 0, world: int = 1):
        """Enqueue the count into a CUDA uint64/int64 tensor of n_tasks+1 entries (last = total)."""
        assert d_counts.is_cuda and d_counts.numel() >= self.n_tasks + 1 and d_counts.element_size() == 8
        L.check(L.bbtc_count_async(self.ctx.handle, self._h, rank, world, ctypes.c_void_p(d_counts.data_ptr())))

    def close(self):
        if getattr(self, "_h", None) and L is not None and L.lib is not None:
            L.bbtc_plan_free(self._h)
        self._h = None

    def __del__(self):
        self.close()


def count_triangles(src, dst, n_hint: int = 0, p: int = 1, cuts=None, device: int = 0, ctx: Context | None = None):
    """One-shot: returns dict(total, per_task, cuts, n, m)."""
    ctx = ctx or Context(device)
    g = Graph.from_edges(ctx, src, dst, n_hint)
    plan = Plan(ctx, g, p, cuts)
    tot, pt = plan.count()
    st = g.stats()
    return dict(total=tot, per_task=pt, cuts=plan.cuts(), n=st["n"], m=st["m"], plan=plan, graph=g)
