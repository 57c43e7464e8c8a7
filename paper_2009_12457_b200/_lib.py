"""ctypes binding to libbbtc.so — argument marshalling only (include/bbtc.h).

Every function here has the C-ABI name and forwards to it; all arithmetic runs
in the library's CUDA kernels.  Importing this module never falls back to a CPU
path: if libbbtc.so is missing it raises immediately.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# BBTC_LIB overrides the library path (A/B builds of the same ABI); the default is in-tree.
LIB_PATH = os.environ.get("BBTC_LIB") or os.path.join(_HERE, "libbbtc.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
                      "there is no CPU fallback")

lib = ctypes.CDLL(LIB_PATH)

c_u32 = ctypes.c_uint32
c_u64 = ctypes.c_uint64
_u32p = ctypes.POINTER(c_u32)
_u64p = ctypes.POINTER(c_u64)
_vp = ctypes.c_void_p
_pp = ctypes.POINTER(ctypes.c_void_p)

STATUS = {0: "BBTC_OK", -1: "BBTC_EINVAL", -2: "BBTC_ENOMEM", -3: "BBTC_EIO", -4: "BBTC_EPARSE",
          -5: "BBTC_ERANGE", -6: "BBTC_ECUDA", -7: "BBTC_ENCCL", -8: "BBTC_ESTATE"}
MEM_HOST, MEM_DEVICE = 0, 1
PLAN_STATS = 1
PLAN_ROWMAJOR = 2
PLAN_SPARSE = 4
FMT_TEXT, FMT_MM, FMT_BIN = 0, 1, 2


class BBTCError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class bbtc_ctx_opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("stream", _vp), ("copy_streams", c_u32), ("reserved", c_u32)]


class bbtc_graph_stats(ctypes.Structure):
    _fields_ = [("n", c_u32), ("n_nonisolated", c_u32), ("m", c_u64), ("raw_edges", c_u64), ("d_max", c_u32),
                ("dplus_max", c_u32)]


class bbtc_plan_info(ctypes.Structure):
    _fields_ = [("p", c_u32), ("clamped", c_u32), ("n_tasks", c_u64), ("n_blocks", c_u64), ("m", c_u64),
                ("m_max", c_u64), ("lambda_", ctypes.c_double), ("dmax_blk", c_u32), ("host_blocks", c_u32),
                ("block_bytes", c_u64), ("max_task_bytes", c_u64), ("b_alg", c_u64), ("visits", c_u64),
                ("work_items", c_u64), ("sum_a", c_u64), ("sum_b", c_u64),
                ("dense_tasks", c_u32), ("dense_bits", c_u32), ("dense_bytes", c_u64), ("stream_bytes", c_u64),
                ("list_read_bytes", c_u64), ("dense_edge_bytes", c_u64), ("slot_bytes", c_u64)]


class bbtc_edge_list(ctypes.Structure):
    _fields_ = [("src", _u32p), ("dst", _u32p), ("n_edges", c_u64), ("n_hint", c_u32), ("reserved", c_u32)]


class bbtc_edge_map(ctypes.Structure):
    _fields_ = [("pairs", _u32p), ("n_edges", c_u64), ("base", _vp), ("bytes", c_u64)]


class bbtc_timing(ctypes.Structure):
    _fields_ = [("t_total_ms", ctypes.c_double), ("t_h2d_ms", ctypes.c_double), ("t_kernel_ms", ctypes.c_double),
                ("h2d_bytes", c_u64), ("launches", c_u64), ("t_dense_ms", ctypes.c_double)]


class bbtc_block_ptrs(ctypes.Structure):
    _fields_ = [("edge", _vp * 3), ("n_edge_arrays", c_u32), ("reserved", c_u32), ("nnz", c_u64),
                ("rowptr", _vp), ("rowptr_len", c_u64)]


class bbtc_hybrid_opts(ctypes.Structure):
    _fields_ = [("cpu_threads", c_u32), ("gpu_chunk", c_u32), ("cutoff", ctypes.c_double)]


class bbtc_hybrid_stats(ctypes.Structure):
    _fields_ = [("cpu_tasks", c_u64), ("gpu_tasks", c_u64), ("gpu_launches", c_u64), ("cpu_triangles", c_u64),
                ("t_cpu_ms", ctypes.c_double), ("t_gpu_ms", ctypes.c_double)]


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_st = ctypes.c_int
bbtc_ctx_create = _sig("bbtc_ctx_create", _st, ctypes.POINTER(bbtc_ctx_opts), _pp)
bbtc_ctx_free = _sig("bbtc_ctx_free", None, _vp)
bbtc_ctx_sync = _sig("bbtc_ctx_sync", _st, _vp)
bbtc_ctx_stream = _sig("bbtc_ctx_stream", _st, _vp, ctypes.POINTER(_vp))
bbtc_ctx_launches = _sig("bbtc_ctx_launches", c_u64, _vp)
bbtc_graph_from_edges = _sig("bbtc_graph_from_edges", _st, _vp, _vp, _vp, c_u64, c_u32, ctypes.c_int, _pp)
bbtc_graph_stats_get = _sig("bbtc_graph_stats_get", _st, _vp, ctypes.POINTER(bbtc_graph_stats))
bbtc_graph_size = _sig("bbtc_graph_size", _st, _vp, _u32p, _u64p)
bbtc_graph_rank = _sig("bbtc_graph_rank", _st, _vp, _vp, _u32p)
bbtc_graph_csr = _sig("bbtc_graph_csr", _st, _vp, _vp, _u64p, _u32p)
bbtc_graph_free = _sig("bbtc_graph_free", None, _vp)
bbtc_edges_read = _sig("bbtc_edges_read", _st, ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(bbtc_edge_list))
bbtc_edges_free = _sig("bbtc_edges_free", None, ctypes.POINTER(bbtc_edge_list))
bbtc_graph_load = _sig("bbtc_graph_load", _st, _vp, ctypes.c_char_p, ctypes.c_int, c_u32, _pp)
bbtc_edges_map = _sig("bbtc_edges_map", _st, ctypes.c_char_p, ctypes.POINTER(bbtc_edge_map))
bbtc_edges_unmap = _sig("bbtc_edges_unmap", None, ctypes.POINTER(bbtc_edge_map))
bbtc_graph_from_pairs = _sig("bbtc_graph_from_pairs", _st, _vp, _vp, c_u64, c_u32, ctypes.c_int, _pp)
bbtc_graph_load_mapped = _sig("bbtc_graph_load_mapped", _st, _vp, ctypes.c_char_p, c_u32, _pp)
bbtc_plan_create = _sig("bbtc_plan_create", _st, _vp, _vp, c_u32, _u32p, c_u32, _pp)
bbtc_plan_auto_p = _sig("bbtc_plan_auto_p", _st, _vp, _vp, c_u64, c_u32, c_u32, _u32p)
bbtc_plan_info_get = _sig("bbtc_plan_info_get", _st, _vp, ctypes.POINTER(bbtc_plan_info))
bbtc_plan_cuts = _sig("bbtc_plan_cuts", _st, _vp, _u32p)
bbtc_plan_block = _sig("bbtc_plan_block", _st, _vp, _vp, c_u32, c_u32, _u32p, _u32p, _u32p, _u64p)
bbtc_plan_to_host = _sig("bbtc_plan_to_host", _st, _vp, _vp)
bbtc_plan_set_budget = _sig("bbtc_plan_set_budget", _st, _vp, c_u64)
bbtc_plan_free = _sig("bbtc_plan_free", None, _vp)
bbtc_n_tasks = _sig("bbtc_n_tasks", c_u64, c_u32)
bbtc_task_index = _sig("bbtc_task_index", _st, c_u32, c_u32, c_u32, c_u32, _u64p)
bbtc_task_ijk = _sig("bbtc_task_ijk", _st, c_u32, c_u64, _u32p, _u32p, _u32p)
bbtc_count_async = _sig("bbtc_count_async", _st, _vp, _vp, c_u32, c_u32, _vp)
bbtc_count = _sig("bbtc_count", _st, _vp, _vp, c_u32, c_u32, c_u32, _u64p, _u64p, ctypes.POINTER(bbtc_timing))
bbtc_count_hybrid = _sig("bbtc_count_hybrid", _st, _vp, _vp, ctypes.POINTER(bbtc_hybrid_opts), _u64p, _u64p,
                         ctypes.POINTER(bbtc_timing), ctypes.POINTER(bbtc_hybrid_stats))
bbtc_plan_block_nnz = _sig("bbtc_plan_block_nnz", _st, _vp, _u64p)
bbtc_task_times = _sig("bbtc_task_times", _st, _vp, _vp, ctypes.POINTER(ctypes.c_double))
bbtc_cuts_refine = _sig("bbtc_cuts_refine", _st, _vp, _vp, c_u32, _u32p, c_u32, _u32p, _u64p)
bbtc_stage = _sig("bbtc_stage", _st, _vp, _vp)
bbtc_unstage = _sig("bbtc_unstage", _st, _vp, _vp)
bbtc_stage_blocks = _sig("bbtc_stage_blocks", _st, _vp, _vp, _u32p, c_u32, c_u32)
bbtc_shard_canon = _sig("bbtc_shard_canon", _st, _vp, _vp, _vp, c_u64, ctypes.c_int, c_u32, c_u32, _vp, _u64p,
                        _u32p)
bbtc_shard_graph = _sig("bbtc_shard_graph", _st, _vp, _vp, c_u64, c_u32, _vp, _pp)
bbtc_shard_rank = _sig("bbtc_shard_rank", _st, _vp, _vp, _vp, c_u64)
bbtc_shard_block_sizes = _sig("bbtc_shard_block_sizes", _st, _vp, _vp, c_u32, _u32p, _vp, _u32p, _u32p)
bbtc_shard_assign = _sig("bbtc_shard_assign", _st, c_u32, _u32p, _u64p, c_u32, _u32p, _u32p)
bbtc_shard_by_block = _sig("bbtc_shard_by_block", _st, _vp, _vp, c_u32, _u32p, _u32p, c_u32, _vp, _u64p)
bbtc_plan_create_shard = _sig("bbtc_plan_create_shard", _st, _vp, _vp, _vp, c_u64, c_u32, _u32p, _u64p, _u32p,
                              c_u32, c_u32, c_u32, _pp)
bbtc_plan_block_ptrs = _sig("bbtc_plan_block_ptrs", _st, _vp, c_u32, ctypes.POINTER(bbtc_block_ptrs))
bbtc_last_error = _sig("bbtc_last_error", ctypes.c_char_p)
bbtc_version = _sig("bbtc_version", ctypes.c_char_p)

EXPORTS = [n for n in dir() if n.startswith("bbtc_") and callable(globals()[n]) and
           not isinstance(globals()[n], type)]


def check(rc: int):
    if rc != 0:
        raise BBTCError(rc, (bbtc_last_error() or b"").decode())
