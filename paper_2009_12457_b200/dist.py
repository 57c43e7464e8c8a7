"""Multi-GPU glue: one process per GPU, torch.distributed for the
plumbing (NCCL over NVLink on GPUs; gloo, staged through host memory, for CPU-side
and shared-GPU tests).  Every arithmetic step runs in libbbtc's kernels; this module
only moves buffers between ranks and calls the C-ABI in order.

Sharded build (`build_sharded`): each rank starts from its own 1/N of
the raw edges (resident or in pinned host memory: only that share crosses its PCIe
link) and
  1. canonicalises + de-duplicates it and groups the keys by a hash owner rank
     (bbtc_shard_canon)                                   -> all-to-all #1 (NCCL)
  2. de-duplicates what it received, partial degrees (bbtc_shard_graph)
                                                          -> all-reduce of degrees
  3. ranks every vertex and orients its edges (bbtc_shard_rank)
  4. cuts + its per-block edge counts (bbtc_shard_block_sizes) -> all-reduce
  5. task -> rank and block -> owner, LPT with block affinity (bbtc_shard_assign;
     identical on every rank)
  6. groups its oriented edges by block owner (bbtc_shard_by_block) -> all-to-all #2
  7. builds the blocks it owns in the global layout (bbtc_plan_create_shard)
  8. forwards each block from its owner to the other ranks whose tasks read it
     (point-to-point over NVLink: NCCL send/recv batched in one group).
Then `plan.count_async(counts, rank, world)` counts this rank's tasks and one
all-reduce of the uint64 per-task counters (int64 bit pattern: two's-complement
addition is bit-identical) gives every rank the full result.
"""
from __future__ import annotations

import ctypes
import time

import numpy as np


def _dist():
    import torch.distributed as dist
    return dist


def _world_rank(group=None):
    dist = _dist()
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def _nccl(group=None) -> bool:
    return _dist().get_backend(group) == "nccl"


def reduce_counts(counts, group=None):
    """In-place sum of the per-task counter tensor over all ranks (one collective)."""
    dist = _dist()
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        _all_reduce(counts, dist.ReduceOp.SUM, group)
    return counts


def _all_reduce(t, op, group=None):
    dist = _dist()
    if t.is_cuda and not _nccl(group):      # gloo: through host memory
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)
    return t


def count_distributed(plan, counts, group=None):
    """Enqueue this rank's share of the count and combine the ranks' counters.

    counts: CUDA int64 tensor of plan.n_tasks + 1 entries (last = total)."""
    world, rank = _world_rank(group)
    plan.count_async(counts, rank, world)
    _after_ctx_stream(plan.ctx, counts)
    return reduce_counts(counts, group)


def _after_ctx_stream(ctx, counts):
    """Make torch's current stream (the one NCCL/gloo order the collective after) wait
    for the count enqueued on the context's stream; a no-op when they are the same."""
    if not getattr(counts, "is_cuda", False):
        return
    import torch
    cur = torch.cuda.current_stream(counts.device)
    h = ctx.stream
    if h and h != cur.cuda_stream:
        ev = torch.cuda.Event()
        ev.record(torch.cuda.ExternalStream(h, device=counts.device))
        cur.wait_event(ev)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank timing (multi-GPU times are max over ranks)."""
    import torch
    dist = _dist()
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    _all_reduce(t, dist.ReduceOp.MAX, group)
    return float(t.item())


# ---- buffer movement ---------------------------------------------------------------
def exchange(send, send_counts, group=None):
    """All-to-all of a grouped int64 buffer: send[0:send_counts[0]] goes to rank 0, the
    next send_counts[1] to rank 1, ...  Returns (received tensor, received counts)."""
    import torch
    dist = _dist()
    world, _ = _world_rank(group)
    sc = torch.tensor([int(x) for x in send_counts], dtype=torch.int64)
    nccl = _nccl(group) and send.is_cuda
    if nccl:
        rc_d = torch.empty_like(sc, device=send.device)
        dist.all_to_all_single(rc_d, sc.to(send.device), group=group)
        rc = rc_d.cpu()
    else:
        rc = torch.empty_like(sc)
        dist.all_to_all_single(rc, sc, group=group)
    n_out, n_in = int(sc.sum()), int(rc.sum())
    recv = torch.empty(max(n_in, 1), dtype=torch.int64, device=send.device)
    ins, outs = sc.tolist(), rc.tolist()
    if nccl:
        dist.all_to_all_single(recv[:n_in], send[:n_out], output_split_sizes=outs, input_split_sizes=ins, group=group)
    else:
        h = torch.empty(n_in, dtype=torch.int64)
        dist.all_to_all_single(h, send[:n_out].cpu(), output_split_sizes=outs, input_split_sizes=ins, group=group)
        recv[:n_in].copy_(h)
    return recv[:n_in], outs


class _DevArray:
    """__cuda_array_interface__ over library-owned device memory (a zero-copy view)."""

    def __init__(self, ptr: int, count: int, typestr: str = "<u4"):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (ptr, False),
                                         "version": 2, "strides": None}


def _view_u32(ptr: int, count: int, device):
    import torch
    t = torch.as_tensor(_DevArray(ptr, count, "<i4"), device=device)
    assert t.data_ptr() == ptr
    return t


def task_blocks(p: int):
    """(canonical index, (b_ij, b_ik, b_jk)) of every task, Alg. 4 order."""
    bid = lambda i, j: j * (j + 1) // 2 + i  # noqa: E731
    out = []
    for i in range(p):
        for j in range(i, p):
            for k in range(j, p):
                out.append((bid(i, j), bid(i, k), bid(j, k)))
    return out


def block_readers(p: int, task_rank):
    """{block: set of ranks whose tasks read it}."""
    need = {}
    for t, bl in enumerate(task_blocks(p)):
        for b in bl:
            need.setdefault(b, set()).add(int(task_rank[t]))
    return need


def block_routes(p: int, task_rank, block_rank, block_nnz):
    """[(block, owner, [receiving ranks])] for every non-empty block some other rank needs."""
    need = block_readers(p, task_rank)
    routes = []
    for b in sorted(need):
        if int(block_nnz[b]) == 0:
            continue
        o = int(block_rank[b])
        dst = sorted(r for r in need[b] if r != o)
        if dst:
            routes.append((b, o, dst))
    return routes


def forward_blocks(plan, routes, device, group=None):
    """Point-to-point delivery of blocks from their owners (NCCL send/recv over NVLink,
    one batched group; gloo through host memory).  Returns (bytes sent, bytes received)."""
    import torch
    from . import _lib as L
    dist = _dist()
    _, rank = _world_rank(group)
    nccl = _nccl(group)
    ops, post, sent, recvd = [], [], 0, 0
    for b, owner, dsts in routes:
        if rank != owner and rank not in dsts:
            continue
        bp = L.bbtc_block_ptrs()
        L.check(L.bbtc_plan_block_ptrs(plan._h, b, ctypes.byref(bp)))
        spans = [(bp.edge[x], bp.nnz) for x in range(bp.n_edge_arrays)] + [(bp.rowptr, bp.rowptr_len)]
        for ptr, cnt in spans:
            if cnt == 0:
                continue
            view = _view_u32(int(ptr), int(cnt), device)
            if rank == owner:
                for q in dsts:
                    src = view if nccl else view.cpu()
                    ops.append(dist.P2POp(dist.isend, src, q, group=group))
                    sent += 4 * int(cnt)
            else:
                buf = view if nccl else torch.empty(int(cnt), dtype=torch.int32)
                ops.append(dist.P2POp(dist.irecv, buf, owner, group=group))
                if not nccl:
                    post.append((view, buf))
                recvd += 4 * int(cnt)
    if ops and nccl:
        for w in dist.batch_isend_irecv(ops):   # one NCCL group: every transfer in flight at once
            w.wait()
    else:
        for w in [op.op(op.tensor, op.peer, group=group) for op in ops]:
            w.wait()
    for view, buf in post:
        view.copy_(buf)
    torch.cuda.synchronize(device)
    return sent, recvd


def shard_assign(p: int, cuts, block_nnz, world: int):
    """bbtc_shard_assign: (task_rank uint32[n_tasks], block_rank uint32[p(p+1)/2])."""
    from . import _lib as L
    nt = p * (p + 1) * (p + 2) // 6
    nb = p * (p + 1) // 2
    c = np.ascontiguousarray(cuts, dtype=np.uint32)
    bn = np.ascontiguousarray(block_nnz, dtype=np.uint64)
    tr = np.empty(nt, np.uint32)
    br = np.empty(nb, np.uint32)
    L.check(L.bbtc_shard_assign(p, c.ctypes.data_as(L._u32p), bn.ctypes.data_as(L._u64p), world,
                                tr.ctypes.data_as(L._u32p), br.ctypes.data_as(L._u32p)))
    return tr, br


def build_sharded(ctx, src, dst, n_hint: int, p: int, cuts=None, group=None, flags: int = 0):
    """The §8(e) sharded a1-a5 (module docstring).  src/dst: this rank's share of the raw
    edges (CUDA int32 tensors, or host arrays: then the share is copied H2D here).
    Returns (graph shard, shard plan, info dict)."""
    import torch
    from . import Graph, Plan, _ptr
    from . import _lib as L
    dist = _dist()
    world, rank = _world_rank(group)
    device = torch.device("cuda", ctx.device)
    times = {}
    t0 = time.perf_counter()

    def mark(name):
        torch.cuda.synchronize(device)
        times[name] = (time.perf_counter() - t0) * 1e3

    ps, pd = _ptr(src, np.uint32), _ptr(dst, np.uint32)
    E = ps[1]
    host_in = ps[2] == L.MEM_HOST
    keys = torch.empty(max(E, 1), dtype=torch.int64, device=device)
    sc = np.zeros(world, np.uint64)
    mx = ctypes.c_uint32()
    L.check(L.bbtc_shard_canon(ctx.handle, ps[0], pd[0], E, ps[2], n_hint, world, ctypes.c_void_p(keys.data_ptr()),
                               sc.ctypes.data_as(L._u64p), ctypes.byref(mx)))
    nv = torch.tensor([max(n_hint, mx.value)], dtype=torch.int64, device=device)
    _all_reduce(nv, dist.ReduceOp.MAX, group)
    n = int(nv.item())
    mark("canon")
    recv, _ = exchange(keys, sc, group)
    del keys
    mark("exchange_keys")
    deg = torch.empty(max(n, 1), dtype=torch.int32, device=device)
    h = ctypes.c_void_p()
    L.check(L.bbtc_shard_graph(ctx.handle, ctypes.c_void_p(recv.data_ptr()), recv.numel(), n,
                               ctypes.c_void_p(deg.data_ptr()), ctypes.byref(h)))
    g = Graph(ctx, h)
    del recv
    m_local = g.m
    mt = torch.tensor([m_local], dtype=torch.int64, device=device)
    _all_reduce(mt, dist.ReduceOp.SUM, group)
    _all_reduce(deg, dist.ReduceOp.SUM, group)
    m_total = int(mt.item())
    mark("dedup_degrees")
    L.check(L.bbtc_shard_rank(ctx.handle, g._h, ctypes.c_void_p(deg.data_ptr()), m_total))
    del deg
    mark("rank_orient")
    cut_arr = None if cuts is None else np.ascontiguousarray(cuts, dtype=np.uint32)
    preq = p if cut_arr is None else len(cut_arr) - 1
    cuts_h = np.empty(preq + 1, np.uint32)
    pe = ctypes.c_uint32()
    nb_max = preq * (preq + 1) // 2
    bnnz = torch.empty(max(nb_max, 1), dtype=torch.int64, device=device)
    L.check(L.bbtc_shard_block_sizes(ctx.handle, g._h, preq, None if cut_arr is None else cut_arr.ctypes.data_as(L._u32p),
                                     ctypes.c_void_p(bnnz.data_ptr()), cuts_h.ctypes.data_as(L._u32p), ctypes.byref(pe)))
    pe = pe.value
    nb = pe * (pe + 1) // 2
    cuts_h = cuts_h[:pe + 1].copy()
    bn = bnnz[:nb].contiguous()
    _all_reduce(bn, dist.ReduceOp.SUM, group)
    bnnz_h = bn.cpu().numpy().view(np.uint64).copy()
    task_rank, block_rank = shard_assign(pe, cuts_h, bnnz_h, world)
    mark("cuts_assign")
    out = torch.empty(max(m_local, 1), dtype=torch.int64, device=device)
    sc2 = np.zeros(world, np.uint64)
    L.check(L.bbtc_shard_by_block(ctx.handle, g._h, pe, cuts_h.ctypes.data_as(L._u32p),
                                  block_rank.ctypes.data_as(L._u32p), world, ctypes.c_void_p(out.data_ptr()),
                                  sc2.ctypes.data_as(L._u64p)))
    recv2, _ = exchange(out, sc2, group)
    del out
    mark("exchange_blocks")
    hp = ctypes.c_void_p()
    L.check(L.bbtc_plan_create_shard(ctx.handle, g._h, ctypes.c_void_p(recv2.data_ptr()), recv2.numel(), pe,
                                     cuts_h.ctypes.data_as(L._u32p), bnnz_h.ctypes.data_as(L._u64p),
                                     task_rank.ctypes.data_as(L._u32p), rank, world, flags, ctypes.byref(hp)))
    del recv2
    plan = Plan.__new__(Plan)
    plan.ctx = ctx
    plan._h = hp
    ctx._children.add(plan)
    mark("build_blocks")
    routes = block_routes(pe, task_rank, block_rank, bnnz_h)
    sent, got = forward_blocks(plan, routes, device, group)
    mark("forward_blocks")
    info = {"n": n, "m": m_total, "m_local": m_local, "p": pe, "cuts": cuts_h, "task_rank": task_rank,
            "block_rank": block_rank, "block_nnz": bnnz_h, "h2d_bytes": 8 * E if host_in else 0,
            "nvlink_bytes_sent": sent, "nvlink_bytes_recv": got, "times_ms": times,
            "tasks_here": int((task_rank == rank).sum())}
    return g, plan, info



def count_owner_h2d(ctx, plan, info, counts, group=None):
    """§8(e) "copy each block H2D once, by its owner, and forward it over NVLink", for a
    shard plan whose blocks are in pinned host memory (plan.to_host()): this rank copies
    the blocks it owns that some task reads (bbtc_stage_blocks), receives the others it
    needs from their owners (NCCL P2P), counts its tasks and joins the all-reduce.
    Returns (h2d bytes of this rank, NVLink bytes received)."""
    import torch
    world, rank = _world_rank(group)
    p = info["p"]
    need = block_readers(p, info["task_rank"])
    owned = [b for b, rs in sorted(need.items()) if int(info["block_rank"][b]) == rank and int(info["block_nnz"][b])]
    cuts = info["cuts"]
    h2d = 0
    for b in owned:
        j = int((np.sqrt(8 * b + 1) - 1) // 2)
        while (j + 1) * (j + 2) // 2 <= b:
            j += 1
        i = b - j * (j + 1) // 2
        h2d += 12 * int(info["block_nnz"][b]) + 4 * (int(cuts[i + 1] - cuts[i]) + 1)
    plan.unstage()
    plan.stage_blocks(owned)
    routes = block_routes(p, info["task_rank"], info["block_rank"], info["block_nnz"])
    _, got = forward_blocks(plan, routes, torch.device("cuda", ctx.device), group)
    plan.stage_blocks([], resident=True)
    plan.count_async(counts, rank, world)
    _after_ctx_stream(ctx, counts)
    reduce_counts(counts, group)
    return h2d, got
