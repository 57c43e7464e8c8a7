"""Multi-GPU glue (a8): one rank per GPU, one all-reduce of the per-task counters.

Each rank counts the work items r, r+N, ... of the same plan (bbtc_count_async
with rank/world) into an int64[n_tasks+1] device tensor (the uint64 bit pattern:
two's-complement addition is bit-identical), and `reduce_counts` sums the
tensors over the process group — NCCL over NVLink on GPUs, gloo on CPU tests.
"""
from __future__ import annotations


def reduce_counts(counts, group=None):
    """In-place sum of the per-task counter tensor over all ranks (one collective)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def count_distributed(plan, counts, group=None):
    """Enqueue this rank's share of the count and combine the ranks' counters.

    counts: CUDA int64 tensor of plan.n_tasks + 1 entries (last = total)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(group), dist.get_world_size(group)
    else:
        rank, world = 0, 1
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
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
