"""N > 1 path on CPU: world-size-2 gloo ranks combine partial per-task counters with
the same reduce_counts the GPU bench uses (NCCL there).  Partial counters come from
the oracle split by rank (task t -> rank t % world), standing in for the device
count's rank split; the reduction must reproduce the full counters bit-exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs
import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2009_12457_b200.dist import max_over_ranks, reduce_counts
    s, d = inputs.rmat(11, 16, 5)
    g = oracle.OracleGraph(s, d, 1 << 11)
    tot, pt, _, cuts = g.count(6)
    mine = np.zeros(len(pt) + 1, np.uint64)
    for t in range(len(pt)):
        if t % world == rank:
            mine[t] = pt[t]
    mine[-1] = mine[:-1].sum()
    buf = torch.from_numpy(mine.view(np.int64).copy())
    reduce_counts(buf)
    out = buf.numpy().view(np.uint64)
    ok = bool(np.array_equal(out[:-1], pt)) and int(out[-1]) == tot
    mx = max_over_ranks(float(rank + 1))
    q.put((rank, ok, mx))
    dist.destroy_process_group()


def test_gloo_world2_reduce_counts():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res)
    assert all(mx == 2.0 for _, _, mx in res)


def test_count_rows_strides_sum_to_total():
    s, d = inputs.rmat(12, 16, 2)
    g = oracle.OracleGraph(s, d, 1 << 12)
    T = g.count(1)[0]
    assert sum(g.count_rows(r, g.n, 5)[0] for r in range(5)) == T
