"""N > 1 on the GPU: world-2 ranks (both on cuda:0 — this box has one GPU — reducing
with gloo instead of NCCL) each count their share of the work items through the
C-ABI, and one all-reduce of the per-task counters gives the oracle's counts."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

import inputs
import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import paper_2009_12457_b200 as bb
    from paper_2009_12457_b200.dist import count_distributed
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    s, d = inputs.rmat(15, 16, 4)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = bb.Context(0, stream=stream.cuda_stream)
    g = bb.Graph.from_edges(ctx, s, d, 1 << 15)
    plan = bb.Plan(ctx, g, 7)
    counts = torch.zeros(plan.n_tasks + 1, dtype=torch.int64, device="cuda")
    plan.count_async(counts, rank, world)
    torch.cuda.synchronize()
    partial = int(counts[-1].item())
    count_distributed(plan, counts)   # recount + all-reduce through the bench's path
    torch.cuda.synchronize()
    q.put((rank, partial, counts.cpu().numpy().view(np.uint64).tolist(), plan.cuts().tolist()))
    dist.destroy_process_group()


def test_two_ranks_sum_to_oracle(gpu):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    s, d = inputs.rmat(15, 16, 4)
    og = oracle.OracleGraph(s, d, 1 << 15)
    otot, opt, _, _ = og.count(cuts=np.asarray(res[0][3], np.uint32))
    assert res[0][1] + res[1][1] == otot and 0 < res[0][1] < otot
    for _, _, full, _ in res:
        assert full[-1] == otot and full[:-1] == [int(x) for x in opt]


def test_bench_two_ranks_one_gpu(gpu):
    """The bench's N>1 path end to end (torchrun, 2 ranks sharing the GPU, gloo)."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--config", "rmat16", "--steps", "3", "--warmup", "3", "--e2e-steps", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    import json
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["value"] > 0
    s, d = inputs.rmat(16, 16, 1)
    og = oracle.OracleGraph(s, d, 1 << 16)
    assert rec["triangles"] == og.count(4)[0]
