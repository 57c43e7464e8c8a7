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


def _shard_worker(rank, world, port, q, spec, p, host_input, backend):
    """One rank of the §8(e) sharded pipeline (dist.build_sharded) on cuda:0."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import paper_2009_12457_b200 as bb
    from paper_2009_12457_b200.dist import build_sharded, count_distributed
    torch.cuda.set_device(0)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, n_hint = spec
    a, b = cfg.shard(rank, world)
    s, d = cfg.generate_range(a, b - a, seed=3)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = bb.Context(0, stream=stream.cuda_stream)
    if not host_input:
        s = torch.from_numpy(s.view(np.int32)).cuda()
        d = torch.from_numpy(d.view(np.int32)).cuda()
    g, plan, info = build_sharded(ctx, s, d, n_hint, p)
    counts = torch.zeros(plan.n_tasks + 1, dtype=torch.int64, device="cuda")
    plan.count_async(counts, rank, world)
    torch.cuda.synchronize()
    mine = counts.cpu().numpy().view(np.uint64).copy()
    count_distributed(plan, counts)
    torch.cuda.synchronize()
    full = counts.cpu().numpy().view(np.uint64).tolist()
    # incl. H2D: blocks in pinned host memory, each copied once by its owner, forwarded
    from paper_2009_12457_b200.dist import count_owner_h2d
    plan.to_host()
    h2d_blocks, _ = count_owner_h2d(ctx, plan, info, counts)
    torch.cuda.synchronize()
    full_h = counts.cpu().numpy().view(np.uint64).tolist()
    q.put((rank, full, mine.tolist(), info["cuts"].tolist(),
           info["h2d_bytes"], b - a, info["tasks_here"], info["nvlink_bytes_recv"], info["m"], info["n"],
           full_h, h2d_blocks, plan.info()["block_bytes"]))
    dist.destroy_process_group()


def _run_shards(world, spec, p, host_input, backend="gloo"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q, spec, p, host_input, backend))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for pr in procs:
        pr.join(timeout=120)
    return res


@pytest.mark.parametrize("world,host_input", [(2, True), (3, False), (5, True)])
def test_sharded_build_matches_oracle(gpu, world, host_input):
    """§8(e): each rank holds 1/N of the raw edges (only that share crosses its PCIe link
    for host input), the sharded a1-a5 + block forwarding + a rank's own tasks, and one
    all-reduce: per-task counts equal the oracle's (several ranks share cuda:0, gloo)."""
    cfg = inputs.CONFIGS["rmat16"]
    res = _run_shards(world, (cfg, 1 << 16), 6, host_input)
    s, d = cfg.generate(seed=3)
    og = oracle.OracleGraph(s, d, 1 << 16)
    cuts = np.asarray(res[0][3], np.uint32)
    assert np.array_equal(cuts, og.default_cuts(6))                 # global default rule
    otot, opt, _, _ = og.count(cuts=cuts)
    partial = np.zeros(len(opt), np.uint64)
    h2d_total = 0
    for rank, full, mine, c, h2d, share, ntasks, got, m, n, full_h, h2d_blocks, block_bytes in res:
        assert full[-1] == otot and full[:-1] == [int(x) for x in opt]
        assert full_h == full                                          # owner-copy + NVLink path
        h2d_total += h2d_blocks
        assert h2d_blocks < block_bytes                                # no rank copies every block
        assert c == res[0][3] and (m, n) == (og.m, og.n)
        assert h2d == (8 * share if host_input else 0)               # per-rank H2D = its share
        partial += np.asarray(mine[:-1], np.uint64)
        assert 0 < ntasks < len(opt)
    assert np.array_equal(partial, opt)                                # ranks' tasks are disjoint
    assert sum(r[6] for r in res) == len(opt)
    assert h2d_total <= res[0][12]                                     # every block crosses PCIe at most once


def test_sharded_build_user_cuts_and_karate(gpu):
    """Karate over 2 ranks (each with half the raw pairs) gives the golden per-task counts."""
    import json
    cfg = inputs.CONFIGS["karate"]
    res = _run_shards(2, (cfg, 34), 2, True)
    G = json.load(open(os.path.join(ROOT, "tests", "golden", "karate.json")))
    assert res[0][3] == G["default_cuts"]["2"]
    assert res[0][1][:-1] == G["per_task"][0]["counts"] and res[0][1][-1] == 45
    assert res[0][10] == res[0][1]


def test_nccl_single_rank_path(gpu):
    """The NCCL branch (all-to-all, all-reduce, the batched P2P group) executes: world 1
    over NCCL on the one GPU of this box gives the oracle's counts."""
    cfg = inputs.CONFIGS["rmat16"]
    res = _run_shards(1, (cfg, 1 << 16), 4, False, backend="nccl")
    s, d = cfg.generate(seed=3)
    og = oracle.OracleGraph(s, d, 1 << 16)
    otot, opt, _, _ = og.count(cuts=np.asarray(res[0][3], np.uint32))
    assert res[0][1][-1] == otot and res[0][1][:-1] == [int(x) for x in opt]
