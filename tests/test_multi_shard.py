"""§8(e) host logic on CPU (no GPU): the multi-GPU scheduler (bbtc_shard_assign, a
host-only C-ABI call) and the buffer movement of dist.py over world-size-2 gloo."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2009_12457_b200 import dist as bdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _random_blocks(rng, p, n=10000):
    cuts = np.concatenate([[0], np.sort(rng.integers(0, n + 1, size=p - 1)), [n]]).astype(np.uint32)
    nb = p * (p + 1) // 2
    bnnz = rng.integers(0, 5000, size=nb).astype(np.uint64)
    bnnz[rng.random(nb) < 0.2] = 0
    return cuts, bnnz


def _work(p, cuts, bnnz):
    """The scheduler's documented LPT weight (capi.cpp shard_assign): a
    task counted through bit rows (isDense with the default 8192 dense bits and ratio 4:
    bit-row stride S = the power of two >= |V_k| / 32 in [8, 512], δ(G_ik) >= 4·S/32)
    weighs 0.145·nnz(G_ij)·(S + 35); any other nnz(G_ij)·(16 + δ(G_ik)) +
    2·min(nnz(G_ij), |V_j|)·δ(G_jk)."""
    rows = np.diff(cuts.astype(np.float64))
    bid = lambda i, j: j * (j + 1) // 2 + i  # noqa: E731
    d = lambda i, j: bnnz[bid(i, j)] / rows[i] if rows[i] else 0.0  # noqa: E731

    def stride(k):
        if rows[k] == 0 or rows[k] > 8192:
            return 0
        s = 8
        while s * 32 < rows[k]:
            s *= 2
        return s if s <= 512 else 0

    def cost(i, j, k):
        nij = float(bnnz[bid(i, j)])
        S = stride(k)
        if S and nij > 0 and d(i, k) >= 4 * S / 32:
            return 0.145 * nij * (S + 35)
        return nij * (16 + d(i, k)) + 2 * min(nij, rows[j]) * d(j, k)
    return [cost(i, j, k) for i in range(p) for j in range(i, p) for k in range(j, p)]


@pytest.mark.parametrize("p,world,seed", [(1, 2, 0), (4, 2, 1), (8, 3, 2), (12, 8, 3), (16, 8, 4), (30, 5, 5)])
def test_shard_assign_valid_balanced_deterministic(p, world, seed):
    rng = np.random.default_rng(seed)
    cuts, bnnz = _random_blocks(rng, p)
    tr, br = bdist.shard_assign(p, cuts, bnnz, world)
    tr2, br2 = bdist.shard_assign(p, cuts, bnnz, world)
    assert np.array_equal(tr, tr2) and np.array_equal(br, br2)        # same on every rank
    nt = p * (p + 1) * (p + 2) // 6
    assert len(tr) == nt and tr.max() < world and br.max() < world
    w = np.array(_work(p, cuts, bnnz))
    load = np.bincount(tr, weights=w, minlength=world)
    # LPT bound: no rank above max(1.02 x ideal share, ideal + the largest task)
    assert load.max() <= max(1.02 * w.sum() / world, w.sum() / world + w.max()) + 1e-6
    # every non-empty block's owner is a rank that reads it (when some rank does)
    routes = bdist.block_routes(p, tr, br, bnnz)
    readers = {}
    for t, bl in enumerate(bdist.task_blocks(p)):
        for b in bl:
            readers.setdefault(b, set()).add(int(tr[t]))
    for b, rs in readers.items():
        assert int(br[b]) in rs
    for b, o, dsts in routes:
        assert bnnz[b] > 0 and o not in dsts and set(dsts) | {o} == readers[b]


def test_shard_assign_affinity_beats_round_robin():
    """Block affinity: fewer block copies cross NVLink than a plain round-robin split."""
    rng = np.random.default_rng(9)
    p, world = 16, 8
    cuts, bnnz = _random_blocks(rng, p, 100000)
    tr, br = bdist.shard_assign(p, cuts, bnnz, world)
    moved = sum(len(d) * int(bnnz[b]) for b, _, d in bdist.block_routes(p, tr, br, bnnz))
    rr = np.arange(len(tr), dtype=np.uint32) % world
    need = {}
    for t, bl in enumerate(bdist.task_blocks(p)):
        for b in bl:
            need.setdefault(b, set()).add(int(rr[t]))
    moved_rr = sum((len(s) - 1) * int(bnnz[b]) for b, s in need.items())
    assert moved < moved_rr


def test_shard_assign_rejects_bad_input():
    import paper_2009_12457_b200 as bb
    with pytest.raises(bb.BBTCError):
        bdist.shard_assign(3, [0, 5, 2, 9], np.zeros(6, np.uint64), 2)
    with pytest.raises(bb.BBTCError):
        bdist.shard_assign(2, [0, 1, 2], np.zeros(3, np.uint64), 0)


def _exchange_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(rank)
    counts = rng.integers(0, 50, size=world)
    counts[(rank + 1) % world] = 0                                   # an empty split
    send = torch.cat([torch.full((int(c),), rank * 1000 + d, dtype=torch.int64) for d, c in enumerate(counts)])
    recv, rc = bdist.exchange(send, counts)
    ok = recv.numel() == sum(rc)
    off = 0
    for src, c in enumerate(rc):
        ok = ok and bool((recv[off:off + c] == src * 1000 + rank).all())
        off += c
    t = torch.tensor([rank + 1], dtype=torch.int64)
    bdist.reduce_counts(t)
    q.put((rank, ok, int(t.item()), bdist.max_over_ranks(float(rank))))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_exchange_all_to_all(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _, _ in res)
    assert all(s == world * (world + 1) // 2 and mx == world - 1 for _, _, s, mx in res)


def test_generate_range_matches_full():
    import inputs
    for name in ("rmat16",):
        cfg = inputs.CONFIGS[name]
        s, d = cfg.generate(seed=3)
        for r in range(3):
            a, b = cfg.shard(r, 3)
            s2, d2 = cfg.generate_range(a, b - a, seed=3)
            assert np.array_equal(s[a:b], s2) and np.array_equal(d[a:b], d2)
    cfg = inputs.Config("cl", "chunglu", p=2, n=5000, m=40000, gamma=2.2, dmax=300)
    s, d = cfg.generate(seed=2)
    a, b = cfg.shard(1, 4)
    s2, d2 = cfg.generate_range(a, b - a, seed=2)
    assert np.array_equal(s[a:b], s2) and np.array_equal(d[a:b], d2)
    assert math.isclose(sum(cfg.shard(r, 4)[1] - cfg.shard(r, 4)[0] for r in range(4)), cfg.n_samples)
