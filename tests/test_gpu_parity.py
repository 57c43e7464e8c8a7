"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, bit-exact.

Every count is an integer, so totals and per-task counts must match exactly
(SURVEY.md §8(c) A18).  Inputs are seeded and synthetic (inputs/).
"""
import json
import os

import numpy as np
import pytest

import inputs
import oracle

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def ctx(gpu):
    import paper_2009_12457_b200 as bb
    return bb.Context(0)


def run(ctx, s, d, n_hint, p=1, cuts=None, stats=False, row_major=False):
    import paper_2009_12457_b200 as bb
    g = bb.Graph.from_edges(ctx, s, d, n_hint)
    plan = bb.Plan(ctx, g, p, cuts, stats=stats, row_major=row_major)
    tot, pt = plan.count()
    return g, plan, tot, pt


def check(ctx, s, d, n_hint, p=1, cuts=None, og=None, row_major=False):
    og = og or oracle.OracleGraph(s, d, n_hint)
    g, plan, tot, pt = run(ctx, s, d, n_hint, p, cuts, row_major=row_major)
    ocuts = og.default_cuts(p) if cuts is None else np.asarray(cuts, np.uint32)
    assert np.array_equal(plan.cuts(), ocuts)
    otot, opt, _, _ = og.count(cuts=ocuts)
    assert tot == otot
    assert np.array_equal(pt, opt)
    return g, plan


def test_karate_golden(ctx):
    G = json.load(open(os.path.join(GOLD, "karate.json")))
    s, d = inputs.karate()
    g, plan, tot, pt = run(ctx, s, d, 34, 2)
    assert tot == G["total"] == 45
    assert list(plan.cuts()) == G["default_cuts"]["2"]
    rank = g.rank()
    order = np.empty(34, np.int64)
    order[rank] = np.arange(34)
    assert list(order) == G["order_new_to_old"]
    for case in G["per_task"]:
        _, _, tot, pt = run(ctx, s, d, 34, cuts=case["cuts"])
        assert list(pt) == case["counts"] and tot == 45


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("row_major", [False, True])
def test_rmat16_p_grid(ctx, seed, row_major):
    s, d = inputs.rmat(16, 16, seed)
    og = oracle.OracleGraph(s, d, 1 << 16)
    for p in (1, 2, 3, 4, 5, 8, 16):
        check(ctx, s, d, 1 << 16, p, og=og, row_major=row_major)


def test_rmat16_preprocessing_matches_oracle(ctx):
    s, d = inputs.rmat(16, 16, 1)
    og = oracle.OracleGraph(s, d, 1 << 16)
    import paper_2009_12457_b200 as bb
    g = bb.Graph.from_edges(ctx, s, d, 1 << 16)
    st = g.stats()
    assert (st["n"], st["m"]) == (og.n, og.m)
    assert st["d_max"] == int(og.degrees().max())
    assert st["n_nonisolated"] == int((og.degrees() > 0).sum())
    assert np.array_equal(g.rank(), og.rank())
    row, col = g.csr()
    orow, ocol = og.csr()
    assert np.array_equal(row, orow) and np.array_equal(col, ocol)
    assert st["dplus_max"] == int(np.diff(orow.astype(np.int64)).max())   # d+_max
    assert g.size() == (og.n, og.m)


def test_blocks_round_trip(ctx):
    """Every block G_ij holds exactly the oriented edges with u in V_i, v in V_j."""
    s, d = inputs.rmat(12, 16, 4)
    og = oracle.OracleGraph(s, d, 1 << 12)
    g, plan, _, _ = run(ctx, s, d, 1 << 12, 5)
    cuts = plan.cuts()
    orow, ocol = og.csr()
    src = np.repeat(np.arange(og.n), np.diff(orow).astype(np.int64))
    seen = 0
    for j in range(5):
        for i in range(j + 1):
            rp, col, row = plan.block(i, j)
            assert rp[0] == 0 and rp[-1] == len(col) and np.all(np.diff(rp.astype(np.int64)) >= 0)
            assert np.array_equal(np.repeat(np.arange(len(rp) - 1), np.diff(rp).astype(np.int64)), row)
            sel = (src >= cuts[i]) & (src < cuts[i + 1]) & (ocol >= cuts[j]) & (ocol < cuts[j + 1])
            assert np.array_equal(row.astype(np.int64) + cuts[i], src[sel])
            # rows ascending; the columns inside a row are a set (no order promised)
            got = np.lexsort((col, row))
            assert np.array_equal(col[got].astype(np.int64) + cuts[j], ocol[sel].astype(np.int64))
            seen += len(col)
    assert seen == og.m


@pytest.mark.parametrize("seed", range(8))
def test_random_graphs_random_cuts(ctx, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(20, 400))
    s, d = inputs.gnp(n, float(rng.uniform(0.02, 0.4)), seed=seed)
    og = oracle.OracleGraph(s, d, n)
    for p in (1, 2, 3, 6):
        inner = np.sort(rng.integers(0, og.n + 1, size=p - 1))
        cuts = np.concatenate([[0], inner, [og.n]]).astype(np.uint32)
        check(ctx, s, d, n, cuts=cuts, og=og)
        check(ctx, s, d, n, p=p, og=og)


@pytest.mark.parametrize("row_major", [False, True])
def test_dense_rows_exceed_slab(ctx, row_major):
    """K_n with long rows forces the global-memory search path (|list| > 1024 words)."""
    n = 1400
    iu = np.triu_indices(n, 1)
    s, d = iu[0].astype(np.uint32), iu[1].astype(np.uint32)
    g, plan, tot, pt = run(ctx, s, d, n, 1, row_major=row_major)
    assert tot == n * (n - 1) * (n - 2) // 6
    _, _, tot3, pt3 = run(ctx, s, d, n, cuts=[0, 300, 1400], row_major=row_major)
    sz = [300, 1100]
    want = [300 * 299 * 298 // 6, 300 * 299 // 2 * 1100, 300 * 1100 * 1099 // 2, 1100 * 1099 * 1098 // 6]
    assert list(pt3) == want and tot3 == tot


def test_degenerate_inputs(ctx):
    import paper_2009_12457_b200 as bb
    e = np.zeros(0, np.uint32)
    _, plan, tot, pt = run(ctx, e, e, 0, 3)
    assert tot == 0 and plan.p == 1
    _, plan, tot, pt = run(ctx, e, e, 9, 4)
    assert tot == 0 and plan.p == 4 and len(pt) == 20
    loops = np.array([1, 5, 5, 7], np.uint32)
    g, plan, tot, _ = run(ctx, loops, loops, 0, 2)
    assert tot == 0 and g.stats()["m"] == 0 and g.stats()["n"] == 8
    tri = np.array([0, 1, 2, 1, 0], np.uint32), np.array([1, 2, 0, 0, 0], np.uint32)
    g, plan, tot, pt = run(ctx, tri[0], tri[1], 0, 7)          # p > n clamps to n = 3
    assert tot == 1 and plan.p == 3 and plan.info()["clamped"] == 1 and int(pt.sum()) == 1
    with pytest.raises(bb.BBTCError):
        run(ctx, tri[0], tri[1], 0, cuts=[0, 2, 1, 3])           # non-monotone cuts
    with pytest.raises(bb.BBTCError):
        run(ctx, tri[0], tri[1], 0, cuts=[0, 2])                 # cuts[p] != n
    with pytest.raises(bb.BBTCError):
        run(ctx, tri[0], tri[1], 0, 0)                           # p == 0
    bad = np.array([0xFFFFFFFF], np.uint32)
    with pytest.raises(bb.BBTCError):
        run(ctx, bad, np.array([1], np.uint32), 0, 1)


@pytest.mark.parametrize("row_major", [False, True])
def test_device_input_streaming_and_ranks(ctx, row_major):
    """Device-resident input, host-streamed blocks (a6) and a rank split all agree."""
    import torch
    import paper_2009_12457_b200 as bb
    s, d = inputs.rmat(15, 16, 9)
    og = oracle.OracleGraph(s, d, 1 << 15)
    otot, opt, _, _ = og.count(cuts=og.default_cuts(6))
    ts = torch.from_numpy(s.view(np.int32)).cuda()
    td = torch.from_numpy(d.view(np.int32)).cuda()
    g = bb.Graph.from_edges(ctx, ts, td, 1 << 15)
    plan = bb.Plan(ctx, g, 6, stats=True, row_major=row_major)
    tot, pt = plan.count()
    assert tot == otot and np.array_equal(pt, opt)
    info = plan.info()
    assert info["b_alg"] > 0 and info["visits"] >= info["m"]
    # rank split: partial counts sum to the full result
    acc = np.zeros_like(pt)
    for r in range(3):
        t_r, pt_r = plan.count(rank=r, world=3)
        acc += pt_r
    assert np.array_equal(acc, opt)
    # async into a device tensor
    dc = torch.zeros(plan.n_tasks + 1, dtype=torch.int64, device="cuda")
    plan.count_async(dc)
    torch.cuda.synchronize()
    h = dc.cpu().numpy().view(np.uint64)
    assert int(h[-1]) == otot and np.array_equal(h[:-1], opt)
    # out-of-core form: blocks in pinned host memory, streamed on count
    plan.to_host()
    assert plan.info()["host_blocks"] == 1
    tot2, pt2, tm = plan.count(timing=True)
    assert tot2 == otot and np.array_equal(pt2, opt) and tm["h2d_bytes"] > 0
    # streamed counts take the tasks in unlock order: a rank split still sums to the total
    acc = np.zeros_like(pt)
    for r in range(3):
        plan.unstage()
        acc += plan.count(rank=r, world=3)[1]
    assert np.array_equal(acc, opt)
    # column-major blocks ship their column ids as column offsets (fewer bytes than
    # the blocks' device form); row-major blocks travel as they are
    info = plan.info()
    assert tm["h2d_bytes"] == info["stream_bytes"]
    # (and the leading zero run of every block's row offsets is set on the device)
    if row_major:
        assert info["stream_bytes"] <= info["block_bytes"]
    else:
        assert info["stream_bytes"] < info["block_bytes"]
    tot3, pt3, tm3 = plan.count(timing=True)           # now resident: no copies
    assert tot3 == otot and tm3["h2d_bytes"] == 0
    plan.unstage()
    plan.stage()
    assert plan.count()[0] == otot


def child(spec, p, modes, env=None, row_major=False, timeout=1500):
    """Counts through tests/gpu_child.py in a fresh process (own environment)."""
    import subprocess
    import sys
    cmd = [sys.executable, os.path.join(os.path.dirname(__file__), "gpu_child.py"), spec, str(p), ",".join(modes)]
    if row_major:
        cmd.append("rowmajor")
    r = subprocess.run(cmd, env={**os.environ, **(env or {})}, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def assert_modes(res, modes, otot, opt):
    for mode in modes:
        tot, *pt = res[mode]
        assert tot == otot, (mode, tot, otot)
        assert pt == [int(x) for x in opt], mode


@pytest.mark.slow
@pytest.mark.parametrize("name", ["orkut", "rmat24", "friendster"])
def test_full_size_configs(ctx, name):
    """BASELINE.json configs 3-5 at full size, per-task parity with the oracle in every
    mode: blocks resident (the bench's launch), a 3-rank split, streamed from pinned host
    memory (a6), streamed by 3 ranks, and out of core at 1/4 of the plan's bytes (or
    just above the largest task where that is more)."""
    cfg = inputs.CONFIGS[name]
    s, d = cfg.generate(seed=1)
    og = oracle.OracleGraph(s, d, cfg.n_hint)
    modes = ["resident", "ranks3", "streamed", "sranks3", "ooc25"]
    res = child(name, cfg.p, modes)
    cuts = np.asarray(res["cuts"], np.uint32)
    assert np.array_equal(cuts, og.default_cuts(cfg.p))
    otot, opt, _, _ = og.count(cuts=cuts)
    assert_modes(res, modes, otot, opt)
    assert res["streamed_h2d"] == res["stream_bytes"] > 0


@pytest.mark.parametrize("row_major", [False, True])
def test_streamed_modes_under_serialised_launches(gpu, row_major):
    """The streamed and out-of-core counts may not depend on kernels running beside the
    persistent count kernel (only copy-engine work sits ahead of a ready flag): they must
    give the oracle's counts with every launch serialised (CUDA_LAUNCH_BLOCKING=1) and the
    count kernel at full occupancy (BBTC_CTAS_PER_SM=8 caps nothing)."""
    s, d = inputs.rmat(16, 16, 9)
    og = oracle.OracleGraph(s, d, 1 << 16)
    modes = ["streamed", "sranks3", "ooc25", "ooc50", "stage", "resident", "ranks3"]
    for env in ({"CUDA_LAUNCH_BLOCKING": "1", "BBTC_CTAS_PER_SM": "8"}, {"BBTC_CTAS_PER_SM": "8"}):
        res = child("rmat:16:16:9", 7, modes, env=env, row_major=row_major, timeout=600)
        otot, opt, _, _ = og.count(cuts=np.asarray(res["cuts"], np.uint32))
        assert_modes(res, modes, otot, opt)


def test_empty_graph_plan_info(ctx):
    """m = 0: lambda = 1 (>= 1 always), no tasks carry work."""
    import paper_2009_12457_b200 as bb
    e = np.zeros(0, np.uint32)
    g = bb.Graph.from_edges(ctx, e, e, 12)
    plan = bb.Plan(ctx, g, 3)
    info = plan.info()
    assert info["lambda"] == 1.0 and info["m"] == 0
    assert plan.count()[0] == 0


@pytest.mark.parametrize("row_major", [False, True])
def test_huge_part_uses_sorted_path(ctx, row_major):
    """A part with >= 2^27 vertices disables the hash keys: the sorted-slab kernel must agree."""
    s, d = inputs.rmat(14, 16, 3)
    spread = (s.astype(np.uint64) * 8209 % (1 << 27)).astype(np.uint32), \
             (d.astype(np.uint64) * 8209 % (1 << 27)).astype(np.uint32)
    n = (1 << 27) + 5
    og = oracle.OracleGraph(spread[0], spread[1], n)
    check(ctx, spread[0], spread[1], n, p=1, og=og, row_major=row_major)
    check(ctx, spread[0], spread[1], n, cuts=[0, (1 << 27) + 1, n], og=og, row_major=row_major)


@pytest.mark.parametrize("n_hint", [0, 1, 5, 1000, 1 << 20])
def test_n_hint_does_not_matter_except_isolated(ctx, n_hint):
    """Narrow sort keys are sized from n_hint; a wrong hint must not change results."""
    s, d = inputs.rmat(10, 16, 7)
    og = oracle.OracleGraph(s, d, n_hint)
    check(ctx, s, d, n_hint, p=3, og=og)


@pytest.mark.parametrize("frac", [0.25, 0.5, 0.9])
@pytest.mark.parametrize("row_major", [False, True])
def test_out_of_core_budget(ctx, frac, row_major):
    """Host-resident plan counted with a device budget below the plan size."""
    import paper_2009_12457_b200 as bb
    s, d = inputs.rmat(15, 16, 21)
    og = oracle.OracleGraph(s, d, 1 << 15)
    otot, opt, _, ocuts = og.count(8)
    g = bb.Graph.from_edges(ctx, s, d, 1 << 15)
    plan = bb.Plan(ctx, g, 8, row_major=row_major)
    total_bytes = plan.info()["block_bytes"]
    plan.to_host()
    plan.set_budget(int(total_bytes * frac))
    for _ in range(2):   # twice: the second count reuses nothing (cache dies with the call)
        tot, pt, tm = plan.count(timing=True)
        assert tot == otot and np.array_equal(pt, opt)
        assert tm["h2d_bytes"] >= plan.info()["stream_bytes"] > 0   # every block at least once
    plan.set_budget(1024)   # smaller than any task's blocks
    with pytest.raises(bb.BBTCError):
        plan.count()


def test_hash_canonicalisation_option(gpu):
    """BBTC_DEDUP=hash (hash-set canonicalisation) yields the same graph and counts."""
    import subprocess
    import sys
    code = ("import sys, numpy as np; sys.path.insert(0, %r); import inputs, paper_2009_12457_b200 as bb; "
            "s, d = inputs.rmat(14, 16, 3); s = np.concatenate([s, d[:999], s[:5]]); d = np.concatenate([d, s[:999], s[:5]]); "
            "ctx = bb.Context(0); g = bb.Graph.from_edges(ctx, s, d, 1 << 14); p = bb.Plan(ctx, g, 5); "
            "t, pt = p.count(); print(t, ','.join(map(str, pt)), g.stats()['m'])") % os.path.dirname(GOLD.rstrip('/golden'))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = code.replace(repr(os.path.dirname(GOLD.rstrip('/golden'))), repr(root))
    out = subprocess.run([sys.executable, "-c", code], env={**os.environ, "BBTC_DEDUP": "hash"},
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    tot, pts, m = out.stdout.split()
    s, d = inputs.rmat(14, 16, 3)
    s2 = np.concatenate([s, d[:999], s[:5]])
    d2 = np.concatenate([d, s[:999], s[:5]])
    og = oracle.OracleGraph(s2, d2, 1 << 14)
    otot, opt, _, _ = og.count(5)
    assert int(tot) == otot and int(m) == og.m
    assert [int(x) for x in pts.split(",")] == [int(x) for x in opt]


def test_many_parts(ctx):
    """p = 100 (171,700 tasks, 5,050 blocks) and a user cut vector with many empty parts."""
    s, d = inputs.rmat(13, 16, 12)
    og = oracle.OracleGraph(s, d, 1 << 13)
    check(ctx, s, d, 1 << 13, p=100, og=og)
    rng = np.random.default_rng(3)
    cuts = np.concatenate([[0], np.sort(rng.integers(0, og.n + 1, size=119)), [og.n]]).astype(np.uint32)
    check(ctx, s, d, 1 << 13, cuts=cuts, og=og)


def test_host_input_stream_sort(ctx):
    """Host input large enough for the piecewise sort + merge path (> 2^26 raw pairs)."""
    import paper_2009_12457_b200 as bb
    s, d = inputs.rmat(22, 20, 5)          # 83.9 M raw pairs -> 2 pieces
    og = oracle.OracleGraph(s, d, 1 << 22)
    g = bb.Graph.from_edges(ctx, s, d, 1 << 22)
    st = g.stats()
    assert (st["n"], st["m"]) == (og.n, og.m)
    assert np.array_equal(g.rank(), og.rank())
    plan = bb.Plan(ctx, g, 6)
    tot, pt = plan.count()
    otot, opt, _, _ = og.count(cuts=plan.cuts())
    assert tot == otot and np.array_equal(pt, opt)


@pytest.mark.parametrize("seed", [1, 2])
def test_dense_and_sparse_tasks_agree(ctx, seed):
    """isDense: bit-row tasks and list tasks give the oracle's counts."""
    import paper_2009_12457_b200 as bb
    s, d = inputs.rmat(16, 16, seed)
    og = oracle.OracleGraph(s, d, 1 << 16)
    g = bb.Graph.from_edges(ctx, s, d, 1 << 16)
    for p in (2, 4, 8, 16):
        otot, opt, _, _ = og.count(cuts=og.default_cuts(p))
        dense = bb.Plan(ctx, g, p)
        sparse = bb.Plan(ctx, g, p, sparse=True)
        assert sparse.info()["dense_tasks"] == 0
        assert dense.info()["dense_tasks"] > 0     # the top parts of R-MAT are small
        for plan in (dense, sparse):
            tot, pt = plan.count()
            assert tot == otot and np.array_equal(pt, opt)
        assert dense.info()["dense_bytes"] > 0
        # streamed (a6): list kernel on the sparse tasks while blocks arrive, then the
        # bit rows are built from the landed blocks and the dense tasks counted
        dense.to_host()
        tot, pt, tm = dense.count(timing=True)
        assert tot == otot and np.array_equal(pt, opt)
        assert tm["h2d_bytes"] > 0 and tm["t_dense_ms"] > 0 and dense.info()["dense_bytes"] > 0
        dense.unstage()
        tot, pt = dense.count()                     # streamed again after dropping the bit rows
        assert tot == otot and np.array_equal(pt, opt)


def test_dense_strides(gpu):
    """Bit rows of every stride (8..256 words): parts of 100..6000 vertices, dense up to 8192."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sizes = [6000, 3000, 1500, 700, 300, 100, 31, 1]
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r); import inputs, paper_2009_12457_b200 as bb\n"
        "s, d = inputs.rmat(15, 16, 4); ctx = bb.Context(0); g = bb.Graph.from_edges(ctx, s, d, 1 << 15)\n"
        "n = g.stats()['n']; sizes = %r; cuts = [0, n - sum(sizes)]\n"
        "for z in sizes: cuts.append(cuts[-1] + z)\n"
        "p = bb.Plan(ctx, g, cuts=np.array(cuts, np.uint32)); t, pt = p.count()\n"
        "t0, _ = p.count(0, 2); t1, _ = p.count(1, 2); assert t0 + t1 == t\n"
        "print(t, ','.join(map(str, pt)), p.info()['dense_tasks'], ','.join(map(str, cuts)))\n") % (root, sizes)
    out = subprocess.run([sys.executable, "-c", code], env={**os.environ, "BBTC_DENSE_BITS": "8192"},
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    tot, pts, nd, cuts = out.stdout.split()
    s, d = inputs.rmat(15, 16, 4)
    og = oracle.OracleGraph(s, d, 1 << 15)
    otot, opt, _, _ = og.count(cuts=np.array([int(x) for x in cuts.split(",")], np.uint32))
    assert int(tot) == otot
    assert [int(x) for x in pts.split(",")] == [int(x) for x in opt]
    assert int(nd) > 60   # of 165 tasks: every one with k >= 1 and a non-empty G_ij


def test_auto_p_from_budget(ctx):
    """bbtc_plan_auto_p: the smallest p whose largest task fits the budget."""
    import paper_2009_12457_b200 as bb
    s, d = inputs.rmat(16, 16, 5)
    og = oracle.OracleGraph(s, d, 1 << 16)
    g = bb.Graph.from_edges(ctx, s, d, 1 << 16)
    whole = bb.Plan(ctx, g, 1).info()["max_task_bytes"]
    assert bb.auto_p(ctx, g, whole, depth=1) == 1
    for frac, depth in ((0.4, 1), (0.4, 2), (0.15, 1)):
        budget = int(whole * frac)
        p = bb.auto_p(ctx, g, budget, depth=depth)
        assert p > 1
        assert bb.Plan(ctx, g, p).info()["max_task_bytes"] * depth <= budget
        for q in range(1, p):   # smallest such p
            assert bb.Plan(ctx, g, q).info()["max_task_bytes"] * depth > budget
    p = bb.auto_p(ctx, g, int(whole * 0.4), depth=1)
    plan = bb.Plan(ctx, g, p)
    otot, opt, _, _ = og.count(p)
    plan.to_host()
    plan.set_budget(int(whole * 0.4) * 3)   # a few tasks' blocks at a time
    tot, pt = plan.count()
    assert tot == otot and np.array_equal(pt, opt)
    with pytest.raises(bb.BBTCError) as ei:
        bb.auto_p(ctx, g, 1000)
    assert ei.value.code == -5


def test_packed_transpose_keys(gpu):
    """Packed transpose keys (per-block column ranges minus the isolated prefix of each
    part): forced on, with isolated vertices spanning several parts of user cuts."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s, d = inputs.rmat(14, 16, 6)
    n = 1 << 16                                   # 3/4 of the ids isolated (lowest ranks)
    og = oracle.OracleGraph(s, d, n)
    n_iso = int((og.degrees() == 0).sum())
    cuts_user = np.unique(np.concatenate([[0], np.linspace(0, n_iso + 2000, 9).astype(np.int64),
                                          np.linspace(n_iso + 2000, og.n, 8).astype(np.int64), [og.n]]))
    code = ("import sys, json, numpy as np; sys.path.insert(0, %r); import inputs, paper_2009_12457_b200 as bb\n"
            "s, d = inputs.rmat(14, 16, 6); ctx = bb.Context(0); g = bb.Graph.from_edges(ctx, s, d, %d)\n"
            "out = []\n"
            "for p, cuts in ((16, None), (12, None), (None, %s)):\n"
            "    plan = bb.Plan(ctx, g, p or 1, None if cuts is None else np.array(cuts, np.uint32))\n"
            "    t, pt = plan.count(); out.append([t, pt.tolist(), plan.cuts().tolist()])\n"
            "print(json.dumps(out))\n") % (root, n, cuts_user.tolist())
    res = subprocess.run([sys.executable, "-c", code], env={**os.environ, "BBTC_PACKED_TRANSPOSE": "1"},
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    for tot, pt, cuts in json.loads(res.stdout.strip().splitlines()[-1]):
        otot, opt, _, _ = og.count(cuts=np.asarray(cuts, np.uint32))
        assert tot == otot and pt == [int(x) for x in opt]


@pytest.mark.parametrize("cutoff,threads", [(0.0, 4), (0.5, 0), (1.0, 2), (0.25, 1), (0.0, 16)])
def test_hybrid_cpu_gpu(ctx, cutoff, threads):
    """§8(f)#3 (Alg. 8): GPU from the heavy end of the ExecTime queue, host
    threads from the light end up to the cut-off — every task exactly once."""
    import paper_2009_12457_b200 as bb
    for spec, p in ((("karate", None), 2), (("rmat", 16), 8), (("rmat", 14), 12)):
        if spec[0] == "karate":
            s, d = inputs.karate()
            n = 34
        else:
            s, d = inputs.rmat(spec[1], 16, 5)
            n = 1 << spec[1]
        og = oracle.OracleGraph(s, d, n)
        g = bb.Graph.from_edges(ctx, s, d, n)
        plan = bb.Plan(ctx, g, p)
        otot, opt, _, _ = og.count(cuts=plan.cuts())
        with pytest.raises(bb.BBTCError):
            plan.count_hybrid(threads, cutoff)                      # needs host arenas
        plan.to_host()
        plan.stage()
        tot, pt, st = plan.count_hybrid(threads, cutoff)
        assert tot == otot and np.array_equal(pt, opt)
        sparse = plan.n_tasks - plan.info()["dense_tasks"]
        assert st["cpu_tasks"] + st["gpu_tasks"] == sparse
        if cutoff == 1.0:
            assert st["cpu_tasks"] == 0
        assert st["gpu_tasks"] >= int(np.ceil(cutoff * sparse)) or sparse == 0


def test_cut_refinement_and_study_tools(ctx):
    """§8(f)#4: PBD-like refinement returns valid cuts whose largest block is no larger
    than the default rule's (and the count is the oracle's); block sizes and per-task
    times are reported for every task."""
    import paper_2009_12457_b200 as bb
    s, d = inputs.rmat(16, 16, 2)
    og = oracle.OracleGraph(s, d, 1 << 16)
    g = bb.Graph.from_edges(ctx, s, d, 1 << 16)
    for p in (2, 5, 8):
        base = bb.Plan(ctx, g, p)
        mm0 = int(base.block_nnz().max())
        cuts, mm = bb.refine_cuts(ctx, g, p, max_evals=120)
        assert cuts[0] == 0 and cuts[-1] == og.n and np.all(np.diff(cuts.astype(np.int64)) >= 0)
        plan = bb.Plan(ctx, g, cuts=cuts)
        bn = plan.block_nnz()
        assert int(bn.max()) == mm <= mm0 and int(bn.sum()) == og.m
        otot, opt, _, _ = og.count(cuts=cuts)
        tot, pt = plan.count()
        assert tot == otot and np.array_equal(pt, opt)
        tt = plan.task_times()
        assert len(tt) == plan.n_tasks and np.all(tt >= 0) and tt.max() > 0
    cuts, mm = bb.refine_cuts(ctx, g, 3, cuts=[0, 10, 20, og.n], max_evals=60)
    assert mm <= int(bb.Plan(ctx, g, cuts=[0, 10, 20, og.n]).block_nnz().max())


@pytest.mark.parametrize("heavy_dup", [False, True])
def test_bucket_dedup(ctx, heavy_dup):
    """a1 de-duplication in hashed buckets (device input, >= 2^22 raw pairs): the same
    graph as the oracle's; one edge repeated 20,000 times overflows its bucket and the
    sort path takes over — same result."""
    import torch
    import paper_2009_12457_b200 as bb
    s, d = inputs.rmat(18, 20, 7)                       # 5.2 M raw pairs, K = 36 bits
    if heavy_dup:
        s = np.concatenate([s, np.full(20000, 5, np.uint32)])
        d = np.concatenate([d, np.full(20000, 77, np.uint32)])
    og = oracle.OracleGraph(s, d, 1 << 18)
    ts = torch.from_numpy(s.view(np.int32)).cuda()
    td = torch.from_numpy(d.view(np.int32)).cuda()
    os.environ["BBTC_BUCKET"] = "1"                   # (an option, off by default: DESIGN §7)
    try:
        g = bb.Graph.from_edges(ctx, ts, td, 1 << 18)
    finally:
        del os.environ["BBTC_BUCKET"]
    assert g.size() == (og.n, og.m)
    assert np.array_equal(g.rank(), og.rank())
    row, col = g.csr()
    orow, ocol = og.csr()
    assert np.array_equal(row, orow) and np.array_equal(col, ocol)
    plan = bb.Plan(ctx, g, 6)
    tot, pt = plan.count()
    otot, opt, _, _ = og.count(cuts=plan.cuts())
    assert tot == otot and np.array_equal(pt, opt)


def test_counting_sort_options(gpu):
    """The measured-and-dropped preprocessing options stay correct: bucket
    de-duplication, CSR and transpose by counting sort (BBTC_BUCKET / BBTC_CSR_COUNT /
    BBTC_TRANSPOSE_COUNT), on device input large enough for the buckets."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, json, numpy as np, torch; sys.path.insert(0, %r); import inputs, paper_2009_12457_b200 as bb\n"
            "s, d = inputs.rmat(18, 20, 7); ctx = bb.Context(0)\n"
            "g = bb.Graph.from_edges(ctx, torch.from_numpy(s.view(np.int32)).cuda(), torch.from_numpy(d.view(np.int32)).cuda(), 1 << 18)\n"
            "row, col = g.csr(); plan = bb.Plan(ctx, g, 6); t, pt = plan.count()\n"
            "print(json.dumps([t, pt.tolist(), plan.cuts().tolist(), g.rank().tolist()[:1000], int(row[-1])]))\n") % root
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                         env={**os.environ, "BBTC_BUCKET": "1", "BBTC_CSR_COUNT": "1", "BBTC_TRANSPOSE_COUNT": "1"})
    assert res.returncode == 0, res.stderr[-2000:]
    tot, pt, cuts, rank0, m = json.loads(res.stdout.strip().splitlines()[-1])
    s, d = inputs.rmat(18, 20, 7)
    og = oracle.OracleGraph(s, d, 1 << 18)
    otot, opt, _, _ = og.count(cuts=np.asarray(cuts, np.uint32))
    assert tot == otot and pt == [int(x) for x in opt] and m == og.m
    assert rank0 == og.rank().tolist()[:1000]



@pytest.mark.parametrize("spec,p", [("rmat:16:16:9", 4), ("rmat:15:16:3", 7), ("gnp:3000:0.004:5", 3)])
def test_probe_slots(gpu, spec, p):
    """Probe slots: forced onto every block with at least one edge per row on
    average, so rows of <= 6 entries are probed inline and longer ones through the CSR
    offset in their slot — the oracle's per-task counts in every mode (streamed and
    out-of-core counts run without slots, staged counts on rebuilt arenas)."""
    kind, *a = spec.split(":")
    if kind == "rmat":
        s, d = inputs.rmat(int(a[0]), int(a[1]), int(a[2]))
        n_hint = 1 << int(a[0])
    else:
        s, d = inputs.gnp(int(a[0]), float(a[1]), int(a[2]))
        n_hint = int(a[0])
    og = oracle.OracleGraph(s, d, n_hint)
    modes = ["resident", "ranks3", "streamed", "ooc50", "stage"]
    env = {"BBTC_SLOTS": "1", "BBTC_SLOT_MIN_ROWS": "1", "BBTC_SLOT_MIN_DEG": "0.5", "BBTC_SLOT_MAX_DEG": "1e9"}
    res = child(spec, p, modes, env=env)
    otot, opt, _, _ = og.count(cuts=np.asarray(res["cuts"], np.uint32))
    assert_modes(res, modes, otot, opt)
    assert res.get("slots", 1) > 0
