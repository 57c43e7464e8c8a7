"""Pins for the CPU oracle.  CPU only."""
import json
import math
import os

import numpy as np
import pytest

import inputs
import oracle
from brute import per_task_bruteforce, simple_graph, triangles_dense

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def rand_cuts(rng, n, p):
    inner = np.sort(rng.integers(0, n + 1, size=p - 1))
    return np.concatenate([[0], inner, [n]]).astype(np.uint32)


# ---- P3: karate -----------------------------------------------------------------
def test_karate_golden():
    G = load("karate.json")
    s, d = inputs.karate()
    g = oracle.OracleGraph(s, d, 34)
    assert (g.n, g.m) == (G["n"], G["m"])
    assert list(g.degrees()) == G["degrees_by_id"]
    rank = g.rank()
    order = np.empty(34, np.int64)
    order[rank] = np.arange(34)
    assert list(order) == G["order_new_to_old"]
    row, _ = g.csr()
    assert list(np.diff(row)) == G["outdeg_by_new_id"]
    for p, cuts in G["default_cuts"].items():
        assert list(g.default_cuts(int(p))) == cuts
    tot, pt, pv, _ = g.count(2, per_vertex=True)
    assert tot == G["total"] and int(pv.sum()) == G["sum_per_vertex"]
    for case in G["per_task"]:
        tot, pt, _, _ = g.count(cuts=case["cuts"])
        assert list(pt) == case["counts"], case
        assert tot == 45


def test_karate_prefix_golden_consistent():
    """The golden prefix sums are the App. A degrees in App. A rank order (guards the fixture)."""
    G = load("karate.json")
    w = [G["degrees_by_id"][o] for o in G["order_new_to_old"]]
    assert G["prefix_degrees_by_rank"] == [sum(w[:r]) for r in range(35)]


# ---- default cut rule: closed form on regular graphs --------------------------------
def _regular(kind, n):
    if kind == "cycle":
        return cycle(n)
    if kind == "complete":
        return [(a, b) for a in range(n) for b in range(a + 1, n)]
    if kind == "prism":                                          # C_{n/2} x K_2, 3-regular
        h = n // 2
        return cycle(h) + [(h + a, h + b) for a, b in cycle(h)] + [(a, a + h) for a in range(h)]
    raise ValueError(kind)


@pytest.mark.parametrize("kind,n", [("cycle", 6), ("cycle", 12), ("cycle", 35), ("complete", 9),
                                    ("complete", 13), ("prism", 10), ("prism", 22)])
def test_default_cuts_regular_closed_form(kind, n):
    """For a d-regular graph P[r] = r*d, so min{r : r*d >= ceil(i*n*d/p)} = ceil(ceil(i*n*d/p)/d)
    = ceil(i*n/p) (nested ceilings).  Exact targets (d | i*n*d/p) pin the '>=' side of the rule,
    ragged ones pin the ceiling (SURVEY §8(c) default cut rule)."""
    s, d = _edges(_regular(kind, n))
    g = oracle.OracleGraph(s, d)
    assert g.n == n
    for p in range(1, n + 1):
        want = [-(-i * n // p) for i in range(p + 1)]
        assert list(g.default_cuts(p)) == want, (kind, n, p)


# ---- P1: brute force ------------------------------------------------------------
@pytest.mark.parametrize("seed", range(12))
def test_bruteforce_random(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(5, 45))
    q = float(rng.uniform(0.05, 0.6))
    s, d = inputs.gnp(n, q, seed=seed + 100)
    # add raw noise: reversed pairs, duplicates, self-loops
    s2 = np.concatenate([s, d[: len(d) // 3], s[:5], np.arange(3, dtype=np.uint32)])
    d2 = np.concatenate([d, s[: len(s) // 3], d[:5], np.arange(3, dtype=np.uint32)])
    A = simple_graph(s2, d2, n)
    T, pv_ref = triangles_dense(A)
    g = oracle.OracleGraph(s2, d2, n)
    assert g.m == int(A.sum()) // 2
    for p in (1, 2, 3, 5):
        cuts = rand_cuts(rng, g.n, p)
        tot, pt, pv, _ = g.count(cuts=cuts, per_vertex=True)
        assert tot == T
        assert np.array_equal(pv, pv_ref)
        assert np.array_equal(pt.astype(np.int64), per_task_bruteforce(A, cuts))


# ---- P2: K_n closed forms ---------------------------------------------------------
@pytest.mark.parametrize("n,cuts", [(7, [0, 7]), (9, [0, 2, 5, 9]), (12, [0, 0, 4, 4, 12]), (20, [0, 3, 8, 14, 20])])
def test_complete_graph(n, cuts):
    iu = np.triu_indices(n, 1)
    s, d = iu[0].astype(np.uint32), iu[1].astype(np.uint32)
    g = oracle.OracleGraph(s, d)
    tot, pt, pv, _ = g.count(cuts=cuts, per_vertex=True)
    assert tot == math.comb(n, 3)
    assert all(int(x) == math.comb(n - 1, 2) for x in pv)
    sz = np.diff(cuts)
    p = len(cuts) - 1
    t = 0
    for i in range(p):
        for j in range(i, p):
            for k in range(j, p):
                if i < j < k:
                    want = sz[i] * sz[j] * sz[k]
                elif i == j < k:
                    want = math.comb(sz[i], 2) * sz[k]
                elif i < j == k:
                    want = sz[i] * math.comb(sz[j], 2)
                else:
                    want = math.comb(sz[i], 3)
                assert int(pt[t]) == want, (i, j, k)
                t += 1


# ---- P7: graph families ---------------------------------------------------------
def _edges(pairs):
    a = np.asarray(pairs, dtype=np.uint32).reshape(-1, 2)
    return a[:, 0].copy(), a[:, 1].copy()


def tripartite(a, b, c):
    A, B, C = range(a), range(a, a + b), range(a + b, a + b + c)
    return [(x, y) for X, Y in ((A, B), (B, C), (A, C)) for x in X for y in Y]


def wheel(k):
    return [(0, i) for i in range(1, k + 1)] + [(i, i % k + 1) for i in range(1, k + 1)]


def friendship(k):
    return [e for t in range(k) for e in ((0, 2 * t + 1), (0, 2 * t + 2), (2 * t + 1, 2 * t + 2))]


def cycle(k):
    return [(i, (i + 1) % k) for i in range(k)]


@pytest.mark.parametrize("pairs,want", [
    (tripartite(2, 3, 4), 24), (tripartite(5, 1, 7), 35), (wheel(4), 4), (wheel(9), 9),
    (friendship(1), 1), (friendship(6), 6), (cycle(3), 1), (cycle(4), 0), (cycle(11), 0),
    ([(0, i) for i in range(1, 30)], 0),                                # star
    ([(i, i + 1) for i in range(40)], 0),                               # path
    ([(i, (i - 1) // 2) for i in range(1, 63)], 0),                     # binary tree
    ([(x, y) for x in range(6) for y in range(6, 13)], 0),              # K_{6,7}
])
def test_families(pairs, want):
    s, d = _edges(pairs)
    g = oracle.OracleGraph(s, d)
    for p in (1, 2, 3):
        tot, pt, _, _ = g.count(p)
        assert tot == want and int(pt.sum()) == want


def test_empty_and_degenerate():
    e = np.zeros(0, np.uint32)
    g = oracle.OracleGraph(e, e, 0)
    assert (g.n, g.m) == (0, 0)
    assert g.count(1)[0] == 0
    g = oracle.OracleGraph(e, e, 10)
    tot, pt, _, cuts = g.count(4)
    assert tot == 0 and len(pt) == 20 and list(cuts)[-1] == 10
    s = np.array([3, 3, 5], np.uint32)                                  # only self-loops
    g = oracle.OracleGraph(s, s)
    assert (g.n, g.m) == (6, 0)
    assert g.count(2)[0] == 0


# ---- P5: blocked = unblocked, any p and cuts ------------------------------------
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_blocked_equals_unblocked(seed):
    s, d = inputs.rmat(10, 16, seed)
    g = oracle.OracleGraph(s, d, 1 << 10)
    T = g.count(1)[0]
    rng = np.random.default_rng(seed)
    for p in (2, 3, 4, 5, 8, 16):
        tot, pt, _, cuts = g.count(p)
        assert tot == T and int(pt.sum()) == T
        assert len(cuts) == p + 1
    s6, d6 = inputs.rmat(6, 8, seed)                                    # p = n and p > n (clamped)
    g6 = oracle.OracleGraph(s6, d6, 64)
    T6 = g6.count(1)[0]
    for p in (64, 71):
        tot, pt, _, cuts = g6.count(p)
        assert tot == T6 and int(pt.sum()) == T6 and len(cuts) == 65
    for p in (2, 3, 7, 16):
        cuts = rand_cuts(rng, g.n, p)
        tot, pt, _, _ = g.count(cuts=cuts)
        assert tot == T and int(pt.sum()) == T


def test_single_task_matches_full():
    s, d = inputs.rmat(11, 16, 5)
    g = oracle.OracleGraph(s, d, 1 << 11)
    _, pt, _, cuts = g.count(5)
    tl = oracle.task_list(5)
    for t, (i, j, k) in enumerate(tl):
        assert g.count_task(cuts, int(i), int(j), int(k)) == int(pt[t])


# ---- P10: independent sparse-matrix cross-check -----------------------------------
def test_scipy_block_products():
    sp = pytest.importorskip("scipy.sparse")
    s, d = inputs.rmat(12, 16, 7)
    n = 1 << 12
    keep = s != d
    a, b = np.minimum(s, d)[keep].astype(np.int64), np.maximum(s, d)[keep].astype(np.int64)
    M = sp.coo_matrix((np.ones(len(a)), (a, b)), shape=(n, n)).tocsr()
    M.data[:] = 1
    S = ((M + M.T) > 0).astype(np.int64)
    deg = np.asarray(S.sum(1)).ravel()
    order = np.lexsort((np.arange(n), deg))
    rank = np.empty(n, np.int64)
    rank[order] = np.arange(n)
    C = S.tocoo()
    up = rank[C.row] < rank[C.col]
    U = sp.csr_matrix((np.ones(up.sum(), np.int64), (rank[C.row[up]], rank[C.col[up]])), shape=(n, n))
    T = int(U.multiply(U @ U).sum())
    g = oracle.OracleGraph(s, d, n)
    tot, pt, _, cuts = g.count(4)
    assert tot == T
    t = 0
    for i in range(4):
        for j in range(i, 4):
            for k in range(j, 4):
                Bij = U[cuts[i]:cuts[i + 1], cuts[j]:cuts[j + 1]]
                Bjk = U[cuts[j]:cuts[j + 1], cuts[k]:cuts[k + 1]]
                Bik = U[cuts[i]:cuts[i + 1], cuts[k]:cuts[k + 1]]
                assert int(Bik.multiply(Bij @ Bjk).sum()) == int(pt[t]), (i, j, k)
                t += 1


# ---- P8: invariances -----------------------------------------------------------
def test_invariances():
    s, d = inputs.rmat(10, 8, 11)
    g0 = oracle.OracleGraph(s, d, 1 << 10)
    T, pt0, _, _ = g0.count(3)
    rng = np.random.default_rng(0)
    perm = rng.permutation(1 << 10).astype(np.uint32)
    assert oracle.OracleGraph(perm[s], perm[d], 1 << 10).count(3)[0] == T     # relabelling
    sh = rng.permutation(len(s))
    g1 = oracle.OracleGraph(np.concatenate([d[sh], s[:100], s[:7]]),          # shuffle+reverse+dup+loops
                            np.concatenate([s[sh], d[:100], s[:7]]), 1 << 10)
    T1, pt1, _, _ = g1.count(3)
    assert T1 == T and np.array_equal(pt1, pt0)


# ---- P6: tasks ---------------------------------------------------------------------
def test_task_enumeration():
    P = load("paper_tasks.json")
    assert oracle.task_list(3).tolist() == P["fig2_p3_tasks"]
    for tiles, tasks in P["table3_tiles_tasks"]:
        p = math.isqrt(tiles)
        assert p * p == tiles and len(oracle.task_list(p)) == tasks == p * (p + 1) * (p + 2) // 6


# ---- P9: generator shape (not parity) ---------------------------------------------
def test_rmat_shape_table3():
    ref = load("rmat_table3.json")["scale18"]
    s, d = inputs.rmat(18, 16, 1)
    g = oracle.OracleGraph(s, d, 1 << 18)
    V = int((g.degrees() > 0).sum())
    T = g.count(1)[0]
    assert abs(V / ref["V"] - 1) < 0.01
    assert abs(g.m / ref["E"] - 1) < 0.01
    assert abs(T / ref["T"] - 1) < 0.02


def test_vertex_count_rule():
    """R21: n = max(n_hint, 1 + largest raw id); ids above the hint are vertices, a
    larger hint adds isolated vertices (lowest ranks, part 0)."""
    s, d = _edges(wheel(9))                                           # ids 0..9, 9 triangles
    for hint, n in ((0, 10), (3, 10), (10, 10), (25, 25)):
        g = oracle.OracleGraph(s, d, hint)
        assert g.n == n
        tot, pt, _, cuts = g.count(2)
        assert tot == 9 and cuts[-1] == n
        assert list(g.degrees()[10:]) == [0] * (n - 10)
        assert sorted(g.rank()[10:]) == list(range(n - 10))            # isolated: lowest ranks
    s = np.array([7], np.uint32)                                      # a self-loop still names vertex 7
    assert oracle.OracleGraph(s, s, 2).n == 8
