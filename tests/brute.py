"""Independent brute-force references for pinning the oracle (tests only).

Written from the definitions (PAPER.md P:238-242 triangle; P:244-262 parts and
blocks; P:438-446 degree ordering), sharing nothing with oracle/ or the library.
"""
import itertools

import numpy as np


def simple_graph(src, dst, n_hint=0):
    """Dense symmetric 0/1 adjacency of the simple graph behind raw pairs."""
    n = max([n_hint] + [int(x) + 1 for x in src] + [int(x) + 1 for x in dst])
    A = np.zeros((n, n), dtype=np.int64)
    for a, b in zip(src, dst):
        if a != b:
            A[a, b] = A[b, a] = 1
    return A


def triangles_dense(A):
    """T = trace(A^3)/6 and per-vertex participations diag(A^3)/2."""
    A3 = A @ A @ A
    return int(np.trace(A3)) // 6, np.diag(A3) // 2


def degree_rank(A):
    deg = A.sum(1)
    order = sorted(range(len(deg)), key=lambda x: (int(deg[x]), x))
    rank = np.empty(len(deg), dtype=np.int64)
    rank[order] = np.arange(len(deg))
    return rank


def task_index(p):
    idx, t = {}, 0
    for i in range(p):
        for j in range(i, p):
            for k in range(j, p):
                idx[(i, j, k)] = t
                t += 1
    return idx


def per_task_bruteforce(A, cuts):
    """O(n^3): every mutually adjacent triple, rank-sorted, binned by parts."""
    n = A.shape[0]
    p = len(cuts) - 1
    rank = degree_rank(A)
    part = np.zeros(n, dtype=np.int64)
    for i in range(p):
        part[cuts[i]:cuts[i + 1]] = i
    idx = task_index(p)
    out = np.zeros(len(idx), dtype=np.int64)
    for a, b, c in itertools.combinations(range(n), 3):
        if A[a, b] and A[b, c] and A[a, c]:
            u, v, w = sorted((rank[a], rank[b], rank[c]))
            out[idx[(part[u], part[v], part[w])]] += 1
    return out
