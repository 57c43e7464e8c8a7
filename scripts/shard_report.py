"""§8(e) scheduler report (CPU only): for a config's real block sizes, what the sharded
multi-GPU step moves per rank at N = 1, 2, 4, 8 — raw-edge H2D share, blocks built
(owned), blocks forwarded over NVLink, and the LPT load balance — from the product's
host scheduler (bbtc_shard_assign) and dist.block_routes.  Block sizes come from the
oracle's CSR and default cuts (analysis only; the GPU path computes them itself).

    python scripts/shard_report.py rmat24 10 [orkut 8 ...] > profiles/r02/shard_report.jsonl
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import inputs  # noqa: E402
import oracle  # noqa: E402
from paper_2009_12457_b200 import dist as bdist  # noqa: E402


def block_sizes(og, cuts):
    row, col = og.csr()
    p = len(cuts) - 1
    part = np.searchsorted(cuts, np.arange(og.n, dtype=np.int64), side="right") - 1
    src = np.repeat(np.arange(og.n, dtype=np.int64), np.diff(row).astype(np.int64))
    i, j = part[src], part[col.astype(np.int64)]
    del src
    b = j * (j + 1) // 2 + i
    return np.bincount(b, minlength=p * (p + 1) // 2).astype(np.uint64)


def work(p, cuts, bn):
    rows = np.diff(cuts.astype(np.float64))
    bid = lambda i, j: j * (j + 1) // 2 + i  # noqa: E731
    d = lambda i, j: bn[bid(i, j)] / rows[i] if rows[i] else 0.0  # noqa: E731
    out = []
    for i in range(p):
        for j in range(i, p):
            for k in range(j, p):
                nij = float(bn[bid(i, j)])
                run = min(1.0, rows[j] / nij) if nij > 0 else 1.0
                out.append(nij * (4 + d(i, k) + run * d(j, k)))
    return np.array(out)


args = sys.argv[1:]
for name, p in zip(args[::2], args[1::2]):
    p = int(p)
    cfg = inputs.CONFIGS[name]
    s, d = cfg.generate(seed=1)
    og = oracle.OracleGraph(s, d, cfg.n_hint)
    del s, d
    cuts = og.default_cuts(p).astype(np.int64)
    bn = block_sizes(og, cuts)
    rows = np.diff(cuts)
    bbytes = [12 * int(bn[b]) + 4 * (int(rows[[i for j in range(p) for i in range(j + 1)][b]]) + 1) for b in range(len(bn))]
    w = work(p, cuts, bn)
    for N in (1, 2, 4, 8):
        tr, br = bdist.shard_assign(p, cuts.astype(np.uint32), bn, N)
        load = np.bincount(tr, weights=w, minlength=N)
        routes = bdist.block_routes(p, tr, br, bn)
        recv = np.zeros(N)
        for b, o, dsts in routes:
            for q in dsts:
                recv[q] += bbytes[b]
        owned = np.zeros(N)
        for b in range(len(bn)):
            owned[br[b]] += bbytes[b]
        print(json.dumps({"config": name, "p": p, "N": N, "m": og.m, "raw_h2d_bytes_per_rank": 8 * cfg.n_samples / N,
                          "owned_block_bytes_max": owned.max(), "nvlink_recv_bytes_max": recv.max(),
                          "nvlink_recv_bytes_total": recv.sum(), "all_block_bytes": float(sum(bbytes)),
                          "load_imbalance": float(load.max() / max(load.mean(), 1e-9)),
                          "tasks_per_rank": np.bincount(tr, minlength=N).tolist()}), flush=True)
    del og
