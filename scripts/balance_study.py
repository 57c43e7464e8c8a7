"""Multi-GPU balance of the §8(e) task assignment, from one GPU: per-task device times of
the bench configuration (bbtc_task_times: each task's warp time inside an ordinary
resident count, both kernels), summed per rank under the library's own assignment
(bbtc_shard_assign: LPT on the kernel-aware per-edge cost with block affinity) for
N = 2, 4, 8, against the same LPT run on the measured times (the best a cost model
could do) — max / mean per-rank time (1 = perfect balance).

    python scripts/balance_study.py rmat24:10 orkut:8 friendster:4
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import inputs  # noqa: E402
import paper_2009_12457_b200 as bb  # noqa: E402
from paper_2009_12457_b200.dist import shard_assign  # noqa: E402


def lpt(times, world):
    load = np.zeros(world)
    for t in np.argsort(-times, kind="stable"):
        load[np.argmin(load)] += times[t]
    return load


for spec in sys.argv[1:]:
    name, _, p = spec.partition(":")
    cfg = inputs.CONFIGS[name]
    p = int(p) if p else cfg.p
    s, d = cfg.generate(seed=1)
    ctx = bb.Context(0)
    g = bb.Graph.from_edges(ctx, s, d, cfg.n_hint)
    del s, d
    plan = bb.Plan(ctx, g, p)
    plan.count()
    times = np.median(np.stack([plan.task_times() for _ in range(3)]), axis=0)
    cuts = plan.cuts()
    bnnz = plan.block_nnz()
    for world in (2, 4, 8):
        tr, _ = shard_assign(plan.p, cuts, bnnz, world)
        per_rank = np.bincount(tr.astype(np.int64), weights=times, minlength=world)
        best = lpt(times, world)
        print(json.dumps({"config": name, "p": plan.p, "world": world,
                          "imbalance_library": float(per_rank.max() / per_rank.mean()),
                          "imbalance_lpt_on_measured": float(best.max() / best.mean()),
                          "per_rank_ms": per_rank.tolist(), "tasks_per_rank": np.bincount(tr, minlength=world).tolist(),
                          "sum_task_ms": float(times.sum()), "largest_task_share": float(times.max() / times.sum())}),
              flush=True)
    plan.close()
    g.close()
    ctx.close()
