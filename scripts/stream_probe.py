"""Streamed count (a6) of a config: where the time goes.

Prints, per setting, the count time with blocks resident (excl. H2D), the time to
stage every block alone (the H2D floor), and the streamed count (incl. H2D) with
the time its last copy landed (t_h2d_ms), for 1, 2 and 4 copy streams."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402
import paper_2009_12457_b200 as bb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "rmat24"
cfg = inputs.CONFIGS[name]
s, d = cfg.generate(seed=1)
for ncs in (2, 1, 4):
    ctx = bb.Context(0, copy_streams=ncs)
    g = bb.Graph.from_edges(ctx, s, d, cfg.n_hint)
    plan = bb.Plan(ctx, g, cfg.p)
    ref, _, tm_ex = plan.count(timing=True)
    plan.to_host()
    for rep in range(3):
        plan.unstage()
        ctx.sync()
        t0 = time.perf_counter()
        plan.stage()
        t_stage = (time.perf_counter() - t0) * 1e3
        plan.unstage()
        tot, _, tm = plan.count(timing=True)
        assert tot == ref
        print(json.dumps({"config": name, "copy_streams": ncs, "rep": rep, "excl_ms": tm_ex["t_kernel_ms"],
                          "stage_ms": t_stage, "incl_ms": tm["t_kernel_ms"], "incl_wall_ms": tm["t_total_ms"],
                          "last_copy_ms": tm["t_h2d_ms"], "dense_ms": tm["t_dense_ms"],
                          "h2d_GB": tm["h2d_bytes"] / 1e9}), flush=True)
    del plan, g, ctx
