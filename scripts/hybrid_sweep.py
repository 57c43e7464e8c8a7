"""§8(f)#3 measurement: hybrid CPU+GPU count vs the GPU alone (resident blocks, "excl.
H2D"), over the paper's cut-off grid k/8 of the task queue (§7.7) and
host thread counts.  One JSON line per point.

    python scripts/hybrid_sweep.py karate rmat16 orkut > gpurun_out/hybrid.jsonl
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402
import paper_2009_12457_b200 as bb  # noqa: E402

cores = len(os.sched_getaffinity(0))
for name in sys.argv[1:] or ["karate", "rmat16"]:
    cfg = inputs.CONFIGS[name]
    s, d = cfg.generate(seed=1)
    ctx = bb.Context(0)
    g = bb.Graph.from_edges(ctx, s, d, cfg.n_hint)
    plan = bb.Plan(ctx, g, cfg.p)
    ref, _ = plan.count()
    plan.to_host()
    plan.stage()
    gpu = [plan.count(timing=True)[2]["t_total_ms"] for _ in range(7)]
    print(json.dumps({"config": name, "mode": "gpu_only", "t_ms": statistics.median(gpu), "cores": cores}),
          flush=True)
    for threads in sorted({1, 4, cores}):
        for k in range(9):
            cut = k / 8
            reps = []
            for _ in range(5):
                tot, _, st = plan.count_hybrid(threads, cut)
                assert tot == ref
                reps.append(st)
            med = statistics.median(r["t_total_ms"] for r in reps)
            r = reps[0]
            print(json.dumps({"config": name, "mode": "hybrid", "threads": threads, "cutoff": cut, "t_ms": med,
                              "cpu_tasks": r["cpu_tasks"], "gpu_tasks": r["gpu_tasks"],
                              "gpu_launches": r["gpu_launches"], "t_cpu_ms": r["t_cpu_ms"], "t_gpu_ms": r["t_gpu_ms"],
                              "gpu_only_ms": statistics.median(gpu)}), flush=True)
    plan.close()
    g.close()
    ctx.close()
