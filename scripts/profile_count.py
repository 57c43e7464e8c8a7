"""Build one plan for a config and run the count kernel twice (for ncu: profile launch 2).

    ncu --set full -k regex:k_count -s 1 -c 1 -o gpurun_out/prof python scripts/profile_count.py orkut
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402
import paper_2009_12457_b200 as bb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "orkut"
p = int(sys.argv[2]) if len(sys.argv) > 2 else inputs.CONFIGS[name].p
cfg = inputs.CONFIGS[name]
s, d = cfg.generate(seed=1)
ctx = bb.Context(0)
g = bb.Graph.from_edges(ctx, s, d, cfg.n_hint)
plan = bb.Plan(ctx, g, p, stats=True)
for _ in range(2):
    tot, pt, tm = plan.count(timing=True)
    print(name, "p", p, "triangles", tot, "kernel_ms", tm["t_kernel_ms"], "info", plan.info(), flush=True)
