"""Build one plan for a config and run the resident count twice (bench.py's in-run
ncu traffic capture profiles these launches; the second count is the steady state).

    ncu --set full -k regex:k_count -s 2 -c 1 -o gpurun_out/prof python scripts/profile_count.py orkut [p] [seed]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402
import paper_2009_12457_b200 as bb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "orkut"
cfg = inputs.CONFIGS[name]
p = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else cfg.p
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 1
s, d = cfg.generate(seed=seed)
ctx = bb.Context(0)
g = bb.Graph.from_edges(ctx, s, d, cfg.n_hint)
plan = bb.Plan(ctx, g, p, stats=True)
for _ in range(2):
    tot, pt, tm = plan.count(timing=True)
    print(name, "p", p, "triangles", tot, "kernel_ms", tm["t_kernel_ms"], "dense_ms", tm["t_dense_ms"], flush=True)
