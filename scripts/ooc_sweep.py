"""Out-of-core count time and H2D volume vs device budget (fraction of the plan's bytes)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2009_12457_b200 as bb  # noqa: E402

name = sys.argv[1]
fracs = [float(x) for x in sys.argv[2:]] or [0.25, 0.5, 0.75]
cfg = inputs.CONFIGS[name]
s, d = cfg.generate(seed=1)
ctx = bb.Context(0)
g = bb.Graph.from_edges(ctx, s, d, cfg.n_hint)
plan = bb.Plan(ctx, g, cfg.p)
total = plan.info()["block_bytes"]
ref, _ = plan.count()
plan.to_host()
for f in fracs:
    plan.set_budget(int(total * f))
    plan.unstage()
    tot, _, tm = plan.count(timing=True)
    assert tot == ref
    print(json.dumps({"config": name, "fill": os.environ.get("BBTC_OOC_FILL", "0.5"), "budget_frac": f,
                      "ms": tm["t_total_ms"], "h2d_GB": tm["h2d_bytes"] / 1e9, "h2d_x_plan": tm["h2d_bytes"] / total}),
          flush=True)
