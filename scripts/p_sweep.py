"""Time the whole step (prep + count) for several p on one config.

    python scripts/p_sweep.py friendster 4 8 16
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2009_12457_b200 as bb  # noqa: E402

name = sys.argv[1]
ps = [int(x) for x in sys.argv[2:]] or [inputs.CONFIGS[name].p]
cfg = inputs.CONFIGS[name]
s, d = cfg.generate(seed=1)
ds = torch.from_numpy(s.view(np.int32)).cuda()
dd = torch.from_numpy(d.view(np.int32)).cuda()
del s, d
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = bb.Context(0, stream=stream.cuda_stream)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
for p in ps:
    counts = torch.zeros(bb.n_tasks(p) + 1, dtype=torch.int64, device="cuda")
    res = []
    for it in range(4):
        a, b, c = ev(), ev(), ev()
        a.record(stream)
        g = bb.Graph.from_edges(ctx, ds, dd, cfg.n_hint)
        plan = bb.Plan(ctx, g, p, stats=(it == 0), row_major=bool(os.environ.get("ROW_MAJOR")))
        b.record(stream)
        plan.count_async(counts)
        c.record(stream)
        tot = int(counts[-1].item())
        if it == 0:
            info = plan.info()   # (dense_bytes is set once the bit rows exist: after the count)
        else:
            res.append((a.elapsed_time(b), b.elapsed_time(c)))
        plan.close()
        g.close()
    prep = float(np.median([r[0] for r in res]))
    cnt = float(np.median([r[1] for r in res]))
    print(json.dumps({"config": name, "p": p, "triangles": tot, "prep_ms": prep, "count_ms": cnt,
                      "step_ms": prep + cnt, "edges_per_s": info["m"] / ((prep + cnt) / 1e3),
                      "b_alg_GBps": info["b_alg"] / cnt / 1e6, "visits": info["visits"], "lambda": info["lambda"],
                      "dmax_blk": info["dmax_blk"], "block_bytes": info["block_bytes"],
                      "sum_a": info["sum_a"], "sum_b": info["sum_b"], "dense_tasks": info["dense_tasks"],
                      "dense_bytes": info["dense_bytes"]}), flush=True)
