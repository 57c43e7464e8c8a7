"""Preprocessing trace: a1-a2 (graph) and a3-a5 (plan) of one config, device input, as the
bench step runs them, with BBTC_TRACE=1 phase events and the bench's own CUDA events.

    BBTC_TRACE=1 python scripts/trace_prep.py rmat24 [p] [reps]
"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2009_12457_b200 as bb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "rmat24"
cfg = inputs.CONFIGS[name]
p = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "0" else cfg.p
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
s, d = cfg.generate(seed=1)
ds = torch.from_numpy(s.view("int32")).cuda()
dd = torch.from_numpy(d.view("int32")).cuda()
del s, d
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = bb.Context(0, stream=stream.cuda_stream)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
rows = []
for r in range(reps + 1):
    torch.cuda.synchronize()
    e0, e1, e2 = ev(), ev(), ev()
    h0 = time.perf_counter()
    e0.record(stream)
    g = bb.Graph.from_edges(ctx, ds, dd, cfg.n_hint)
    e1.record(stream)
    h1 = time.perf_counter()
    plan = bb.Plan(ctx, g, p)
    e2.record(stream)
    h2 = time.perf_counter()
    torch.cuda.synchronize()
    if r:
        rows.append((e0.elapsed_time(e1), e1.elapsed_time(e2), (h1 - h0) * 1e3, (h2 - h1) * 1e3))
    plan.close()
    g.close()
med = [statistics.median(x[i] for x in rows) for i in range(4)]
print(f"{name} p={p}: graph {med[0]:.2f} ms (host {med[2]:.2f}), plan {med[1]:.2f} ms (host {med[3]:.2f})", flush=True)
