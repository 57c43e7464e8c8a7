"""One warm step, then one profiled step of the whole hot path (for ncu launch lists).

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python scripts/profile_step.py rmat24
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2009_12457_b200 as bb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "rmat24"
cfg = inputs.CONFIGS[name]
p = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.p
s, d = cfg.generate(seed=1)
ds = torch.from_numpy(s.view(np.int32)).cuda()
dd = torch.from_numpy(d.view(np.int32)).cuda()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = bb.Context(0, stream=stream.cuda_stream)
counts = torch.zeros(bb.n_tasks(p) + 1, dtype=torch.int64, device="cuda")


def step():
    g = bb.Graph.from_edges(ctx, ds, dd, cfg.n_hint)
    plan = bb.Plan(ctx, g, p)
    plan.count_async(counts)
    tot = int(counts[-1].item())
    plan.close()
    g.close()
    return tot


step()
torch.cuda.synchronize()
l0 = ctx.launches
torch.cuda.profiler.start()
tot = step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"{name} p={p} triangles={tot} library_launch_calls={ctx.launches - l0}")
