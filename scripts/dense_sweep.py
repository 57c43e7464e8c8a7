"""Dense-task sweep: count time vs BBTC_DENSE_BITS (largest |V_k| counted on bit rows).

    python scripts/dense_sweep.py rmat24 [p] > gpurun_out/dense_rmat24.jsonl
First count of a plan includes building the bit rows (build_ms = first - median of the rest).
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402
import paper_2009_12457_b200 as bb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "rmat24"
cfg = inputs.CONFIGS[name]
p = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.p
bits_list = [int(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else "0,512,1024,2048,4096,8192".split(","))]
s, d = cfg.generate(seed=1)
ctx = bb.Context(0)
g = bb.Graph.from_edges(ctx, s, d, cfg.n_hint)
ref = None
for bits in bits_list:
    os.environ["BBTC_DENSE_BITS"] = str(bits)
    plan = bb.Plan(ctx, g, p)
    ts = []
    for _ in range(4):
        tot, pt, tm = plan.count(timing=True)
        ts.append(tm["t_kernel_ms"])
        ref = tot if ref is None else ref
        assert tot == ref, (tot, ref)
    info = plan.info()
    med = statistics.median(ts[1:])
    print(json.dumps({"config": name, "p": p, "dense_bits": bits, "kernel_ms": med, "first_ms": ts[0],
                      "build_ms": ts[0] - med, "dense_tasks": info["dense_tasks"],
                      "dense_bytes": info["dense_bytes"], "triangles": tot}), flush=True)
    plan.close()
