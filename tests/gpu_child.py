"""Child process for GPU parity tests that need their own environment (e.g.
CUDA_LAUNCH_BLOCKING=1): counts one seeded input in several modes through the C-ABI
and prints one JSON line {mode: [total, per_task...]}.  Never imports the oracle.

    python tests/gpu_child.py rmat:15:16:9 6 resident,streamed,ooc25,ooc50,stage,ranks3
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import inputs  # noqa: E402
import paper_2009_12457_b200 as bb  # noqa: E402


def edges(spec):
    kind, *a = spec.split(":")
    if kind == "rmat":
        scale, ef, seed = map(int, a)
        return (*inputs.rmat(scale, ef, seed), 1 << scale)
    if kind == "gnp":
        n, q, seed = int(a[0]), float(a[1]), int(a[2])
        return (*inputs.gnp(n, q, seed), n)
    cfg = inputs.CONFIGS[kind]
    s, d = cfg.generate(seed=int(a[0]) if a else 1)
    return s, d, cfg.n_hint


def run(spec, p, modes, row_major=False):
    s, d, n_hint = edges(spec)
    ctx = bb.Context(0)
    g = bb.Graph.from_edges(ctx, s, d, n_hint)
    plan = bb.Plan(ctx, g, p, row_major=row_major)
    out = {"cuts": plan.cuts().tolist(), "slots": plan.info()["slot_bytes"]}
    whole = plan.info()["block_bytes"]
    max_task = plan.info()["max_task_bytes"]
    host = False

    def res(t, pt):
        return [int(t)] + [int(x) for x in pt]

    for mode in modes:
        if mode == "resident":
            out[mode] = res(*plan.count())
        elif mode.startswith("ranks") or mode.startswith("sranks"):
            # a rank split: resident blocks, or (sranks) streamed from host memory per rank
            w = int(mode.split("ranks")[1])
            if mode[0] == "s" and not host:
                plan.to_host()
                host = True
            acc = None
            for r in range(w):
                if mode[0] == "s":
                    plan.set_budget(0)
                    plan.unstage()
                t, pt = plan.count(r, w)
                acc = pt.astype(np.uint64) if acc is None else acc + pt
            out[mode] = res(int(acc.sum()), acc)
        else:
            if not host:
                plan.to_host()
                host = True
            plan.unstage()
            if mode == "streamed":
                plan.set_budget(0)
                t, pt, tm = plan.count(timing=True)
                out[mode] = res(t, pt)
                out[mode + "_h2d"] = int(tm["h2d_bytes"])
            elif mode.startswith("ooc"):
                frac = int(mode[3:]) / 100
                budget = max(int(whole * frac), int(max_task * 2))
                plan.set_budget(budget)
                t, pt, tm = plan.count(timing=True)
                plan.set_budget(0)
                out[mode] = res(t, pt)
                out[mode + "_budget"] = budget
            elif mode == "stage":
                plan.stage()
                out[mode] = res(*plan.count())
    out["stream_bytes"] = int(plan.info()["stream_bytes"]) if host else 0
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    rm = len(sys.argv) > 4 and sys.argv[4] == "rowmajor"
    run(sys.argv[1], int(sys.argv[2]), sys.argv[3].split(","), rm)
