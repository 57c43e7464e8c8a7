"""Count-kernel A/B across library builds (BBTC_LIB) and configs: per (lib, config) one
process builds the resident plan and reports median list / bit-row kernel ms of 5 counts.

    python scripts/ab_variants.py rmat24,orkut,friendster paper_2009_12457_b200/libbbtc.so build_ab/min6/libbbtc.so

A variant may also be the default library under environment knobs: `env:K=V[;K2=V2]`
(e.g. `env:BBTC_L2_FETCH=32`).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, os, statistics, sys
sys.path.insert(0, %r)
import inputs, paper_2009_12457_b200 as bb
name = sys.argv[1]; p = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "0" else inputs.CONFIGS[name].p
cfg = inputs.CONFIGS[name]
s, d = cfg.generate(seed=1)
ctx = bb.Context(0)
g = bb.Graph.from_edges(ctx, s, d, cfg.n_hint)
del s, d
plan = bb.Plan(ctx, g, p)
ref = plan.count()[0]
reps = [plan.count(timing=True)[2] for _ in range(5)]
print(json.dumps({"config": name, "p": p, "lib": os.environ.get("BBTC_VARIANT", os.environ.get("BBTC_LIB", "default")), "triangles": ref,
                  "list_ms": statistics.median(r["t_kernel_ms"] - r["t_dense_ms"] for r in reps),
                  "dense_ms": statistics.median(r["t_dense_ms"] for r in reps),
                  "count_ms": statistics.median(r["t_kernel_ms"] for r in reps)}), flush=True)
''' % ROOT

configs = sys.argv[1].split(",")
libs = sys.argv[2:]
for cfgp in configs:
    name, _, p = cfgp.partition(":")
    for lib in libs:
        if lib.startswith("env:"):
            kv = dict(x.split("=", 1) for x in lib[4:].split(";") if x)
            env = {**os.environ, **kv, "BBTC_VARIANT": lib, "BBTC_LIB": os.path.abspath("paper_2009_12457_b200/libbbtc.so")}
        else:
            env = {**os.environ, "BBTC_LIB": os.path.abspath(lib)}
        r = subprocess.run([sys.executable, "-c", CHILD, name, p or "0"], env=env, capture_output=True, text=True,
                           timeout=1200)
        out = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        print(out[-1] if out else json.dumps({"config": name, "lib": lib, "error": r.stderr[-500:]}), flush=True)
