"""A/B of the list kernel's column source on resident blocks: per-edge ccv vs column
offsets (kCP, the streamed walk).  Run twice: plain and with BBTC_FORCE_CP=1."""
import json, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import inputs  # noqa: E402
import paper_2009_12457_b200 as bb  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "rmat24"
cfg = inputs.CONFIGS[name]
s, d = cfg.generate(seed=1)
ctx = bb.Context(0)
g = bb.Graph.from_edges(ctx, s, d, cfg.n_hint)
plan = bb.Plan(ctx, g, cfg.p)
ref = plan.count()[0]
plan.to_host()
plan.stage()
reps = [plan.count(timing=True) for _ in range(6)][1:]
assert all(r[0] == ref for r in reps)
print(json.dumps({"config": name, "force_cp": bool(os.environ.get("BBTC_FORCE_CP")),
                  "list_ms": statistics.median(r[2]["t_kernel_ms"] - r[2]["t_dense_ms"] for r in reps),
                  "dense_ms": statistics.median(r[2]["t_dense_ms"] for r in reps)}), flush=True)
