"""Which tasks does the column-offset walk (kCP) slow down?  Per-task times with and
without BBTC_FORCE_CP on the same staged host plan."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import inputs, paper_2009_12457_b200 as bb
name = sys.argv[1] if len(sys.argv) > 1 else "rmat24"
cfg = inputs.CONFIGS[name]
s, d = cfg.generate(seed=1)
ctx = bb.Context(0)
g = bb.Graph.from_edges(ctx, s, d, cfg.n_hint)
plan = bb.Plan(ctx, g, cfg.p, sparse=True)
os.environ["BBTC_FORCE_CP"] = "1"
plan.to_host()
plan.stage()
t_cp = np.median([plan.task_times() for _ in range(3)], axis=0)
del os.environ["BBTC_FORCE_CP"]
t_pl = np.median([plan.task_times() for _ in range(3)], axis=0)
p = plan.p
bn = plan.block_nnz()
cuts = plan.cuts()
bid = lambda i, j: j * (j + 1) // 2 + i
tr = [(i, j, k) for i in range(p) for j in range(i, p) for k in range(j, p)]
print("sum plain %.3f ms, sum cp %.3f ms" % (t_pl.sum(), t_cp.sum()))
for x in np.argsort(-(t_cp - t_pl))[:15]:
    i, j, k = tr[x]
    print(tr[x], "plain %.3f cp %.3f" % (t_pl[x], t_cp[x]), "nnz_ij", bn[bid(i, j)], "|V_j|", cuts[j + 1] - cuts[j],
          "|V_i|", cuts[i + 1] - cuts[i])
