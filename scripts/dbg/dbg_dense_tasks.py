"""Which dense (bit-row) tasks carry the bit-row kernel's time: per-task warp time
(bbtc_task_times) with block sizes and G_ij density."""
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
plan = bb.Plan(ctx, g, cfg.p)
plan.count()
tt = plan.task_times()
p = plan.p
cuts = plan.cuts().astype(np.int64)
sz = np.diff(cuts)
bn = plan.block_nnz()
bid = lambda i, j: j * (j + 1) // 2 + i
tr = [(i, j, k) for i in range(p) for j in range(i, p) for k in range(j, p)]
tot = tt.sum()
print("total warp-ms %.1f, dense tasks %d" % (tot, plan.info()["dense_tasks"]))
for x in np.argsort(-tt)[:30]:
    i, j, k = tr[x]
    dens = bn[bid(i, j)] / max(1, sz[i] * sz[j])
    print(tr[x], "warp-ms %.1f (%.1f%%)" % (tt[x], 100 * tt[x] / tot), "nnz_ij", bn[bid(i, j)], "|V_i|", sz[i], "|V_j|", sz[j],
          "|V_k|", sz[k], "dens_ij %.4f" % dens, "nnz_ik", bn[bid(i, k)], "nnz_jk", bn[bid(j, k)])
