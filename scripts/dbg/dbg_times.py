import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import inputs, paper_2009_12457_b200 as bb
s, d = inputs.rmat(20, 16, 1)
ctx = bb.Context(0)
g = bb.Graph.from_edges(ctx, s, d, 1 << 20)
plan = bb.Plan(ctx, g, 8, sparse=True, stats=True)
tot, pt = plan.count()
tt = plan.task_times()
bn = plan.block_nnz()
p = plan.p
bid = lambda i, j: j * (j + 1) // 2 + i
tr = [(i, j, k) for i in range(p) for j in range(i, p) for k in range(j, p)]
order = np.argsort(-tt)
for x in order[:12]:
    i, j, k = tr[x]
    print(x, (i, j, k), "t_ms %.4f" % tt[x], "nnz_ij", bn[bid(i, j)], "nnz_ik", bn[bid(i, k)], "nnz_jk", bn[bid(j, k)], "tri", pt[x])
print("cuts", plan.cuts())
for x in np.argsort(tt)[:5]:
    print("fast", x, tr[x], tt[x], bn[bid(tr[x][0], tr[x][1])])
