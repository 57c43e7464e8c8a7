"""Exit-time teardown check: module-level context, graph, plan alive at exit."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import inputs, paper_2009_12457_b200 as bb
s, d = inputs.rmat(16, 16, 1)
ctx = bb.Context(0)
g = bb.Graph.from_edges(ctx, s, d, 1 << 16)
plan = bb.Plan(ctx, g, 8)
print(plan.count()[0], plan.task_times().sum() > 0, flush=True)
