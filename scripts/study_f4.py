"""§8(f)#4: partition and estimator study on the synthetic configs (PAPER §7.2 and §7.6).

    python scripts/study_f4.py psweep rmat24 4 8 12 16 24 32      > gpurun_out/psweep_rmat24.jsonl
    python scripts/study_f4.py estim  rmat24 16                    > gpurun_out/estim_rmat24.jsonl

psweep: for each p, the default cut rule and the PBD-like refinement (bbtc_cuts_refine,
minimising m_max): λ, m_max, d'_avg, c = d_avg/d'_avg, λp/c (the O(λp/c · m^1.5) bound,
P:603-608), and the measured prep / count times of the resident step.

estim: per-task device times (bbtc_task_times) against the paper's four workload
estimators — NNZ (nonzeros of the task's three blocks), Density (sum of
nonzeros per unit area of the blocks), Degree (sum of the blocks' average degrees),
ExecTime (nnz(G_ij)·max(δ(G_ik), δ(G_jk))) — plus the per-edge cost this
build sizes work items with (nnz(G_ij)·(8 + δ(G_ik) + δ(G_jk))).  Reported as the
paper's metric: the least fraction of the estimator-sorted task list that covers the x
most time-consuming tasks, x = 1..32 (lower is better), and Spearman's ρ.
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2009_12457_b200 as bb  # noqa: E402


def triples(p):
    return [(i, j, k) for i in range(p) for j in range(i, p) for k in range(j, p)]


def bid(i, j):
    return j * (j + 1) // 2 + i


def time_step(ctx, ds, dd, cfg, p, cuts, stream, counts, reps=3):
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    out = []
    for it in range(reps + 1):
        a, b, c = ev(), ev(), ev()
        a.record(stream)
        g = bb.Graph.from_edges(ctx, ds, dd, cfg.n_hint)
        plan = bb.Plan(ctx, g, p, cuts)
        b.record(stream)
        plan.count_async(counts)
        c.record(stream)
        tot = int(counts[-1].item())
        if it:
            out.append((a.elapsed_time(b), b.elapsed_time(c)))
        plan.close()
        g.close()
    return tot, statistics.median(x[0] for x in out), statistics.median(x[1] for x in out)


def psweep(name, ps):
    cfg = inputs.CONFIGS[name]
    s, d = cfg.generate(seed=1)
    ds = torch.from_numpy(s.view(np.int32)).cuda()
    dd = torch.from_numpy(d.view(np.int32)).cuda()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = bb.Context(0, stream=stream.cuda_stream)
    g = bb.Graph.from_edges(ctx, ds, dd, cfg.n_hint)
    st = g.stats()
    n_ne, m = st["n_nonisolated"], st["m"]
    d_avg = 2 * m / max(n_ne, 1)
    for p in ps:
        counts = torch.zeros(bb.n_tasks(p) + 1, dtype=torch.int64, device="cuda")
        for rule in ("default", "refined"):
            if rule == "default":
                cuts = bb.Plan(ctx, g, p).cuts()
            else:
                cuts, _ = bb.refine_cuts(ctx, g, p, max_evals=int(os.environ.get("REFINE_EVALS", "200")))
            plan = bb.Plan(ctx, g, cuts=cuts)
            info = plan.info()
            bn = plan.block_nnz().astype(np.float64)
            sizes = np.diff(cuts.astype(np.int64))
            rows_sum = sum(sizes[i] for j in range(len(sizes)) for i in range(j + 1))
            d_avg_blk = m / max(rows_sum, 1)          # nnz per block row, averaged over blocks
            c = d_avg / d_avg_blk
            plan.close()
            tot, prep, cnt = time_step(ctx, ds, dd, cfg, p, cuts, stream, counts)
            print(json.dumps({"study": "psweep", "config": name, "p": int(len(cuts) - 1), "rule": rule,
                              "lambda": info["lambda"], "m_max": int(bn.max()), "d_avg": d_avg,
                              "d_avg_blk": d_avg_blk, "c": c, "lambda_p_over_c": info["lambda"] * p / c,
                              "prep_ms": prep, "count_ms": cnt, "step_ms": prep + cnt, "triangles": tot,
                              "dense_tasks": info["dense_tasks"], "cuts": cuts.tolist() if p <= 16 else None}),
                  flush=True)


def coverage(order, times, xs=range(1, 33)):
    """Least fraction of the estimator-sorted list whose prefix holds the x slowest tasks."""
    top = np.argsort(-times, kind="stable")
    pos = np.empty(len(order), np.int64)
    pos[order] = np.arange(len(order))
    return [float((pos[top[:x]].max() + 1) / len(order)) for x in xs if x <= len(order)]


def spearman(a, b):
    ra = np.argsort(np.argsort(a, kind="stable"), kind="stable").astype(np.float64)
    rb = np.argsort(np.argsort(b, kind="stable"), kind="stable").astype(np.float64)
    ra -= ra.mean()
    rb -= rb.mean()
    return float((ra * rb).sum() / np.sqrt((ra * ra).sum() * (rb * rb).sum()))


def estim(name, p):
    cfg = inputs.CONFIGS[name]
    s, d = cfg.generate(seed=1)
    ctx = bb.Context(0)
    g = bb.Graph.from_edges(ctx, s, d, cfg.n_hint)
    del s, d
    for sparse in (True, False):
        plan = bb.Plan(ctx, g, p, sparse=sparse)
        plan.count()
        times = np.median(np.stack([plan.task_times() for _ in range(3)]), axis=0)
        cuts = plan.cuts().astype(np.float64)
        sz = np.diff(cuts)
        bn = plan.block_nnz().astype(np.float64)
        tr = triples(plan.p)
        idx = np.arange(len(tr))
        delta = lambda i, j: bn[bid(i, j)] / sz[i] if sz[i] else 0.0  # noqa: E731
        dens = lambda i, j: bn[bid(i, j)] / (sz[i] * sz[j]) if sz[i] * sz[j] else 0.0  # noqa: E731
        est = {
            "NNZ": [bn[bid(i, j)] + bn[bid(i, k)] + bn[bid(j, k)] for i, j, k in tr],
            "Density": [dens(i, j) + dens(i, k) + dens(j, k) for i, j, k in tr],
            "Degree": [delta(i, j) + delta(i, k) + delta(j, k) for i, j, k in tr],
            "ExecTime": [bn[bid(i, j)] * max(delta(i, k), delta(j, k)) for i, j, k in tr],
            "ItemCost": [bn[bid(i, j)] * (8 + delta(i, k) + delta(j, k)) for i, j, k in tr],
            # kernel-aware: probe words per edge, staged list once per column run of G_ij
            "ProbeCost": [bn[bid(i, j)] * (4 + delta(i, k)) + min(bn[bid(i, j)], sz[j]) * delta(j, k)
                          for i, j, k in tr],
        }
        for e, v in est.items():
            v = np.asarray(v)
            order = idx[np.lexsort((idx, -v))]          # non-increasing estimate, ties by index
            cov = coverage(order, times)
            print(json.dumps({"study": "estimators", "config": name, "p": plan.p, "kernels": "list only" if sparse
                              else "list + bit rows", "estimator": e, "spearman": spearman(v, times),
                              "coverage_top_x": cov, "mean_coverage": float(np.mean(cov)),
                              "tasks": len(tr), "sum_task_ms": float(times.sum()),
                              "times_ms": times.tolist(), "estimate": v.tolist(),
                              "top_task_share": float(np.sort(times)[-1] / times.sum())}), flush=True)
        plan.close()


if __name__ == "__main__":
    kind, name = sys.argv[1], sys.argv[2]
    args = [int(x) for x in sys.argv[3:]]
    if kind == "psweep":
        psweep(name, args or [inputs.CONFIGS[name].p])
    else:
        estim(name, args[0] if args else inputs.CONFIGS[name].p)
