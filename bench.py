#!/usr/bin/env python
"""bench.py — BBTC on B200: whole hot path per step, JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config rmat24] [--impl ours|reference]

A step is one pass of every §8(a) row over the config's synthetic raw edge list
(already resident in HBM): canonicalise + degree rank + orient (a1-a2), cuts +
BCSR + tasks (a3-a5), the intersection kernel over this rank's work items (a7)
and, for N > 1, one NCCL all-reduce of the uint64 per-task counters (a8).
`value` = unique undirected edges / step time (the paper's rate, P:1029-1031 read
as m/t, R9), whole job.  `e2e` = the same through the C-ABI with the
raw edges in pinned HOST memory (H2D inside the step) and the per-task counts
read back to the host.  Extra keys report the paper's split: count time with
blocks resident ("excl. H2D") and with blocks streamed from pinned host memory
("incl. H2D").

Multi-GPU (torchrun, one rank per GPU): every rank builds the plan (replicated
preprocessing), counts the work items r, r+N, ... and the counters are summed
with one all-reduce; time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402

METRIC = "TC wall time (s) and edges/s, excl./incl. H2D copy, at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="rmat24", choices=sorted(inputs.CONFIGS))
    ap.add_argument("--p", type=int, default=0, help="override the config's p")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(config):
    path = os.path.join(ROOT, "profiles", f"ncu_count_{config}.json")
    try:
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
                self.lines = [ln for ln in out.splitlines() if ln.strip()]
            except Exception:
                pass

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
                for nm, v in zip(names, f[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            except Exception:
                continue
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(cfg, s, d, threads_hint=0, target_s=8.0):
    """The oracle as it stands, on the box's host cores, on a bounded sample:
    full oracle preprocessing (canonicalise, rank, orient) + the node-iterator
    count on every stride-th row, extrapolated to all rows."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    og = oracle.OracleGraph(s, d, cfg.n_hint, threads_hint)
    t_build = time.perf_counter() - t0
    m = og.m
    stride = 1024
    t_s = 0.0
    while True:
        t1 = time.perf_counter()
        og.count_rows(0, og.n, stride)
        t_s = time.perf_counter() - t1
        if t_s * 2 > target_s or stride == 1:
            break
        stride = max(1, stride // 4)
    t_full = t_build + t_s * stride
    del og
    return {"value": m / t_full, "unit": "edges/s", "cores": cores, "kind": "oracle",
            "sample": f"{cfg.name}: full oracle build ({t_build:.2f} s) + node-iterator count on every "
                      f"{stride}-th row ({t_s:.2f} s), extrapolated x{stride}",
            "t_build_s": t_build, "t_count_sample_s": t_s, "stride": stride, "t_extrapolated_s": t_full}


def run_reference(args):
    """--impl reference: the oracle, on rank 0 only, on this config."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = inputs.CONFIGS[args.config]
    s, d = cfg.generate(seed=args.seed)
    import oracle
    cores = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    og = oracle.OracleGraph(s, d, cfg.n_hint)
    t_build = time.perf_counter() - t0
    # stride sized so one sample step is ~2 s of CPU work
    stride = 256
    for _ in range(8):
        t1 = time.perf_counter()
        og.count_rows(0, og.n, stride)
        ts = time.perf_counter() - t1
        if ts > 1.0 or stride == 1:
            break
        stride = max(1, stride // 4)
    for _ in range(args.warmup):
        og.count_rows(0, og.n, stride)
    times = []
    for k in range(args.steps):
        t1 = time.perf_counter()
        og.count_rows(k % stride, og.n, stride)
        times.append(time.perf_counter() - t1)
    t_step = t_build + statistics.median(times) * stride
    v = og.m / t_step
    line = {"metric": METRIC, "impl": "reference", "value": v, "unit": "edges/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": cfg.name, "desc": cfg.desc, "p": cfg.p, "seed": args.seed,
                       "l2": "inputs larger than L2 (CPU run)"},
            "e2e": {"value": v, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "cpu_baseline": {"value": v, "unit": "edges/s", "cores": cores, "kind": "oracle",
                             "sample": f"oracle build once ({t_build:.2f} s) + per step the node-iterator count "
                                       f"on every {stride}-th row, extrapolated x{stride}"},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_2009_12457_b200 as bb
    from paper_2009_12457_b200.dist import count_distributed, max_over_ranks, reduce_counts

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # One rank per GPU (NCCL over NVLink).  More ranks than GPUs (a functional check of
    # the N>1 path on a small box) share devices and reduce with gloo instead.
    ndev = torch.cuda.device_count()
    local = local % max(ndev, 1)
    torch.cuda.set_device(local)
    if world > 1:
        if world <= ndev:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    cfg = inputs.CONFIGS[args.config]
    p = args.p or cfg.p
    E = cfg.n_samples
    # Raw edges: pinned host copy (for e2e) and a device copy (for the device-resident step).
    hs = torch.empty(E, dtype=torch.int32, pin_memory=True)
    hd = torch.empty(E, dtype=torch.int32, pin_memory=True)
    t0 = time.perf_counter()
    cfg.generate(seed=args.seed, out=(hs.numpy().view(np.uint32), hd.numpy().view(np.uint32)))
    t_gen = time.perf_counter() - t0
    ds = hs.to("cuda", non_blocking=True)
    dd = hd.to("cuda", non_blocking=True)
    # A dedicated stream shared by torch (events, all-reduce) and the library.
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = bb.Context(local, stream=stream.cuda_stream)
    nt = bb.n_tasks(p)
    counts = torch.zeros(nt + 1, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    kern_ms = []

    step_ev = []   # per timed step: events at start, after a1-a2, after a3-a5, after a7, end

    def step(src, dst, record):
        e0, e1, e2 = ev(), ev(), ev()
        e0.record(stream)
        g = bb.Graph.from_edges(ctx, src, dst, cfg.n_hint)
        e1.record(stream)
        plan = bb.Plan(ctx, g, p)
        e2.record(stream)
        a, b = ev(), ev()
        a.record(stream)
        plan.count_async(counts, rank, world)
        b.record(stream)
        reduce_counts(counts)
        e3 = ev()
        e3.record(stream)
        tot = int(counts[-1].item())
        if record:
            kern_ms.append(a.elapsed_time(b))
            step_ev.append((e0, e1, e2, b, e3))
        info = plan.info()
        st = g.stats()
        plan.close()
        g.close()
        return tot, info, st

    for _ in range(args.warmup):
        tot, info, st = step(ds, dd, False)
    kern_ms.clear()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = ctx.launches
    with Clocks(local) as clk:
        s0, s1 = ev(), ev()
        s0.record(stream)
        for _ in range(args.steps):
            tot, info, st = step(ds, dd, True)
        s1.record(stream)
        torch.cuda.synchronize()
    launches = (ctx.launches - l0) // args.steps
    ms = s0.elapsed_time(s1) / args.steps
    if world > 1:
        dist.barrier()
    ms = max_over_ranks(ms, device="cuda")
    m = st["m"]
    value = m / (ms / 1e3)
    kern = statistics.mean(kern_ms)
    per_step = [e0.elapsed_time(e3) for e0, _, _, _, e3 in step_ev]
    t_graph = statistics.median(e0.elapsed_time(e1) for e0, e1, _, _, _ in step_ev)
    t_plan = statistics.median(e1.elapsed_time(e2) for _, e1, e2, _, _ in step_ev)

    # e2e: host (pinned) raw edges -> H2D inside the step -> per-task counts back on the host
    e2e_ms = []
    for x in range(args.e2e_steps + 1):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = ev(), ev()
        a.record(stream)
        g = bb.Graph.from_edges(ctx, hs, hd, cfg.n_hint)
        plan = bb.Plan(ctx, g, p)
        count_distributed(plan, counts)
        host_counts = counts.cpu()
        b.record(stream)
        torch.cuda.synchronize()
        assert int(host_counts[-1]) == tot
        plan.close()
        g.close()
        if x:
            e2e_ms.append(a.elapsed_time(b))
    e2e = max_over_ranks(statistics.median(e2e_ms), device="cuda")

    # The paper's split (one plan, stats on): count with blocks resident vs streamed.
    g = bb.Graph.from_edges(ctx, ds, dd, cfg.n_hint)
    plan = bb.Plan(ctx, g, p, stats=True)
    pinfo = plan.info()
    plan.count(rank, world)                      # builds the dense tasks' bit rows
    # The paper's convention: median of 5 runs after a warm-up, plus the minimum.
    reps_x = [plan.count(rank, world, timing=True) for _ in range(5)]
    tot_x, _, tm_x = reps_x[0]
    dinfo = plan.info()
    plan.to_host()
    reps_i = []
    for _ in range(6):                           # first: warm-up of the host plan's streaming order
        plan.unstage()
        reps_i.append(plan.count(rank, world, timing=True))
    reps_i = reps_i[1:]
    tot_i, _, tm_i = reps_i[0]
    sinfo = plan.info()
    t_x = [r[2]["t_total_ms"] for r in reps_x]
    t_i = [r[2]["t_total_ms"] for r in reps_i]
    t_h2d = [r[2]["t_h2d_ms"] for r in reps_i]
    # Out of core: the device may hold only half of the blocks.
    plan.unstage()
    plan.set_budget(pinfo["block_bytes"] // 2)
    plan.count(rank, world)                      # first use of the cache arenas' sizes
    tot_o, _, tm_o = plan.count(rank, world, timing=True)
    # Streaming (unlock order) and the budget re-order the tasks, so a rank's share of
    # the items differs between modes; the sums over ranks agree.
    sums = torch.tensor([tot_x, tot_i, tot_o], dtype=torch.int64, device="cuda")
    if world > 1:
        dist.all_reduce(sums)
    assert int(sums[0]) == int(sums[1]) == int(sums[2]) == tot
    plan.close()
    g.close()

    peak, peak_src = load_peaks()
    b_alg_launch = pinfo["b_alg"] / world
    achieved = b_alg_launch / (kern / 1e3) / 1e9
    traffic = ncu_traffic(cfg.name)
    line = {
        "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": cfg.name, "desc": cfg.desc, "p": p, "seed": args.seed, "raw_edges": E,
                   "n": st["n"], "m": m, "tasks": nt, "parallelism": f"tasks/{world}",
                   "l2": "inputs larger than L2 (no flush needed)"},
        "e2e": {"value": m / (e2e / 1e3), "unit": "edges/s", "ms_per_step": e2e,
                "h2d_bytes_per_step": 8 * E, "d2h_bytes_per_step": 8 * (nt + 1)},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "k_count + k_count_dense", "kernel_ms": kern,
                     "b_alg_bytes_per_launch": b_alg_launch, "peak_source": peak_src,
                     "note": "one count = the list kernel (k_count, sparse tasks) then the bit-row kernel "
                             "(k_count_dense, dense tasks), timed together. achieved/frac are logical (B_alg = "
                             "bytes Alg. 5 reads per edge, SURVEY 8(d)); staged lists reused across a run of "
                             "edges and bit rows replacing long lists let it exceed 1. physical_frac = ncu DRAM "
                             "bytes of both kernels per count / this time / peak.",
                     "physical_frac": (traffic / world / (kern / 1e3) / 1e9 / peak) if traffic else None},
        "clocks": clk.summary(),
        "triangles": tot,
        "paper_split": {
            "note": "count only (a7-a8), blocks already built: excl = all blocks resident; incl = blocks in "
                    "pinned host memory, streamed H2D inside the timing (P:37-40, DESIGN R10). Median of 5 "
                    "after a warm-up, and min (P:1028-1029). edges/s = m / t (R9).",
            "t_excl_ms": statistics.median(t_x), "t_excl_min_ms": min(t_x),
            "t_incl_ms": statistics.median(t_i), "t_incl_min_ms": min(t_i),
            "edges_per_s_excl": m / (statistics.median(t_x) / 1e3) if world == 1 else None,
            "edges_per_s_incl": m / (statistics.median(t_i) / 1e3) if world == 1 else None,
            "h2d_bytes": tm_i["h2d_bytes"], "h2d_last_copy_ms": statistics.median(t_h2d),
            "h2d_GBps": tm_i["h2d_bytes"] / (statistics.median(t_h2d) / 1e3) / 1e9 if t_h2d[0] > 0 else None,
            "block_bytes_device": pinfo["block_bytes"], "stream_bytes": sinfo["stream_bytes"]},
        "breakdown_ms": {"step": ms, "step_median": statistics.median(per_step), "step_min": min(per_step),
                         "graph_a1_a2": t_graph, "plan_a3_a5": t_plan,
                         "count_kernel": kern, "prep_and_plan": ms - kern,
                         "count_list_kernel": tm_x["t_kernel_ms"] - tm_x["t_dense_ms"],
                         "count_dense_kernel": tm_x["t_dense_ms"], "dense_tasks": dinfo["dense_tasks"],
                         "dense_bit_row_bytes": dinfo["dense_bytes"],
                         "count_excl_h2d": statistics.median(t_x), "count_incl_h2d": statistics.median(t_i),
                         "h2d_bytes_blocks": tm_i["h2d_bytes"],
                         "count_out_of_core_half_budget": tm_o["t_total_ms"], "h2d_bytes_out_of_core": tm_o["h2d_bytes"],
                         "gen_s": t_gen},
        "plan": {"lambda": pinfo["lambda"], "dmax_blk": pinfo["dmax_blk"], "visits": pinfo["visits"],
                 "b_alg": pinfo["b_alg"], "work_items": pinfo["work_items"], "block_bytes": pinfo["block_bytes"]},
        "paper_context": "BBTC on 8xV100 DGX-1 hybrid, copy incl.: R-MAT scale24 1.154 s = 2.3e8 edges/s "
                         "(P:1182-1186); Friendster 3.133 s = 5.8e8 edges/s (P:1200-1204). Other hardware.",
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, hs.numpy().view(np.uint32), hd.numpy().view(np.uint32))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
