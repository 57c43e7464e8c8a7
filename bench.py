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

Multi-GPU (torchrun, one rank per GPU, NCCL): the sharded step of SURVEY §8(e)
(main_sharded): each rank holds 1/N of the raw edges, a1-a5 run
sharded with two all-to-alls and block forwarding over NVLink, every rank counts
the tasks the LPT/block-affinity scheduler gave it, and one all-reduce sums the
per-task counters; time is the max over ranks.
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
    ap.add_argument("--no-ncu", action="store_true", help="skip the in-run ncu traffic capture")
    ap.add_argument("--e2e-steps", type=int, default=3)
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def live_traffic(cfg, p, seed, timeout=900):
    """DRAM bytes per launch of the two count kernels, measured in THIS run: an ncu
    subprocess (dram__bytes_read/write.sum, gpu__time_duration.sum, L2 hit rate) over
    scripts/profile_count.py, which builds the same plan and counts twice; the second
    count's launches are used (the first builds the bit rows).  ncu times are
    serialised and cold-cache: only the bytes (and L2 hit rate) are taken from it."""
    import csv
    import shutil
    import tempfile
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, "ncu not found"
    with tempfile.TemporaryDirectory() as tmp:
        log = os.path.join(tmp, "ncu.csv")
        cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
               "lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,"
               "lts__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active",
               "--clock-control", "none", "-k", "regex:k_count", "--csv",
               "--log-file", log, sys.executable, os.path.join(ROOT, "scripts", "profile_count.py"), cfg.name,
               str(p), str(seed)]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
        except Exception as ex:  # noqa: BLE001
            return None, f"ncu failed: {ex}"
        if r.returncode != 0 or not os.path.exists(log):
            return None, f"ncu rc={r.returncode}: {(r.stderr or r.stdout)[-300:]}"
        rows = [ln for ln in open(log) if ln.startswith('"')]
    launches = {}
    for row in csv.DictReader(rows):
        try:
            lid = int(row["ID"])
        except (KeyError, ValueError):
            continue
        d = launches.setdefault(lid, {"kernel": row.get("Kernel Name", "")})
        v = float(str(row["Metric Value"]).replace(",", ""))
        unit = row.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                 "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1.0)
        d[row["Metric Name"]] = v * scale
    out = {}
    for lid in sorted(launches):           # later launches overwrite: the second count's
        d = launches[lid]
        kind = "dense" if "k_count_dense" in d["kernel"] else "list"
        out[kind] = {"dram_bytes": d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0),
                     "dram_read_bytes": d.get("dram__bytes_read.sum", 0),
                     "ncu_ms": d.get("gpu__time_duration.sum"), "l2_hit_pct": d.get("lts__t_sector_hit_rate.pct"),
                     "warp_inst": d.get("smsp__inst_executed.sum"),
                     "l1tex_pct": d.get("l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
                     "l2_pct": d.get("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                     "issue_active_pct": d.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                     "launch_id": lid}
    return out, "ncu " + " ".join(cmd[1:9])


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


def oracle_full_pass(og, pieces):
    """One full node-iterator count by the oracle, as `pieces` contiguous row ranges of
    equal edge count (a partition of the rows: nothing extrapolated).  Returns
    (triangles, per-piece seconds).  Strided row samples were measured to inflate the
    time by 1.4-2x (cache locality, serial tails)."""
    row, _ = og.csr()
    K = max(1, pieces)
    cuts = np.searchsorted(row, np.linspace(0, og.m, K + 1), side="left").astype(np.int64)
    cuts[0], cuts[-1] = 0, og.n
    cuts = np.maximum.accumulate(cuts)
    del row
    times, tri = [], 0
    for k in range(K):
        t1 = time.perf_counter()
        tri += og.count_rows(int(cuts[k]), int(cuts[k + 1]), 1)[0]
        times.append(time.perf_counter() - t1)
    return tri, times, cuts


def cpu_baseline(cfg, s, d, pieces=20):
    """The oracle as it stands, on the box's host cores, over the WHOLE workload (not
    extrapolated): oracle build (canonicalise, rank, orient) + one full node-iterator
    count — the same measurement as the reference arm (`--impl reference`, K = 20 steps).
    edges/s = m / (build + count), like the GPU step (a1-a7)."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    og = oracle.OracleGraph(s, d, cfg.n_hint)
    t_build = time.perf_counter() - t0
    tri, times, _ = oracle_full_pass(og, pieces)
    m = og.m
    del og
    t_count = sum(times)
    return {"value": m / (t_build + t_count), "unit": "edges/s", "cores": cores, "kind": "oracle",
            "sample": f"{cfg.name}: the whole workload, not extrapolated: oracle build ({t_build:.2f} s) + one full "
                      f"node-iterator count as {pieces} row ranges of equal edge count ({t_count:.2f} s) on "
                      f"{cores} threads (the reference arm's measurement)",
            "t_build_s": t_build, "t_count_s": t_count, "triangles": tri}


def run_reference(args):
    """--impl reference: the oracle (this tier has no reference code), rank 0 only.
    The oracle graph is built once (timed); the K timed steps are K contiguous row
    ranges of equal edge count — a partition of the rows, so the K steps together are
    exactly one full node-iterator count (nothing extrapolated; strided row samples
    were measured to inflate the time by 1.4-2x: cache locality and serial tails).
    value = m / (build + sum of the K step times); W warm-up steps repeat pieces untimed."""
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
    del s, d
    K = max(1, args.steps)
    if args.warmup:   # untimed: the first min(W, K) pieces
        row, _ = og.csr()
        wc = np.searchsorted(row, np.linspace(0, og.m, K + 1), side="left").astype(np.int64)
        wc[0], wc[-1] = 0, og.n
        del row
        for w in range(min(args.warmup, K)):
            og.count_rows(int(wc[w]), int(max(wc[w], wc[w + 1])), 1)
    tri, times, _ = oracle_full_pass(og, K)
    t_all = t_build + sum(times)
    v = og.m / t_all
    sample = (f"{cfg.name}: the whole workload as {K} contiguous row ranges of equal edge count (one full "
              f"node-iterator count, {sum(times):.2f} s) + oracle build once ({t_build:.2f} s), {cores} threads")
    line = {"metric": METRIC, "impl": "reference", "value": v, "unit": "edges/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_all / K * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": cfg.name, "desc": cfg.desc, "p": args.p or cfg.p, "seed": args.seed,
                       "l2": "inputs larger than L2 (CPU run)"},
            "e2e": {"value": v, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "cpu_baseline": {"value": v, "unit": "edges/s", "cores": cores, "kind": "oracle", "sample": sample},
            "triangles": int(tri), "step_s": times, "t_build_s": t_build, "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def main_sharded(args, world, rank, local):
    """N > 1: the §8(e) sharded step.  Every rank starts from its own 1/N
    of the raw edges (generated for its sample range) resident in its HBM; a step =
    sharded a1-a5 (two all-to-alls, two all-reduces, block forwarding over NVLink) +
    this rank's tasks + one all-reduce of the per-task counters.  Time = max over ranks
    of the CUDA-event step time; value = m / time (whole job)."""
    import torch
    import torch.distributed as dist

    import paper_2009_12457_b200 as bb
    from paper_2009_12457_b200.dist import build_sharded, count_owner_h2d, max_over_ranks, reduce_counts
    cfg = inputs.CONFIGS[args.config]
    p = args.p or cfg.p
    # At least 8 tasks per rank (unless --p is given): friendster's p = 4 has 20 tasks, whose
    # best split over 8 ranks is 1.42x the mean load (scripts/balance_study.py).
    while not args.p and bb.n_tasks(p) < 8 * world:
        p += 1
    a, b = cfg.shard(rank, world)
    E = b - a
    hs = torch.empty(max(E, 1), dtype=torch.int32, pin_memory=True)[:E]
    hd = torch.empty(max(E, 1), dtype=torch.int32, pin_memory=True)[:E]
    t0 = time.perf_counter()
    cfg.generate_range(a, E, seed=args.seed, out=(hs.numpy().view(np.uint32), hd.numpy().view(np.uint32)))
    t_gen = time.perf_counter() - t0
    ds = hs.to("cuda", non_blocking=True)
    dd = hd.to("cuda", non_blocking=True)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = bb.Context(local, stream=stream.cuda_stream)
    nt = bb.n_tasks(p)
    counts = torch.zeros(nt + 1, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    kern_ms, infos = [], []

    def step(src, dst, record):
        g, plan, info = build_sharded(ctx, src, dst, cfg.n_hint, p)
        a_, b_ = ev(), ev()
        a_.record(stream)
        plan.count_async(counts, rank, world)
        b_.record(stream)
        reduce_counts(counts)
        tot = int(counts[-1].item())
        if record:
            kern_ms.append(a_.elapsed_time(b_))
            infos.append(info)
        return tot, g, plan, info

    for _ in range(args.warmup):
        tot, g, plan, info = step(ds, dd, False)
        plan.close()
        g.close()
    dist.barrier()
    torch.cuda.synchronize()
    l0 = ctx.launches
    with Clocks(local) as clk:
        s0, s1 = ev(), ev()
        s0.record(stream)
        for _ in range(args.steps):
            tot, g, plan, info = step(ds, dd, True)
            plan.close()
            g.close()
        s1.record(stream)
        torch.cuda.synchronize()
    launches = (ctx.launches - l0) // args.steps
    ms = s0.elapsed_time(s1) / args.steps
    dist.barrier()
    ms = max_over_ranks(ms, device="cuda")
    m = infos[-1]["m"]
    value = m / (ms / 1e3)
    kern = max_over_ranks(statistics.mean(kern_ms), device="cuda")
    # e2e: the share in pinned host memory -> H2D inside the step -> counters on the host
    e2e_ms = []
    for x in range(args.e2e_steps + 1):
        torch.cuda.synchronize()
        dist.barrier()
        a_, b_ = ev(), ev()
        a_.record(stream)
        g, plan, info = build_sharded(ctx, hs.numpy().view(np.uint32), hd.numpy().view(np.uint32), cfg.n_hint, p)
        plan.count_async(counts, rank, world)
        reduce_counts(counts)
        host_counts = counts.cpu()
        b_.record(stream)
        torch.cuda.synchronize()
        assert int(host_counts[-1]) == tot
        h2d_rank = info["h2d_bytes"]
        plan.close()
        g.close()
        if x:
            e2e_ms.append(a_.elapsed_time(b_))
    e2e = max_over_ranks(statistics.median(e2e_ms), device="cuda")
    # The paper's split on the shard plans: excl. = blocks resident (the count of
    # this rank's tasks + the all-reduce); incl. = blocks in pinned host memory, each copied
    # H2D once by its owner and forwarded over NVLink to the ranks that read it
    # (dist.count_owner_h2d), then counted.  CUDA-event times, max over ranks.
    g, plan, info = build_sharded(ctx, ds, dd, cfg.n_hint, p)
    t_x, t_i = [], []
    for x in range(6):
        dist.barrier()
        a_, b_ = ev(), ev()
        a_.record(stream)
        plan.count_async(counts, rank, world)
        reduce_counts(counts)
        b_.record(stream)
        torch.cuda.synchronize()
        if x:
            t_x.append(a_.elapsed_time(b_))
    plan.to_host()
    for x in range(6):
        plan.unstage()
        torch.cuda.synchronize()
        dist.barrier()
        a_, b_ = ev(), ev()
        a_.record(stream)
        h2d_blocks, _ = count_owner_h2d(ctx, plan, info, counts)
        b_.record(stream)
        torch.cuda.synchronize()
        assert int(counts[-1].item()) == tot
        if x:
            t_i.append(a_.elapsed_time(b_))
    plan.close()
    g.close()
    t_excl = max_over_ranks(statistics.median(t_x), device="cuda")
    t_incl = max_over_ranks(statistics.median(t_i), device="cuda")
    per_rank = {"h2d_raw_bytes": h2d_rank, "h2d_block_bytes": h2d_blocks,
                "nvlink_bytes_recv": info["nvlink_bytes_recv"], "nvlink_bytes_sent": info["nvlink_bytes_sent"],
                "tasks": info["tasks_here"], "build_ms": info["times_ms"], "count_kernel_ms": statistics.mean(kern_ms),
                "t_excl_ms": statistics.median(t_x), "t_incl_ms": statistics.median(t_i)}
    gathered = [None] * world
    dist.all_gather_object(gathered, per_rank)
    line = {
        "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": cfg.name, "desc": cfg.desc, "p": p, "seed": args.seed, "raw_edges": cfg.n_samples,
                   "n": infos[-1]["n"], "m": m, "tasks": nt,
                   "parallelism": f"sharded a1-a5 + tasks by LPT/block affinity over {world} ranks",
                   "l2": "inputs larger than L2 (no flush needed)"},
        "e2e": {"value": m / (e2e / 1e3), "unit": "edges/s", "ms_per_step": e2e,
                "h2d_bytes_per_step": 8 * cfg.n_samples, "h2d_bytes_per_rank": 8 * E,
                "d2h_bytes_per_step": 8 * (nt + 1) * world},
        "gpu_launches": launches, "count_kernel_ms_max": kern, "clocks": clk.summary(), "triangles": tot,
        "per_rank": gathered, "gen_s": t_gen,
        "paper_split": {"note": "count only: excl = shard plans resident (this rank's tasks + all-reduce); incl = "
                                "blocks in pinned host memory, each copied H2D once by its owner and forwarded over "
                                "NVLink (P:37-40, DESIGN 9). Median of 5 after a warm-up, max over ranks.",
                        "t_excl_ms": t_excl, "t_incl_ms": t_incl, "edges_per_s_excl": m / (t_excl / 1e3),
                        "edges_per_s_incl": m / (t_incl / 1e3),
                        "h2d_bytes_total": sum(r["h2d_block_bytes"] for r in gathered)},
        "roofline": {"bound": "hbm", "kernel": "k_count", "note": "ncu traffic is captured at N=1 only",
                     "achieved": None, "peak": load_peaks()[0], "unit": "GB/s", "frac": None, "traffic": None},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


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
        return main_sharded(args, world, rank, local)
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
        st = None if record else g.stats()   # (stats computes d+_max: kept out of the timed steps)
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
            tot, info, _ = step(ds, dd, True)
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
    # Out of core: the device may hold only half of the blocks (or just the
    # largest task's three blocks where that is more: small p).
    plan.unstage()
    ooc_budget = max(pinfo["block_bytes"] // 2, int(pinfo["max_task_bytes"] * 1.05))
    plan.set_budget(ooc_budget)
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

    t_list = statistics.median(r[2]["t_kernel_ms"] - r[2]["t_dense_ms"] for r in reps_x)
    t_dense = statistics.median(r[2]["t_dense_ms"] for r in reps_x)
    del ds, dd
    torch.cuda.synchronize()
    ctx.close()
    torch.cuda.empty_cache()

    peak, peak_src = load_peaks()
    # Roofline of the dominant kernel (the list kernel), physical: DRAM bytes per launch
    # measured by ncu in this run / the launch's CUDA-event time (median of the 5 counts
    # above) / the measured HBM peak.  compulsory_* = the bytes the kernel must read at
    # least once (the distinct blocks it reads; for the bit-row kernel the bit rows and
    # its G_ij iteration arrays); b_alg_* = SURVEY 8(d)'s logical bytes (Alg. 5 reading
    # both lists of every edge), which staged-list reuse and bit rows undercut.
    traffic, traffic_src = (None, "skipped (N>1: ncu on one GPU only)")
    if rank == 0 and world == 1 and not args.no_ncu:
        traffic, traffic_src = live_traffic(cfg, p, args.seed)

    def kern_roof(kind, t_ms, compulsory, b_alg=None):
        tr = (traffic or {}).get(kind) if traffic else None
        d = {"kernel_ms": t_ms, "compulsory_bytes": compulsory,
             "compulsory_GBps": compulsory / (t_ms / 1e3) / 1e9 if t_ms > 0 else None}
        d["compulsory_frac"] = d["compulsory_GBps"] / peak if t_ms > 0 else None
        if tr:
            d.update({"traffic": tr["dram_bytes"], "achieved": tr["dram_bytes"] / (t_ms / 1e3) / 1e9,
                      "l2_hit_pct": tr["l2_hit_pct"], "ncu_ms_cold_serialised": tr["ncu_ms"],
                      "traffic_over_compulsory": tr["dram_bytes"] / compulsory if compulsory else None})
            d["frac"] = d["achieved"] / peak
            # the other limits the kernel runs into (ncu, same launch): warp instructions
            # issued per second of the CUDA-event time against the SMs x 4 schedulers x the
            # measured SM clock, and ncu's L1/TEX and L2 throughput fractions
            sm_mhz = (clk.summary() or {}).get("sm_mhz") or 1965.0
            if tr.get("warp_inst"):
                peak_issue = torch.cuda.get_device_properties(local).multi_processor_count * 4 * sm_mhz * 1e6
                d["issue"] = {"warp_inst": tr["warp_inst"], "rate": tr["warp_inst"] / (t_ms / 1e3),
                              "peak": peak_issue, "frac": tr["warp_inst"] / (t_ms / 1e3) / peak_issue,
                              "ncu_issue_active_pct": tr.get("issue_active_pct")}
            d["ncu_l1tex_pct"] = tr.get("l1tex_pct")
            d["ncu_l2_pct"] = tr.get("l2_pct")
        if b_alg is not None:
            d["b_alg_bytes"] = b_alg
            d["b_alg_logical_frac"] = b_alg / (t_ms / 1e3) / 1e9 / peak if t_ms > 0 else None
        return d

    lst = kern_roof("list", t_list, dinfo["list_read_bytes"], pinfo["b_alg"] / world)
    dns = kern_roof("dense", t_dense, dinfo["dense_bytes"] + dinfo["dense_edge_bytes"])
    line = {
        "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": cfg.name, "desc": cfg.desc, "p": p, "seed": args.seed, "raw_edges": E,
                   "n": st["n"], "m": m, "d_max": st["d_max"], "dplus_max": st["dplus_max"], "tasks": nt,
                   "parallelism": f"tasks/{world}",
                   "l2": "inputs larger than L2 (no flush needed)"},
        "e2e": {"value": m / (e2e / 1e3), "unit": "edges/s", "ms_per_step": e2e,
                "h2d_bytes_per_step": 8 * E, "d2h_bytes_per_step": 8 * (nt + 1)},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": "k_count (list kernel, sparse tasks)", "unit": "GB/s", "peak": peak,
                     "achieved": lst.get("achieved"), "frac": lst.get("frac"), "traffic": lst.get("traffic"),
                     "compulsory_frac": lst["compulsory_frac"], "peak_source": peak_src,
                     "traffic_source": traffic_src, "kernels": {"list": lst, "dense": dns},
                     "note": "physical: achieved = ncu DRAM bytes (read+write) per launch, measured in this run, "
                             "/ the launch's CUDA-event time; compulsory_frac = distinct bytes the kernel must read "
                             "/ time / peak; b_alg_logical_frac = SURVEY 8(d) B_alg / time / peak (logical, can "
                             "exceed 1); kernels.*.issue = warp instructions per launch / its event time vs SMs x 4 "
                             "schedulers x the sampled SM clock, ncu_l1tex_pct / ncu_l2_pct = ncu throughput "
                             "fractions of the same launch: the list kernel's limits where L2 serves most sectors "
                             "(DESIGN 8)."},
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
                         "count_list_kernel": t_list, "count_dense_kernel": t_dense,
                         "dense_tasks": dinfo["dense_tasks"], "dense_bit_row_bytes": dinfo["dense_bytes"],
                         "count_excl_h2d": statistics.median(t_x), "count_incl_h2d": statistics.median(t_i),
                         "h2d_bytes_blocks": tm_i["h2d_bytes"],
                         "count_out_of_core_half_budget": tm_o["t_total_ms"], "h2d_bytes_out_of_core": tm_o["h2d_bytes"],
                         "out_of_core_budget_bytes": ooc_budget,
                         "gen_s": t_gen},
        "plan": {"lambda": pinfo["lambda"], "dmax_blk": pinfo["dmax_blk"], "visits": pinfo["visits"],
                 "b_alg": pinfo["b_alg"], "work_items": pinfo["work_items"], "block_bytes": pinfo["block_bytes"],
                 "slot_bytes": pinfo.get("slot_bytes", 0)},
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
