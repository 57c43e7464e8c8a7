"""Summarise an ncu report (raw metrics + top SASS lines by stall samples) as JSON/text.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json] [--top 25]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "sm__maximum_warps_per_active_cycle_pct", "launch__grid_size"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")][:80]}
        for k in KEYS:
            if k in h:
                d[k] = r[h.index(k)]
                d[k + ".unit"] = units[h.index(k)]
        res.append(d)
    return res


def sass_top(rep, top):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ie, src, smp = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")

    def num(x):
        try:
            float(x or 0)
            return True
        except ValueError:
            return False
    # several kernels: their tables are concatenated (header rows repeat); pool the lines
    data = [r for r in rows[2:] if len(r) > smp and num(r[smp])]
    tot = sum(float(r[smp] or 0) for r in data)
    order = sorted(range(len(data)), key=lambda i: -float(data[i][smp] or 0))[:top]
    return [{"idx": i, "sass": data[i][src].strip(), "inst": data[i][ie],
             "stall_pct": round(100 * float(data[i][smp] or 0) / max(tot, 1), 2)} for i in order]


if __name__ == "__main__":
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
    summary = {"report": rep, "launches": raw(rep), "top_stalls": sass_top(rep, top)}
    if "--traffic" in sys.argv:
        # profiles/ncu_count_<config>.json for bench.py: DRAM bytes of ONE count (the
        # report must hold exactly one k_count and at most one k_count_dense launch).
        cfg, out = sys.argv[sys.argv.index("--traffic") + 1: sys.argv.index("--traffic") + 3]
        ks = [L for L in summary["launches"] if "k_count" in L["kernel"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        b = lambda L, k: float(L[k]) * scale[L[k + ".unit"]]  # noqa: E731
        rd = sum(b(L, "dram__bytes_read.sum") for L in ks)
        wr = sum(b(L, "dram__bytes_write.sum") for L in ks)
        ms = sum(float(L["gpu__time_duration.sum"]) * (1e-3 if L["gpu__time_duration.sum.unit"] == "us" else 1)
                 for L in ks)
        with open(out, "w") as f:
            json.dump({"config": cfg, "kernel": " + ".join(L["kernel"][:60] for L in ks), "source": rep,
                       "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
                       "duration_ms_ncu": ms,
                       "per_kernel": [{k: L[k] for k in L} for L in ks]}, f, indent=1)
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(summary, f, indent=1)
    for L in summary["launches"]:
        for k, v in L.items():
            if not k.endswith(".unit"):
                print(f"{k:60s} {v} {L.get(k + '.unit', '')}")
    for s in summary["top_stalls"]:
        print(f"{s['stall_pct']:6.2f}% {s['inst']:>12s}  {s['sass']}")
