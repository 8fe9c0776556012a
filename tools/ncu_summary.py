"""Summarise ncu outputs into profiles/ (tracked):
  python tools/ncu_summary.py launches <launches.csv> <out.md>
  python tools/ncu_summary.py full <report.ncu-rep> <config> <format> <alg_bytes> <out_prefix>
The `full` mode also writes profiles/ncu_traffic_<config>.json, which bench.py
reads for the roofline `traffic` field (DRAM bytes per launch)."""
import collections
import csv
import io
import json
import subprocess
import sys

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= max(ki, vi, ui):
            continue
        name = r[ki]
        short = name.split("(")[0].replace("void ", "")
        us = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    lines = ["| kernel | launches | total µs | share | avg µs |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f}% | {t / n:.2f} |")
    lines.append(f"| **total** | {sum(a[0] for a in agg.values())} | {tot:.1f} | 100% | |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__occupancy_limit_registers", "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "local_load_bytes"]


def full(rep, config, fmt, alg_bytes, prefix):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    launches_ = []
    for r in rows[2:]:
        d = {}
        for i, n in enumerate(h):
            if n in WANT or n == "Kernel Name":
                d[n] = (r[i], units[i])
        launches_.append(d)

    def val(d, k):
        v, u = d.get(k, ("nan", ""))
        x = float(v.replace(",", "")) if v not in ("", "n/a") else float("nan")
        mult = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}.get(u, 1.0)
        if k == "gpu__time_duration.sum":
            mult = SCALE.get(u, 1.0)
        return x * mult

    traffic = [val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum") for d in launches_]
    times = [val(d, "gpu__time_duration.sum") for d in launches_]
    mean_t = sum(traffic) / len(traffic)
    summary = {"config": config, "format": fmt, "report": rep, "launches": len(launches_),
               "dram_bytes_per_launch": mean_t, "alg_bytes_per_launch": float(alg_bytes),
               "traffic_over_alg": mean_t / float(alg_bytes), "duration_us": times,
               "dram_GBps_under_ncu": [t / (u * 1e-6) / 1e9 for t, u in zip(traffic, times)],
               "metrics": [{k: " ".join(v) for k, v in d.items()} for d in launches_]}
    json.dump(summary, open(f"{prefix}.json", "w"), indent=1)
    # per-config traffic file, one entry per format label (bench.py reads its own)
    tpath = f"profiles/ncu_traffic_{config}.json"
    try:
        tj = json.load(open(tpath))
    except (OSError, ValueError):
        tj = {}
    if "format" in tj:  # legacy single-format layout
        tj = {tj["format"]: {"dram_bytes_per_launch": tj["dram_bytes_per_launch"], "source": tj.get("source")}}
    tj[fmt] = {"dram_bytes_per_launch": mean_t, "source": rep}
    json.dump(tj, open(tpath, "w"), indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "metrics"}, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(*sys.argv[2:7])
