"""ncu DRAM traffic of the SpMV kernels, per launch, keyed by the exact kernel
label the bench reports (profiles/ncu_traffic_<cfg>.json; SURVEY §8(d) "ncu
evidence for each (config, format, best variant)").

For each label: tools/kernel_one.py runs the format (launch-tuned, or the
given launch) and brackets REPS SpMVs with cudaProfilerStart/Stop; ncu
(--profile-from-start off, --clock-control none) collects per kernel launch
dram__bytes_read/write, duration, L2 hit rate, L1TEX throughput and sectors
per request. Per label the launches of one SpMV (main kernel + helpers such as
the fixup) are summed; the x DRAM re-read factor is
(dram read − stored matrix bytes) / x bytes.

python tools/ncu_traffic.py c2 ELL-16 SELL-16 ELL [--out profiles/ncu_traffic_c2.json]
Runs on the GPU box (needs ncu and a GPU)."""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "lts__t_sector_hit_rate.pct",
           "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
           "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "launch__registers_per_thread",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed"]

# label -> kernel_one arguments
LABELS = {
    "ELL": ["ELL", "--index16", "0"], "ELL-16": ["ELL", "--index16", "1"], "ELL-8": ["ELL", "--index16", "2"],
    "SELL": ["SELL", "--index16", "0"], "SELL-16": ["SELL", "--index16", "1"], "SELL-8": ["SELL", "--index16", "2"],
    "CSR-vector": ["CSR", "--csr-alg", "2"], "CSR-merge": ["CSR", "--csr-alg", "3"],
    "CSR-stream": ["CSR", "--csr-alg", "4"], "COO": ["COO"], "HYB": ["HYB"],
    "BELL-2": ["BELL", "--bell-b", "2"], "BELL-3": ["BELL", "--bell-b", "3"],
}


def capture(cfg, label, reps=3, launch=""):
    args = [sys.executable, os.path.join(HERE, "kernel_one.py"), cfg] + LABELS[label] + [str(reps)]
    args += ["--launch", launch] if launch else ["--tune"]
    log = os.path.join(ROOT, "gpurun_out", f"ncu_{cfg}_{label}.csv")
    cmd = ["ncu", "--profile-from-start", "off", "--clock-control", "none", "--metrics", ",".join(METRICS), "--csv",
           "--log-file", log] + args
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1800)
    meta = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    rows = list(csv.DictReader(io.StringIO("".join(ln for ln in open(log) if ln.startswith('"')))))
    launches = {}
    for row in rows:
        k = (row["ID"], row["Kernel Name"])
        launches.setdefault(k, {})[row["Metric Name"]] = float(row["Metric Value"].replace(",", "") or 0)
    # group the launches of one SpMV: REPS repetitions of the same kernel sequence
    seq = sorted(launches.items(), key=lambda kv: int(kv[0][0]))
    per = len(seq) // reps if reps else len(seq)
    one = seq[-per:] if per else seq
    tot = lambda m: sum(v.get(m, 0.0) for _, v in one)  # noqa: E731
    main = max(one, key=lambda kv: kv[1].get("gpu__time_duration.sum", 0.0))
    stored = meta["info"]["stored_bytes"]
    alg = stored + meta["x_bytes"] + meta["y_bytes"]
    dram = tot("dram__bytes_read.sum") + tot("dram__bytes_write.sum")
    req = main[1].get("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", 0.0)
    return {"label": label, "launch": meta["launch"], "kernels": [k[1] for k, _ in one],
            "dram_bytes_per_launch": int(dram), "dram_read": int(tot("dram__bytes_read.sum")),
            "dram_write": int(tot("dram__bytes_write.sum")), "alg_bytes": int(alg),
            "traffic_over_alg": round(dram / alg, 4) if alg else None,
            "x_reread_factor": round((tot("dram__bytes_read.sum") - stored) / meta["x_bytes"], 3),
            "duration_us_ncu": round(tot("gpu__time_duration.sum") / 1e3, 2),
            "main_kernel": main[0][1], "main_duration_us_ncu": round(main[1]["gpu__time_duration.sum"] / 1e3, 2),
            "l2_hit_pct": main[1].get("lts__t_sector_hit_rate.pct"),
            "l1tex_pct": main[1].get("l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
            "dram_pct": main[1].get("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
            "sectors_per_request": round(main[1].get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", 0) / req, 2)
            if req else None,
            "registers": main[1].get("launch__registers_per_thread"),
            "source": "ncu --clock-control none, cold-cache serialised replay (times are not bench values)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("labels", nargs="+")
    ap.add_argument("--out", default="")
    ap.add_argument("--launch", default="", help="label=b,r,c,k;label=...")
    a = ap.parse_args()
    launches = dict(kv.split("=") for kv in a.launch.split(";") if kv)
    out = os.path.join(ROOT, "profiles", f"ncu_traffic_{a.config}.json") if not a.out else a.out
    res = json.load(open(out)) if os.path.exists(out) else {}
    res = {k: v for k, v in res.items() if isinstance(v, dict) and "label" in v}  # drop legacy layouts
    for lab in a.labels:
        try:
            res[lab] = capture(a.config, lab, launch=launches.get(lab, ""))
        except Exception as ex:  # report, keep going
            res[lab] = {"label": lab, "error": repr(ex)[:300]}
        print(a.config, json.dumps(res[lab]), flush=True)
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
