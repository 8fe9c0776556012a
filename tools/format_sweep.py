"""Per-format kernel throughput on the BASELINE configs (SURVEY §8(d) pass bar:
every format >= 70% of HBM roofline on its best-suited matrix).

For each config and format: convert (c_latency), launch-tune that format
(spmv_tune LAUNCH), then time the tuned kernel with CUDA events (alpha=1,
beta=0, median of 5 batches) and report GB/s over the algorithmic bytes
(format stored bytes + x + y), the fraction of the measured HBM peak and
GFLOP/s. Writes JSON + a markdown table."""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2302_05662_b200 as P  # noqa: E402
import spmv_inputs as si  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0

VARIANTS = [("CSR-vector", P.FMT_CSR, dict(csr_alg=P.CSR_VECTOR)),
            ("CSR-merge", P.FMT_CSR, dict(csr_alg=P.CSR_MERGE)),
            ("CSR-stream", P.FMT_CSR, dict(csr_alg=P.CSR_STREAM)),
            ("ELL", P.FMT_ELL, dict(index16=0)),
            ("ELL-16", P.FMT_ELL, dict(index16=1)),
            ("ELL-8", P.FMT_ELL, dict(index16=2)),
            ("SELL", P.FMT_SELL, dict(index16=0)),
            ("SELL-16", P.FMT_SELL, dict(index16=1)),
            ("SELL-8", P.FMT_SELL, dict(index16=2)),
            ("SELL-sigma", P.FMT_SELL, dict(sell_sigma=-1)),
            ("HYB", P.FMT_HYB, {}),
            ("COO", P.FMT_COO, {}),
            ("BELL-2", P.FMT_BELL, dict(bell_b=2)),
            ("BELL-3", P.FMT_BELL, dict(bell_b=3))]


def time_kernel(h, fmt, x, y, reps=None):
    s = torch.cuda.current_stream()
    for _ in range(3):
        P.spmv_run(h, 1.0, x, 0.0, y, fmt=fmt)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    P.spmv_run(h, 1.0, x, 0.0, y, fmt=fmt)
    e1.record(s)
    torch.cuda.synchronize()
    one = e0.elapsed_time(e1)
    reps = reps or max(5, min(500, int(20.0 / max(one, 1e-3))))
    ts = []
    for _ in range(5):
        e0.record(s)
        for _ in range(reps):
            P.spmv_run(h, 1.0, x, 0.0, y, fmt=fmt)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / reps)
    return statistics.median(ts) * 1e-3


# Extra matrices for the "best-suited matrix" pass bar: each
# family's large member, every format measured on every one of them, all
# arrays > L2 (126 MB).
EXTRA = {
    # short regular rows (5 per row): COO's entry-order gathers stay within 3 x lines per 32 entries
    "lap2d_4096": lambda: si.stencil_device(si.LAP2D, 4096, random_values=True),
    # long contiguous rows (64 per row): warp-per-row CSR-vector reads whole lines of col/val and x
    "band64_2M": lambda: si.dense_band(1 << 21, 32),
    # short/long-row mix (5-point rows + every 2048th row with 2048 more local entries): HYB / merge-path
    "lap2d_long_4096": lambda: si.lap2d_long_rows(4096, 2048, 2048),
}


def load(name):
    if name in EXTRA:
        coo = EXTRA[name]()
        return coo
    return si.config_device(name)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4", help="BASELINE configs and/or " + ",".join(EXTRA))
    ap.add_argument("--out", default="gpurun_out/format_sweep")
    ap.add_argument("--no-tune", action="store_true")
    ap.add_argument("--formats", default="", help="comma list of variant names (default all)")
    args = ap.parse_args()
    results = []
    for cfg in args.configs.split(","):
        coo = load(cfg)
        if isinstance(coo.val, np.ndarray):
            coo = si.COO(coo.rows, coo.cols, torch.from_numpy(coo.row).cuda(), torch.from_numpy(coo.col).cuda(),
                         torch.from_numpy(coo.val).cuda())
        dt = coo.val.dtype
        vb = 4 if dt == torch.float32 else 8
        x = si.vector_device(coo.cols, dtype=dt)
        y = torch.empty(coo.rows, dtype=dt, device="cuda")
        h = P.spmv_create(coo.rows, coo.cols, coo.row, coo.col, coo.val)
        feats = P.spmv_features(h)
        del coo
        torch.cuda.empty_cache()
        for name, fmt, params in VARIANTS:
            if args.formats and name not in args.formats.split(","):
                continue
            if name.startswith("BELL") and (feats["std"] > feats["mean"] or feats["mean"] < 4):
                continue  # block formats only make sense on block-structured matrices
            params = dict(params)
            if params.get("sell_sigma") == -1:
                if feats["std"] <= 0.5 * feats["mean"]:
                    continue  # sorting only matters for skewed rows
                C = 128 if vb == 4 else 64
                params["sell_sigma"] = C * 512
            rec = {"config": cfg, "format": name, "dtype": "f32" if vb == 4 else "f64", "n": feats["n_rows"],
                   "nnz": feats["nnz"]}
            try:
                P.spmv_convert(h, fmt, **params)
            except P.SpmvError as e:
                rec["error"] = str(e)[:160]
                results.append(rec)
                print(json.dumps(rec), flush=True)
                continue
            _, c_lat = P.spmv_overheads(h)
            info = P.spmv_format_info(h, fmt)
            if not args.no_tune:
                P.spmv_tune(h, P.TUNE_LAUNCH, 1000)
            launch = P.spmv_get_launch(h, fmt)
            t = time_kernel(h, fmt, x, y)
            alg = info["stored_bytes"] + feats["n_cols"] * vb + feats["n_rows"] * vb
            csr_min = (feats["n_rows"] + 1) * 4 + feats["nnz"] * (4 + vb) + feats["n_cols"] * vb + feats["n_rows"] * vb
            rec.update({"launch": launch, "t_us": round(t * 1e6, 2), "alg_bytes": alg,
                        "GBps": round(alg / t / 1e9, 1), "frac_measured_peak": round(alg / t / 1e9 / PEAK, 4),
                        "frac_8TBs": round(alg / t / 1e9 / 8000, 4), "useful_GBps": round(csr_min / t / 1e9, 1),
                        "GFLOPs": round(2 * feats["nnz"] / t / 1e9, 1),
                        "c_latency_ms": round(c_lat[P.FORMAT_NAMES[fmt]] * 1e3, 3),
                        "padding": (round(1 - feats["nnz"] / info["slots"], 4)
                                    if info["slots"] and fmt in (P.FMT_ELL, P.FMT_SELL, P.FMT_BELL) else None)})
            results.append(rec)
            print(json.dumps(rec), flush=True)
            if fmt not in (P.FMT_CSR,):
                P.spmv_convert(h, P.FMT_CSR)  # keep memory bounded: rebuild formats per variant
        f_lat, _ = P.spmv_overheads(h)
        results.append({"config": cfg, "features": feats, "f_latency_ms": round(f_lat * 1e3, 3)})
        P.spmv_destroy(h)
        P.lib().spmv_trim_pool(0)
        torch.cuda.empty_cache()
    json.dump(results, open(args.out + ".json", "w"), indent=1)
    lines = ["| config | format | dtype | launch (block,maxreg,carve,knob) | µs | GB/s (alg) | frac of measured peak | frac of 8 TB/s | useful GB/s | GFLOP/s | padding | c_latency ms |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in results:
        if "format" not in r:
            continue
        if "error" in r:
            lines.append(f"| {r['config']} | {r['format']} | {r['dtype']} | — | infeasible: {r['error'][:60]} | | | | | | | |")
            continue
        lines.append(f"| {r['config']} | {r['format']} | {r['dtype']} | {tuple(r['launch'])} | {r['t_us']} | {r['GBps']} | "
                     f"{r['frac_measured_peak']:.3f} | {r['frac_8TBs']:.3f} | {r['useful_GBps']} | {r['GFLOPs']} | "
                     f"{r['padding']} | {r['c_latency_ms']} |")
    open(args.out + ".md", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
