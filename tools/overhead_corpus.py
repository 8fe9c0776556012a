"""Warm conversion and feature-extraction latencies on the selector corpus
(the overhead estimators of the run-time mode, P:452,
fig:overhead_prediction P:461-516).

Round 1 stored one conversion per format, cold for the first build of each
kernel in the process (lazy module loading, e.g. 1.2 ms for a 5 K-entry ELL);
the overhead regressors fit to that did not generalise (CV R² ≤ 0.16). Here
every latency is the median of 3 warm repetitions:
  f_latency: 3 fresh handles, spmv_features each (device time of the kernels);
  c_latency(fmt): convert (auto column encoding, as the run-time mode
  converts), back to CSR, 3 times.
Writes one JSON record per matrix with the predictors the estimators use
(nnz, n_rows, ELL slots = n_pad·max_len) and each format's stored bytes.
python tools/overhead_corpus.py [--out gpurun_out/overhead_corpus.jsonl]"""
import argparse
import json
import os
import statistics
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2302_05662_b200 as P  # noqa: E402
from selector_corpus import corpus_specs  # noqa: E402

FORMATS = [("ELL", P.FMT_ELL, dict(index16=-1)), ("SELL", P.FMT_SELL, dict(index16=-1)), ("HYB", P.FMT_HYB, {}),
           ("COO", P.FMT_COO, {}), ("BELL-2", P.FMT_BELL, dict(bell_b=2)), ("BELL-3", P.FMT_BELL, dict(bell_b=3))]


def measure(name, coo):
    row = torch.from_numpy(coo.row).cuda()
    col = torch.from_numpy(coo.col).cuda()
    val = torch.from_numpy(np.asarray(coo.val, np.float64)).cuda()
    n = coo.rows
    f_lat = []
    feats = None
    for _ in range(4):
        h = P.spmv_create(n, coo.cols, row, col, val)
        feats = P.spmv_features(h)
        f_lat.append(P.spmv_overheads(h)[0])
        P.spmv_destroy(h)
    rec = {"name": name, "n": n, "nnz": int(coo.row.shape[0]), "features": feats,
           "f_latency_s": statistics.median(f_lat[1:]), "formats": {}}
    rec["ell_slots"] = (n + 127) // 128 * 128 * int(feats["max_len"])
    for vname, fmt, params in FORMATS:
        r = {}
        if vname.startswith("BELL") and (feats["mean"] < 4 or feats["std"] > feats["mean"]):
            r["skipped"] = "not block-like"
        elif fmt == P.FMT_ELL and rec["ell_slots"] > 4 * max(feats["nnz"], 1) + (1 << 20):
            r["skipped"] = "ELL padding > 4x nnz"
        if "skipped" not in r:
            try:
                lat = []
                for _ in range(4):  # a fresh handle per repetition: every conversion really builds
                    h = P.spmv_create(n, coo.cols, row, col, val)
                    try:
                        P.spmv_features(h)
                        P.spmv_convert(h, fmt, **params)
                        lat.append(P.spmv_overheads(h)[1][P.FORMAT_NAMES[fmt]])
                        info = P.spmv_format_info(h, fmt)
                    finally:
                        P.spmv_destroy(h)
                r["c_latency_s"] = statistics.median(lat[1:])
                r["c_latency_all_s"] = lat
                r["stored_bytes"] = info["stored_bytes"]
                r["index_bytes"] = info["index_bytes"]
            except P.SpmvError as e:
                r["error"] = str(e)[:160]
        rec["formats"][vname] = r
    P.lib().spmv_trim_pool(0)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "overhead_corpus.jsonl"))
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        for name, gen in corpus_specs():
            t0 = time.time()
            try:
                rec = measure(name, gen())
            except Exception as e:  # record and continue
                rec = {"name": name, "error": repr(e)[:200]}
            rec["wall_s"] = round(time.time() - t0, 2)
            f.write(json.dumps(rec) + "\n")
            f.flush()
            print(name, rec.get("nnz"), {k: v.get("c_latency_s") for k, v in rec.get("formats", {}).items()},
                  rec.get("f_latency_s"), flush=True)


if __name__ == "__main__":
    main()
