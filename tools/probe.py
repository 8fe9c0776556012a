"""Diagnostics (not part of the bench contract): per-mode kernel timings for
launch variants and a synced per-phase breakdown of one bench step."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2302_05662_b200 as P  # noqa: E402
import spmv_inputs as si  # noqa: E402


def timeit(fn, reps=200):
    s = torch.cuda.current_stream()
    for _ in range(5):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--formats", default="SELL,ELL")
    ap.add_argument("--launches", default="256,255,-1,0;512,64,0,0;256,128,-1,0;128,255,-1,0;1024,64,-1,0")
    args = ap.parse_args()
    coo = si.config_device(args.config)
    dt = coo.val.dtype
    x = si.vector_device(coo.cols, dtype=dt)
    y = torch.empty(coo.rows, dtype=dt, device="cuda")
    sums_prev = torch.zeros(2, dtype=torch.float64, device="cuda")
    sums = torch.zeros(2, dtype=torch.float64, device="cuda")
    out = {}
    # phase breakdown (synced)
    ph = {}
    torch.cuda.synchronize()
    t = time.perf_counter()
    h = P.spmv_create(coo.rows, coo.cols, coo.row, coo.col, coo.val)
    torch.cuda.synchronize(); ph["create"] = time.perf_counter() - t; t = time.perf_counter()
    P.spmv_features(h)
    torch.cuda.synchronize(); ph["features"] = time.perf_counter() - t; t = time.perf_counter()
    P.spmv_convert(h, P.FMT_SELL)
    torch.cuda.synchronize(); ph["convert_sell"] = time.perf_counter() - t; t = time.perf_counter()
    P.spmv_destroy(h)
    torch.cuda.synchronize(); ph["destroy"] = time.perf_counter() - t
    out["phases_ms_synced"] = {k: round(v * 1e3, 3) for k, v in ph.items()}
    f, c = P.spmv_overheads(h) if False else (None, None)
    h = P.spmv_create(coo.rows, coo.cols, coo.row, coo.col, coo.val)
    P.spmv_norm2(h, x, sums_prev)
    for fname in args.formats.split(","):
        fmt = P.FORMATS[fname]
        P.spmv_convert(h, fmt)
        for L in args.launches.split(";"):
            lv = [int(v) for v in L.split(",")]
            try:
                P.spmv_set_launch(h, fmt, *lv)
                t_run = timeit(lambda: P.spmv_run(h, 1.0, x, 0.0, y))
                t_pow = timeit(lambda: P.spmv_power_step(h, x, y, sums_prev, sums))
            except P.SpmvError as e:
                t_run = t_pow = str(e)
            out[f"{fname} {L}"] = {"run_us": t_run, "power_us": t_pow}
    P.spmv_destroy(h)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
