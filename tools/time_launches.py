"""Time one format's SpMV at explicit launch variants (CUDA events, median of 5).
python tools/time_launches.py c2 CSR --csr-alg 3 256,255,-1,264 128,255,50,8 ..."""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2302_05662_b200 as P  # noqa: E402
import spmv_inputs as si  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("format")
ap.add_argument("launches", nargs="+")
ap.add_argument("--csr-alg", type=int, default=0)
ap.add_argument("--index16", type=int, default=0)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
coo = si.config_device(a.config)
x = si.vector_device(coo.cols, dtype=coo.val.dtype)
y = torch.empty(coo.rows, dtype=coo.val.dtype, device="cuda")
h = P.spmv_create(coo.rows, coo.cols, coo.row, coo.col, coo.val)
fmt = P.FORMATS[a.format]
kw = {"csr_alg": a.csr_alg} if fmt == P.FMT_CSR else {}
if fmt in (P.FMT_ELL, P.FMT_SELL):
    kw["index16"] = a.index16
P.spmv_convert(h, fmt, **kw)
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for L in a.launches:
    try:
        P.spmv_set_launch(h, fmt, *[int(v, 0) for v in L.split(",")])
        for _ in range(3):
            P.spmv_run(h, 1.0, x, 0.0, y)
        ts = []
        for _ in range(5):
            e0.record(s)
            for _ in range(a.reps):
                P.spmv_run(h, 1.0, x, 0.0, y)
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / a.reps * 1e3)
        print(f"{a.config} {a.format} alg={a.csr_alg} launch={L}: {statistics.median(ts):.2f} us", flush=True)
    except P.SpmvError as ex:
        torch.cuda.synchronize()
        print(f"{a.config} {a.format} launch={L}: {ex}", flush=True)
P.spmv_destroy(h)
