"""Run one format's SpMV kernel on a config N times (for ncu captures).

python tools/kernel_one.py c3 COO 8 [--launch 64,128,0,8] [--csr-alg 3] [--index16 1] [--tune]
The SpMV launches are bracketed by cudaProfilerStart/Stop, so
`ncu --profile-from-start off` sees only them (not generation, conversion
or tuning). Prints the format, launch and format info as one JSON line."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2302_05662_b200 as P  # noqa: E402
import spmv_inputs as si  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("format")
ap.add_argument("reps", type=int)
ap.add_argument("--launch", default="")
ap.add_argument("--csr-alg", type=int, default=0)
ap.add_argument("--sigma", type=int, default=0)
ap.add_argument("--index16", type=int, default=-1)
ap.add_argument("--bell-b", type=int, default=0)
ap.add_argument("--tune", action="store_true", help="launch-tune the format first (outside the profiled range)")
a = ap.parse_args()
coo = si.config_device(a.config)
x = si.vector_device(coo.cols, dtype=coo.val.dtype)
y = torch.empty(coo.rows, dtype=coo.val.dtype, device="cuda")
h = P.spmv_create(coo.rows, coo.cols, coo.row, coo.col, coo.val)
del coo
torch.cuda.empty_cache()
fmt = P.FORMATS[a.format]
kw = {}
if fmt == P.FMT_CSR:
    kw["csr_alg"] = a.csr_alg
if fmt == P.FMT_SELL and a.sigma:
    kw["sell_sigma"] = a.sigma
if fmt in (P.FMT_ELL, P.FMT_SELL):
    kw["index16"] = a.index16
if fmt == P.FMT_BELL and a.bell_b:
    kw["bell_b"] = a.bell_b
P.spmv_convert(h, fmt, **kw)
if a.launch:
    P.spmv_set_launch(h, fmt, *[int(v) for v in a.launch.split(",")])
elif a.tune:
    P.spmv_tune(h, P.TUNE_LAUNCH, 1000)
for _ in range(2):
    P.spmv_run(h, 1.0, x, 0.0, y)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(a.reps):
    P.spmv_run(h, 1.0, x, 0.0, y)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
info = P.spmv_format_info(h, fmt)
print(json.dumps({"format": P.FORMAT_NAMES[fmt], "launch": list(P.spmv_get_launch(h, fmt)), "info": info,
                  "n": int(y.numel()), "x_bytes": int(x.numel() * x.element_size()),
                  "y_bytes": int(y.numel() * y.element_size())}))
P.spmv_destroy(h)
