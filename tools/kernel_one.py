"""Run one format's SpMV kernel on a config N times (for ncu captures).
python tools/kernel_one.py c3 COO 8 [--launch 64,128,0,8] [--csr-alg 3]"""
import argparse
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
a = ap.parse_args()
coo = si.config_device(a.config)
x = si.vector_device(coo.cols, dtype=coo.val.dtype)
y = torch.empty(coo.rows, dtype=coo.val.dtype, device="cuda")
h = P.spmv_create(coo.rows, coo.cols, coo.row, coo.col, coo.val)
fmt = P.FORMATS[a.format]
kw = {}
if fmt == P.FMT_CSR:
    kw["csr_alg"] = a.csr_alg
if fmt == P.FMT_SELL and a.sigma:
    kw["sell_sigma"] = a.sigma
P.spmv_convert(h, fmt, **kw)
if a.launch:
    P.spmv_set_launch(h, fmt, *[int(v) for v in a.launch.split(",")])
for _ in range(a.reps):
    P.spmv_run(h, 1.0, x, 0.0, y)
torch.cuda.synchronize()
print(P.FORMAT_NAMES[fmt], P.spmv_get_launch(h, fmt), P.spmv_format_info(h, fmt))
P.spmv_destroy(h)
