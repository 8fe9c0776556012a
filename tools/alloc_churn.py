"""Does re-allocating the matrix every step change the SpMV kernel's speed?
(c5 bench steps create/convert/destroy 77 GB per step.)

A: one handle, E back-to-back plain SpMVs, 5 batches (CUDA events).
B: N steps of create -> convert -> the same E SpMVs -> destroy.
python tools/alloc_churn.py c5 ELL 2 --E 20 --steps 6 [--launch b,r,c,k]"""
import argparse
import json
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
ap.add_argument("index16", type=int)
ap.add_argument("--E", type=int, default=20)
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--launch", default="")
ap.add_argument("--trim", action="store_true", help="trim the pool after every destroy")
a = ap.parse_args()
coo = si.config_device(a.config)
x = si.vector_device(coo.cols, dtype=coo.val.dtype)
y = torch.empty(coo.rows, dtype=coo.val.dtype, device="cuda")
fmt = P.FORMATS[a.format]
kw = {"index16": a.index16} if fmt in (P.FMT_ELL, P.FMT_SELL) else {}
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def run_E(h):
    e0.record(s)
    for _ in range(a.E):
        P.spmv_run(h, 1.0, x, 0.0, y)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.E


def make():
    h = P.spmv_create(coo.rows, coo.cols, coo.row, coo.col, coo.val)
    P.spmv_convert(h, fmt, **kw)
    if a.launch:
        P.spmv_set_launch(h, fmt, *[int(v, 0) for v in a.launch.split(",")])
    return h


out = {"config": a.config, "format": a.format, "index16": a.index16, "E": a.E}
h = make()
run_E(h)
out["A_ms"] = [round(run_E(h), 4) for _ in range(5)]
P.spmv_destroy(h)
torch.cuda.synchronize()
B = []
for i in range(a.steps):
    h = make()
    run_E(h)  # warm
    B.append(round(run_E(h), 4))
    P.spmv_destroy(h)
    if a.trim:
        P.lib().spmv_trim_pool(0)
    torch.cuda.synchronize()
out["B_ms"] = B
print(json.dumps(out), flush=True)
