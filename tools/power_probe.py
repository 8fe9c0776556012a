"""Plain SpMV vs power step (fused Σz², Σx·z epilogue, device α, PDL) on the
same handle and launch: how much of the in-loop kernel time is the epilogue.
python tools/power_probe.py c5 ELL 2 --launch 512,64,0,65664 --E 20"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2302_05662_b200 as P  # noqa: E402
import spmv_inputs as si  # noqa: E402
from paper_2302_05662_b200.dist import Layout, native_power_iteration  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("format")
ap.add_argument("index16", type=int)
ap.add_argument("--launch", default="")
ap.add_argument("--E", type=int, default=20)
a = ap.parse_args()
coo = si.config_device(a.config)
n = coo.rows
x = si.vector_device(coo.cols, dtype=coo.val.dtype)
y = torch.empty(n, dtype=coo.val.dtype, device="cuda")
h = P.spmv_create(coo.rows, coo.cols, coo.row, coo.col, coo.val)
del coo
torch.cuda.empty_cache()
fmt = P.FORMATS[a.format]
P.spmv_convert(h, fmt, **({"index16": a.index16} if fmt in (P.FMT_ELL, P.FMT_SELL) else {}))
if a.launch:
    P.spmv_set_launch(h, fmt, *[int(v, 0) for v in a.launch.split(",")])
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
bufs = {"cur": torch.zeros(n, dtype=x.dtype, device="cuda"), "nxt": torch.zeros(n, dtype=x.dtype, device="cuda"),
        "chunk": torch.zeros(1, dtype=x.dtype, device="cuda"),
        "sums": torch.zeros(a.E + 1, 2, dtype=torch.float64, device="cuda")}
lay = Layout.from_bounds([0, n])
out = {"plain_ms": [], "power_ms": []}
for rep in range(4):
    P.spmv_run(h, 1.0, x, 0.0, y)
    e0.record(s)
    for _ in range(a.E):
        P.spmv_run(h, 1.0, x, 0.0, y)
    e1.record(s)
    torch.cuda.synchronize()
    out["plain_ms"].append(round(e0.elapsed_time(e1) / a.E, 4))
    z, sums, _, lms = native_power_iteration(h, lay, 0, x, bufs, a.E, None, time_loop=True)
    out["power_ms"].append(round(lms / a.E, 4))
print(json.dumps(out))
P.spmv_destroy(h)
