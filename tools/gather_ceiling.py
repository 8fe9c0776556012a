"""Measured x-gather ceiling of a config's own column stream.

Times, over the column array as CSR/COO store it (and as ELL stores it for
c4), only the gathers x[col[k]] — no values, no FMA, no y — through the LSU
(two orders) and through the TMA unit (tile::gather4, 16-byte bulk copies).
Also counts the distinct 128-byte x lines per 32 consecutive stored entries
(the L1TEX wavefronts a warp-order gather instruction costs).

python tools/gather_ceiling.py c3 c4 [--reps 20] [--json out.json]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

MODES = {0: "lsu_warp_order", 1: "lsu_lane_order", 2: "tma_gather4", 3: "tma_bulk16"}


def lib():
    import build_tools  # noqa: F401  (same directory)
    path = build_tools.build()
    L = ctypes.CDLL(path)
    L.gather_ceiling.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                 ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p]
    L.gather_ceiling.restype = ctypes.c_int
    return L


sys.path.insert(0, HERE)


def lines_per_warp(col, vbytes):
    """Mean distinct 128-byte x lines per group of 32 consecutive entries."""
    import torch
    n = (col.numel() // 32) * 32
    ln = (col[:n].long() * vbytes) >> 7
    ln = ln.view(-1, 32).sort(dim=1).values
    d = (ln[:, 1:] != ln[:, :-1]).sum(dim=1) + 1
    return float(d.double().mean().item())


def measure(col, nnz, x, n, vbytes, reps=20, modes=(0, 1, 2, 3)):
    import torch
    L = lib()
    out = {}
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for m in modes:
        ms = ctypes.c_double()
        rc = L.gather_ceiling(m, 0 if vbytes == 8 else 1, ctypes.c_void_p(col.data_ptr()), nnz,
                              ctypes.c_void_p(x.data_ptr()), n, reps, ctypes.byref(ms), st)
        out[MODES[m]] = {"us": round(ms.value * 1e3, 2), "gathers_per_ns": round(nnz / (ms.value * 1e6), 2)} \
            if rc == 0 else {"error": rc}
    ok = [v["us"] for v in out.values() if "us" in v]
    out["ceiling_us"] = min(ok) if ok else None
    out["lines_per_32"] = round(lines_per_warp(col, vbytes), 2)
    return out


def ell_order_cols(coo, K):
    """Column array in ELL order (k-major over rows) for a fixed-length-K matrix."""
    return coo.col.view(coo.rows, K).t().contiguous().view(-1)


def main():
    import torch
    import spmv_inputs as si
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    res = {}
    for cfg in a.configs:
        coo = si.config_device(cfg)
        vb = coo.val.element_size()
        x = si.vector_device(coo.cols, dtype=coo.val.dtype)
        r = {"nnz": coo.nnz, "csr_order": measure(coo.col, coo.nnz, x, coo.cols, vb, a.reps)}
        if cfg == "c4":
            ce = ell_order_cols(coo, 32)
            r["ell_order"] = measure(ce, coo.nnz, x, coo.cols, vb, a.reps)
            del ce
        res[cfg] = r
        print(cfg, json.dumps(r), flush=True)
        del coo, x
        torch.cuda.empty_cache()
    if a.json:
        json.dump(res, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
