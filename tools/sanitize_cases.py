"""Small end-to-end driver for compute-sanitizer (memcheck / racecheck /
initcheck / synccheck): every format, both dtypes, unsorted ingest, features,
power steps and a short tune, on small ragged matrices."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2302_05662_b200 as P  # noqa: E402
import spmv_inputs as si  # noqa: E402
from gpu_cases import corpus  # noqa: E402

# (format, params, launch or None): every kernel family incl. the round-2 tile,
# merge-stream and 8-bit dictionary variants
FMTS = [(P.FMT_CSR, dict(csr_alg=P.CSR_VECTOR), None), (P.FMT_CSR, dict(csr_alg=P.CSR_SCALAR), None),
        (P.FMT_CSR, dict(csr_alg=P.CSR_MERGE), None), (P.FMT_CSR, dict(csr_alg=P.CSR_MERGE), (128, 255, -1, 0x108)),
        (P.FMT_CSR, dict(csr_alg=P.CSR_MERGE), (128, 255, -1, 0x208)),
        (P.FMT_ELL, dict(index16=0), None), (P.FMT_SELL, dict(index16=0), None),
        (P.FMT_SELL, dict(sell_C=32, sell_sigma=64, index16=0), None), (P.FMT_HYB, {}, None),
        (P.FMT_HYB, {}, (256, 255, -1, 0x108)), (P.FMT_COO, {}, None), (P.FMT_COO, {}, (256, 255, -1, 0x108)),
        (P.FMT_CSR, dict(csr_alg=P.CSR_STREAM), None), (P.FMT_BELL, dict(bell_b=2), None),
        (P.FMT_BELL, dict(bell_b=3), None),
        (P.FMT_ELL, dict(index16=-1), None), (P.FMT_SELL, dict(index16=-1), None),
        (P.FMT_SELL, dict(sell_C=32, sell_sigma=64, index16=-1), None)]


def main():
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["ragged_empty", "long_rows", "appendix_d", "empty_7x5",
                                                              "rmat10", "mixed_tiles"]
    cases = {n: c for n, c in corpus()}
    for name in names:
        coo = cases[name]
        for dtype, tdt in (("f64", torch.float64), ("f32", torch.float32)):
            sh = si.shuffled(coo, 3)
            r = torch.from_numpy(sh.row).cuda()
            c = torch.from_numpy(sh.col).cuda()
            v = torch.from_numpy(sh.val).to(tdt).cuda()
            h = P.spmv_create(coo.rows, coo.cols, r, c, v)
            if coo.rows > 0:
                P.spmv_features(h)
            x = torch.from_numpy(si.vector(max(coo.cols, 1))[:coo.cols]).to(tdt).cuda()
            y = torch.ones(coo.rows, dtype=tdt, device="cuda")
            for fmt, params, launch in FMTS:
                if coo.rows == 0 and fmt != P.FMT_CSR:
                    continue
                P.spmv_convert(h, fmt, **params)
                P.spmv_set_launch(h, fmt, *(launch or (0, 0, -1, 0)))
                P.spmv_run(h, 2.5, x, -0.5, y)
                P.spmv_run(h, 1.0, x, 0.0, y)
                if coo.rows == coo.cols and coo.rows > 0:
                    s0 = torch.zeros(2, dtype=torch.float64, device="cuda")
                    s1 = torch.zeros(2, dtype=torch.float64, device="cuda")
                    P.spmv_norm2(h, x, s0)
                    z = torch.empty_like(x)
                    P.spmv_power_step(h, x, z, s0, s1)
            torch.cuda.synchronize()
            P.spmv_destroy(h)
        print("ok", name, flush=True)
    coo = si.lap2d(12, random_values=True)
    h = P.spmv_create(coo.rows, coo.cols, torch.from_numpy(coo.row).cuda(), torch.from_numpy(coo.col).cuda(),
                      torch.from_numpy(coo.val).cuda())
    P.spmv_tune(h, P.TUNE_FORMAT, 100)
    P.spmv_destroy(h)
    h = P.spmv_create(coo.rows, coo.cols, torch.from_numpy(coo.row).cuda(), torch.from_numpy(coo.col).cuda(),
                      torch.from_numpy(coo.val).cuda())
    P.spmv_tune(h, P.TUNE_FORMAT | P.TUNE_PREDICT, 100)
    P.spmv_destroy(h)
    print("ok tune")
    # distributed plan: 3 in-process ranks, overlap + halo lists, direct and staged exchange
    from test_gpu_plan import run_plan
    for staged in ("0", "1"):
        os.environ["SPMV_PLAN_FORCE_STAGED"] = staged
        for flags in (P.PLAN_OVERLAP | P.PLAN_HALO, 0):
            run_plan(si.stencil27(8, random_values=True), 3, flags, [2], P.FMT_SELL, {"index16": -1})
    os.environ.pop("SPMV_PLAN_FORCE_STAGED", None)
    print("ok plan")


if __name__ == "__main__":
    main()
