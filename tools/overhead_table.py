"""Device analog of the paper's `tab:overhead`: f_latency
(feature extraction) and c_latency (conversion out of the COO input) on one
B200, for synthetic 27-point stencils whose nnz match the paper's 30 matrices
(0.8 M - 19.2 M nnz). The paper's CPU/NumPy seconds are printed beside as
context (other hardware, other code): they are the quantity the run-time
mode's gate must amortise, and the reason SURVEY §8 moves
features and conversions onto the device.

Measured per matrix (CUDA events on the handle's stream, warm: the first
matrix's numbers are discarded as module-loading warm-up):
  ingest  = spmv_create from device-resident COO (validate, order check,
            CSR row pointers) — the paper's input is COO;
  f       = spmv_features (the handle's own event-timed f_latency);
  c(ELL), c(SELL) = spmv_convert (event-timed c_latency).
python tools/overhead_table.py [--out gpurun_out/overhead]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2302_05662_b200 as P  # noqa: E402
import spmv_inputs as si  # noqa: E402

# (matrix, nnz, f_latency s, c_latency s) — tab:overhead
PAPER = [("shar_te2-b3", 800800, 1.71875, 1.625), ("rim", 1014951, 1.578125, 2.046875),
         ("bcsstk32", 1029655, 1.71, 2.125), ("il2010", 1082232, 3.625, 2.5),
         ("viscorocks", 1162244, 1.90625, 2.4375), ("cant", 2034917, 3.4531, 4.59),
         ("parabolic_fem", 2100225, 5.46875, 4.984375), ("pkustk04", 2137125, 3.78, 4.53125),
         ("apache2", 2766523, 7.84, 6.06), ("consph", 3046907, 5.375, 6.65625),
         ("wiki-talk-temporal", 3309592, 10.4375, 7.3281), ("amazon0601", 3387388, 7.125, 7.171875),
         ("Chevron3", 3413113, 7.0625, 7.328125), ("xenon2", 3866688, 6.75, 9.375),
         ("x104", 5138004, 9.093, 11.76563), ("crankseg_1", 5333507, 9.78025, 11.75),
         ("Si87H76", 5451000, 9.828125, 11.90625), ("Hamrle3", 5514242, 15.09375, 12.89063),
         ("pwtk", 5926171, 11.39, 13.8593), ("Chevron4", 6376412, 13.76563, 14.71875),
         ("Hardesty1", 6539157, 15.09375, 14.5625), ("rgg_n_2_20_s0", 6891620, 15.32813, 15.34375),
         ("crankseg_2", 7106348, 13.03125, 15.25), ("CurlCurl_3", 7382096, 17.89063, 18.8125),
         ("human_gene2", 9041364, 17.01563, 21.70313), ("af_shell6", 9046865, 18.78125, 21.4687),
         ("atmosmodm", 10319760, 24.14063, 23.90625), ("kim2", 11330020, 22.70313, 27.10938),
         ("test1", 12968200, 23.78125, 30.03125), ("eu-2005", 19235140, 39.82813, 47.98438)]


def stencil_n_for(nnz):
    """Smallest N whose 27-point stencil has at least nnz entries (27·N³ minus the boundary)."""
    n = 2
    while 27 * n ** 3 - 27 * n ** 2 * 2 < nnz:
        n += 1
    return n


def run_one(N):
    coo = si.stencil_device(si.STENCIL27, N, random_values=True)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    h = P.spmv_create(coo.rows, coo.cols, coo.row, coo.col, coo.val)
    e1.record(s)
    torch.cuda.synchronize()
    ingest = e0.elapsed_time(e1) * 1e-3
    P.spmv_features(h)
    f_lat, _ = P.spmv_overheads(h)
    c = {}
    for name, fmt in (("ELL", P.FMT_ELL), ("SELL", P.FMT_SELL)):
        P.spmv_convert(h, fmt)  # warm: main() ran one matrix through every kernel first
        _, cl = P.spmv_overheads(h)
        c[name] = cl[name]
    P.spmv_destroy(h)
    return coo.nnz, ingest, f_lat, c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/overhead")
    a = ap.parse_args()
    run_one(20)  # warm-up (module loading, pool)
    rows = []
    for name, nnz_p, f_p, c_p in PAPER:
        N = stencil_n_for(nnz_p)
        nnz, ingest, f, c = run_one(N)
        r = {"paper_matrix": name, "paper_nnz": nnz_p, "paper_f_s": f_p, "paper_c_s": c_p,
             "stencil_N": N, "nnz": nnz, "ingest_ms": ingest * 1e3, "f_ms": f * 1e3,
             "c_ell_ms": c["ELL"] * 1e3, "c_sell_ms": c["SELL"] * 1e3}
        r["ratio_f_plus_c"] = (f_p + c_p) / (f + min(c["ELL"], c["SELL"]))
        rows.append(r)
        print(json.dumps(r), flush=True)
    json.dump(rows, open(a.out + ".json", "w"), indent=1)
    lines = ["| paper matrix | paper nnz | paper f+c (s, CPU/NumPy) | stencil N | nnz | ingest ms | f ms | c(ELL) ms | c(SELL) ms | f+c(best) ms | paper ÷ B200 |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        fc = r["f_ms"] + min(r["c_ell_ms"], r["c_sell_ms"])
        lines.append(f"| {r['paper_matrix']} | {r['paper_nnz']:,} | {r['paper_f_s'] + r['paper_c_s']:.2f} | "
                     f"{r['stencil_N']} | {r['nnz']:,} | {r['ingest_ms']:.3f} | {r['f_ms']:.3f} | "
                     f"{r['c_ell_ms']:.3f} | {r['c_sell_ms']:.3f} | {fc:.3f} | {r['ratio_f_plus_c']:,.0f}× |")
    open(a.out + ".md", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
