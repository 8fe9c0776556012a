"""Distributed-plan schedule on ONE GPU.

W ranks = W host threads of this process joined by the in-process
communicator group (spmv_dist_local_group); every rank runs the real plan
(interior/halo split, overlap stream schedule, halo lists) on its own stream,
the collectives are device copies. All ranks share one GPU, so the total work
is the 1-GPU problem (strong scaling onto the same device): the sweep shows
what each schedule costs on top of the SpMV — the all-gather moves
(W-1)·n values per step in total, the halo exchange only the halo planes —
and that overlap hides the exchange behind the interior kernel.

Output: JSON lines + a markdown table (ms per power step = max over ranks of
the loop time / E, GFLOP/s = 2·nnz·E / that time)."""
import argparse
import json
import os
import sys
import threading
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2302_05662_b200 as P  # noqa: E402
import spmv_inputs as si  # noqa: E402

FLAGS = {"allgather": 0, "allgather+overlap": P.PLAN_OVERLAP, "halo": P.PLAN_HALO,
         "halo+overlap": P.PLAN_OVERLAP | P.PLAN_HALO}


def row_lengths(cfg):
    c = si.CONFIGS[cfg]
    kind = si.LAP2D if c["kind"] == "lap2d" else si.STENCIL27
    n = c["N"] ** (2 if kind == si.LAP2D else 3)
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    import ctypes
    si.lib().gen_dev_stencil_rowlen(kind, c["N"], 0, n, out.data_ptr(),
                                    ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    return out.cpu().numpy(), kind, c["N"], n


def run(cfg, world, flag_names, fmt, E, reps):
    lengths, kind, N, n = row_lengths(cfg)
    bounds = P.spmv_dist_partition_lengths(lengths, world)
    chunk = int(np.max(np.diff(bounds)))
    comms = P.spmv_dist_local_group(world, [0] * world)
    x0g = si.vector_device(n)
    lock = threading.Lock()
    results = {}

    def rank_main(r):
        torch.cuda.set_device(0)
        st = torch.cuda.Stream()
        a, b = int(bounds[r]), int(bounds[r + 1])
        with torch.cuda.stream(st):
            coo = si.stencil_device(kind, N, a, b, random_values=True)
            if world > 1:
                P.spmv_dist_remap_columns(coo.col, bounds, stream=st)
            h = P.spmv_create(b - a, world * chunk, coo.row, coo.col, coo.val, stream=st)
            del coo
            P.spmv_convert(h, fmt)
            x0 = torch.zeros(world * chunk, dtype=torch.float64, device="cuda")
            for q in range(world):
                qa, qb = int(bounds[q]), int(bounds[q + 1])
                x0[q * chunk: q * chunk + (qb - qa)] = x0g[qa:qb]
            b0, b1 = torch.empty_like(x0), torch.empty_like(x0)
            sums = torch.zeros(E + 1, 2, dtype=torch.float64, device="cuda")
            out = {}
            for name in flag_names:
                plan = P.spmv_dist_plan_create(h, comms[r], chunk, FLAGS[name])
                info = P.spmv_dist_plan_info(plan)
                P.spmv_dist_plan_iterate(plan, x0, b0, b1, 5, sums)  # warm-up
                ts, ims = [], []
                for _ in range(reps):
                    _, lms, im = P.spmv_dist_plan_iterate(plan, x0, b0, b1, E, sums, time_loop=True,
                                                          time_interior=True)
                    ts.append(lms)
                    ims.append(float(np.mean(im)))
                lam = float(sums[E, 1].item() / np.sqrt(sums[E - 1, 0].item()))
                P.spmv_dist_plan_destroy(plan)
                out[name] = dict(loop_ms=float(np.median(ts)), interior_ms=float(np.median(ims)), info=info, lam=lam)
            P.spmv_destroy(h)
        st.synchronize()
        with lock:
            results[r] = out

    try:
        with ThreadPoolExecutor(world) as ex:
            list(ex.map(rank_main, range(world)))
    finally:
        for c in comms:
            P.spmv_dist_destroy(c)
    nnz = int(lengths.sum())
    rows = []
    for name in flag_names:
        loop = max(results[r][name]["loop_ms"] for r in range(world))
        inf0 = results[0][name]["info"]
        rows.append(dict(config=cfg, world=world, schedule=name, format=P.FORMAT_NAMES[fmt], E=E,
                         ms_per_step=loop / E, gflops=2.0 * nnz * E / (loop * 1e-3) / 1e9,
                         interior_us=1e3 * max(results[r][name]["interior_ms"] for r in range(world)),
                         recv_bytes_per_step_rank0=inf0["recv_bytes_per_step"], halo=inf0["halo"],
                         part_rows_rank0=inf0["part_rows"], lam=results[0][name]["lam"]))
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--format", default="SELL")
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "plan_sweep"))
    a = ap.parse_args()
    fmt = P.FORMATS[a.format]
    all_rows = []
    for w in [int(v) for v in a.worlds.split(",")]:
        names = list(FLAGS) if w > 1 else ["allgather"]
        rows = run(a.config, w, names, fmt, a.iters, a.reps)
        for r in rows:
            print(json.dumps(r), flush=True)
        all_rows += rows
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(all_rows, open(a.out + ".json", "w"), indent=1)
    with open(a.out + ".md", "w") as f:
        f.write("| config | ranks | schedule | ms/step | GFLOP/s | interior kernel µs | recv B/step (rank 0) | "
                "rank-0 rows interior/lo/hi |\n|---|---|---|---|---|---|---|---|\n")
        for r in all_rows:
            f.write(f"| {r['config']} | {r['world']} | {r['schedule']} | {r['ms_per_step']:.4f} | {r['gflops']:.1f} | "
                    f"{r['interior_us']:.1f} | {r['recv_bytes_per_step_rank0']} | "
                    f"{'/'.join(str(v) for v in r['part_rows_rank0'])} |\n")


if __name__ == "__main__":
    main()
