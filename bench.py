#!/usr/bin/env python
"""bench.py — whole-path throughput of the B200 SpMV library (one JSON line).

A step is one pass of the whole hot path (SURVEY.md §8(a) rows a1–a8) over
one synthetic matrix, as the paper's run-time mode applies it to an
iterative solver:
  a1/a2 spmv_create   device COO -> validated canonical COO + CSR
  a3    spmv_features device Table 2 features
  a6/a7 the tuner/selector's decision for this workload (format + launch),
        measured once before timing with spmv_tune and replayed per step
  a4    spmv_convert  CSR -> chosen format
  a5/a8 E power-iteration steps (spmv_power_step: one SpMV kernel with the
        fused norm epilogue; NCCL all-gather/all-reduce when N > 1)
  spmv_destroy.
value = useful GFLOP/s = 2·nnz·E·K / (max-over-ranks device time of K steps).

`--impl reference` times the CPU oracle (oracle/, the only reference this
tier has) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpMV GFLOP/s & HBM GB/s vs 8 TB/s per format at 1/2/4/8 B200; MFLOPS/W"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--iters", type=int, default=100, help="power-iteration steps per step (E)")
    ap.add_argument("--format", default="auto", help="auto (spmv_tune) or COO/CSR/CSR-vector/CSR-merge/CSR-stream/ELL/HYB/SELL/BELL")
    ap.add_argument("--no-tune-launch", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--launch", default="", help="block,maxreg,carveout,knob (skips the launch sweep)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-serial", action="store_true", help="e2e one step at a time (default at N=1: two in flight)")
    ap.add_argument("--index16", type=int, default=-1, choices=[-1, 0, 1],
                    help="ELL/SELL column storage with --format: -1 auto (16-bit offsets when they fit), 0 int32, 1 16-bit")
    ap.add_argument("--plan", default="overlap,halo",
                    help="N>1 schedule: comma list of overlap (interior SpMV overlaps the exchange) and halo "
                         "(exchange only referenced remote entries); 'none' = split + all-gather, serialised")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks / energy

class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled DURING the timed
    region by an in-process NVML thread (an nvidia-smi -lms subprocess
    measurably stalls the CUDA launch path, so it is not used)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, index=0, period_s=0.25):
        import threading
        self.samples = []
        self.stop_ev = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.h = None
            return
        self.period = period_s
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nv
        while not self.stop_ev.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                try:
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            self.stop_ev.wait(self.period)

    def stop(self):
        if self.h is None:
            return None
        self.stop_ev.set()
        self.t.join(timeout=2)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        sm = [s for s, _ in self.samples]
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        loaded = [s for s in sm if s > 0.5 * self.max_mhz] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(sm), "source": "NVML thread, 250 ms"}


class Energy:
    def __init__(self, index=0):
        self.h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self.h = None

    def read_j(self):
        if self.h is None:
            return None
        try:
            return self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h) / 1000.0
        except Exception:
            return None


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ----------------------------------------------------------------------------- CPU oracle arm

CPU_SAMPLE = {"c1": ("lap2d", 64), "c2": ("stencil27", 64), "c3": ("rmat", 16), "c4": ("uniform", 1 << 18),
              "c5": ("stencil27", 64)}


def oracle_pipeline(cfg, iters, seconds_cap=None):
    """The oracle (as it stands) on a bounded sample of the workload:
    canonicalize -> CSR -> features -> format build -> E power steps.
    Returns (flops, seconds, description)."""
    import oracle
    import spmv_inputs as si
    kind, size = CPU_SAMPLE[cfg]
    if kind == "lap2d":
        coo = si.lap2d(size, random_values=True)
    elif kind == "stencil27":
        coo = si.stencil27(size, random_values=True)
    elif kind == "rmat":
        coo = si.rmat(size, dtype=np.float64)
    else:
        coo = si.uniform_k(size, 32)
    x = si.vector(coo.cols)
    t0 = time.perf_counter()
    st, R, C, V = oracle.canonicalize(coo.rows, coo.cols, coo.row, coo.col, coo.val)
    rp = oracle.csr(coo.rows, R)
    _, f = oracle.features(coo.rows, coo.cols, rp, C)
    if kind in ("stencil27", "lap2d", "uniform"):
        oracle.sell(coo.rows, rp, C, V, 64, 1)
    z = x / np.linalg.norm(x)
    for k in range(iters):
        y, z, lam, s = oracle.power_step(coo.rows, rp, C, V, z)
    t = time.perf_counter() - t0
    desc = (f"oracle (1 thread, fp64, naive C) on {kind}({size}) n={coo.rows} nnz={coo.nnz}: canonicalize+CSR+"
            f"features+SELL build+{iters} power steps")
    return 2.0 * coo.nnz * iters, t, desc


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    iters = args.iters
    times = []
    flops = 0.0
    desc = ""
    for i in range(args.warmup + args.steps):
        fl, t, desc = oracle_pipeline(args.config, iters)
        if i >= args.warmup:
            times.append(t)
            flops = fl
    tot = sum(times)
    val = flops * len(times) / tot / 1e9
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(val, 4), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000 * tot / len(times), 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "power_iterations_per_step": iters, "sample": CPU_SAMPLE[args.config]},
        "cpu_baseline": {"value": round(val, 4), "unit": "GFLOP/s", "cores": 1, "kind": "oracle", "sample": desc},
        "e2e": {"value": round(val, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ----------------------------------------------------------------------------- GPU arm

def setup_dist(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def gen_slab(cfg, bounds, rank, layout):
    """Row slab [b_r, b_{r+1}) of the config on this device, columns remapped
    into the padded all-gather layout (identity for world = 1)."""
    import torch
    import paper_2302_05662_b200 as P
    import spmv_inputs as si
    a, b = int(bounds[rank]), int(bounds[rank + 1])
    c = si.CONFIGS[cfg]
    dt = torch.float32 if c["dtype"] == "f32" else torch.float64
    if c["kind"] in ("lap2d", "stencil27"):
        kind = si.LAP2D if c["kind"] == "lap2d" else si.STENCIL27
        coo = si.stencil_device(kind, c["N"], a, b, random_values=True, dtype=dt)
        n = c["N"] ** (2 if kind == si.LAP2D else 3)
    else:
        full = si.config_device(cfg)
        n = full.rows
        if a == 0 and b == n:
            coo = full
        else:
            rr = full.row.long()
            lo = int(torch.searchsorted(rr, torch.tensor([a], device=rr.device)).item())
            hi = int(torch.searchsorted(rr, torch.tensor([b], device=rr.device)).item())
            coo = si.COO(b - a, n, (full.row[lo:hi] - a).contiguous(), full.col[lo:hi].contiguous(),
                         full.val[lo:hi].contiguous())
    if layout.world > 1:
        P.spmv_dist_remap_columns(coo.col, layout.bounds)
    coo.cols = layout.padded_n if layout.world > 1 else n
    coo.rows = b - a
    return coo, n


def row_lengths(cfg):
    import spmv_inputs as si
    import torch
    c = si.CONFIGS[cfg]
    if c["kind"] in ("lap2d", "stencil27"):
        kind = si.LAP2D if c["kind"] == "lap2d" else si.STENCIL27
        n = c["N"] ** (2 if kind == si.LAP2D else 3)
        out = torch.empty(n, dtype=torch.int64, device="cuda")
        import ctypes
        si.lib().gen_dev_stencil_rowlen(kind, c["N"], 0, n, out.data_ptr(),
                                        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        return out.cpu().numpy()
    full = si.config_device(cfg)
    return torch.bincount(full.row.long(), minlength=full.rows).cpu().numpy()


def summarize_decisions(log):
    out = {}
    for r in log or []:
        if r.get("kind") == "format_select":
            out["chosen"] = r.get("chosen")
            out["gate"] = r.get("gate")
            out["candidates"] = [{k: c.get(k) for k in ("format", "alg", "t_s", "rejected") if k in c}
                                 for c in r.get("candidates", [])]
        elif r.get("kind") == "launch_sweep":
            out["launch_variants"] = len(r.get("variants", []))
            out["launch_best"] = r.get("best")
            out["launch_best_t_s"] = r.get("t_best_s")
    return out


def stored_bytes_power(info_bytes, rows, cols, vb):
    # format arrays (padding included) + x read once + y written
    return info_bytes + cols * vb + rows * vb


def run_ours(args):
    import torch
    import paper_2302_05662_b200 as P
    from paper_2302_05662_b200.dist import Layout, NativeComm, PowerIteration, native_power_iteration
    import spmv_inputs as si

    world, rank, local = setup_dist(args)
    dev = torch.device("cuda", local)
    cfgd = si.CONFIGS[args.config]
    dtype = "f32" if cfgd["dtype"] == "f32" else "f64"
    tdt = torch.float32 if dtype == "f32" else torch.float64
    vb = 4 if dtype == "f32" else 8
    E = args.iters

    lengths = row_lengths(args.config)
    bounds = P.spmv_dist_partition_lengths(lengths, world)
    layout = Layout.from_bounds(bounds)
    coo, n_global = gen_slab(args.config, bounds, rank, layout)
    nnz_local = coo.nnz
    del lengths
    torch.cuda.empty_cache()

    # x0 (global, padded layout), generated on device
    x0g = si.vector_device(n_global, dtype=tdt, device=dev)
    x0 = torch.zeros(layout.padded_n if world > 1 else n_global, dtype=tdt, device=dev)
    if world > 1:
        for r in range(world):
            a, b = layout.rows_of(r)
            x0[r * layout.chunk: r * layout.chunk + (b - a)] = x0g[a:b]
    else:
        x0.copy_(x0g)
    del x0g

    # ---- a6/a7 decision, measured once before timing (replayed every step)
    h = P.spmv_create(coo.rows, coo.cols, coo.row, coo.col, coo.val)
    P.spmv_features(h)
    if args.format == "auto":
        flags = P.TUNE_FORMAT | (0 if args.no_tune_launch else P.TUNE_LAUNCH)
        rep = P.spmv_tune(h, flags, expected_iterations=E)
        fmt = rep.format
        params = dict(csr_alg=rep.params.csr_alg, csr_T=rep.params.csr_T, sell_C=rep.params.sell_C,
                      sell_sigma=rep.params.sell_sigma, hyb_K=rep.params.hyb_K, bell_b=rep.params.bell_b,
                      index16=rep.params.index16)
        launch = P.spmv_get_launch(h, fmt)
        decision = P.spmv_decision_log(h)
    else:
        csr_algs = {"CSR-vector": P.CSR_VECTOR, "CSR-merge": P.CSR_MERGE, "CSR-stream": P.CSR_STREAM}
        fmt = P.FMT_CSR if args.format in csr_algs else P.FORMATS[args.format]
        params = {"index16": args.index16} if fmt in (P.FMT_ELL, P.FMT_SELL) else {}
        if args.format in csr_algs:
            params = {"csr_alg": csr_algs[args.format]}
        P.spmv_convert(h, fmt, **params)
        if args.launch:
            P.spmv_set_launch(h, fmt, *[int(v) for v in args.launch.split(",")])
        elif not args.no_tune_launch:
            P.spmv_tune(h, P.TUNE_LAUNCH, expected_iterations=E)
        launch = P.spmv_get_launch(h, fmt)
        decision = P.spmv_decision_log(h)
    P.spmv_destroy(h)
    if fmt != P.FMT_CSR:
        params = {k: v for k, v in params.items() if k != "csr_alg" or fmt == P.FMT_CSR}
    if fmt == P.FMT_SELL:
        params = dict(sell_C=params.get("sell_C", 0), sell_sigma=params.get("sell_sigma", 0),
                      index16=params.get("index16", 0))
    elif fmt == P.FMT_ELL:
        params = dict(index16=params.get("index16", 0))
    elif fmt == P.FMT_BELL:
        params = dict(bell_b=params.get("bell_b", 0))
    elif fmt == P.FMT_HYB:
        params = dict(hyb_K=params.get("hyb_K", -1))
    elif fmt == P.FMT_CSR:
        params = dict(csr_alg=params.get("csr_alg", 0), csr_T=params.get("csr_T", 0))
    else:
        params = {}
    fmt_label = P.FORMAT_NAMES[fmt] + ({P.CSR_MERGE: "-merge", P.CSR_STREAM: "-stream", P.CSR_VECTOR: "-vector"}
                                       .get(params.get("csr_alg", 0), "") if fmt == P.FMT_CSR else "")

    stream = torch.cuda.current_stream()
    state = {"kms": []}
    comm = NativeComm(rank, world, local) if world > 1 else None
    bufs = {
        "cur": torch.zeros(layout.padded_n if world > 1 else n_global, dtype=tdt, device=dev),
        "nxt": torch.zeros(layout.padded_n if world > 1 else n_global, dtype=tdt, device=dev),
        "chunk": torch.zeros(layout.chunk, dtype=tdt, device=dev),
        "sums": torch.zeros(E + 1, 2, dtype=torch.float64, device=dev)}

    plan_flags = 0
    for f in (args.plan or "").split(","):
        plan_flags |= {"overlap": P.PLAN_OVERLAP, "halo": P.PLAN_HALO}.get(f.strip(), 0)

    def power(h, x_start, bufs=bufs):
        # N = 1: one event pair around the E back-to-back SpMV launches (no
        # events between kernels); N > 1: the distributed plan (interior/halo
        # split, overlap, halo exchange) with events around each interior kernel.
        timing = state.get("time_kernels", False)
        if world > 1:
            plan = P.spmv_dist_plan_create(h, comm.comm, layout.chunk, plan_flags)
            if state.get("want_plan_info"):
                state["plan_info"] = P.spmv_dist_plan_info(plan)
                part0 = P.spmv_dist_plan_part(plan, 0)
                state["part0_info"] = P.spmv_format_info(part0, fmt) if part0 is not None else None
            fb, _, ims = P.spmv_dist_plan_iterate(plan, x_start, bufs["cur"], bufs["nxt"], E, bufs["sums"],
                                                  time_interior=timing)
            P.spmv_dist_plan_destroy(plan)
            if ims:
                state["kms"].extend(ims)
            return (bufs["cur"] if fb == 0 else bufs["nxt"]), bufs["sums"]
        res = native_power_iteration(h, layout, rank, x_start, bufs, E, comm,
                                     time_kernels=timing and world > 1, time_loop=timing and world == 1)
        z, sums, kms = res[:3]
        lms = res[3] if len(res) > 3 else None
        if kms:
            state["kms"].extend(kms)
        if lms is not None and timing:
            state["kms"].extend([lms / E] * E)
        return z, sums

    phases = {} if os.environ.get("BENCH_PHASES") else None

    def mark(name):
        if phases is not None:
            torch.cuda.synchronize()
            phases.setdefault(name, []).append(time.perf_counter())

    ev_names = ["create", "features", "convert", "power", "destroy"]

    def ev_mark(i):
        # CUDA events at phase boundaries on the stream (no synchronisation)
        if state.get("phase_events") is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            state["phase_events"][-1].append(e)

    def one_step(coo_in, want_info=False):
        if state.get("phase_events") is not None:
            state["phase_events"].append([])
        mark("0_start")
        ev_mark(0)
        h = P.spmv_create(coo_in.rows, coo_in.cols, coo_in.row, coo_in.col, coo_in.val)
        state["h"] = h
        mark("1_create")
        ev_mark(1)
        P.spmv_features(h)
        mark("2_features")
        ev_mark(2)
        P.spmv_convert(h, fmt, **params)
        P.spmv_set_launch(h, fmt, *launch)
        info = P.spmv_format_info(h, fmt) if want_info else None  # (reads sizes back: not in the timed loop)
        state["want_plan_info"] = want_info
        mark("3_convert")
        ev_mark(3)
        power(h, x0)
        mark("4_power")
        ev_mark(4)
        P.spmv_destroy(h)
        state["h"] = None
        mark("5_destroy")
        ev_mark(5)
        return info

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    info = None
    for w in range(args.warmup):
        info = one_step(coo, want_info=(w == args.warmup - 1)) or info
    if info is None:
        info = one_step(coo, want_info=True)
    barrier()

    clocks = ClockSampler(local) if not os.environ.get("BENCH_NO_CLOCKS") else None
    energy = Energy(local)
    state["time_kernels"] = not os.environ.get("BENCH_NO_KEVENTS")
    state["kms"] = []
    state["phase_events"] = []
    l0 = P.launch_count()
    e_j0 = energy.read_j()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    barrier()
    state["host_t0"] = time.perf_counter()
    t_start.record(stream)
    for _ in range(args.steps):
        one_step(coo)
    t_end.record(stream)
    barrier()
    e_j1 = energy.read_j()
    launches = P.launch_count() - l0
    clk = clocks.stop() if clocks else None
    state["time_kernels"] = False
    ms = t_start.elapsed_time(t_end)
    host_s = time.perf_counter() - state.get("host_t0", time.perf_counter())
    if phases is not None and rank == 0:
        keys = sorted(phases)
        n = min(len(phases[k]) for k in keys)
        rep = {}
        for a, b in zip(keys[:-1], keys[1:]):
            d = [phases[b][i] - phases[a][i] for i in range(n)]
            rep[b] = {"first_ms": round(d[0] * 1e3, 3), "last_ms": round(d[-1] * 1e3, 3),
                      "median_ms": round(statistics.median(d) * 1e3, 3)}
        print("PHASES", json.dumps(rep), file=sys.stderr, flush=True)
    kernel_ms = list(state["kms"])
    phase_ms = {}
    pe = state.pop("phase_events", None) or []
    state["phase_events"] = None
    for i, name in enumerate(ev_names):
        vals = [st[i].elapsed_time(st[i + 1]) for st in pe if len(st) > i + 1]
        if vals:
            phase_ms[name] = round(statistics.median(vals), 4)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        nnz_t = torch.tensor([nnz_local], dtype=torch.float64, device=dev)
        dist.all_reduce(nnz_t)
        nnz_total = nnz_t.item()
    else:
        nnz_total = nnz_local
    ms_max = ms_t.item()
    flops = 2.0 * nnz_total * E * args.steps
    value = flops / (ms_max * 1e-3) / 1e9

    # ---- roofline of the dominant kernel (the SpMV of the chosen format)
    rows_local = coo.rows
    if world > 1 and state.get("part0_info"):
        # interior kernel: its stored arrays + the own chunk of x + its rows of y
        p0rows = state["plan_info"]["part_rows"][0]
        alg_bytes = state["part0_info"]["stored_bytes"] + rows_local * vb + p0rows * vb
    else:
        alg_bytes = stored_bytes_power(info["stored_bytes"], rows_local, n_global, vb)
    k_avg_ms = statistics.mean(kernel_ms) if kernel_ms else float("nan")
    achieved = alg_bytes / (k_avg_ms * 1e-3) / 1e9
    peak, peak_kind = measured_peaks()
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            key = fmt_label if fmt == P.FMT_CSR else P.FORMAT_NAMES[fmt]
            if pj.get("format") == key:  # legacy single-format layout
                traffic = pj.get("dram_bytes_per_launch")
            elif isinstance(pj.get(key), dict):
                traffic = pj[key].get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    kernel_share = sum(kernel_ms) / ms if ms > 0 else None

    # ---- e2e: same metric through the C ABI with HOST buffers (rank 0 .. all ranks)
    e2e = None
    try:
        if args.no_e2e:
            raise RuntimeError("e2e skipped (--no-e2e)")
        host_row = coo.row.cpu().pin_memory()
        host_col = coo.col.cpu().pin_memory()
        host_val = coo.val.cpu().pin_memory()
        host_x0 = x0.cpu().pin_memory()
        # N = 1: two steps in flight on two streams (one host thread each, the
        # C calls release the GIL), so step k+1's host->device copy overlaps
        # step k's kernels; every step still copies its own inputs in and its
        # result out. N > 1: one step at a time (the ranks' collectives are
        # issued in step order on one communicator).
        free_b, _ = torch.cuda.mem_get_info(dev)
        step_b = 3 * coo.nnz * (8 + vb)  # COO + format + scratch, per step in flight (upper estimate)
        depth = 2 if world == 1 and not args.e2e_serial and 2 * step_b < 0.8 * free_b else 1
        lanes = []
        for i in range(depth):
            lanes.append({
                "stream": torch.cuda.Stream(device=dev),
                "bufs": bufs if i == 0 else {k: torch.zeros_like(v) for k, v in bufs.items()},
                "y_host": torch.empty(layout.padded_n if world > 1 else n_global, dtype=tdt).pin_memory(),
                "s_host": torch.empty(E + 1, 2, dtype=torch.float64).pin_memory()})
        y_host, s_host = lanes[0]["y_host"], lanes[0]["s_host"]

        import threading
        ingest_lock = threading.Lock()

        def e2e_step(lane):
            torch.cuda.set_device(dev)
            st = lane["stream"]
            with torch.cuda.stream(st):
                # one ingest at a time: the host link is the shared resource, so
                # the lanes settle into copy(k+1) || kernels(k) instead of both
                # copying, then both computing, in lockstep; one FIFO per
                # copy engine (the x upload is queued with the matrix, not behind
                # the other lane's next matrix upload)
                xdev = torch.empty_like(x0)
                with ingest_lock:
                    h = P.spmv_create(coo.rows, coo.cols, host_row.numpy(), host_col.numpy(), host_val.numpy(),
                                      device=dev.index if dev.index is not None else 0, stream=st)
                    xdev.copy_(host_x0, non_blocking=True)
                try:
                    P.spmv_features(h)
                    P.spmv_convert(h, fmt, **params)
                    P.spmv_set_launch(h, fmt, *launch)
                    z, sums = power(h, xdev, lane["bufs"])
                    lane["y_host"].copy_(z, non_blocking=True)
                    lane["s_host"].copy_(sums, non_blocking=True)
                    st.synchronize()
                finally:
                    P.spmv_destroy(h)

        def run_lane(i, count):
            for _ in range(count):
                e2e_step(lanes[i])

        from concurrent.futures import ThreadPoolExecutor
        pool = ThreadPoolExecutor(max_workers=depth)  # the same host threads warm up and run

        def run_all(total):
            counts = [total // depth + (1 if i < total % depth else 0) for i in range(depth)]
            for f in [pool.submit(run_lane, i, counts[i]) for i in range(depth)]:
                f.result()

        run_all(max(2 * depth, args.warmup))
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        run_all(args.steps)
        torch.cuda.synchronize()
        barrier()
        t_e2e = time.perf_counter() - t0
        pool.shutdown()
        tt = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
        if world > 1:
            import torch.distributed as dist
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": round(flops / tt.item() / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(coo.nnz * (8 + vb) + x0.numel() * vb),
               "d2h_bytes_per_step": int(y_host.numel() * vb + s_host.numel() * 8),
               "steps_in_flight": depth}
        lam = PowerIteration.lambdas(s_host)
    except Exception as ex:  # report, never fall back
        e2e = {"value": None, "unit": "GFLOP/s", "error": repr(ex)[:200]}
        lam = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        fl, t, desc = oracle_pipeline(args.config, E)
        cpu = {"value": round(fl / t / 1e9, 4), "unit": "GFLOP/s", "cores": 1, "kind": "oracle", "sample": desc}

    mflops_w = None
    if e_j0 is not None and e_j1 is not None and e_j1 > e_j0:
        joules = (e_j1 - e_j0)
        mflops_w = flops / 1e6 / joules / (world if world > 1 else 1)

    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": dtype,
            "data": "synthetic",
            "config": {"workload": args.config, "desc": cfgd["desc"], "n": n_global, "nnz": int(nnz_total),
                       "power_iterations_per_step": E, "format": fmt_label, "format_params": params,
                       "launch": {"block": launch[0], "maxreg": launch[1], "carveout_pct": launch[2],
                                  "knob": launch[3]},
                       "partition": "row, nnz-balanced" if world > 1 else "none",
                       "plan": ({"flags": args.plan, **{k: state["plan_info"][k] for k in
                                 ("h0", "h1", "part_rows", "halo", "recv_bytes_per_step")}}
                                if world > 1 and state.get("plan_info") else None),
                       "l2": "inputs larger than L2 (matrix arrays > 126 MB; x stays L2-resident by design)"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "kernel": f"{fmt_label} SpMV (power-step epilogue)" + (
                             "" if world == 1 else ", interior rows"),
                         "kernel_timing": ("CUDA events around the E back-to-back SpMV launches of each step / E "
                                           "(includes launch gaps)") if world == 1 else
                                          "CUDA events around each interior SpMV (overlapping the exchange)",
                         "alg_bytes_per_launch": int(alg_bytes), "kernel_avg_us": round(k_avg_ms * 1e3, 2),
                         "kernel_share_of_step": round(kernel_share, 4) if kernel_share else None,
                         "peak_source": peak_kind, "frac_of_8TBs": round(achieved / 8000.0, 4)},
            "hbm_gbs": round(achieved, 1),
            "step_phases_ms": phase_ms,
            "mflops_per_w": round(mflops_w, 1) if mflops_w else None,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "host_ms_per_step": round(host_s * 1e3 / args.steps, 3),
            "clocks": clk,
            "lambda_last": float(lam[-1]) if lam is not None and len(lam) else None,
            "tuner": summarize_decisions(decision),
        }
        print(json.dumps(out), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    run_ours(args)


if __name__ == "__main__":
    main()
