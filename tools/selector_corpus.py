"""Training corpus for the learned format selector (the
paper's run-time-mode pipeline, P:442-452 and §5.4, applied to a
self-measured B200 corpus instead of SuiteSparse).

For each synthetic matrix (families of SURVEY §8(d) plus random / banded /
power-law / arrow structures, 10^4..10^8 nnz): device features
(spmv_features, Table 2) and f_latency, then for every candidate
format: conversion latency (c_latency), the launch sweep (spmv_tune LAUNCH)
and the tuned kernel time (CUDA events, median of 5 batches). Writes one JSON
record per matrix. Inputs are seeded; nothing here is the method's arithmetic."""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2302_05662_b200 as P  # noqa: E402
import spmv_inputs as si  # noqa: E402

VARIANTS = [("CSR-vector", P.FMT_CSR, dict(csr_alg=P.CSR_VECTOR)),
            ("CSR-merge", P.FMT_CSR, dict(csr_alg=P.CSR_MERGE)),
            ("ELL", P.FMT_ELL, {}),
            ("SELL", P.FMT_SELL, {}),
            ("HYB", P.FMT_HYB, {}),
            ("COO", P.FMT_COO, {}),
            ("BELL-2", P.FMT_BELL, dict(bell_b=2)),
            ("BELL-3", P.FMT_BELL, dict(bell_b=3)),
            ("CSR-stream", P.FMT_CSR, dict(csr_alg=P.CSR_STREAM))]


# ---------------------------------------------------------------- inputs (seeded, vectorised numpy)

def _values(rng, m):
    return si.value_of(rng.integers(0, np.iinfo(np.uint64).max, size=m, dtype=np.uint64, endpoint=True))


def from_lengths(n, cols, lengths, seed, col_fn):
    """Rows with the given lengths; col_fn(rng, row_ids) draws columns; dedupe."""
    rng = np.random.Generator(np.random.PCG64(seed))
    lengths = np.minimum(np.asarray(lengths, np.int64), cols)
    r = np.repeat(np.arange(n, dtype=np.int64), lengths)
    c = col_fn(rng, r).astype(np.int64)
    c = np.clip(c, 0, cols - 1)
    key = np.unique(r * cols + c)
    r = (key // cols).astype(np.int32)
    c = (key % cols).astype(np.int32)
    return si.COO(n, cols, r, c, _values(rng, r.shape[0]))


def banded(n, k, width, seed):
    return from_lengths(n, n, np.full(n, k), seed,
                        lambda rng, r: r + rng.integers(-width, width + 1, size=r.shape[0]))


def powerlaw(n, mean, alpha, seed):
    rng = np.random.Generator(np.random.PCG64(seed + 7))
    L = np.minimum(rng.zipf(alpha, size=n), n // 2).astype(np.int64)
    L = np.maximum((L * mean / max(L.mean(), 1e-9)).astype(np.int64), 0)
    return from_lengths(n, n, L, seed, lambda rng, r: rng.integers(0, n, size=r.shape[0]))


def poisson_rows(n, mean, seed):
    rng = np.random.Generator(np.random.PCG64(seed + 11))
    return from_lengths(n, n, rng.poisson(mean, size=n), seed, lambda rng, r: rng.integers(0, n, size=r.shape[0]))


def arrow(n, k, dense_rows, seed):
    rng = np.random.Generator(np.random.PCG64(seed + 13))
    L = np.full(n, k, np.int64)
    L[rng.choice(n, size=dense_rows, replace=False)] = n // 4
    return from_lengths(n, n, L, seed, lambda rng, r: r + rng.integers(-64, 65, size=r.shape[0]))


def corpus_specs(scale=1.0):
    S = []
    for N in [32, 64, 128, 256, 512, 1024, 2048, 3072]:
        S.append((f"lap2d_{N}", lambda N=N: si.lap2d(N, random_values=True)))
    for N in [12, 24, 40, 64, 96, 128, 160]:
        S.append((f"stencil27_{N}", lambda N=N: si.stencil27(N, random_values=True)))
    for N, B in [(16, 2), (32, 2), (64, 2), (96, 2), (16, 3), (32, 3), (64, 3), (80, 3), (16, 4), (40, 4)]:
        S.append((f"block27_{N}x{B}", lambda N=N, B=B: si.block27(N, B, random_values=True)))
    for lg in [14, 17, 20, 22]:
        for k in [3, 8, 16, 32, 64]:
            if lg == 22 and k == 64:
                continue
            S.append((f"uniform_{lg}_{k}", lambda lg=lg, k=k: si.uniform_k(1 << lg, k)))
    for sc in [12, 14, 16, 18, 20, 22]:
        for ef in [4, 16]:
            S.append((f"rmat_{sc}_{ef}", lambda sc=sc, ef=ef: si.rmat(sc, ef)))
    for n, k, w in [(1 << 14, 8, 64), (1 << 17, 16, 1000), (1 << 20, 12, 300), (1 << 19, 40, 50000),
                    (1 << 21, 6, 20), (1 << 18, 64, 4000)]:
        S.append((f"banded_{n}_{k}_{w}", lambda n=n, k=k, w=w: banded(n, k, w, 101)))
    for n, m, a in [(1 << 14, 8, 2.0), (1 << 17, 12, 2.2), (1 << 20, 10, 1.8), (1 << 19, 30, 2.5),
                    (1 << 21, 5, 2.0)]:
        S.append((f"powerlaw_{n}_{m}_{a}", lambda n=n, m=m, a=a: powerlaw(n, m, a, 202)))
    for n, m in [(1 << 14, 5), (1 << 17, 20), (1 << 20, 8), (1 << 20, 16)]:
        S.append((f"poisson_{n}_{m}", lambda n=n, m=m: poisson_rows(n, m, 303)))
    for n, k, d in [(1 << 16, 8, 4), (1 << 19, 16, 8), (1 << 20, 6, 32)]:
        S.append((f"arrow_{n}_{k}_{d}", lambda n=n, k=k, d=d: arrow(n, k, d, 404)))
    return S


# ---------------------------------------------------------------- measurement

def time_kernel(h, fmt, x, y):
    s = torch.cuda.current_stream()
    for _ in range(3):
        P.spmv_run(h, 1.0, x, 0.0, y, fmt=fmt)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    P.spmv_run(h, 1.0, x, 0.0, y, fmt=fmt)
    e1.record(s)
    torch.cuda.synchronize()
    one = e0.elapsed_time(e1)
    reps = max(5, min(300, int(10.0 / max(one, 1e-3))))
    ts = []
    for _ in range(5):
        e0.record(s)
        for _ in range(reps):
            P.spmv_run(h, 1.0, x, 0.0, y, fmt=fmt)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / reps)
    return statistics.median(ts) * 1e-3


def measure(name, coo, tune=True, variants=None, rec=None):
    t0 = time.time()
    row = torch.from_numpy(coo.row).cuda()
    col = torch.from_numpy(coo.col).cuda()
    val = torch.from_numpy(np.asarray(coo.val, np.float64)).cuda()
    n, m = coo.rows, coo.cols
    x = torch.from_numpy(si.vector(m)).cuda()
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    h = P.spmv_create(n, m, row, col, val)
    feats = P.spmv_features(h)
    f_lat, _ = P.spmv_overheads(h)
    if rec is None:  # a fresh record (else: add the requested variants to an existing one)
        rec = {"name": name, "n": n, "cols": m, "nnz": int(coo.row.shape[0]), "formats": {}}
        rec["features"] = feats
        rec["f_latency_s"] = f_lat
    else:
        assert rec["features"] == feats, name  # the same seeded matrix
    del row, col, val
    for vname, fmt, params in VARIANTS:
        if variants and vname not in variants:
            continue
        r = {}
        if vname.startswith("BELL") and (feats["mean"] < 4 or feats["std"] > feats["mean"]):
            r["skipped"] = "not block-like (mean < 4 or std > mean)"
        elif fmt == P.FMT_ELL and (n + 127) // 128 * 128 * feats["max_len"] > 4 * max(feats["nnz"], 1) + (1 << 20):
            r["skipped"] = "ELL padding > 4x nnz"
        if "skipped" in r:
            rec["formats"][vname] = r
            continue
        try:
            P.spmv_convert(h, fmt, **params)
            _, c_lat = P.spmv_overheads(h)
            info = P.spmv_format_info(h, fmt)
            if fmt == P.FMT_BELL and info["stored_bytes"] > 4 * (feats["nnz"] * 12 + 8 * n):
                r["skipped"] = "BELL block padding > 4x"
            else:
                if tune:
                    P.spmv_tune(h, P.TUNE_LAUNCH, 1000)
                r["t_s"] = time_kernel(h, fmt, x, y)
                r["launch"] = P.spmv_get_launch(h, fmt)
                r["c_latency_s"] = c_lat[P.FORMAT_NAMES[fmt]] if fmt != P.FMT_CSR else 0.0
                r["stored_bytes"] = info["stored_bytes"]
        except P.SpmvError as e:
            r["error"] = str(e)[:160]
        rec["formats"][vname] = r
        if fmt != P.FMT_CSR:
            P.spmv_convert(h, P.FMT_CSR)
    P.spmv_destroy(h)
    P.lib().spmv_trim_pool(0)
    rec["wall_s"] = round(time.time() - t0, 2)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "selector_corpus.jsonl"))
    ap.add_argument("--only", default="", help="comma list of name prefixes")
    ap.add_argument("--no-tune", action="store_true")
    ap.add_argument("--variants", default="", help="comma list of variant names to measure (default all)")
    ap.add_argument("--merge", default="", help="existing corpus .jsonl: add the measured variants to its records")
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    variants = a.variants.split(",") if a.variants else None
    old = {}
    if a.merge:
        for line in open(a.merge):
            r = json.loads(line)
            old[r["name"]] = r
    with open(a.out, "w") as f:
        for name, gen in corpus_specs():
            if a.only and not any(name.startswith(p) for p in a.only.split(",")):
                continue
            try:
                coo = gen()
                prev = old.get(name)
                rec = measure(name, coo, tune=not a.no_tune, variants=variants,
                              rec=prev if prev and "formats" in prev else None)
            except Exception as e:  # record and continue
                rec = {"name": name, "error": repr(e)[:200]}
            f.write(json.dumps(rec) + "\n")
            f.flush()
            best = min(((k, v["t_s"]) for k, v in rec.get("formats", {}).items() if "t_s" in v),
                       key=lambda kv: kv[1], default=(None, None))
            print(name, rec.get("nnz"), best, rec.get("wall_s"), flush=True)


if __name__ == "__main__":
    main()
