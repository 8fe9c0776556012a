"""spmv_inputs — seeded synthetic inputs for the B200 SpMV path (INPUTS ONLY).

This module holds none of the SpMV method's arithmetic. It generates the
matrices and vectors of SURVEY.md §8(d) ("Synthetic inputs") from a
counter-based splitmix64 hash, on the host (gen_host.c, numpy results) or on
the device (gen_dev.cu, torch results), bit-identically. Both the oracle
tests and the product tests/bench draw their inputs from here; the product
library and the oracle never import each other.

Configs (BASELINE.json `configs`):
  c1  lap2d(64)                   5-point Laplacian 64x64, fp64
  c2  stencil27(128)              27-point stencil 128^3, fp64
  c3  rmat(23, 16)                Graph500 RMAT, fp32
  c4  uniform_k(2**22, 32)        uniform random 32/row, fp64
  c5  stencil27(512)              27-point stencil 512^3, fp64 (row slabs)
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libspmvinputs.so")

MATRIX_SEED = 0x2302056620230211
X_SEED = 0x5EEDC0FFEE000001
Y_SEED = 0x5EEDC0FFEE000002

LAP2D, STENCIL27, BLOCK27 = 0, 1, 100
# Graph500 RMAT quadrant probabilities.
RMAT_ABC = (0.57, 0.19, 0.19)

_SOURCES = ["gen_common.h", "gen_host.c", "gen_dev.cu"]


def build(force: bool = False) -> str:
    """Compile libspmvinputs.so (host generator + device twin)."""
    srcs = [os.path.join(HERE, s) for s in _SOURCES]
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(s) for s in srcs)):
        return LIB_PATH
    bdir = os.path.join(HERE, "_build")
    os.makedirs(bdir, exist_ok=True)
    host_o = os.path.join(bdir, "gen_host.o")
    dev_o = os.path.join(bdir, "gen_dev.o")
    subprocess.check_call(["gcc", "-O2", "-fPIC", "-fopenmp", "-std=c11", "-c",
                           srcs[1], "-o", host_o])
    subprocess.check_call(["nvcc", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
                           "-gencode", "arch=compute_100a,code=sm_100a", "-c", srcs[2],
                           "-o", dev_o])
    tmp = LIB_PATH + ".tmp"
    subprocess.check_call(["nvcc", "-shared", "-Wno-deprecated-gpu-targets", "-Xcompiler", "-fopenmp", host_o, dev_o,
                           "-o", tmp, "-lgomp"])
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        i64, u64, i32, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
        L.gen_stencil_nnz.argtypes = [i32, i64, i64, i64]
        L.gen_stencil_nnz.restype = i64
        L.gen_stencil.argtypes = [i32, i64, i64, i64, i64, i32, u64, vp, vp, vp]
        L.gen_uniform.argtypes = [i64, i32, u64, i64, i64, i64, vp, vp, vp]
        L.gen_vector.argtypes = [u64, i64, vp]
        L.gen_rmat.argtypes = [i32, i32, u64, u64, u64, u64, vp, vp, vp]
        L.gen_rmat.restype = i64
        L.gen_dev_stencil_rowlen.argtypes = [i32, i64, i64, i64, vp, vp]
        L.gen_dev_stencil_fill.argtypes = [i32, i64, i64, i64, i64, vp, vp, vp, vp, i32, i32, u64, vp]
        L.gen_dev_uniform.argtypes = [i64, i32, u64, i64, i64, i64, vp, vp, vp, i32, vp]
        L.gen_dev_rmat_keys.argtypes = [i32, i32, u64, u64, u64, u64, vp, vp]
        L.gen_dev_pair_values.argtypes = [i64, vp, vp, u64, vp, i32, vp]
        L.gen_dev_vector.argtypes = [u64, i64, vp, i32, vp]
        _lib = L
    return _lib


def _ptr(a) -> int:
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


@dataclass
class COO:
    """Sorted, duplicate-free COO triplets (host numpy or device torch arrays)."""
    rows: int
    cols: int
    row: object
    col: object
    val: object

    @property
    def nnz(self) -> int:
        return int(self.row.shape[0])


def rmat_thresholds(a=RMAT_ABC[0], b=RMAT_ABC[1], c=RMAT_ABC[2]):
    t1 = int(a * 2.0 ** 53)
    t2 = int((a + b) * 2.0 ** 53)
    t3 = int((a + b + c) * 2.0 ** 53)
    return t1, t2, t3


# ----------------------------------------------------------------------------- host

def _stencil_n(kind, N):
    if kind == LAP2D:
        return N * N
    if kind > BLOCK27:
        return (kind - BLOCK27) * N ** 3
    return N ** 3


def stencil(kind: int, N: int, r0: int = 0, r1: int | None = None, random_values: bool = False,
            seed: int = MATRIX_SEED, row_base: int | None = None, dtype=np.float64) -> COO:
    n = _stencil_n(kind, N)
    r1 = n if r1 is None else r1
    row_base = r0 if row_base is None else row_base
    L = lib()
    nnz = L.gen_stencil_nnz(kind, N, r0, r1)
    row = np.empty(nnz, np.int32)
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    L.gen_stencil(kind, N, r0, r1, row_base, int(random_values), seed, _ptr(row), _ptr(col), _ptr(val))
    return COO(r1 - r0 if row_base == r0 else n, n, row, col, val.astype(dtype, copy=False))


def block27(N: int, B: int, **kw) -> COO:
    """27-point stencil with B unknowns per point and dense B×B blocks."""
    return stencil(BLOCK27 + B, N, **kw)


def lap2d(N: int, **kw) -> COO:
    return stencil(LAP2D, N, **kw)


def stencil27(N: int, **kw) -> COO:
    return stencil(STENCIL27, N, **kw)


def uniform_k(n: int, k: int, seed: int = MATRIX_SEED, dtype=np.float64) -> COO:
    assert n & (n - 1) == 0 and 0 < k <= 64 and k <= n
    row = np.empty(n * k, np.int32)
    col = np.empty(n * k, np.int32)
    val = np.empty(n * k, np.float64)
    lib().gen_uniform(n, k, seed, 0, n, 0, _ptr(row), _ptr(col), _ptr(val))
    return COO(n, n, row, col, val.astype(dtype, copy=False))


def rmat(scale: int, ef: int = 16, seed: int = MATRIX_SEED, dtype=np.float32) -> COO:
    m = ef << scale
    row = np.empty(m, np.int32)
    col = np.empty(m, np.int32)
    val = np.empty(m, np.float64)
    t1, t2, t3 = rmat_thresholds()
    k = lib().gen_rmat(scale, ef, seed, t1, t2, t3, _ptr(row), _ptr(col), _ptr(val))
    n = 1 << scale
    return COO(n, n, row[:k].copy(), col[:k].copy(), val[:k].astype(dtype))


def vector(n: int, seed: int = X_SEED, dtype=np.float64) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().gen_vector(seed, n, _ptr(out))
    return out.astype(dtype, copy=False)


def value_of(h: np.ndarray) -> np.ndarray:
    """Vectorised gen_value for numpy uint64 hashes (same rule as gen_common.h)."""
    h = h.astype(np.uint64)
    v = 1.0 + (h & np.uint64(0xFFFFF)).astype(np.float64) / 1048576.0
    return np.where((h >> np.uint64(63)) != 0, -v, v)


def random_coo(rows: int, cols: int, nnz: int, seed: int, dtype=np.float64,
               lengths: np.ndarray | None = None) -> COO:
    """Random sorted unique triplets for the parity corpus (numpy PCG64).

    With `lengths`, row i gets exactly lengths[i] distinct columns (ragged /
    power-law / empty-row mixes); otherwise nnz cells are drawn uniformly."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if lengths is None:
        nnz = min(nnz, rows * cols)
        cells = rng.choice(rows * cols, size=nnz, replace=False) if nnz else np.zeros(0, np.int64)
        cells.sort()
        r = (cells // max(cols, 1)).astype(np.int32)
        c = (cells % max(cols, 1)).astype(np.int32)
    else:
        lengths = np.minimum(np.asarray(lengths, np.int64), cols)
        rs, cs = [], []
        for i, L in enumerate(lengths):
            if L == 0:
                continue
            cc = np.sort(rng.choice(cols, size=int(L), replace=False))
            rs.append(np.full(int(L), i, np.int32))
            cs.append(cc.astype(np.int32))
        r = np.concatenate(rs) if rs else np.zeros(0, np.int32)
        c = np.concatenate(cs) if cs else np.zeros(0, np.int32)
    v = value_of(rng.integers(0, np.iinfo(np.uint64).max, size=r.shape[0], dtype=np.uint64,
                              endpoint=True))
    return COO(rows, cols, r, c, v.astype(dtype))


def dense_band(n: int, half: int, seed: int = MATRIX_SEED, dtype=np.float64) -> COO:
    """Row i holds every column of [i - half, i + half) inside [0, n): a
    banded matrix with long, contiguous rows (2·half entries away from the
    edges) — the long-row case of the §8(d) families."""
    w = 2 * half
    r = np.repeat(np.arange(n, dtype=np.int64), w)
    c = r - half + np.tile(np.arange(w, dtype=np.int64), n)
    keep = (c >= 0) & (c < n)
    r, c = r[keep].astype(np.int32), c[keep].astype(np.int32)
    rng = np.random.Generator(np.random.PCG64(seed))
    v = value_of(rng.integers(0, np.iinfo(np.uint64).max, size=r.shape[0], dtype=np.uint64, endpoint=True))
    return COO(n, n, r, c, v.astype(dtype))


def lap2d_long_rows(N: int, every: int, extra: int, seed: int = MATRIX_SEED, dtype=np.float64) -> COO:
    """2D 5-point stencil on an N×N grid where every `every`-th row also holds
    columns i+2 .. i+1+extra (extra < N-2; none of them is a stencil column):
    short regular rows mixed with a few long local rows (the short/long-row
    mix of the §8(d) families). Rows sorted, columns sorted within a row."""
    assert extra < N - 2
    base = lap2d(N, random_values=True, dtype=np.float64)
    n = base.rows
    long_rows = np.arange(0, n, every, dtype=np.int64)
    er = np.repeat(long_rows, extra)
    ec = er + 2 + np.tile(np.arange(extra, dtype=np.int64), long_rows.shape[0])
    keep = ec < n
    er, ec = er[keep], ec[keep]
    r = np.concatenate([base.row.astype(np.int64), er])
    c = np.concatenate([base.col.astype(np.int64), ec])
    order = np.argsort(r * n + c, kind="stable")
    r, c = r[order].astype(np.int32), c[order].astype(np.int32)
    rng = np.random.Generator(np.random.PCG64(seed))
    v = value_of(rng.integers(0, np.iinfo(np.uint64).max, size=r.shape[0], dtype=np.uint64, endpoint=True))
    return COO(n, n, r, c, v.astype(dtype))


def shuffled(coo: COO, seed: int) -> COO:
    rng = np.random.Generator(np.random.PCG64(seed))
    p = rng.permutation(coo.nnz)
    return COO(coo.rows, coo.cols, coo.row[p].copy(), coo.col[p].copy(), coo.val[p].copy())


# ----------------------------------------------------------------------------- device

def _stream(torch):
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _check(rc):
    if rc != 0:
        raise RuntimeError(f"spmv_inputs device generator failed: cuda error {rc}")


def stencil_device(kind: int, N: int, r0: int = 0, r1: int | None = None,
                   random_values: bool = False, seed: int = MATRIX_SEED,
                   row_base: int | None = None, dtype=None, device="cuda") -> COO:
    import torch
    dtype = dtype or torch.float64
    n = _stencil_n(kind, N)
    r1 = n if r1 is None else r1
    row_base = r0 if row_base is None else row_base
    L = lib()
    lens = torch.empty(max(r1 - r0, 1), dtype=torch.int64, device=device)
    _check(L.gen_dev_stencil_rowlen(kind, N, r0, r1, lens.data_ptr(), _stream(torch)))
    lens = lens[: r1 - r0]
    offs = torch.zeros(r1 - r0 + 1, dtype=torch.int64, device=device)
    torch.cumsum(lens, 0, out=offs[1:])
    nnz = int(offs[-1].item()) if r1 > r0 else 0
    row = torch.empty(nnz, dtype=torch.int32, device=device)
    col = torch.empty(nnz, dtype=torch.int32, device=device)
    val = torch.empty(nnz, dtype=dtype, device=device)
    _check(L.gen_dev_stencil_fill(kind, N, r0, r1, row_base, offs.data_ptr(), row.data_ptr(),
                                  col.data_ptr(), val.data_ptr(), int(dtype == torch.float32),
                                  int(random_values), seed, _stream(torch)))
    del lens, offs
    return COO(r1 - r0 if row_base == r0 else n, n, row, col, val)


def uniform_k_device(n: int, k: int, seed: int = MATRIX_SEED, dtype=None, device="cuda") -> COO:
    import torch
    dtype = dtype or torch.float64
    row = torch.empty(n * k, dtype=torch.int32, device=device)
    col = torch.empty(n * k, dtype=torch.int32, device=device)
    val = torch.empty(n * k, dtype=dtype, device=device)
    _check(lib().gen_dev_uniform(n, k, seed, 0, n, 0, row.data_ptr(), col.data_ptr(), val.data_ptr(),
                                 int(dtype == torch.float32), _stream(torch)))
    return COO(n, n, row, col, val)


def rmat_device(scale: int, ef: int = 16, seed: int = MATRIX_SEED, dtype=None, device="cuda") -> COO:
    import torch
    dtype = dtype or torch.float32
    m = ef << scale
    keys = torch.empty(m, dtype=torch.int64, device=device)
    t1, t2, t3 = rmat_thresholds()
    _check(lib().gen_dev_rmat_keys(scale, ef, seed, t1, t2, t3, keys.data_ptr(), _stream(torch)))
    keys = torch.unique(keys, sorted=True)  # dedupe (input generation only)
    row = (keys >> 32).to(torch.int32)
    col = (keys & 0xFFFFFFFF).to(torch.int32)
    del keys
    val = torch.empty(row.shape[0], dtype=dtype, device=device)
    _check(lib().gen_dev_pair_values(row.shape[0], row.data_ptr(), col.data_ptr(), seed + 1,
                                     val.data_ptr(), int(dtype == torch.float32), _stream(torch)))
    n = 1 << scale
    return COO(n, n, row, col, val)


def vector_device(n: int, seed: int = X_SEED, dtype=None, device="cuda"):
    import torch
    dtype = dtype or torch.float64
    out = torch.empty(n, dtype=dtype, device=device)
    _check(lib().gen_dev_vector(seed, n, out.data_ptr(), int(dtype == torch.float32), _stream(torch)))
    return out


# ----------------------------------------------------------------------------- configs

CONFIGS = {
    "c1": dict(desc="2D 5-point Laplacian 64x64 fp64", kind="lap2d", N=64, dtype="f64"),
    "c2": dict(desc="3D 27-point stencil 128^3 fp64", kind="stencil27", N=128, dtype="f64"),
    "c3": dict(desc="RMAT scale 23 edgefactor 16 fp32", kind="rmat", scale=23, ef=16, dtype="f32"),
    "c4": dict(desc="uniform random n=2^22, 32/row fp64", kind="uniform", n=1 << 22, k=32, dtype="f64"),
    "c5": dict(desc="3D 27-point stencil 512^3 fp64", kind="stencil27", N=512, dtype="f64"),
    # extra workloads (not BASELINE configs): block-structured matrices for BELL
    "b2": dict(desc="27-point stencil 100^3 x 2 dof (2x2 blocks) fp64", kind="block27", N=100, B=2, dtype="f64"),
    "b3": dict(desc="27-point stencil 80^3 x 3 dof (3x3 blocks) fp64", kind="block27", N=80, B=3, dtype="f64"),
}


def config_device(name: str, random_values: bool = True, device="cuda", r0: int = 0, r1=None,
                  **override) -> COO:
    """Generate a BASELINE.json config on the device (values random ±[1,2))."""
    import torch
    cfg = dict(CONFIGS[name], **override)
    dt = torch.float32 if cfg["dtype"] == "f32" else torch.float64
    if cfg["kind"] == "lap2d":
        return stencil_device(LAP2D, cfg["N"], r0, r1, random_values=random_values, dtype=dt, device=device)
    if cfg["kind"] == "stencil27":
        return stencil_device(STENCIL27, cfg["N"], r0, r1, random_values=random_values, dtype=dt, device=device)
    if cfg["kind"] == "block27":
        return stencil_device(BLOCK27 + cfg["B"], cfg["N"], r0, r1, random_values=random_values, dtype=dt,
                              device=device)
    if cfg["kind"] == "rmat":
        return rmat_device(cfg["scale"], cfg["ef"], dtype=dt, device=device)
    if cfg["kind"] == "uniform":
        return uniform_k_device(cfg["n"], cfg["k"], dtype=dt, device=device)
    raise KeyError(name)


def config_host(name: str, random_values: bool = True, **override) -> COO:
    cfg = dict(CONFIGS[name], **override)
    dt = np.float32 if cfg["dtype"] == "f32" else np.float64
    if cfg["kind"] == "lap2d":
        return lap2d(cfg["N"], random_values=random_values, dtype=dt)
    if cfg["kind"] == "stencil27":
        return stencil27(cfg["N"], random_values=random_values, dtype=dt)
    if cfg["kind"] == "block27":
        return block27(cfg["N"], cfg["B"], random_values=random_values, dtype=dt)
    if cfg["kind"] == "rmat":
        return rmat(cfg["scale"], cfg["ef"], dtype=dt)
    if cfg["kind"] == "uniform":
        return uniform_k(cfg["n"], cfg["k"], dtype=dt)
    raise KeyError(name)
