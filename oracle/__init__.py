"""oracle — the CPU oracle for the B200 SpMV path.

TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` leg may import this package. The product
package (paper_2302_05662_b200) never imports it and shares no code with it.

Thin numpy/ctypes wrapper over oracle/oracle.c (plain C, fp64, naive loops,
each function citing the PAPER.md passage it follows). The O9 parity check
 is written here in numpy because it is a comparison rule,
not a computation of the method.

Parity-pin status: O1–O8, O10–O12 are pinned by
tests/test_oracle_pins.py. The tuner/selector *choices* and energy numbers
are "parity unpinned" (they depend on hardware timing, not on arithmetic).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.c")
LIB_PATH = os.path.join(HERE, "liboracle.so")

OK, INVALID_ARG, INDEX_OUT_OF_RANGE, DUPLICATE, UNSUPPORTED = 0, 1, 2, 3, 4
STATUS_NAMES = {0: "OK", 1: "INVALID_ARG", 2: "INDEX_OUT_OF_RANGE", 3: "DUPLICATE",
                4: "UNSUPPORTED"}


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= os.path.getmtime(SRC):
        return LIB_PATH
    tmp = LIB_PATH + ".tmp"
    subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-fno-fast-math",
                           "-ffp-contract=off", "-fopenmp", SRC, "-o", tmp, "-lm", "-lgomp"])
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


class _Features(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in
                ("n_rows", "n_cols", "nnz", "max_len", "min_len", "n_empty", "mode",
                 "bw_lower", "bw_upper", "bandwidth")] + \
               [(n, ctypes.c_double) for n in ("mean", "var", "std", "ell_ratio", "median")]


FEATURE_FIELDS = [f[0] for f in _Features._fields_]

_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        i64, vp, d = ctypes.c_int64, ctypes.c_void_p, ctypes.c_double
        L.oracle_canonicalize.argtypes = [i64, i64, i64, vp, vp, vp, vp, vp, vp]
        L.oracle_canonicalize.restype = ctypes.c_int
        L.oracle_csr.argtypes = [i64, i64, vp, vp]
        L.oracle_features.argtypes = [i64, i64, vp, vp, ctypes.POINTER(_Features)]
        L.oracle_features.restype = ctypes.c_int
        L.oracle_ell_npad.argtypes = [i64]
        L.oracle_ell_npad.restype = i64
        L.oracle_ell.argtypes = [i64, vp, vp, vp, i64, i64, vp, vp]
        L.oracle_sell_perm.argtypes = [i64, vp, i64, i64, vp]
        L.oracle_sell_perm.restype = ctypes.c_int
        L.oracle_sell_nslices.argtypes = [i64, i64]
        L.oracle_sell_nslices.restype = i64
        L.oracle_sell_slice_ptr.argtypes = [i64, vp, vp, i64, vp]
        L.oracle_sell_slice_ptr.restype = i64
        L.oracle_sell_fill.argtypes = [i64, vp, vp, vp, vp, i64, vp, vp, vp]
        L.oracle_hyb_auto_k.argtypes = [i64, vp]
        L.oracle_hyb_auto_k.restype = i64
        L.oracle_hyb_tail_nnz.argtypes = [i64, vp, i64]
        L.oracle_hyb_tail_nnz.restype = i64
        L.oracle_hyb_tail.argtypes = [i64, vp, vp, vp, i64, vp, vp, vp]
        L.oracle_bell_kb.argtypes = [i64, vp, vp, i64, i64]
        L.oracle_bell_kb.restype = i64
        L.oracle_bell.argtypes = [i64, vp, vp, vp, i64, i64, i64, i64, vp, vp]
        L.oracle_spmv_csr.argtypes = [i64, vp, vp, vp, vp, d, d, vp, vp, vp]
        L.oracle_dense_spmv.argtypes = [i64, i64, i64, vp, vp, vp, vp, vp]
        L.oracle_power_step.argtypes = [i64, vp, vp, vp, vp, vp, vp,
                                        ctypes.POINTER(d), ctypes.POINTER(d)]
        L.oracle_partition.argtypes = [i64, vp, i64, vp]
        L.oracle_spmv_csr_omp.argtypes = L.oracle_spmv_csr.argtypes
        L.oracle_power_step_omp.argtypes = L.oracle_power_step.argtypes
        L.oracle_omp_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a):
    return a.ctypes.data if a is not None else None


# --------------------------------------------------------------------------- O1/O2

def canonicalize(rows, cols, r, c, v):
    """O1: returns (status, R, C, V) — sorted by (row, col); V in fp64."""
    r, c, v = _c(r, np.int32), _c(c, np.int32), _c(v, np.float64)
    n = r.shape[0]
    R, C, V = np.empty(n, np.int32), np.empty(n, np.int32), np.empty(n, np.float64)
    st = lib().oracle_canonicalize(rows, cols, n, _p(r), _p(c), _p(v), _p(R), _p(C), _p(V))
    return st, R, C, V


def csr(rows, R):
    """O2: row_ptr (int64, rows+1) from the canonical row array."""
    R = _c(R, np.int32)
    rp = np.empty(rows + 1, np.int64)
    lib().oracle_csr(rows, R.shape[0], _p(R), _p(rp))
    return rp


# --------------------------------------------------------------------------- O3

def features(rows, cols, row_ptr, col):
    """O3: Table 2 features + max/min/#empty/bandwidth, as a dict."""
    rp, col = _c(row_ptr, np.int64), _c(col, np.int32)
    f = _Features()
    st = lib().oracle_features(rows, cols, _p(rp), _p(col), ctypes.byref(f))
    if st != OK:
        return st, None
    return st, {name: getattr(f, name) for name in FEATURE_FIELDS}


# --------------------------------------------------------------------------- O4–O7

def ell_npad(rows):
    return lib().oracle_ell_npad(rows)


def ell(rows, row_ptr, col, val, K=None):
    """O4: (K, n_pad, colE, valE) column-major [K][n_pad]."""
    rp, col, val = _c(row_ptr, np.int64), _c(col, np.int32), _c(val, np.float64)
    if K is None:
        K = int(np.max(np.diff(rp))) if rows > 0 else 0
    n_pad = ell_npad(rows)
    colE = np.empty(K * n_pad, np.int32)
    valE = np.empty(K * n_pad, np.float64)
    lib().oracle_ell(rows, _p(rp), _p(col), _p(val), K, n_pad, _p(colE), _p(valE))
    return K, n_pad, colE, valE


def sell(rows, row_ptr, col, val, C, sigma):
    """O5: (perm, slice_ptr, colS, valS) for SELL-C-sigma."""
    rp, col, val = _c(row_ptr, np.int64), _c(col, np.int32), _c(val, np.float64)
    perm = np.empty(max(rows, 1), np.int32)
    st = lib().oracle_sell_perm(rows, _p(rp), C, sigma, _p(perm))
    if st != OK:
        raise ValueError(f"oracle_sell_perm: {STATUS_NAMES[st]}")
    perm = perm[:rows]
    ns = lib().oracle_sell_nslices(rows, C)
    sp = np.empty(ns + 1, np.int64)
    total = lib().oracle_sell_slice_ptr(rows, _p(rp), _p(perm), C, _p(sp))
    colS = np.empty(total, np.int32)
    valS = np.empty(total, np.float64)
    lib().oracle_sell_fill(rows, _p(rp), _p(col), _p(val), _p(perm), C, _p(sp), _p(colS), _p(valS))
    return perm, sp, colS, valS


def hyb_auto_k(rows, row_ptr):
    rp = _c(row_ptr, np.int64)
    return lib().oracle_hyb_auto_k(rows, _p(rp))


def hyb(rows, row_ptr, col, val, K=None):
    """O6: (K, n_pad, colE, valE, tail_row, tail_col, tail_val)."""
    rp, col, val = _c(row_ptr, np.int64), _c(col, np.int32), _c(val, np.float64)
    if K is None:
        K = hyb_auto_k(rows, rp)
    K_, n_pad, colE, valE = ell(rows, rp, col, val, K)
    t = lib().oracle_hyb_tail_nnz(rows, _p(rp), K)
    tr, tc, tv = np.empty(t, np.int32), np.empty(t, np.int32), np.empty(t, np.float64)
    lib().oracle_hyb_tail(rows, _p(rp), _p(col), _p(val), K, _p(tr), _p(tc), _p(tv))
    return K, n_pad, colE, valE, tr, tc, tv


def bell(rows, row_ptr, col, val, bh=2, bw=2):
    """O13: (Kb, nbr_pad, bcol[Kb·nbr_pad], bval[Kb·bh·bw·nbr_pad]) — value plane
    e = r·bw + c of slot k at (k·bh·bw + e)·nbr_pad + I."""
    rp, col, val = _c(row_ptr, np.int64), _c(col, np.int32), _c(val, np.float64)
    kb = lib().oracle_bell_kb(rows, _p(rp), _p(col), bh, bw)
    nbr = (rows + bh - 1) // bh
    nbr_pad = (nbr + 127) // 128 * 128
    bcol = np.empty(kb * nbr_pad, np.int32)
    bval = np.empty(kb * bh * bw * nbr_pad, np.float64)
    lib().oracle_bell(rows, _p(rp), _p(col), _p(val), bh, bw, kb, nbr_pad, _p(bcol), _p(bval))
    return kb, nbr_pad, bcol, bval


# --------------------------------------------------------------------------- O8–O12

def spmv_csr(rows, row_ptr, col, val, x, alpha=1.0, beta=0.0, y_in=None, all_cores=False):
    """O8: (y, abs_sum) in fp64; abs_sum_i = Σ|a_ik x_k|. `all_cores` runs the
    same per-row loop under OpenMP (timing leg; bitwise the same y)."""
    rp, col, val, x = _c(row_ptr, np.int64), _c(col, np.int32), _c(val, np.float64), _c(x, np.float64)
    y = np.empty(rows, np.float64)
    a = np.empty(rows, np.float64)
    yin = _c(y_in, np.float64) if (y_in is not None and beta != 0.0) else None
    fn = lib().oracle_spmv_csr_omp if all_cores else lib().oracle_spmv_csr
    fn(rows, _p(rp), _p(col), _p(val), _p(x), alpha, beta, _p(yin), _p(y), _p(a))
    return y, a


def omp_threads() -> int:
    """Threads the all-core leg uses (OMP_NUM_THREADS or the host's cores)."""
    return int(lib().oracle_omp_threads())


def dense_spmv(rows, cols, r, c, v, x):
    """O10: dense brute force (tiny sizes only)."""
    r, c, v, x = _c(r, np.int32), _c(c, np.int32), _c(v, np.float64), _c(x, np.float64)
    y = np.empty(rows, np.float64)
    lib().oracle_dense_spmv(rows, cols, r.shape[0], _p(r), _p(c), _p(v), _p(x), _p(y))
    return y


def power_step(rows, row_ptr, col, val, x, all_cores=False):
    """O11: (y, x_next, lambda, s)."""
    rp, col, val, x = _c(row_ptr, np.int64), _c(col, np.int32), _c(val, np.float64), _c(x, np.float64)
    y, xn = np.empty(rows, np.float64), np.empty(rows, np.float64)
    lam, s = ctypes.c_double(), ctypes.c_double()
    (lib().oracle_power_step_omp if all_cores else lib().oracle_power_step)(rows, _p(rp), _p(col), _p(val), _p(x), _p(y), _p(xn),
                            ctypes.byref(lam), ctypes.byref(s))
    return y, xn, lam.value, s.value


def partition(rows, row_ptr, P):
    """O12: nnz-balanced row bounds (P+1)."""
    rp = _c(row_ptr, np.int64)
    b = np.empty(P + 1, np.int64)
    lib().oracle_partition(rows, _p(rp), P, _p(b))
    return b


# --------------------------------------------------------------------------- O9

TAU = {"f64": 1e-12, "f32": 1e-5}


def parity_check(y, y_ref, abs_ref, alpha, beta, y_in, tau):
    """O9: per row, NaN<->NaN, ±Inf exact, else
    |y − y_ref| <= tau·(|α|·a_i + |β|·|y_in_i|). Returns (ok, worst_ratio, bad_rows)."""
    y = np.asarray(y, np.float64)
    y_ref = np.asarray(y_ref, np.float64)
    bound = tau * (abs(alpha) * np.asarray(abs_ref, np.float64))
    if beta != 0.0 and y_in is not None:
        bound = bound + tau * abs(beta) * np.abs(np.asarray(y_in, np.float64))
    nan_ref = np.isnan(y_ref)
    inf_ref = np.isinf(y_ref)
    fin = ~(nan_ref | inf_ref)
    bad = np.zeros(y.shape, bool)
    bad |= nan_ref & ~np.isnan(y)
    bad |= inf_ref & (y != y_ref)
    err = np.where(fin, np.abs(y - np.where(fin, y_ref, 0.0)), 0.0)
    err = np.where(np.isnan(err), np.inf, err)
    bad |= fin & (err > bound)
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(fin & (err > 0), err / np.where(bound > 0, bound, np.inf), 0.0)
        ratio = np.where(fin & (err > 0) & (bound == 0), np.inf, ratio)
    worst = float(ratio.max()) if ratio.size else 0.0
    return (not bad.any()), worst, np.nonzero(bad)[0]
