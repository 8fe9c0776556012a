"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself:
the Appendix D worked example, closed forms, textbook
examples, invariants, and pure-Python brute force on tiny
inputs. No GPU. Each test names the oracle item (O1–O12) it pins.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import spmv_inputs as si

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "appendix_d.json")))


def golden_coo():
    t = np.array(GOLD["triplets_shuffled"], dtype=np.float64)
    return GOLD["rows"], GOLD["cols"], t[:, 0].astype(np.int32), t[:, 1].astype(np.int32), t[:, 2]


def dense_of(rows, cols, r, c, v):
    D = [[0.0] * cols for _ in range(rows)]
    for a, b, w in zip(r, c, v):
        D[int(a)][int(b)] = float(w)
    return D


def build(coo):
    st, R, C, V = oracle.canonicalize(coo.rows, coo.cols, coo.row, coo.col, coo.val)
    assert st == oracle.OK
    return oracle.csr(coo.rows, R), C, V


# ------------------------------------------------------------------ O1 / O2

def test_appendix_d_canonical_and_csr():
    rows, cols, r, c, v = golden_coo()
    st, R, C, V = oracle.canonicalize(rows, cols, r, c, v)
    assert st == oracle.OK
    rp = oracle.csr(rows, R)
    assert rp.tolist() == GOLD["row_ptr"]
    assert C.tolist() == GOLD["col"]
    assert V.tolist() == GOLD["val"]


@pytest.mark.parametrize("seed", range(8))
def test_canonicalize_bruteforce_and_permutation_invariance(seed):
    coo = si.random_coo(13, 11, 40, seed)
    sh = si.shuffled(coo, seed + 100)
    st, R, C, V = oracle.canonicalize(sh.rows, sh.cols, sh.row, sh.col, sh.val)
    assert st == oracle.OK
    ref = sorted(zip(sh.row.tolist(), sh.col.tolist(), sh.val.tolist()))
    assert list(zip(R.tolist(), C.tolist(), V.tolist())) == ref
    st2, R2, C2, V2 = oracle.canonicalize(coo.rows, coo.cols, coo.row, coo.col, coo.val)
    assert (R2 == R).all() and (C2 == C).all() and (V2 == V).all()


def test_canonicalize_errors_and_zeros():
    r = np.array([0, 1, 0], np.int32); c = np.array([1, 1, 1], np.int32)
    v = np.array([1.0, 0.0, 2.0])
    assert oracle.canonicalize(2, 2, r, c, v)[0] == oracle.DUPLICATE
    assert oracle.canonicalize(2, 2, np.array([2], np.int32), np.array([0], np.int32),
                               np.array([1.0]))[0] == oracle.INDEX_OUT_OF_RANGE
    assert oracle.canonicalize(2, 2, np.array([0], np.int32), np.array([-1], np.int32),
                               np.array([1.0]))[0] == oracle.INDEX_OUT_OF_RANGE
    assert oracle.canonicalize(-1, 2, r[:0], c[:0], v[:0])[0] == oracle.INVALID_ARG
    assert oracle.canonicalize(2 ** 31, 2, r[:0], c[:0], v[:0])[0] == oracle.UNSUPPORTED
    st, R, C, V = oracle.canonicalize(2, 2, r[:2], c[:2], v[:2])                 # explicit zero kept
    assert st == oracle.OK and V.tolist() == [1.0, 0.0]


def test_csr_textbook_examples():
    # identity -> [0,1,2,3]; empty 4x4 -> [0,0,0,0,0]
    assert oracle.csr(3, np.array([0, 1, 2], np.int32)).tolist() == [0, 1, 2, 3]
    assert oracle.csr(4, np.zeros(0, np.int32)).tolist() == [0, 0, 0, 0, 0]
    coo = si.random_coo(50, 40, 300, 7, lengths=np.random.default_rng(1).integers(0, 9, 50))
    rp, C, V = build(coo)
    assert rp[-1] == coo.nnz and (np.diff(rp) >= 0).all()
    # reconstruct-dense exact
    D = dense_of(coo.rows, coo.cols, coo.row, coo.col, coo.val)
    for i in range(coo.rows):
        for k in range(rp[i], rp[i + 1]):
            assert D[i][C[k]] == V[k]
    assert sum(1 for row in D for w in row if w != 0.0) == coo.nnz


# ------------------------------------------------------------------ O3 features

def brute_features(rows, cols, rp, col):
    L = [int(rp[i + 1] - rp[i]) for i in range(rows)]
    n = rows
    S1, S2 = sum(L), sum(l * l for l in L)
    s = sorted(L)
    counts = {}
    for l in L:
        counts[l] = counts.get(l, 0) + 1
    best = max(counts.values())
    lo = hi = 0
    for i in range(rows):
        for k in range(rp[i], rp[i + 1]):
            lo = max(lo, i - int(col[k])); hi = max(hi, int(col[k]) - i)
    return dict(nnz=S1, max_len=max(L), min_len=min(L), n_empty=L.count(0),
                mode=min(l for l, c in counts.items() if c == best),
                mean_exact=Fraction(S1, n), var_exact=Fraction(n * S2 - S1 * S1, n * n),
                median_exact=Fraction(s[(n - 1) // 2] + s[n // 2], 2),
                ell_exact=Fraction(S1, n * max(L)) if max(L) else Fraction(1),
                bw_lower=lo, bw_upper=hi)


def ulps(a, b):
    if a == b:
        return 0
    return abs(a - b) / math.ulp(max(abs(a), abs(b)))


def test_features_appendix_d():
    rows, cols = GOLD["rows"], GOLD["cols"]
    st, f = oracle.features(rows, cols, np.array(GOLD["row_ptr"]), np.array(GOLD["col"]))
    assert st == oracle.OK
    for k, v in GOLD["features"].items():
        assert f[k] == v, k
    assert np.float64(f["var"]).view(np.uint64) == 0x4000000000000000
    assert np.float64(f["std"]).view(np.uint64) == 0x3FF6A09E667F3BCD


@pytest.mark.parametrize("seed", range(10))
def test_features_bruteforce_random(seed):
    rng = np.random.default_rng(seed)
    rows = int(rng.integers(1, 60))
    lengths = rng.integers(0, 12, rows) * (rng.random(rows) < 0.8)
    coo = si.random_coo(rows, 40, 0, seed, lengths=lengths)
    rp, C, V = build(coo)
    st, f = oracle.features(coo.rows, coo.cols, rp, C)
    b = brute_features(coo.rows, coo.cols, rp, C)
    for k in ("nnz", "max_len", "min_len", "n_empty", "mode", "bw_lower", "bw_upper"):
        assert f[k] == b[k], k
    assert f["bandwidth"] == max(b["bw_lower"], b["bw_upper"])
    assert f["median"] == float(b["median_exact"])          # exact (half-integers)
    assert ulps(f["mean"], float(b["mean_exact"])) <= 0.5
    assert ulps(f["var"], float(b["var_exact"])) <= 2
    assert ulps(f["ell_ratio"], float(b["ell_exact"])) <= 0.5
    assert abs(f["std"] - math.sqrt(float(b["var_exact"]))) <= 4 * math.ulp(max(f["std"], 1e-300))
    # identity ELL_ratio · max = mean (holds for 28/30 plotted matrices)
    assert abs(f["ell_ratio"] * f["max_len"] - f["mean"]) <= 1e-12 * max(1.0, f["mean"])


def test_features_empty_rows_matrix():
    st, f = oracle.features(4, 4, np.zeros(5, np.int64), np.zeros(0, np.int32))
    assert st == oracle.OK
    assert f["ell_ratio"] == 1.0 and f["max_len"] == 0 and f["n_empty"] == 4
    assert f["median"] == 0.0 and f["mode"] == 0 and f["bandwidth"] == 0
    assert oracle.features(0, 4, np.zeros(1, np.int64), np.zeros(0, np.int32))[0] == oracle.INVALID_ARG


def stencil27_closed_form(N):
    """Appendix B: rows of 27/18/12/8 entries with counts (N-2)^3, 6(N-2)^2, 12(N-2), 8."""
    counts = {27: (N - 2) ** 3, 18: 6 * (N - 2) ** 2, 12: 12 * (N - 2), 8: 8}
    n = N ** 3
    S1 = sum(l * c for l, c in counts.items())
    S2 = sum(l * l * c for l, c in counts.items())
    assert S1 == (3 * N - 2) ** 3
    return n, S1, S2


@pytest.mark.parametrize("N", [3, 16, 33])
def test_features_stencil27_closed_form(N):
    coo = si.stencil27(N)
    rp, C, V = build(coo)
    st, f = oracle.features(coo.rows, coo.cols, rp, C)
    n, S1, S2 = stencil27_closed_form(N)
    assert f["nnz"] == S1 and f["max_len"] == 27 and f["min_len"] == 8
    assert f["mean"] == float(Fraction(S1, n))
    assert ulps(f["var"], float(Fraction(n * S2 - S1 * S1, n * n))) <= 2
    assert f["ell_ratio"] == float(Fraction(S1, 27 * n))
    assert f["bandwidth"] == N * N + N + 1
    counts = [(8, 8), (12, 12 * (N - 2)), (18, 6 * (N - 2) ** 2), (27, (N - 2) ** 3)]
    order = [l for l, c in counts for _ in range(c)]          # sorted lengths, closed form
    assert f["median"] == (order[(n - 1) // 2] + order[n // 2]) / 2
    assert f["mode"] == min(l for l, c in counts if c == max(c for _, c in counts))


def test_features_stencil27_128_appendix_b():
    # SURVEY Appendix B printed values for N = 128 (c2); computed from counts only.
    n, S1, S2 = stencil27_closed_form(128)
    assert S1 == 55_742_968 and S2 == 1_489_355_288
    assert float(Fraction(S1, n)) == 26.580318450927734
    assert abs(float(Fraction(n * S2 - S1 * S1, n * n)) - 3.666614131987444) < 1e-15
    assert abs(float(Fraction(S1, 27 * n)) - 0.9844562389232494) < 1e-16


def test_features_lap2d_64_appendix_b():
    coo = si.lap2d(64)
    rp, C, V = build(coo)
    st, f = oracle.features(coo.rows, coo.cols, rp, C)
    assert f["nnz"] == 20224 and f["mean"] == 4.9375 and f["var"] == 0.060546875
    assert f["max_len"] == 5 and f["min_len"] == 3 and f["ell_ratio"] == 0.9875
    assert f["median"] == 5.0 and f["mode"] == 5 and f["bandwidth"] == 64


def test_features_uniform():
    coo = si.uniform_k(1 << 10, 32)
    rp, C, V = build(coo)
    st, f = oracle.features(coo.rows, coo.cols, rp, C)
    assert f["mean"] == 32.0 and f["var"] == 0.0 and f["ell_ratio"] == 1.0
    assert f["median"] == 32.0 and f["mode"] == 32 and f["min_len"] == 32
    # SPEC S:304 / shar_te2-b3 (P:690/711/731): uniform 4/row -> avg 4, var 0, ELL_ratio 1
    coo4 = si.uniform_k(1 << 8, 4)
    rp, C, V = build(coo4)
    f4 = oracle.features(coo4.rows, coo4.cols, rp, C)[1]
    assert (f4["mean"], f4["var"], f4["ell_ratio"], f4["median"]) == (4.0, 0.0, 1.0, 4.0)


# ------------------------------------------------------------------ O4–O6 layouts

def reconstruct_ell(K, n_pad, colE, valE, rows, cols):
    D = [[0.0] * cols for _ in range(rows)]
    for k in range(K):
        for i in range(n_pad):
            c = colE[k * n_pad + i]
            if c >= 0:
                assert i < rows and D[i][c] == 0.0
                D[i][c] = valE[k * n_pad + i]
            else:
                assert valE[k * n_pad + i] == 0.0
    return D


def test_ell_appendix_d_and_spec_example():
    rp = np.array(GOLD["row_ptr"]); C = np.array(GOLD["col"]); V = np.array(GOLD["val"], float)
    K, n_pad, colE, valE = oracle.ell(5, rp, C, V)
    assert (K, n_pad) == (GOLD["ell"]["K"], GOLD["ell"]["n_pad"])
    for k in range(K):
        assert colE[k * n_pad:k * n_pad + 5].tolist() == GOLD["ell"]["col_rows_0_4"][k]
        assert valE[k * n_pad:k * n_pad + 5].tolist() == GOLD["ell"]["val_rows_0_4"][k]
        assert (colE[k * n_pad + 5:(k + 1) * n_pad] == -1).all()
    # rows {2,4,1} -> K = 4, 5 padded slots before row padding
    rp2 = np.array([0, 2, 6, 7]); C2 = np.array([0, 1, 0, 1, 2, 3, 0]); V2 = np.ones(7)
    K2, n2, colE2, _ = oracle.ell(3, rp2, C2, V2)
    assert K2 == 4 and sum((colE2[k * n2:k * n2 + 3] == -1).sum() for k in range(K2)) == 5
    assert (colE2 == -1).sum() == n2 * K2 - 7


def test_ell_reconstructs_dense():
    coo = si.random_coo(70, 30, 0, 3, lengths=np.random.default_rng(3).integers(0, 7, 70))
    rp, C, V = build(coo)
    K, n_pad, colE, valE = oracle.ell(coo.rows, rp, C, V)
    assert n_pad == 128
    assert reconstruct_ell(K, n_pad, colE, valE, coo.rows, coo.cols) == dense_of(
        coo.rows, coo.cols, coo.row, coo.col, coo.val)


def test_sell_appendix_d():
    rp = np.array(GOLD["row_ptr"]); C = np.array(GOLD["col"]); V = np.array(GOLD["val"], float)
    for key, (c, s) in (("sell_C2_s1", (2, 1)), ("sell_C4_s4", (4, 4))):
        perm, sp, colS, valS = oracle.sell(5, rp, C, V, c, s)
        g = GOLD[key]
        assert perm.tolist() == g["perm"] and sp.tolist() == g["slice_ptr"]
        assert colS.tolist() == g["col"] and valS.tolist() == g["val"]


def reconstruct_sell(perm, sp, colS, valS, C, rows, cols):
    D = [[0.0] * cols for _ in range(rows)]
    for s in range(len(sp) - 1):
        w = (sp[s + 1] - sp[s]) // C
        for k in range(w):
            for j in range(C):
                pos = sp[s] + k * C + j
                if colS[pos] >= 0:
                    i = perm[s * C + j]
                    D[i][colS[pos]] = valS[pos]
    return D


@pytest.mark.parametrize("C,sigma", [(1, 1), (2, 1), (4, 8), (8, 8), (32, 64), (64, 1)])
def test_sell_reconstruct_and_invariants(C, sigma):
    rng = np.random.default_rng(C + sigma)
    coo = si.random_coo(77, 50, 0, 5, lengths=rng.integers(0, 15, 77) * (rng.random(77) < 0.7))
    rp, Ci, V = build(coo)
    perm, sp, colS, valS = oracle.sell(coo.rows, rp, Ci, V, C, sigma)
    assert sorted(perm.tolist()) == list(range(coo.rows))
    L = np.diff(rp)
    for w0 in range(0, coo.rows, sigma):                    # σ-window sort (L desc, row asc)
        win = perm[w0:w0 + sigma].tolist()
        assert sorted(win) == list(range(w0, min(w0 + sigma, coo.rows)))
        assert win == sorted(win, key=lambda i: (-L[i], i))
    for s in range(len(sp) - 1):                            # slice width = max lane length
        lanes = [L[perm[q]] for q in range(s * C, min((s + 1) * C, coo.rows))]
        assert sp[s + 1] - sp[s] == C * max(lanes)
    assert reconstruct_sell(perm, sp, colS, valS, C, coo.rows, coo.cols) == dense_of(
        coo.rows, coo.cols, coo.row, coo.col, coo.val)


def test_sell_spec_examples():
    # rows {3,1,2,2}, C = 2 -> widths [3, 2], 2 padded slots
    rp = np.array([0, 3, 4, 6, 8]); Ci = np.array([0, 1, 2, 0, 0, 1, 1, 2]); V = np.ones(8)
    perm, sp, colS, _ = oracle.sell(4, rp, Ci, V, 2, 1)
    assert np.diff(sp).tolist() == [6, 4] and (colS == -1).sum() == 2
    # one slice of height = rows, σ = 1 has exactly ELL's padding (no phantom rows)
    coo = si.random_coo(128, 40, 0, 9, lengths=np.random.default_rng(9).integers(0, 9, 128))
    rp, Ci, V = build(coo)
    perm, sp, colS, _ = oracle.sell(128, rp, Ci, V, 128, 1)
    K, n_pad, colE, _ = oracle.ell(128, rp, Ci, V)
    assert (colS == -1).sum() == (colE == -1).sum()
    with pytest.raises(ValueError):
        oracle.sell(128, rp, Ci, V, 4, 6)        # σ must be 1 or a multiple of C


def test_hyb_rules():
    rp = np.array(GOLD["row_ptr"]); C = np.array(GOLD["col"]); V = np.array(GOLD["val"], float)
    assert oracle.hyb_auto_k(5, rp) == GOLD["hyb_auto_K"]
    K, n_pad, colE, valE, tr, tc, tv = oracle.hyb(5, rp, C, V, 2)
    assert [list(t) for t in zip(tr.tolist(), tc.tolist(), tv.tolist())] == GOLD["hyb_K2_tail"]
    # Appendix B: c1 -> K_h = 3 with a 7,936-entry tail; c4 -> 32; 27-pt -> 27
    coo = si.lap2d(64)
    rp1, C1, V1 = build(coo)
    assert oracle.hyb_auto_k(coo.rows, rp1) == 3
    K, n_pad, colE, valE, tr, tc, tv = oracle.hyb(coo.rows, rp1, C1, V1)
    assert tr.shape[0] == 7936
    D = reconstruct_ell(K, n_pad, colE, valE, coo.rows, coo.cols)
    for a, b, w in zip(tr, tc, tv):
        assert D[a][b] == 0.0
        D[a][b] = w
    assert D == dense_of(coo.rows, coo.cols, coo.row, coo.col, coo.val)
    assert oracle.hyb_auto_k(1 << 12, build(si.uniform_k(1 << 12, 32))[0]) == 32
    c2 = si.stencil27(24)
    assert oracle.hyb_auto_k(c2.rows, build(c2)[0]) == 27
    # K_h = max -> empty tail; K_h = 0 -> pure COO
    assert oracle.hyb(coo.rows, rp1, C1, V1, 5)[4].shape[0] == 0
    assert oracle.hyb(coo.rows, rp1, C1, V1, 0)[4].shape[0] == coo.nnz


# ------------------------------------------------------------------ O8 SpMV

def test_spmv_appendix_d():
    rp = np.array(GOLD["row_ptr"]); C = np.array(GOLD["col"]); V = np.array(GOLD["val"], float)
    x = np.array(GOLD["x"], float)
    y, a = oracle.spmv_csr(5, rp, C, V, x)
    assert y.tolist() == GOLD["Ax"]
    y, a = oracle.spmv_csr(5, rp, C, V, x, GOLD["alpha"], GOLD["beta"], np.array(GOLD["y_in"], float))
    assert y.tolist() == GOLD["y_axpby"]
    y, a = oracle.spmv_csr(5, rp, C, V, np.ones(6))
    assert y.tolist() == GOLD["A_ones"]
    y, a = oracle.spmv_csr(5, rp, C, V, x, 2.5, 0.0, np.full(5, np.nan))   # β = 0: y not read
    assert np.isfinite(y).all()


@pytest.mark.parametrize("seed", range(6))
def test_spmv_equals_dense_bruteforce(seed):
    rng = np.random.default_rng(seed)
    rows, cols = int(rng.integers(1, 40)), int(rng.integers(1, 40))
    coo = si.random_coo(rows, cols, int(rng.integers(0, rows * cols)), seed)
    # integer values -> every partial sum exact -> Neumaier == plain dense sum exactly
    vi = rng.integers(-8, 9, coo.nnz).astype(float)
    xi = rng.integers(-8, 9, cols).astype(float)
    rp, C, V = build(si.COO(rows, cols, coo.row, coo.col, vi))
    y, a = oracle.spmv_csr(rows, rp, C, V, xi)
    yd = oracle.dense_spmv(rows, cols, coo.row, coo.col, vi, xi)
    D = dense_of(rows, cols, coo.row, coo.col, vi)
    yp = [sum(D[i][j] * xi[j] for j in range(cols)) for i in range(rows)]
    assert (y == yd).all() and y.tolist() == yp
    # random values: within the O9 bound of the dense brute force
    xr = si.vector(cols, seed=seed)
    rp, C, V = build(coo)
    y, a = oracle.spmv_csr(rows, rp, C, V, xr)
    yd = oracle.dense_spmv(rows, cols, coo.row, coo.col, coo.val, xr)
    assert (np.abs(y - yd) <= 4e-16 * 40 * a).all()


def test_spmv_unit_vectors_give_columns():
    coo = si.random_coo(30, 20, 200, 11)
    rp, C, V = build(coo)
    D = dense_of(30, 20, coo.row, coo.col, coo.val)
    for j in range(20):
        e = np.zeros(20); e[j] = 1.0
        y, _ = oracle.spmv_csr(30, rp, C, V, e)
        assert y.tolist() == [D[i][j] for i in range(30)]


def test_spmv_row_sums_stencils():
    # A·1 = row sums: 5-pt interior 0 / edge 1 / corner 2; 27-pt 27 − L
    coo = si.lap2d(16)
    rp, C, V = build(coo)
    y, _ = oracle.spmv_csr(coo.rows, rp, C, V, np.ones(coo.cols))
    L = np.diff(rp)
    assert (y == 5 - L).all()
    coo = si.stencil27(9)
    rp, C, V = build(coo)
    y, _ = oracle.spmv_csr(coo.rows, rp, C, V, np.ones(coo.cols))
    assert (y == 27 - np.diff(rp)).all()


def test_spmv_lap2d_quadratic():
    N = 20
    coo = si.lap2d(N)
    rp, C, V = build(coo)
    gy = np.arange(N * N) // N
    y, _ = oracle.spmv_csr(coo.rows, rp, C, V, (gy ** 2).astype(float))
    interior = [r for r in range(N * N) if 0 < r // N < N - 1 and 0 < r % N < N - 1]
    assert (y[interior] == -2.0).all()


@pytest.mark.parametrize("p,q", [(1, 1), (3, 7)])
def test_spmv_dirichlet_eigenvector(p, q):
    N = 64
    coo = si.lap2d(N)
    rp, C, V = build(coo)
    gx, gy = np.arange(N * N) % N, np.arange(N * N) // N
    v = np.sin(p * np.pi * (gx + 1) / (N + 1)) * np.sin(q * np.pi * (gy + 1) / (N + 1))
    lam = 4 - 2 * np.cos(p * np.pi / (N + 1)) - 2 * np.cos(q * np.pi / (N + 1))
    y, a = oracle.spmv_csr(coo.rows, rp, C, V, v)
    assert (np.abs(y - lam * v) <= 1e-13 * (a + 1e-300) + 1e-15).all()


def test_spmv_alpha_beta_special_cases():
    coo = si.random_coo(25, 25, 120, 4)
    rp, C, V = build(coo)
    yin = si.vector(25, seed=si.Y_SEED)
    y, _ = oracle.spmv_csr(25, rp, C, V, np.zeros(25), 1.0, 0.75, yin)
    assert (y == 0.75 * yin).all()
    y, _ = oracle.spmv_csr(25, rp, C, V, np.full(25, np.inf), 0.0, 2.0, yin)   # α = 0: A not read
    assert (y == 2.0 * yin).all()


# ------------------------------------------------------------------ O9 / O11 / O12

def test_parity_check_rule():
    ok, w, bad = oracle.parity_check([1.0, np.nan, np.inf], [1.0, np.nan, np.inf], [1, 1, 1], 1, 0, None, 1e-12)
    assert ok
    ok, w, bad = oracle.parity_check([1.0 + 1e-11], [1.0], [1.0], 1, 0, None, 1e-12)
    assert not ok and bad.tolist() == [0]
    ok, w, bad = oracle.parity_check([1.0 + 1e-13], [1.0], [1.0], 1, 0, None, 1e-12)
    assert ok and 0 < w < 1
    ok, w, bad = oracle.parity_check([np.nan], [1.0], [1.0], 1, 0, None, 1e-12)
    assert not ok


def test_omp_leg_bitwise():
    """The all-core timing leg (SURVEY §8(d) CPU baseline) sums each row on one
    thread in the same order: y, Σ|a·x| and the power step are bitwise the
    1-thread oracle's, and the closed form A·1 = row sums still holds."""
    coo = si.stencil27(24, random_values=True)
    rp, C, V = build(coo)
    x = si.vector(coo.cols)
    y1, a1 = oracle.spmv_csr(coo.rows, rp, C, V, x, 2.5, -0.5, x[: coo.rows])
    y2, a2 = oracle.spmv_csr(coo.rows, rp, C, V, x, 2.5, -0.5, x[: coo.rows], all_cores=True)
    assert np.array_equal(y1.view(np.int64), y2.view(np.int64)) and np.array_equal(a1, a2)
    p1 = oracle.power_step(coo.rows, rp, C, V, x / np.linalg.norm(x))
    p2 = oracle.power_step(coo.rows, rp, C, V, x / np.linalg.norm(x), all_cores=True)
    assert np.array_equal(p1[0], p2[0]) and np.array_equal(p1[1], p2[1]) and p1[2:] == p2[2:]
    lap = si.stencil27(24)
    rp, C, V = build(lap)
    y, _ = oracle.spmv_csr(lap.rows, rp, C, V, np.ones(lap.cols), all_cores=True)
    assert (y == 27 - np.diff(rp)).all()
    assert oracle.omp_threads() >= 1


def test_power_step_closed_forms():
    N = 64
    coo = si.lap2d(N)
    rp, C, V = build(coo)
    n = N * N
    x0 = np.full(n, 1.0 / 8.0 ** 2)                 # ‖x0‖ = 1 for n = 4096 (1/64 each)
    y, xn, lam, s = oracle.power_step(n, rp, C, V, x0)
    assert (y == (5 - np.diff(rp)) / 64.0).all()    # step 1 = row sums / √n, exact
    gx, gy = np.arange(n) % N, np.arange(n) // N
    v = np.sin(N * np.pi * (gx + 1) / (N + 1)) * np.sin(N * np.pi * (gy + 1) / (N + 1))
    v /= np.linalg.norm(v)
    y, xn, lam, s = oracle.power_step(n, rp, C, V, v)
    assert abs(lam - 7.995328907329307) < 1e-12      # Appendix B λ_max(5-pt, 64²)
    assert abs(np.linalg.norm(xn) - 1.0) < 1e-14


def test_partition_invariants():
    rng = np.random.default_rng(5)
    for P in (1, 2, 3, 4, 8):
        coo = si.random_coo(200, 60, 0, P, lengths=rng.integers(0, 30, 200))
        rp, C, V = build(coo)
        b = oracle.partition(coo.rows, rp, P)
        nnz = int(rp[-1])
        assert b[0] == 0 and b[-1] == coo.rows and (np.diff(b) >= 0).all()
        expect = [int(np.searchsorted(rp, -(-k * nnz // P), side="left")) for k in range(1, P)]
        assert b[1:-1].tolist() == expect
        per = np.diff(rp[b])
        assert per.sum() == nnz
        assert (np.abs(per - nnz / P) <= np.diff(rp).max() + 1).all()


# ------------------------------------------------------------------ O13 BELL

def reconstruct_bell(kb, nbr_pad, bcol, bval, b, rows, cols):
    D = [[0.0] * cols for _ in range(rows)]
    for k in range(kb):
        for I in range(nbr_pad):
            J = bcol[k * nbr_pad + I]
            for r in range(b):
                for c in range(b):
                    v = bval[(k * b * b + r * b + c) * nbr_pad + I]
                    if J < 0:
                        assert v == 0.0
                        continue
                    i, j = I * b + r, J * b + c
                    if i < rows and j < cols:
                        D[i][j] += v
                    else:
                        assert v == 0.0
    return D


def test_bell_spec_examples():
    # 4x4 with nonzeros confined to the top-left 2x2 -> 1 stored block
    rp = np.array([0, 2, 4, 4, 4]); C = np.array([0, 1, 0, 1]); V = np.array([1.0, 2, 3, 4])
    kb, nbr_pad, bcol, bval = oracle.bell(4, rp, C, V, 2, 2)
    assert kb == 1 and (bcol >= 0).sum() == 1 and bcol[0] == 0
    # 4x4 dense -> 4 stored blocks, each fully dense
    rpd = np.array([0, 4, 8, 12, 16]); Cd = np.tile(np.arange(4), 4); Vd = np.arange(1.0, 17.0)
    kb, nbr_pad, bcol, bval = oracle.bell(4, rpd, Cd, Vd, 2, 2)
    assert kb == 2 and (bcol >= 0).sum() == 4
    assert reconstruct_bell(kb, nbr_pad, bcol, bval, 2, 4, 4) == [[float(4 * i + j + 1) for j in range(4)]
                                                                  for i in range(4)]


@pytest.mark.parametrize("b", [2, 3, 4])
@pytest.mark.parametrize("seed", range(4))
def test_bell_bruteforce_and_reconstruct(b, seed):
    rng = np.random.default_rng(seed)
    rows, cols = int(rng.integers(1, 40)), int(rng.integers(1, 40))   # ragged edges
    coo = si.random_coo(rows, cols, int(rng.integers(0, rows * cols // 2 + 1)), seed)
    rp, C, V = build(coo)
    kb, nbr_pad, bcol, bval = oracle.bell(rows, rp, C, V, b, b)
    blocks = {}
    for i, j in zip(coo.row.tolist(), coo.col.tolist()):
        blocks.setdefault(i // b, set()).add(j // b)
    assert kb == max((len(v) for v in blocks.values()), default=0)
    for I in range((rows + b - 1) // b):
        got = [int(bcol[k * nbr_pad + I]) for k in range(kb) if bcol[k * nbr_pad + I] >= 0]
        assert got == sorted(blocks.get(I, set()))                        # increasing block columns
    assert reconstruct_bell(kb, nbr_pad, bcol, bval, b, rows, cols) == dense_of(rows, cols, coo.row, coo.col, coo.val)


def test_block27_generator_block_structure():
    # every stored 3x3 block of the 3-dof 27-point stencil is dense -> zero block padding
    coo = si.block27(5, 3)
    rp, C, V = build(coo)
    kb, nbr_pad, bcol, bval = oracle.bell(coo.rows, rp, C, V, 3, 3)
    nblocks = int((bcol >= 0).sum())
    assert nblocks * 9 == coo.nnz and kb == 27
