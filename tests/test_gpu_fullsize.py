"""Full-size parity at BASELINE.json's configs (c1–c4), in the configuration
bench.py times (selector + launch tuner decision): CSR and features bit-exact
against the oracle over the whole matrix; y checked on sampled rows (random
rows, first/last, the longest rows) whose expected values the oracle computes
one by one; three native power steps checked the same way."""
import numpy as np
import pytest

import oracle
import spmv_inputs as si

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_2302_05662_b200")

pytestmark = pytest.mark.gpu
TAU = {"f64": 1e-12, "f32": 1e-5}


def sub_csr(rp, col, val, rows_sel):
    """CSR of the selected rows (oracle input); columns stay global."""
    L = rp[rows_sel + 1] - rp[rows_sel]
    srp = np.concatenate([[0], np.cumsum(L)]).astype(np.int64)
    idx = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows_sel]) if len(rows_sel) else np.zeros(0, np.int64)
    return srp, col[idx], val[idx]


def sample_rows(rp, n, seed=5, k=3000):
    rng = np.random.default_rng(seed)
    L = np.diff(rp)
    pick = set(rng.choice(n, size=min(k, n), replace=False).tolist())
    pick |= {0, n - 1}
    pick |= set(np.argsort(L)[-16:].tolist())
    return np.array(sorted(pick), np.int64)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4"])
def test_fullsize_selected_format(cfg):
    coo = si.config_device(cfg)
    dtype = si.CONFIGS[cfg]["dtype"]
    dt = coo.val.dtype
    R = coo.row.cpu().numpy()
    Cc = coo.col.cpu().numpy()
    V = coo.val.cpu().numpy().astype(np.float64)
    n = coo.rows
    h = P.spmv_create(coo.rows, coo.cols, coo.row, coo.col, coo.val)
    try:
        # a2: CSR row pointers bit-exact over the whole matrix
        rp = oracle.csr(n, R)
        info = P.spmv_format_info(h, P.FMT_CSR)
        rpd = np.empty(n + 1, np.int64 if info["row_ptr_is64"] else np.int32)
        P.spmv_copy_array(h, P.ARR_CSR_ROW_PTR, rpd)
        assert (rpd.astype(np.int64) == rp).all()
        # a3: features bit-exact
        st, fo = oracle.features(n, coo.cols, rp, Cc)
        fd = P.spmv_features(h)
        for k, v in fo.items():
            same = np.float64(fd[k]).tobytes() == np.float64(v).tobytes() if isinstance(v, float) else fd[k] == v
            assert same, (k, fd[k], v)
        # a6/a7: the configuration bench.py replays
        rep = P.spmv_tune(h, P.TUNE_ALL, expected_iterations=100)
        fmt = rep.format
        # a5: y on sampled rows
        x = si.vector_device(coo.cols, dtype=dt)
        yin = si.vector_device(n, seed=si.Y_SEED, dtype=dt)
        y = yin.clone()
        P.spmv_run(h, 2.5, x, -0.5, y)
        torch.cuda.synchronize()
        rows_sel = sample_rows(rp, n)
        srp, sc, sv = sub_csr(rp, Cc, V, rows_sel)
        xh = x.cpu().numpy().astype(np.float64)
        yinh = yin.cpu().numpy().astype(np.float64)[rows_sel]
        y_ref, a_ref = oracle.spmv_csr(len(rows_sel), srp, sc, sv, xh, 2.5, -0.5, yinh)
        yg = y.cpu().numpy().astype(np.float64)[rows_sel]
        ok, worst, bad = oracle.parity_check(yg, y_ref, a_ref, 2.5, -0.5, yinh, TAU[dtype])
        assert ok, (cfg, P.FORMAT_NAMES[fmt], worst, rows_sel[bad[:5]])
        # a8: three native power steps, each checked against the oracle fed the GPU's own x_k
        if coo.rows == coo.cols:
            from paper_2302_05662_b200.dist import Layout, native_power_iteration
            E = 3
            layout = Layout.from_bounds(np.array([0, n]))
            for steps in range(1, E + 1):
                bufs = {"cur": torch.zeros(n, dtype=dt, device="cuda"), "nxt": torch.zeros(n, dtype=dt, device="cuda"),
                        "chunk": torch.zeros(1, dtype=dt, device="cuda"),
                        "sums": torch.zeros(steps + 1, 2, dtype=torch.float64, device="cuda")}
                z, sums, _ = native_power_iteration(h, layout, 0, x, bufs, steps)
                torch.cuda.synchronize()
                zk = z.cpu().numpy().astype(np.float64)
                if steps > 1:
                    prev_sum = sums[steps - 1, 0].item()
                    xk = zprev / np.sqrt(prev_sum)
                    y_ref, a_ref = oracle.spmv_csr(len(rows_sel), srp, sc, sv, xk, 1.0, 0.0, None)
                    ok, worst, bad = oracle.parity_check(zk[rows_sel], y_ref, a_ref, 1.0, 0.0, None, TAU[dtype])
                    assert ok, (cfg, "power step", steps, worst)
                zprev = zk
    finally:
        P.spmv_destroy(h)


FULL_FORMATS = {
    "c2": [("CSR-vector", P.FMT_CSR, dict(csr_alg=P.CSR_VECTOR)), ("CSR-stream", P.FMT_CSR, dict(csr_alg=P.CSR_STREAM)),
           ("CSR-merge", P.FMT_CSR, dict(csr_alg=P.CSR_MERGE)), ("ELL", P.FMT_ELL, dict(index16=0)),
           ("ELL-16", P.FMT_ELL, dict(index16=1)), ("SELL", P.FMT_SELL, dict(index16=0)),
           ("SELL-16", P.FMT_SELL, dict(index16=1)), ("HYB", P.FMT_HYB, {}), ("COO", P.FMT_COO, {})],
    "c3": [("CSR-vector", P.FMT_CSR, dict(csr_alg=P.CSR_VECTOR)), ("CSR-merge", P.FMT_CSR, dict(csr_alg=P.CSR_MERGE)),
           ("CSR-stream", P.FMT_CSR, dict(csr_alg=P.CSR_STREAM)), ("HYB", P.FMT_HYB, {}), ("COO", P.FMT_COO, {})],
    "c4": [("CSR-vector", P.FMT_CSR, dict(csr_alg=P.CSR_VECTOR)), ("CSR-stream", P.FMT_CSR, dict(csr_alg=P.CSR_STREAM)),
           ("ELL", P.FMT_ELL, {}), ("SELL", P.FMT_SELL, {}), ("COO", P.FMT_COO, {})],
}


@pytest.mark.timeout(900)
@pytest.mark.parametrize("cfg", ["c2", "c3", "c4"])
def test_fullsize_every_format(cfg):
    """Every format's kernel at the full BASELINE size (default launch, the
    TMA-staged CSR-stream included): y on sampled rows against the oracle."""
    coo = si.config_device(cfg)
    dtype = si.CONFIGS[cfg]["dtype"]
    dt = coo.val.dtype
    R = coo.row.cpu().numpy()
    Cc = coo.col.cpu().numpy()
    V = coo.val.cpu().numpy().astype(np.float64)
    n = coo.rows
    h = P.spmv_create(coo.rows, coo.cols, coo.row, coo.col, coo.val)
    del coo
    try:
        rp = oracle.csr(n, R)
        rows_sel = sample_rows(rp, n, seed=9, k=2000)
        srp, sc, sv = sub_csr(rp, Cc, V, rows_sel)
        x = si.vector_device(P.spmv_features(h)["n_cols"], dtype=dt)
        xh = x.cpu().numpy().astype(np.float64)
        yin = si.vector_device(n, seed=si.Y_SEED, dtype=dt)
        yinh = yin.cpu().numpy().astype(np.float64)[rows_sel]
        y_ref, a_ref = oracle.spmv_csr(len(rows_sel), srp, sc, sv, xh, 2.5, -0.5, yinh)
        for name, fmt, params in FULL_FORMATS[cfg]:
            P.spmv_convert(h, fmt, **params)
            y = yin.clone()
            P.spmv_run(h, 2.5, x, -0.5, y)
            torch.cuda.synchronize()
            yg = y.cpu().numpy().astype(np.float64)[rows_sel]
            ok, worst, bad = oracle.parity_check(yg, y_ref, a_ref, 2.5, -0.5, yinh, TAU[dtype])
            assert ok, (cfg, name, worst, rows_sel[bad[:5]])
            if fmt != P.FMT_CSR:
                P.spmv_convert(h, P.FMT_CSR)
    finally:
        P.spmv_destroy(h)


def c5_windows(n, plane):
    """Row windows of c5 checked against the oracle: the first and last rows
    (boundary planes), a plane seam, the middle, and scattered single rows."""
    w = [(0, 700), (n - 700, n), (plane - 350, plane + 350), (n // 2 - 350, n // 2 + 350)]
    rng = np.random.default_rng(11)
    w += [(int(r), int(r) + 1) for r in rng.choice(n - 1, size=40, replace=False)]
    return w


@pytest.mark.timeout(2400)
def test_fullsize_c5_bench_configuration():
    """c5 (27-point 512^3, 3.61e9 nnz, int64 row pointers) on one GPU, in the
    configuration bench.py --config c5 times (spmv_tune decision), plus the
    CSR-stream and ELL kernels: y on sampled row windows against the oracle,
    the window rows regenerated on the host (the full matrix is 58 GB of
    triplets, too large for the oracle); then three native power steps."""
    coo = si.config_device("c5")
    n = coo.rows
    nnz = coo.nnz
    h = P.spmv_create(coo.rows, coo.cols, coo.row, coo.col, coo.val)
    del coo
    torch.cuda.empty_cache()
    try:
        fd = P.spmv_features(h)
        # closed forms for the 27-point stencil on N^3: nnz = (3N-2)^3, bandwidth N^2+N+1
        N = 512
        assert nnz == (3 * N - 2) ** 3 == fd["nnz"] == 3609741304
        assert fd["max_len"] == 27 and fd["min_len"] == 8 and fd["n_empty"] == 0
        assert fd["bandwidth"] == N * N + N + 1 and fd["median"] == 27.0 and fd["mode"] == 27
        assert P.spmv_format_info(h, P.FMT_CSR)["row_ptr_is64"]
        wins = c5_windows(n, N * N)
        x = si.vector_device(n)
        xh = x.cpu().numpy()
        yin = si.vector_device(n, seed=si.Y_SEED)
        refs = []
        for r0, r1 in wins:
            w = si.stencil(si.STENCIL27, N, r0, r1, random_values=True)
            st, R, C, V = oracle.canonicalize(w.rows, w.cols, w.row, w.col, w.val)
            refs.append((r0, r1, oracle.csr(r1 - r0, R), C, V))
        sel = np.concatenate([np.arange(r0, r1) for r0, r1, *_ in refs])

        def check(y, alpha, beta, xv, yinh, label):
            yg = y.cpu().numpy()
            for r0, r1, rp, C, V in refs:
                yi = None if yinh is None else yinh[r0:r1]
                y_ref, a_ref = oracle.spmv_csr(r1 - r0, rp, C, V, xv, alpha, beta, yi)
                ok, worst, bad = oracle.parity_check(yg[r0:r1], y_ref, a_ref, alpha, beta, yi, 1e-12)
                assert ok, (label, r0, worst, bad[:5])

        rep = P.spmv_tune(h, P.TUNE_ALL, expected_iterations=100)
        yinh = yin.cpu().numpy()
        cases = [("tuned:" + P.FORMAT_NAMES[rep.format], None, None),
                 ("CSR-stream", P.FMT_CSR, dict(csr_alg=P.CSR_STREAM)), ("ELL", P.FMT_ELL, {})]
        for label, fmt, params in cases:
            if fmt is not None:
                P.spmv_convert(h, fmt, **params)
            y = yin.clone()
            P.spmv_run(h, 2.5, x, -0.5, y)
            torch.cuda.synchronize()
            check(y, 2.5, -0.5, xh, yinh, label)
            del y
            if fmt == P.FMT_ELL:
                break
            if fmt is not None:
                P.spmv_convert(h, P.FMT_CSR)
        # three native power steps on the ELL kernel (bench's c5 hot loop shape)
        from paper_2302_05662_b200.dist import Layout, native_power_iteration
        layout = Layout.from_bounds(np.array([0, n]))
        zprev = None
        for steps in (1, 2):
            bufs = {"cur": torch.zeros(n, dtype=torch.float64, device="cuda"),
                    "nxt": torch.zeros(n, dtype=torch.float64, device="cuda"),
                    "chunk": torch.zeros(1, dtype=torch.float64, device="cuda"),
                    "sums": torch.zeros(steps + 1, 2, dtype=torch.float64, device="cuda")}
            z, sums, _ = native_power_iteration(h, layout, 0, x, bufs, steps)
            torch.cuda.synchronize()
            zk = z.cpu().numpy()
            if steps == 2:
                xk = zprev / np.sqrt(sums[1, 0].item())
                check(z, 1.0, 0.0, xk, None, "power step 2")
            zprev = zk
            del bufs, z
        assert len(sel) > 2800
    finally:
        P.spmv_destroy(h)
