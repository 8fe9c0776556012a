"""GPU tests: 16-bit column offsets (index16 = 1) and 8-bit dictionary codes
(index16 = 2) for ELL/SELL, and the learned run-time mode (SPMV_TUNE_PREDICT,
SURVEY §8(f) f3).

index16 changes only how the column index is STORED (d = col − row as int16,
pad −32768; or the 8-bit code of d in the matrix's dictionary of distinct
offsets, pad 255): decoded, the layouts must equal the oracle's ELL/SELL
(O4/O5) bit for bit, and every SpMV must pass O9 exactly as the int32
layouts do."""
import numpy as np
import pytest

import oracle
import spmv_inputs as si
from gpu_cases import corpus, oracle_csr, to_device, vec

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_2302_05662_b200")
pytestmark = pytest.mark.gpu

TAU = {"f64": 1e-12, "f32": 1e-5}
CASES = {name: coo for name, coo in corpus()}


def fits16(coo):
    if coo.row.shape[0] == 0:
        return True
    d = coo.col.astype(np.int64) - coo.row.astype(np.int64)
    return int(np.abs(d).max()) <= 32767


def n_offsets(coo):
    """Distinct col − row offsets (the 8-bit dictionary fits iff <= 255)."""
    if coo.row.shape[0] == 0:
        return 0
    return int(np.unique(coo.col.astype(np.int64) - coo.row.astype(np.int64)).shape[0])


def auto_bytes(coo):
    return 1 if n_offsets(coo) <= 255 else (2 if fits16(coo) else 4)


def create(coo, dtype):
    r, c, v = to_device(coo, dtype)
    return P.spmv_create(coo.rows, coo.cols, r, c, v)


def fetch(h, which, n, np_dtype):
    out = np.empty(n, np_dtype)
    if n:
        P.spmv_copy_array(h, which, out)
    return out


def decode(d16, rows_of_slot):
    d = d16.astype(np.int64)
    return np.where(d == -32768, -1, rows_of_slot + d).astype(np.int32)


def decode8(c8, tab, rows_of_slot):
    c = c8.astype(np.int64)
    return np.where(c == 255, -1, rows_of_slot + tab[np.minimum(c, 254)].astype(np.int64)).astype(np.int32)


def sell_rows_of_slot(perm, sp, Cs, rows):
    out = np.zeros(sp[-1], np.int64)
    for s_ in range(len(sp) - 1):
        w = (sp[s_ + 1] - sp[s_]) // Cs
        for j in range(Cs):
            q = s_ * Cs + j
            rr = perm[q] if q < rows else 0
            out[sp[s_] + np.arange(w) * Cs + j] = rr
    return out


@pytest.mark.parametrize("name", [n for n, c in corpus() if c.rows > 0 and n_offsets(c) <= 255])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_index8_layouts_decode_to_oracle(name, dtype):
    """8-bit codes: the dictionary holds exactly the matrix's distinct offsets
    (sorted), the codes decode to the oracle's ELL / SELL columns bit for bit,
    values are the oracle's, and the SpMV passes O9 for every knob."""
    coo = CASES[name]
    h = create(coo, dtype)
    try:
        rp, R, C, V = oracle_csr(coo)
        P.spmv_convert(h, P.FMT_ELL, index16=2)
        K, n_pad, colE, valE = oracle.ell(coo.rows, rp, C, V)
        info = P.spmv_format_info(h, P.FMT_ELL)
        assert info["index_bytes"] == 1 and (info["K"], info["n_pad"]) == (K, n_pad)
        tab = fetch(h, P.ARR_DICT8_TAB, 256, np.int32)
        offs = np.unique(coo.col.astype(np.int64) - coo.row.astype(np.int64))
        assert (tab[: len(offs)] == offs).all()
        rows_of_slot = np.tile(np.arange(n_pad, dtype=np.int64), K)
        assert (decode8(fetch(h, P.ARR_ELL_COL8, K * n_pad, np.uint8), tab, rows_of_slot) == colE).all()
        assert (fetch(h, P.ARR_ELL_VAL, K * n_pad, np.float32 if dtype == "f32" else np.float64)
                .astype(np.float64) == valE).all()
        assert info["stored_bytes"] == K * n_pad * (1 + (4 if dtype == "f32" else 8)) + 1024
        for alpha, beta in [(1.0, 0.0), (2.5, -0.5)]:
            check_y(h, coo, dtype, P.FMT_ELL, alpha, beta)
        for knob in [32, 64, 128, 64 | (1 << 16), 128 | (1 << 16)]:
            P.spmv_set_launch(h, P.FMT_ELL, 256, 64, -1, knob)
            check_y(h, coo, dtype, P.FMT_ELL, 2.5, -0.5)
        for Cs, sigma in ((32, 1), (64, 1), (128, 512), (256, 256)):
            P.spmv_convert(h, P.FMT_SELL, sell_C=Cs, sell_sigma=sigma, index16=2)
            perm, sp, colS, valS = oracle.sell(coo.rows, rp, C, V, Cs, sigma)
            assert P.spmv_format_info(h, P.FMT_SELL)["index_bytes"] == 1
            ros = sell_rows_of_slot(perm, sp, Cs, coo.rows)
            assert (decode8(fetch(h, P.ARR_SELL_COL8, sp[-1], np.uint8), tab, ros) == colS).all()
            check_y(h, coo, dtype, P.FMT_SELL, 2.5, -0.5)
            P.spmv_set_launch(h, P.FMT_SELL, 128, 64, -1, Cs | (1 << 16))
            check_y(h, coo, dtype, P.FMT_SELL, 1.0, 0.0)
    finally:
        P.spmv_destroy(h)


def test_index8_rejected_when_dictionary_overflows():
    coo = si.uniform_k(1 << 12, 16)   # thousands of distinct offsets
    assert n_offsets(coo) > 255
    h = create(coo, "f64")
    try:
        with pytest.raises(P.SpmvError) as e:
            P.spmv_convert(h, P.FMT_ELL, index16=2)
        assert e.value.status == P.ERR_UNSUPPORTED
        P.spmv_convert(h, P.FMT_ELL, index16=-1)
        assert P.spmv_format_info(h, P.FMT_ELL)["index_bytes"] == auto_bytes(coo)
    finally:
        P.spmv_destroy(h)


def check_y(h, coo, dtype, fmt, alpha, beta):
    rp, R, C, V = oracle_csr(coo)
    x = vec(coo.cols, 11, dtype)
    yin = vec(coo.rows, 12, dtype)
    y_ref, a_ref = oracle.spmv_csr(coo.rows, rp, C, V, x.astype(np.float64), alpha, beta, yin.astype(np.float64))
    yd = torch.from_numpy(yin).cuda()
    P.spmv_run(h, alpha, torch.from_numpy(x).cuda(), beta, yd, fmt=fmt)
    torch.cuda.synchronize()
    ok, worst, bad = oracle.parity_check(yd.cpu().numpy().astype(np.float64), y_ref, a_ref, alpha, beta, yin,
                                         TAU[dtype])
    assert ok, (P.FORMAT_NAMES[fmt], alpha, beta, worst)


@pytest.mark.parametrize("name", [n for n, c in corpus() if c.rows > 0 and fits16(c)])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_index16_layouts_decode_to_oracle(name, dtype):
    coo = CASES[name]
    h = create(coo, dtype)
    try:
        rp, R, C, V = oracle_csr(coo)
        P.spmv_convert(h, P.FMT_ELL, index16=1)
        K, n_pad, colE, valE = oracle.ell(coo.rows, rp, C, V)
        info = P.spmv_format_info(h, P.FMT_ELL)
        assert info["index_bytes"] == 2 and (info["K"], info["n_pad"]) == (K, n_pad)
        rows_of_slot = np.tile(np.arange(n_pad, dtype=np.int64), K)
        assert (decode(fetch(h, P.ARR_ELL_COL16, K * n_pad, np.int16), rows_of_slot) == colE).all()
        if K * n_pad:
            with pytest.raises(P.SpmvError):
                fetch(h, P.ARR_ELL_COL, K * n_pad, np.int32)  # int32 columns are not stored
        for Cs, sigma in ((32, 1), (64, 1), (128, 64 * 4), (256, 256)):
            if sigma % Cs and sigma != 1:
                continue
            P.spmv_convert(h, P.FMT_SELL, sell_C=Cs, sell_sigma=sigma, index16=1)
            perm, sp, colS, valS = oracle.sell(coo.rows, rp, C, V, Cs, sigma)
            assert P.spmv_format_info(h, P.FMT_SELL)["index_bytes"] == 2
            # row of each slot: slot (s, j, k) at sp[s] + k·C + j belongs to perm[s·C + j]
            rows_of_slot = np.zeros(sp[-1], np.int64)
            for s in range(len(sp) - 1):
                w = (sp[s + 1] - sp[s]) // Cs
                for j in range(Cs):
                    q = s * Cs + j
                    rr = perm[q] if q < coo.rows else 0
                    rows_of_slot[sp[s] + np.arange(w) * Cs + j] = rr
            assert (decode(fetch(h, P.ARR_SELL_COL16, sp[-1], np.int16), rows_of_slot) == colS).all()
            assert (fetch(h, P.ARR_SELL_VAL, sp[-1], np.float32 if dtype == "f32" else np.float64)
                    .astype(np.float64) == valS).all()
    finally:
        P.spmv_destroy(h)


@pytest.mark.parametrize("name", [n for n, c in corpus() if c.rows > 0])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("fmt,params", [(P.FMT_ELL, {}), (P.FMT_SELL, {}), (P.FMT_SELL, {"sell_C": 32, "sell_sigma": 64}),
                                        (P.FMT_SELL, {"sell_C": 256})])
def test_index16_spmv_parity(name, dtype, fmt, params):
    coo = CASES[name]
    h = create(coo, dtype)
    try:
        if not fits16(coo):
            with pytest.raises(P.SpmvError) as e:
                P.spmv_convert(h, fmt, index16=1, **params)
            assert e.value.status == P.ERR_UNSUPPORTED
            P.spmv_convert(h, fmt, index16=-1, **params)     # auto: 8-bit codes if <= 255 offsets, else int32
            assert P.spmv_format_info(h, fmt)["index_bytes"] == auto_bytes(coo)
        else:
            P.spmv_convert(h, fmt, index16=1, **params)
            assert P.spmv_format_info(h, fmt)["index_bytes"] == 2
        for alpha, beta in [(1.0, 0.0), (2.5, -0.5)]:
            check_y(h, coo, dtype, fmt, alpha, beta)
        for knob in ([32, 64, 128, 128 | (1 << 16)] if fmt == P.FMT_ELL else [0, 64]):
            P.spmv_set_launch(h, fmt, 256, 64, -1, knob)
            check_y(h, coo, dtype, fmt, 1.0, 0.0)
    finally:
        P.spmv_destroy(h)


def test_index16_power_step_and_bytes():
    coo = si.stencil27(20, random_values=True)
    n = coo.rows
    h = create(coo, "f64")
    try:
        P.spmv_convert(h, P.FMT_SELL)
        b32 = P.spmv_format_info(h, P.FMT_SELL)["stored_bytes"]
        P.spmv_convert(h, P.FMT_SELL, index16=1)
        info = P.spmv_format_info(h, P.FMT_SELL)
        assert info["index_bytes"] == 2
        assert info["stored_bytes"] == b32 - 2 * info["slots"]
        P.spmv_convert(h, P.FMT_SELL, index16=-1)   # 27 offsets: the 8-bit dictionary
        info = P.spmv_format_info(h, P.FMT_SELL)
        assert info["index_bytes"] == 1
        assert info["stored_bytes"] == b32 - 3 * info["slots"] + 1024
        rp, R, C, V = oracle_csr(coo)
        x = torch.from_numpy(vec(n, 3, "f64")).cuda()
        s0 = torch.zeros(2, dtype=torch.float64, device="cuda")
        s1 = torch.zeros(2, dtype=torch.float64, device="cuda")
        P.spmv_norm2(h, x, s0)
        z = torch.empty_like(x)
        P.spmv_power_step(h, x, z, s0, s1)
        torch.cuda.synchronize()
        xo = x.cpu().numpy() / np.sqrt(float(s0[0]))
        y_ref, _, lam_ref, _ = oracle.power_step(n, rp, C, V, xo)
        _, a_ref = oracle.spmv_csr(n, rp, C, V, xo)
        ok, worst, _ = oracle.parity_check(z.cpu().numpy(), y_ref, a_ref, 1.0, 0.0, None, 1e-12)
        assert ok, worst
        lam = float(s1[1]) / np.sqrt(float(s0[0]))
        assert abs(lam - lam_ref) <= 1e-10 * abs(lam_ref)
    finally:
        P.spmv_destroy(h)


def test_tuner_uses_narrowest_index_that_fits():
    coo = si.stencil27(40, random_values=True)
    h = create(coo, "f64")
    try:
        rep = P.spmv_tune(h, P.TUNE_FORMAT, expected_iterations=100000)
        fmt = rep.format
        if fmt in (P.FMT_ELL, P.FMT_SELL):
            assert rep.params.index16 == 2     # 27 distinct offsets: 8-bit dictionary codes
            assert P.spmv_format_info(h, fmt)["index_bytes"] == 1
            check_y(h, coo, "f64", fmt, 1.0, 0.0)
    finally:
        P.spmv_destroy(h)


# ---------------------------------------------------------------- learned run-time mode

@pytest.mark.parametrize("case", ["stencil27_40", "rmat14", "lap2d_300", "uniform_16_8"])
def test_predict_mode(case):
    coo = {"stencil27_40": lambda: si.stencil27(40, random_values=True),
           "rmat14": lambda: si.rmat(14, 16, dtype=np.float64),
           "lap2d_300": lambda: si.lap2d(300, random_values=True),
           "uniform_16_8": lambda: si.uniform_k(1 << 16, 8)}[case]()
    h = create(coo, "f64")
    try:
        feats = P.spmv_features(h)
        pred = P.spmv_predict(feats)
        rep = P.spmv_tune(h, P.TUNE_FORMAT | P.TUNE_PREDICT | P.TUNE_LAUNCH, expected_iterations=10 ** 7)
        log = [r for r in P.spmv_decision_log(h) if r.get("kind") == "format_predict"]
        assert len(log) == 1
        rec = log[0]
        assert rec["class"] == pred["class"]
        g = rec["gate"]
        assert g["convert"] == (pred["cls"] != 0 and g["gain_s"] > g["overhead"])
        assert abs(g["c_latency_pred_s"] - (0.0 if pred["class"].startswith("CSR") else pred["c_latency_s"])) <= \
            1e-9 * max(1.0, g["c_latency_pred_s"])
        if g["convert"]:
            assert rep.format == pred["format"]
            assert rec["chosen"] == pred["class"]
        else:
            assert rep.format == P.FMT_CSR and rec["chosen"] == "CSR-vector"
        for alpha, beta in [(1.0, 0.0), (2.5, -0.5)]:
            check_y(h, coo, "f64", rep.format, alpha, beta)
        # one iteration never amortises a conversion
        h2 = create(coo, "f64")
        rep2 = P.spmv_tune(h2, P.TUNE_FORMAT | P.TUNE_PREDICT, expected_iterations=0)
        assert rep2.format == P.FMT_CSR and rep2.converted == 0
        P.spmv_destroy(h2)
    finally:
        P.spmv_destroy(h)


@pytest.mark.parametrize("case", ["stencil27_40", "rmat14"])
def test_predict_decide_only(case):
    """SPMV_TUNE_DECIDE_ONLY reports the PREDICT verdict without converting;
    the t_CSR it gates on comes from a row sample scaled to nnz (the whole
    matrix below 2^26 entries)."""
    coo = {"stencil27_40": lambda: si.stencil27(40, random_values=True),
           "rmat14": lambda: si.rmat(14, 16, dtype=np.float64)}[case]()
    h = create(coo, "f64")
    try:
        feats = P.spmv_features(h)
        pred = P.spmv_predict(feats)
        rep = P.spmv_tune(h, P.TUNE_FORMAT | P.TUNE_PREDICT | P.TUNE_DECIDE_ONLY, expected_iterations=10 ** 7)
        assert P.spmv_get_format(h) == P.FMT_CSR          # nothing converted
        rec = [r for r in P.spmv_decision_log(h) if r.get("kind") == "format_predict"][-1]
        assert rec["t_csr_sample_nnz"] == coo.nnz
        if rec["gate"]["convert"]:
            assert rep.converted == 1 and rep.format == pred["format"]
        else:
            assert rep.converted == 0 and rep.format == P.FMT_CSR
        with pytest.raises(P.SpmvError):
            P.spmv_tune(h, P.TUNE_FORMAT | P.TUNE_DECIDE_ONLY, 100)          # needs PREDICT
        with pytest.raises(P.SpmvError):
            P.spmv_tune(h, P.TUNE_ALL | P.TUNE_PREDICT | P.TUNE_DECIDE_ONLY, 100)  # not with LAUNCH
    finally:
        P.spmv_destroy(h)


def test_predict_mode_rejects_other_objectives():
    coo = si.lap2d(30, random_values=True)
    h = create(coo, "f64")
    try:
        with pytest.raises(P.SpmvError) as e:
            P.spmv_tune(h, P.TUNE_FORMAT | P.TUNE_PREDICT, 100, objective="energy")
        assert e.value.status == P.ERR_UNSUPPORTED
        with pytest.raises(P.SpmvError):
            P.spmv_tune(h, P.TUNE_LAUNCH | P.TUNE_PREDICT, 100)   # PREDICT needs FORMAT
    finally:
        P.spmv_destroy(h)
