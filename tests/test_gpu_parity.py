"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bit-exact: canonical COO/CSR, features, ELL/SELL/HYB/COO layouts.
Tolerance O9: |y − y_ref| <= tau·(|α|·Σ|a·x| + |β|·|y_in|),
tau = 1e-12 (fp64) / 1e-5 (fp32, north star), per row."""
import numpy as np
import pytest

import oracle
import spmv_inputs as si
from gpu_cases import corpus, oracle_csr, small_corpus, to_device, vec

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_2302_05662_b200")

pytestmark = pytest.mark.gpu

TAU = {"f64": 1e-12, "f32": 1e-5}
AB = [(1.0, 0.0), (2.5, -0.5), (0.0, 1.0), (1.0, 1.0)]
CASES = {name: coo for name, coo in corpus()}


def tdt(dtype):
    return torch.float64 if dtype == "f64" else torch.float32


def create(coo, dtype="f64", where="device", shuffle=False):
    if shuffle:
        coo = si.shuffled(coo, 77)
    if where == "device":
        r, c, v = to_device(coo, dtype)
    else:
        r, c = np.ascontiguousarray(coo.row), np.ascontiguousarray(coo.col)
        v = np.ascontiguousarray(coo.val.astype(np.float32 if dtype == "f32" else np.float64))
    return P.spmv_create(coo.rows, coo.cols, r, c, v)


def fetch(h, which, n, np_dtype):
    out = np.empty(n, np_dtype)
    if n:
        P.spmv_copy_array(h, which, out)
    return out


def check_y(h, coo, dtype, fmt, alpha, beta, ref=None, nan_y=False):
    rp, R, C, V = ref if ref is not None else oracle_csr(coo)
    x = vec(coo.cols, 11, dtype)
    yin = vec(coo.rows, 12, dtype)
    y_ref, a_ref = oracle.spmv_csr(coo.rows, rp, C, V, x.astype(np.float64), alpha, beta, yin.astype(np.float64))
    xd = torch.from_numpy(x).cuda()
    yd = torch.from_numpy(yin).cuda()
    if nan_y:
        yd.fill_(float("nan"))
    P.spmv_run(h, alpha, xd, beta, yd, fmt=fmt)
    torch.cuda.synchronize()
    y = yd.cpu().numpy().astype(np.float64)
    ok, worst, bad = oracle.parity_check(y, y_ref, a_ref, alpha, beta, None if nan_y else yin, TAU[dtype])
    assert ok, (P.FORMAT_NAMES[fmt], alpha, beta, worst, bad[:8], y[bad[:4]], y_ref[bad[:4]])
    return y


# ------------------------------------------------------------------ inputs module

def test_generators_host_device_identical():
    for kind, N in ((si.LAP2D, 17), (si.STENCIL27, 7)):
        for rv in (False, True):
            h = si.stencil(kind, N, random_values=rv)
            d = si.stencil_device(kind, N, random_values=rv)
            assert (d.row.cpu().numpy() == h.row).all() and (d.col.cpu().numpy() == h.col).all()
            assert (d.val.cpu().numpy() == h.val).all()
    h = si.stencil(si.STENCIL27, 8, r0=100, r1=300)
    d = si.stencil_device(si.STENCIL27, 8, r0=100, r1=300)
    assert (d.row.cpu().numpy() == h.row).all() and (d.col.cpu().numpy() == h.col).all()
    u, ud = si.uniform_k(1 << 12, 32), si.uniform_k_device(1 << 12, 32)
    assert (ud.col.cpu().numpy() == u.col).all() and (ud.val.cpu().numpy() == u.val).all()
    r, rd = si.rmat(12, dtype=np.float64), si.rmat_device(12, dtype=torch.float64)
    assert (rd.row.cpu().numpy() == r.row).all() and (rd.col.cpu().numpy() == r.col).all()
    assert (rd.val.cpu().numpy() == r.val).all()
    assert (si.vector_device(1000).cpu().numpy() == si.vector(1000)).all()


# ------------------------------------------------------------------ a1/a2 ingest + CSR

@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("where,shuffle", [("device", False), ("host", False), ("device", True)])
def test_create_csr_bit_exact(name, dtype, where, shuffle):
    coo = CASES[name]
    if shuffle and coo.nnz > 20000:
        pytest.skip("large shuffled case covered elsewhere")
    h = create(coo, dtype, where, shuffle)
    try:
        rp, R, C, V = oracle_csr(coo)
        info = P.spmv_format_info(h, P.FMT_CSR)
        rpd = fetch(h, P.ARR_CSR_ROW_PTR, coo.rows + 1, np.int64 if info["row_ptr_is64"] else np.int32)
        assert (rpd.astype(np.int64) == rp).all()
        assert (fetch(h, P.ARR_CSR_COL, coo.nnz, np.int32) == C).all()
        vd = fetch(h, P.ARR_CSR_VAL, coo.nnz, np.float32 if dtype == "f32" else np.float64)
        assert (vd.astype(np.float64) == V).all()
    finally:
        P.spmv_destroy(h)


def test_create_large_unsorted_rmat():
    coo = si.rmat(16, dtype=np.float64)
    h = create(coo, "f64", "device", shuffle=True)
    try:
        rp, R, C, V = oracle_csr(coo)
        assert (fetch(h, P.ARR_CSR_ROW_PTR, coo.rows + 1, np.int32) == rp).all()
        assert (fetch(h, P.ARR_CSR_COL, coo.nnz, np.int32) == C).all()
        assert (fetch(h, P.ARR_CSR_VAL, coo.nnz, np.float64) == V).all()
    finally:
        P.spmv_destroy(h)


def test_create_errors():
    r = torch.tensor([0, 1, 1], dtype=torch.int32, device="cuda")
    c = torch.tensor([0, 2, 2], dtype=torch.int32, device="cuda")
    v = torch.ones(3, dtype=torch.float64, device="cuda")
    with pytest.raises(P.SpmvError) as e:
        P.spmv_create(3, 3, r, c, v)
    assert e.value.status == P.ERR_DUPLICATE
    r2 = torch.tensor([1, 0, 1], dtype=torch.int32, device="cuda")
    c2 = torch.tensor([2, 0, 2], dtype=torch.int32, device="cuda")
    with pytest.raises(P.SpmvError) as e:                       # unsorted + duplicate
        P.spmv_create(3, 3, r2, c2, v)
    assert e.value.status == P.ERR_DUPLICATE
    c3 = torch.tensor([0, 1, 3], dtype=torch.int32, device="cuda")
    with pytest.raises(P.SpmvError) as e:
        P.spmv_create(3, 3, r, c3, v)
    assert e.value.status == P.ERR_INDEX_OUT_OF_RANGE
    r4 = torch.tensor([0, -1, 1], dtype=torch.int32, device="cuda")
    with pytest.raises(P.SpmvError) as e:
        P.spmv_create(3, 3, r4, c, v)
    assert e.value.status == P.ERR_INDEX_OUT_OF_RANGE


# ------------------------------------------------------------------ a3 features

@pytest.mark.parametrize("name", list(CASES))
def test_features_bit_exact(name):
    coo = CASES[name]
    h = create(coo)
    try:
        rp, R, C, V = oracle_csr(coo)
        st, fo = oracle.features(coo.rows, coo.cols, rp, C)
        fd = P.spmv_features(h)
        for k, v in fo.items():
            assert np.float64(fd[k]).tobytes() == np.float64(v).tobytes() if isinstance(v, float) else fd[k] == v, \
                (k, fd[k], v)
    finally:
        P.spmv_destroy(h)


# ------------------------------------------------------------------ a4 layouts

@pytest.mark.parametrize("name", [n for n, _ in small_corpus()])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_layouts_bit_exact(name, dtype):
    coo = CASES[name]
    npv = np.float32 if dtype == "f32" else np.float64
    h = create(coo, dtype)
    try:
        rp, R, C, V = oracle_csr(coo)
        if coo.rows == 0:
            return
        # ELL
        P.spmv_convert(h, P.FMT_ELL)
        K, n_pad, colE, valE = oracle.ell(coo.rows, rp, C, V)
        info = P.spmv_format_info(h, P.FMT_ELL)
        assert (info["K"], info["n_pad"]) == (K, n_pad)
        assert (fetch(h, P.ARR_ELL_COL, K * n_pad, np.int32) == colE).all()
        assert (fetch(h, P.ARR_ELL_VAL, K * n_pad, npv).astype(np.float64) == valE).all()
        # SELL-C-sigma
        for Cs, sigma in ((32, 1), (64, 1), (128, 1), (256, 1), (64, 64), (32, 256), (128, 512)):
            P.spmv_convert(h, P.FMT_SELL, sell_C=Cs, sell_sigma=sigma)
            perm, sp, colS, valS = oracle.sell(coo.rows, rp, C, V, Cs, sigma)
            info = P.spmv_format_info(h, P.FMT_SELL)
            assert info["n_slices"] == len(sp) - 1 and info["slots"] == sp[-1]
            assert (fetch(h, P.ARR_SELL_PERM, coo.rows, np.int32) == perm).all()
            assert (fetch(h, P.ARR_SELL_SLICE_PTR, len(sp), np.int64) == sp).all()
            assert (fetch(h, P.ARR_SELL_COL, sp[-1], np.int32) == colS).all()
            assert (fetch(h, P.ARR_SELL_VAL, sp[-1], npv).astype(np.float64) == valS).all()
        # HYB (auto rule and an explicit width)
        for Kh in (-1, 2):
            P.spmv_convert(h, P.FMT_HYB, hyb_K=Kh)
            K, n_pad, colE, valE, tr, tc, tv = oracle.hyb(coo.rows, rp, C, V, None if Kh < 0 else Kh)
            info = P.spmv_format_info(h, P.FMT_HYB)
            assert (info["K"], info["n_pad"], info["tail_nnz"]) == (K, n_pad, tr.shape[0])
            assert (fetch(h, P.ARR_HYB_ELL_COL, K * n_pad, np.int32) == colE).all()
            assert (fetch(h, P.ARR_HYB_ELL_VAL, K * n_pad, npv).astype(np.float64) == valE).all()
            assert (fetch(h, P.ARR_HYB_TAIL_ROW, tr.shape[0], np.int32) == tr).all()
            assert (fetch(h, P.ARR_HYB_TAIL_COL, tr.shape[0], np.int32) == tc).all()
            assert (fetch(h, P.ARR_HYB_TAIL_VAL, tr.shape[0], npv).astype(np.float64) == tv).all()
        # BELL (b = 2, 3, 4)
        for b in (2, 3, 4):
            P.spmv_convert(h, P.FMT_BELL, bell_b=b)
            kb, nbr_pad, bcol, bval = oracle.bell(coo.rows, rp, C, V, b, b)
            info = P.spmv_format_info(h, P.FMT_BELL)
            assert (info["K"], info["n_pad"], info["block"]) == (kb, nbr_pad, b)
            assert (fetch(h, P.ARR_BELL_COL, kb * nbr_pad, np.int32) == bcol).all()
            assert (fetch(h, P.ARR_BELL_VAL, kb * b * b * nbr_pad, npv).astype(np.float64) == bval).all()
        # COO
        P.spmv_convert(h, P.FMT_COO)
        assert (fetch(h, P.ARR_COO_ROW, coo.nnz, np.int32) == R).all()
        L = np.diff(rp)
        empty = np.nonzero(L == 0)[0]
        assert P.spmv_format_info(h, P.FMT_COO)["n_empty_rows"] == empty.shape[0]
        assert (fetch(h, P.ARR_COO_EMPTY_ROWS, empty.shape[0], np.int32) == empty).all()
    finally:
        P.spmv_destroy(h)


# ------------------------------------------------------------------ a5 SpMV parity

FMTS = [("CSR-vector", P.FMT_CSR, dict(csr_alg=P.CSR_VECTOR)),
        ("CSR-scalar", P.FMT_CSR, dict(csr_alg=P.CSR_SCALAR)),
        ("CSR-merge", P.FMT_CSR, dict(csr_alg=P.CSR_MERGE)),
        ("CSR-stream", P.FMT_CSR, dict(csr_alg=P.CSR_STREAM)),
        ("ELL", P.FMT_ELL, {}),
        ("SELL", P.FMT_SELL, {}),
        ("SELL-sigma", P.FMT_SELL, dict(sell_C=32, sell_sigma=256)),
        ("HYB", P.FMT_HYB, {}),
        ("HYB-K2", P.FMT_HYB, dict(hyb_K=2)),
        ("COO", P.FMT_COO, {}),
        ("BELL-2", P.FMT_BELL, dict(bell_b=2)),
        ("BELL-3", P.FMT_BELL, dict(bell_b=3)),
        ("BELL-4", P.FMT_BELL, dict(bell_b=4))]


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("fname,fmt,params", FMTS, ids=[f[0] for f in FMTS])
def test_spmv_parity(name, dtype, fname, fmt, params):
    coo = CASES[name]
    h = create(coo, dtype)
    try:
        ref = oracle_csr(coo)
        P.spmv_convert(h, fmt, **params)
        for alpha, beta in AB:
            check_y(h, coo, dtype, fmt, alpha, beta, ref)
        check_y(h, coo, dtype, fmt, 2.5, 0.0, ref, nan_y=True)    # beta = 0: y never read
    finally:
        P.spmv_destroy(h)


@pytest.mark.parametrize("fname,fmt,params,knobs", [
    ("CSR-vector", P.FMT_CSR, dict(csr_alg=P.CSR_VECTOR), [1, 2, 4, 8, 16, 32, 0x104, 0x108, 0x110, 0x120]),
    ("CSR-merge", P.FMT_CSR, dict(csr_alg=P.CSR_MERGE), [4, 8, 16, 0x104, 0x108, 0x110, 0x204, 0x208, 0x210,
                                                         0x404, 0x408, 0x808]),
    ("CSR-stream", P.FMT_CSR, dict(csr_alg=P.CSR_STREAM), [16, 32, 64]),
    ("ELL", P.FMT_ELL, {}, [32, 64, 128, 64 | (1 << 16), 256 | (1 << 16)]),
    ("SELL", P.FMT_SELL, {}, [0, 64, 64 | (1 << 16)]),
    ("COO", P.FMT_COO, {}, [2, 4, 8, 0x104, 0x108, 0x110]),
    ("HYB", P.FMT_HYB, {}, [2, 4, 8, 0x104, 0x108, 0x110]),
    ("BELL", P.FMT_BELL, {"bell_b": 3}, [0])])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_launch_variants_parity(fname, fmt, params, knobs, dtype):
    coo = CASES["ragged_empty"]
    h = create(coo, dtype)
    try:
        ref = oracle_csr(coo)
        P.spmv_convert(h, fmt, **params)
        for block in (64, 128, 256, 512, 1024):
            for maxreg in (32, 64, 128, 255):
                for knob in knobs:
                    P.spmv_set_launch(h, fmt, block, maxreg, 25 if block == 128 else -1, knob)
                    try:
                        check_y(h, coo, dtype, fmt, 2.5, -0.5, ref)
                    except P.SpmvError as ex:   # e.g. CSR-stream block × entries over shared memory
                        assert ex.status == P.ERR_UNSUPPORTED
                        torch.cuda.synchronize()
    finally:
        P.spmv_destroy(h)


@pytest.mark.parametrize("case", ["mixed_tiles", "long_rows", "rmat10", "stencil27_9", "ragged_empty"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_csr_stream_tma_all_launches(case, dtype):
    """The TMA-pipelined CSR-stream kernel over every block size, stage size
    and register cap on matrices mixing staged and overflowing tiles, with
    segment starts at every 16-byte residue (bulk-copied interior, lane-copied
    head/tail): O9 parity; block 1024 (+ producer warp) must be refused."""
    coo = CASES[case]
    h = create(coo, dtype)
    try:
        ref = oracle_csr(coo)
        P.spmv_convert(h, P.FMT_CSR, csr_alg=P.CSR_STREAM)
        for block in (64, 128, 256, 512, 1024):
            for maxreg in (32, 255):
                for ept in (16, 32, 64):
                    P.spmv_set_launch(h, P.FMT_CSR, block, maxreg, -1, ept)
                    try:
                        check_y(h, coo, dtype, P.FMT_CSR, 2.5, -0.5, ref)
                        check_y(h, coo, dtype, P.FMT_CSR, 1.0, 0.0, ref, nan_y=True)
                    except P.SpmvError as ex:   # block + producer warp > 1024 or stages > shared memory
                        assert ex.status == P.ERR_UNSUPPORTED
                        assert block == 1024 or block * ept * (12 if dtype == "f64" else 8) * 2 > 200 * 1024
                        torch.cuda.synchronize()
    finally:
        P.spmv_destroy(h)


@pytest.mark.parametrize("case", ["mixed_tiles", "long_rows", "rmat10", "stencil27_9", "ragged_empty"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("fmt", [P.FMT_COO, P.FMT_HYB, "merge", "merge-stream"])
def test_coo_tile_all_launches(case, dtype, fmt):
    """Row-interleaved COO tiles (knob 0x100 | EPT) over every block size and
    tile depth: rows crossing tiles (fixup records), rows longer than the
    thread pass takes (warp-cooperative pass), empty rows, the ragged last
    tile; plain COO, the HYB tail (accumulate mode) and merge-path CSR tiles
    (block·IPT merge items, empty rows written by the tile), also fed by the
    TMA producer warp (0x200 | IPT, two-stage ring, long rows cut into pieces
    summed by all consumer warps): O9 parity and NaN y with beta = 0."""
    coo = CASES[case]
    h = create(coo, dtype)
    try:
        ref = oracle_csr(coo)
        flag = 0x200 if fmt == "merge-stream" else 0x100
        epts = (4, 8, 16, 32)
        if fmt in ("merge", "merge-stream"):
            fmt = P.FMT_CSR
            P.spmv_convert(h, fmt, csr_alg=P.CSR_MERGE)
        else:
            P.spmv_convert(h, fmt)
        for block in (64, 128, 256, 512, 1024):
            for ept in epts:
                P.spmv_set_launch(h, fmt, block, 255 if block <= 256 else 64, -1, flag | ept)
                try:
                    check_y(h, coo, dtype, fmt, 2.5, -0.5, ref)
                    check_y(h, coo, dtype, fmt, 1.0, 0.0, ref, nan_y=True)
                except P.SpmvError as ex:   # tile over the shared-memory cap / block + producer warp > 1024
                    assert ex.status == P.ERR_UNSUPPORTED and (block * ept >= 4096 or block == 1024)
                    torch.cuda.synchronize()
    finally:
        P.spmv_destroy(h)


@pytest.mark.parametrize("case", ["mixed_tiles", "long_rows", "rmat10", "stencil27_9", "ragged_empty"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_csr_nnz_split_all_launches(case, dtype):
    """nnz-split CSR of the merge-path family (knob 0x400 | W): warps of 32·W
    entries with vector loads, rows from the row pointers (binary search in
    the cached partition window, then forward) or (knob 0x808) from the cached
    row map (row-start bits + non-empty row list), lane runs + warp segmented
    scan, rows crossing warps through the fixup, hub rows spanning many warps
    (long-run fixup), empty rows from the handle's list, the ragged last warp:
    O9 parity, NaN y with beta = 0, bitwise repeatable; switching back to a
    merge-path variant recomputes its own partition."""
    coo = CASES[case]
    h = create(coo, dtype)
    try:
        ref = oracle_csr(coo)
        P.spmv_convert(h, P.FMT_CSR, csr_alg=P.CSR_MERGE)
        for block in (64, 128, 256, 512, 1024):
            for knob in (0x404, 0x408, 0x808):   # nnz-split by search, and with the cached row map
                P.spmv_set_launch(h, P.FMT_CSR, block, 64 if block <= 512 else 32, -1, knob)
                check_y(h, coo, dtype, P.FMT_CSR, 2.5, -0.5, ref)
                y1 = check_y(h, coo, dtype, P.FMT_CSR, 1.0, 0.0, ref, nan_y=True)
                y2 = check_y(h, coo, dtype, P.FMT_CSR, 1.0, 0.0, ref, nan_y=True)
                assert y1.tobytes() == y2.tobytes()
                P.spmv_set_launch(h, P.FMT_CSR, 128, 64, -1, 8)           # per-warp merge walk in between
                check_y(h, coo, dtype, P.FMT_CSR, 1.0, 0.0, ref, nan_y=True)
        with pytest.raises(P.SpmvError) as ex:
            P.spmv_set_launch(h, P.FMT_CSR, 128, 64, -1, 0x400 | 16)
            check_y(h, coo, dtype, P.FMT_CSR, 1.0, 0.0, ref)
        assert ex.value.status == P.ERR_INVALID_ARG
        torch.cuda.synchronize()
    finally:
        P.spmv_destroy(h)


@pytest.mark.parametrize("case,fmt,params", [("ragged_empty", P.FMT_ELL, {}), ("stencil27_9", P.FMT_ELL, {"index16": 2}),
                                             ("ragged_empty", P.FMT_SELL, {}), ("ragged_empty", P.FMT_HYB, {}),
                                             ("ragged_empty", P.FMT_BELL, {"bell_b": 2})])
def test_release_csr(case, fmt, params):
    """spmv_release_csr frees CSR/COO after conversion: the active format still
    runs (O9 parity, power steps), features stay cached, everything that reads
    CSR returns NOT_CONVERTED; refused while CSR or COO is active."""
    coo = CASES[case]
    h = create(coo)
    try:
        ref = oracle_csr(coo)
        feats = P.spmv_features(h)
        P.spmv_convert(h, P.FMT_COO)
        with pytest.raises(P.SpmvError) as ex:
            P.spmv_release_csr(h)
        assert ex.value.status == P.ERR_INVALID_ARG
        P.spmv_convert(h, fmt, **params)
        P.spmv_release_csr(h)
        P.spmv_release_csr(h)                                   # no-op
        check_y(h, coo, "f64", fmt, 2.5, -0.5, ref)
        assert P.spmv_features(h) == feats
        for call in (lambda: P.spmv_convert(h, P.FMT_ELL), lambda: P.spmv_tune(h, P.TUNE_LAUNCH, 10),
                     lambda: P.spmv_set_format(h, P.FMT_CSR), lambda: P.spmv_set_format(h, P.FMT_COO),
                     lambda: P.spmv_create_row_slice(h, 0, 10),
                     lambda: P.spmv_copy_array(h, P.ARR_CSR_COL, np.empty(coo.nnz, np.int32))):
            with pytest.raises(P.SpmvError) as ex:
                call()
            assert ex.value.status == P.ERR_NOT_CONVERTED
        torch.cuda.synchronize()
        check_y(h, coo, "f64", fmt, 1.0, 0.0, ref, nan_y=True)
    finally:
        P.spmv_destroy(h)


def test_determinism_bitwise():
    coo = CASES["long_rows"]
    h = create(coo)
    try:
        x = torch.from_numpy(vec(coo.cols, 3, "f64")).cuda()
        for fmt, params in ((P.FMT_CSR, dict(csr_alg=P.CSR_MERGE)), (P.FMT_COO, {}), (P.FMT_HYB, {}),
                            (P.FMT_SELL, {})):
            P.spmv_convert(h, fmt, **params)
            ys = []
            for _ in range(3):
                y = torch.empty(coo.rows, dtype=torch.float64, device="cuda")
                P.spmv_run(h, 1.0, x, 0.0, y)
                ys.append(y.cpu().numpy().tobytes())
            assert ys[0] == ys[1] == ys[2]
    finally:
        P.spmv_destroy(h)


def test_alpha_zero_does_not_read_A_or_x():
    coo = CASES["uniform_rand"]
    h = create(coo)
    try:
        x = torch.full((coo.cols,), float("nan"), dtype=torch.float64, device="cuda")
        yin = torch.from_numpy(vec(coo.rows, 5, "f64")).cuda()
        for fmt in (P.FMT_CSR, P.FMT_ELL, P.FMT_SELL, P.FMT_COO, P.FMT_HYB):
            P.spmv_convert(h, fmt)
            y = yin.clone()
            P.spmv_run(h, 0.0, x, 0.5, y)
            assert torch.equal(y, 0.5 * yin)
    finally:
        P.spmv_destroy(h)


def test_run_argument_errors():
    coo = CASES["uniform_rand"]
    h = create(coo)
    try:
        x = torch.zeros(coo.cols, dtype=torch.float64, device="cuda")
        with pytest.raises(P.SpmvError) as e:
            P.spmv_run(h, 1.0, x, 0.0, x)          # x == y
        assert e.value.status == P.ERR_INVALID_ARG
        with pytest.raises(P.SpmvError) as e:
            P.spmv_run(h, 1.0, x, 0.0, torch.zeros(coo.rows, dtype=torch.float64, device="cuda"), fmt=P.FMT_ELL)
        assert e.value.status == P.ERR_NOT_CONVERTED
        with pytest.raises(P.SpmvError) as e:
            P.spmv_convert(h, P.FMT_SELL, sell_C=48)
        assert e.value.status == P.ERR_UNSUPPORTED
    finally:
        P.spmv_destroy(h)


# ------------------------------------------------------------------ a8 power step

@pytest.mark.parametrize("fname,fmt,params", FMTS, ids=[f[0] for f in FMTS])
def test_power_step_parity(fname, fmt, params):
    coo = si.lap2d(40, random_values=True)
    h = create(coo)
    try:
        rp, R, C, V = oracle_csr(coo)
        P.spmv_convert(h, fmt, **params)
        n = coo.rows
        z_prev = torch.from_numpy(vec(n, 9, "f64")).cuda()          # unnormalised z_{k-1}
        sums_prev = torch.zeros(2, dtype=torch.float64, device="cuda")
        P.spmv_norm2(h, z_prev, sums_prev)
        zp = z_prev.cpu().numpy()
        s_prev = float(sums_prev[0].item())
        assert abs(s_prev - np.dot(zp, zp)) <= 1e-13 * np.dot(zp, zp)
        for step in range(3):
            z = torch.empty(n, dtype=torch.float64, device="cuda")
            sums = torch.zeros(2, dtype=torch.float64, device="cuda")
            P.spmv_power_step(h, z_prev, z, sums_prev, sums)
            torch.cuda.synchronize()
            xk = z_prev.cpu().numpy() / np.sqrt(float(sums_prev[0].item()))   # the GPU's own x_k
            y_ref, xn, lam, s = oracle.power_step(n, rp, C, V, xk)
            _, a_ref = oracle.spmv_csr(n, rp, C, V, xk)
            ok, worst, bad = oracle.parity_check(z.cpu().numpy(), y_ref, a_ref, 1.0, 0.0, None, 1e-12)
            assert ok, (step, worst)
            lam_gpu = float(sums[1].item()) / np.sqrt(float(sums_prev[0].item()))
            assert abs(lam_gpu - lam) <= 1e-10 * abs(lam)
            assert abs(float(sums[0].item()) - s) <= 1e-10 * s
            z_prev, sums_prev = z, sums
    finally:
        P.spmv_destroy(h)


# ------------------------------------------------------------------ a6/a7 tuner + selector


def gate_net_best(sel, objective="latency"):
    """The candidate the gate must pick : the largest net benefit
    gain - overhead over the default CSR (first measured candidate), reading R31."""
    cands = [c for c in sel["candidates"] if "t_s" in c]
    csr, g = cands[0], sel["gate"]
    it, f = g["expected_iterations"], g["f_latency_s"]

    def net(c):
        if objective == "latency":
            return it * (csr["t_s"] - c["t_s"]) - (f + c["c_latency_s"])
        if objective == "power":
            return csr["w"] - c["w"]
        return it * (csr["j_per_spmv"] - c["j_per_spmv"]) - csr["w"] * (f + c["c_latency_s"])
    return max(cands[1:], key=net) if len(cands) > 1 else csr


def test_tune_invariants():
    coo = si.stencil27(24, random_values=True)
    h = create(coo)
    try:
        rep = P.spmv_tune(h, P.TUNE_ALL, expected_iterations=10 ** 6)
        log = P.spmv_decision_log(h)
        sel = [r for r in log if r["kind"] == "format_select"][0]
        names = [c["format"] for c in sel["candidates"] if "t_s" in c]
        assert P.FORMAT_NAMES[rep.format] in names
        g = sel["gate"]
        assert g["convert"] == (g["expected_iterations"] * (g["t_csr_s"] - g["t_best_s"]) >
                                g["f_latency_s"] + g["c_latency_s"])
        assert g["t_best_s"] == gate_net_best(sel)["t_s"]
        sweep = [r for r in log if r["kind"] == "launch_sweep"][-1]
        assert sweep["t_best_s"] <= min(v[4] for v in sweep["variants"]) + 1e-15
        check_y(h, coo, "f64", rep.format, 2.5, -0.5)
        # gate with zero iterations never converts
        rep0 = P.spmv_tune(h, P.TUNE_FORMAT, expected_iterations=0)
        assert rep0.converted == 0 and rep0.format == P.FMT_CSR
    finally:
        P.spmv_destroy(h)


# ------------------------------------------------------------------ native loop (+ NCCL at world 1)

@pytest.mark.parametrize("use_comm", [False, True])
def test_native_power_iterate_matches_stepwise(use_comm):
    from paper_2302_05662_b200.dist import Layout, NativeComm, native_power_iteration
    coo = si.stencil27(10, random_values=True)
    h = create(coo)
    comm = None
    try:
        P.spmv_convert(h, P.FMT_SELL)
        n, E = coo.rows, 7
        x0 = torch.from_numpy(vec(n, 21, "f64")).cuda()
        layout = Layout.from_bounds(np.array([0, n]))
        bufs = {"cur": torch.zeros(n, dtype=torch.float64, device="cuda"),
                "nxt": torch.zeros(n, dtype=torch.float64, device="cuda"),
                "chunk": torch.zeros(n, dtype=torch.float64, device="cuda"),
                "sums": torch.zeros(E + 1, 2, dtype=torch.float64, device="cuda")}
        if use_comm:
            comm = NativeComm(0, 1, 0)
        z, sums, kms = native_power_iteration(h, layout, 0, x0, bufs, E, comm, time_kernels=True)
        torch.cuda.synchronize()
        assert kms is not None and len(kms) == E and all(k > 0 for k in kms)
        # step-by-step through spmv_power_step must give bitwise the same iterates
        zp = x0.clone()
        sp = torch.zeros(2, dtype=torch.float64, device="cuda")
        P.spmv_norm2(h, zp, sp)
        for k in range(E):
            zn = torch.empty_like(zp)
            sn = torch.zeros(2, dtype=torch.float64, device="cuda")
            P.spmv_power_step(h, zp, zn, sp, sn)
            assert torch.equal(sn, sums[k + 1])
            zp, sp = zn, sn
        assert torch.equal(zp, z)
        # and the oracle's lambda (O11) on the same start vector
        rp, R, C, V = oracle_csr(coo)
        x = x0.cpu().numpy() / np.linalg.norm(x0.cpu().numpy())
        lam = []
        for k in range(E):
            y, x, l, s = oracle.power_step(n, rp, C, V, x)
            lam.append(l)
        s_np = sums.cpu().numpy()
        lam_gpu = s_np[1:, 1] / np.sqrt(s_np[:-1, 0])
        assert np.allclose(lam_gpu, lam, rtol=1e-10, atol=0)
    finally:
        if comm is not None:
            comm.close()
        P.spmv_destroy(h)


@pytest.mark.parametrize("B", [2, 3])
def test_bell_block_matrix_parity_and_selection(B):
    """BELL's best-suited matrix (k-dof 27-point stencil): bit-exact layout,
    SpMV parity, power steps, and the selector measures BELL as a candidate."""
    coo = si.block27(24, B, random_values=True)   # large enough that boundary (Kb) padding < 10%
    h = create(coo)
    try:
        ref = oracle_csr(coo)
        P.spmv_convert(h, P.FMT_BELL, bell_b=B)
        info = P.spmv_format_info(h, P.FMT_BELL)
        bcol = fetch(h, P.ARR_BELL_COL, info["K"] * info["n_pad"], np.int32)
        assert (bcol >= 0).sum() * B * B == coo.nnz   # dense blocks: no padding inside stored blocks
        for a, b in AB:
            check_y(h, coo, "f64", P.FMT_BELL, a, b, ref)
        rep = P.spmv_tune(h, P.TUNE_FORMAT, expected_iterations=10 ** 6)
        sel = [r for r in P.spmv_decision_log(h) if r["kind"] == "format_select"][-1]
        assert any(c["format"] == "BELL" and "t_s" in c for c in sel["candidates"]), sel["candidates"]
        check_y(h, coo, "f64", rep.format, 2.5, -0.5, ref)
    finally:
        P.spmv_destroy(h)


def test_tune_skewed_considers_skew_formats():
    """Run-time mode on a power-law matrix: the selector must measure the
    skew-oriented candidates (merge-path CSR, HYB, COO) and its choice must
    still produce oracle-correct y (fp32 data, fp64 accumulation)."""
    coo = si.rmat(15, dtype=np.float32)
    h = create(coo, "f32")
    try:
        rep = P.spmv_tune(h, P.TUNE_ALL, expected_iterations=10 ** 6)
        sel = [r for r in P.spmv_decision_log(h) if r["kind"] == "format_select"][0]
        measured = {(c["format"], c.get("alg")) for c in sel["candidates"] if "t_s" in c}
        assert ("CSR", "merge") in measured and ("HYB", None) in measured and ("COO", None) in measured
        assert sel["gate"]["t_best_s"] == gate_net_best(sel)["t_s"]
        check_y(h, coo, "f32", rep.format, 2.5, -0.5)
    finally:
        P.spmv_destroy(h)


@pytest.mark.parametrize("objective", ["energy", "power", "efficiency"])
def test_tune_objectives(objective):
    """The paper's four objectives: the selector measures
    each candidate with NVML and picks the best for the objective; the gate
    compares the objective's own units; the chosen format stays correct."""
    coo = si.stencil27(48, random_values=True)
    h = create(coo)
    try:
        try:
            rep = P.spmv_tune(h, P.TUNE_ALL, expected_iterations=10 ** 5, objective=objective)
        except P.SpmvError as e:
            if e.status == P.ERR_NVML:
                pytest.skip("NVML not available")
            raise
        log = P.spmv_decision_log(h)
        sel = [r for r in log if r["kind"] == "format_select"][-1]
        assert sel["objective"] == objective and rep.objective == P.OBJECTIVES[objective]
        cands = [c for c in sel["candidates"] if "t_s" in c]
        for c in cands:
            assert c["j_per_spmv"] > 0 and c["w"] > 0 and c["mflops_per_w"] > 0
            # MFLOPS/W is MFLOP per joule
            assert abs(c["mflops_per_w"] - 2 * coo.nnz / 1e6 / c["j_per_spmv"]) <= 1e-6 * c["mflops_per_w"]
        best = gate_net_best(sel, objective)
        g = sel["gate"]
        assert g["convert"] == (g["gain"] > g["overhead"])
        chosen = sel["chosen"].split("-")[0]
        assert chosen == (best["format"] if g["convert"] else "CSR")
        sweep = [r for r in log if r["kind"] == "launch_sweep"][-1]
        assert sweep["objective"] == objective and len(sweep["objective_top"]) >= 1
        assert np.isfinite(rep.energy_j) and np.isfinite(rep.power_w) and np.isfinite(rep.mflops_per_w)
        check_y(h, coo, "f64", rep.format, 1.0, 0.0)
    finally:
        P.spmv_destroy(h)
