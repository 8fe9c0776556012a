"""Distinct handles are independent (include/spmv.h, thread safety): the way
bench.py's end-to-end leg runs two steps in flight — two host threads, each
with its own stream and handle, creating from pinned host COO (64 MB upload
pieces), extracting features, converting and running at the same time. Every
result is checked against the oracle (O9) and the features bit-exactly."""
import threading

import numpy as np
import pytest

import oracle
import spmv_inputs as si
from gpu_cases import oracle_csr, vec

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_2302_05662_b200")
pytestmark = pytest.mark.gpu


def _lane(coo, fmt, params, x, expect, feats_ref, stream, errors, rounds):
    try:
        hr, hc, hv = (torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (coo.row, coo.col, coo.val))
        xd = torch.from_numpy(x).cuda()
        for _ in range(rounds):
            with torch.cuda.stream(stream):
                h = P.spmv_create(coo.rows, coo.cols, hr.numpy(), hc.numpy(), hv.numpy(), stream=stream)
                try:
                    f = P.spmv_features(h)
                    for k, v in feats_ref.items():
                        assert np.float64(f[k]).tobytes() == np.float64(v).tobytes(), (k, f[k], v)
                    P.spmv_convert(h, fmt, **params)
                    y = torch.full((coo.rows,), float("nan"), dtype=torch.float64, device="cuda")
                    P.spmv_run(h, 2.5, xd, 0.0, y)
                    stream.synchronize()
                    y_ref, a_ref = expect
                    ok, worst, bad = oracle.parity_check(y.cpu().numpy(), y_ref, a_ref, 2.5, 0.0, None, 1e-12)
                    assert ok, (P.FORMAT_NAMES[fmt], worst, bad[:5])
                finally:
                    P.spmv_destroy(h)
    except Exception as ex:  # surfaced in the main thread
        errors.append(ex)


def test_two_handles_in_flight():
    cases = [(si.stencil27(40, random_values=True), P.FMT_ELL, {"index16": 1}),
             (si.rmat(14, dtype=np.float64), P.FMT_COO, {})]
    lanes = []
    for coo, fmt, params in cases:
        rp, R, C, V = oracle_csr(coo)
        _, feats_ref = oracle.features(coo.rows, coo.cols, rp, C)
        x = vec(coo.cols, 7, "f64")
        expect = oracle.spmv_csr(coo.rows, rp, C, V, x, 2.5, 0.0, None)
        lanes.append((coo, fmt, params, x, expect, feats_ref))
    errors = []
    threads = [threading.Thread(target=_lane, args=(*ln, torch.cuda.Stream(), errors, 4)) for ln in lanes]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
