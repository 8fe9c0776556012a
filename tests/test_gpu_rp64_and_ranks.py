"""GPU coverage of paths the small corpus cannot reach otherwise:
 * int64 row pointers (used when nnz >= 2^31, e.g. c5) forced on small
   matrices with SPMV_FORCE_RP64=1 in a subprocess, parity vs the oracle;
 * "virtual ranks": P nnz-balanced row slabs with columns
   remapped into the padded all-gather layout, run on one GPU, must give
   bitwise the same y as the single handle for the row-local formats, and the
   power iteration driven through the same exchange must match the oracle."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import spmv_inputs as si
from gpu_cases import oracle_csr, vec

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_2302_05662_b200")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_int64_row_pointers_parity():
    env = dict(os.environ, SPMV_FORCE_RP64="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-x",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                        "-k", "create_csr_bit_exact or features_bit_exact or layouts or spmv_parity or power_step"],
                       env=env, capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    # the subprocess really ran with 64-bit row pointers
    probe = subprocess.run([sys.executable, "-c",
                            "import torch, paper_2302_05662_b200 as P;"
                            "r=torch.tensor([0,1],dtype=torch.int32,device='cuda');"
                            "v=torch.ones(2,dtype=torch.float64,device='cuda');"
                            "h=P.spmv_create(2,2,r,r,v); print(P.spmv_format_info(h,P.FMT_CSR)['row_ptr_is64'])"],
                           env=env, capture_output=True, text=True, cwd=ROOT)
    assert probe.stdout.strip().endswith("1"), probe.stdout + probe.stderr


def slabs(coo, world):
    lengths = np.bincount(coo.row, minlength=coo.rows)
    bounds = P.spmv_dist_partition_lengths(lengths, world)
    chunk = int(np.max(np.diff(bounds)))
    out = []
    for r in range(world):
        a, b = int(bounds[r]), int(bounds[r + 1])
        sel = (coo.row >= a) & (coo.row < b)
        col = coo.col[sel].copy()
        P.spmv_dist_remap_columns(col, bounds)
        out.append((a, b, (coo.row[sel] - a).astype(np.int32), col, coo.val[sel]))
    return bounds, chunk, out


def to_padded(v, bounds, chunk):
    world = len(bounds) - 1
    out = torch.zeros(world * chunk, dtype=v.dtype, device=v.device)
    for r in range(world):
        a, b = int(bounds[r]), int(bounds[r + 1])
        out[r * chunk: r * chunk + (b - a)] = v[a:b]
    return out


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("fmt,params", [(P.FMT_SELL, {}), (P.FMT_ELL, {}), (P.FMT_CSR, {"csr_alg": P.CSR_VECTOR})])
def test_virtual_ranks_bitwise(world, fmt, params):
    coo = si.stencil27(20, random_values=True)
    n = coo.rows
    x = torch.from_numpy(vec(n, 4, "f64")).cuda()
    # single handle
    h = P.spmv_create(n, n, torch.from_numpy(coo.row).cuda(), torch.from_numpy(coo.col).cuda(),
                      torch.from_numpy(coo.val).cuda())
    P.spmv_convert(h, fmt, **params)
    y1 = torch.empty(n, dtype=torch.float64, device="cuda")
    P.spmv_run(h, 1.0, x, 0.0, y1)
    P.spmv_destroy(h)
    # world slabs on the same GPU, x in the padded all-gather layout
    bounds, chunk, parts = slabs(coo, world)
    xp = to_padded(x, bounds, chunk)
    yp = torch.empty(n, dtype=torch.float64, device="cuda")
    for (a, b, rr, cc, vv) in parts:
        hr = P.spmv_create(b - a, world * chunk, torch.from_numpy(rr).cuda(), torch.from_numpy(cc).cuda(),
                           torch.from_numpy(vv).cuda())
        P.spmv_convert(hr, fmt, **params)
        ys = torch.empty(b - a, dtype=torch.float64, device="cuda")
        P.spmv_run(hr, 1.0, xp, 0.0, ys)
        yp[a:b] = ys
        P.spmv_destroy(hr)
    torch.cuda.synchronize()
    assert torch.equal(y1, yp)


def test_virtual_ranks_power_iteration_vs_oracle():
    world, E = 4, 5
    coo = si.lap2d(48, random_values=True)
    n = coo.rows
    bounds, chunk, parts = slabs(coo, world)
    handles = []
    for (a, b, rr, cc, vv) in parts:
        hr = P.spmv_create(b - a, world * chunk, torch.from_numpy(rr).cuda(), torch.from_numpy(cc).cuda(),
                           torch.from_numpy(vv).cuda())
        P.spmv_convert(hr, P.FMT_SELL)
        handles.append((a, b, hr))
    x0 = torch.from_numpy(vec(n, 8, "f64")).cuda()
    cur = to_padded(x0, bounds, chunk)
    S = float((x0 * x0).sum().item())
    sums_prev = torch.tensor([S, 0.0], dtype=torch.float64, device="cuda")
    rp, R, C, V = oracle_csr(coo)
    xo = x0.cpu().numpy() / np.sqrt(S)
    for k in range(E):
        nxt = torch.zeros_like(cur)
        tot = torch.zeros(2, dtype=torch.float64, device="cuda")
        for r, (a, b, hr) in enumerate(handles):
            y = torch.empty(b - a, dtype=torch.float64, device="cuda")
            so = torch.zeros(2, dtype=torch.float64, device="cuda")
            P.spmv_power_step(hr, cur, y, sums_prev, so, r * chunk)
            nxt[r * chunk: r * chunk + (b - a)] = y          # the all-gather
            tot += so                                         # the all-reduce
        torch.cuda.synchronize()
        lam = float(tot[1].item()) / np.sqrt(float(sums_prev[0].item()))
        y_ref, xo_next, lam_ref, s_ref = oracle.power_step(n, rp, C, V, xo)
        assert abs(lam - lam_ref) <= 1e-10 * abs(lam_ref)
        zg = torch.cat([nxt[r * chunk: r * chunk + (b - a)] for r, (a, b, _) in enumerate(handles)]).cpu().numpy()
        _, a_ref = oracle.spmv_csr(n, rp, C, V, xo)
        ok, worst, bad = oracle.parity_check(zg, y_ref, a_ref, 1.0, 0.0, None, 1e-12)
        assert ok, (k, worst)
        xo = zg / np.sqrt(float(tot[0].item()))               # continue from the GPU's own iterate
        cur, sums_prev = nxt, tot
    for _, _, hr in handles:
        P.spmv_destroy(hr)
