"""GPU tests of the distributed power-iteration plan (SURVEY.md §8(e) (i)-(iv),
§8(f) f4) on ONE GPU: W ranks are W host threads of this process, each with
its own stream, joined by the in-process communicator group
(spmv_dist_local_group) — the same loop, split, stream/event schedule and
exchange lists as the NCCL path, with the collectives done by device copies.

Checked against the oracle step by step (O11: each step's z_k against the
oracle's A·x_{k-1} from the GPU's own normalised iterate, O9 tolerance; λ_k
to 1e-10 relative), for every combination of overlap / halo exchange, several
formats, ranks 1-4, stencils (non-empty interior), a general graph (RMAT:
interior may be empty, halo lists fall back to the all-gather) and the
staged (pack/unpack) halo path."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
import spmv_inputs as si
from gpu_cases import oracle_csr, vec

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_2302_05662_b200")
pytestmark = pytest.mark.gpu


def slabs(coo, world):
    lengths = np.bincount(coo.row, minlength=coo.rows)
    bounds = P.spmv_dist_partition_lengths(lengths, world)
    chunk = max(int(np.max(np.diff(bounds))), 1)
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


def run_plan(coo, world, flags, steps_list, fmt, params=None, dtype=torch.float64, x0=None):
    """Runs the plan for each E in steps_list (fresh start from x0 each time);
    returns (infos, {E: (z_E global numpy, sums numpy [E+1, 2])})."""
    params = params or {}
    n = coo.rows
    bounds, chunk, parts = slabs(coo, world)
    comms = P.spmv_dist_local_group(world, [0] * world)
    if x0 is None:
        x0 = torch.from_numpy(vec(n, 8, "f64")).to(dtype).cuda()
    xp = to_padded(x0, bounds, chunk)
    results = {}
    infos = [None] * world

    def rank_main(r):
        torch.cuda.set_device(0)
        st = torch.cuda.Stream()
        a, b, rr, cc, vv = parts[r]
        with torch.cuda.stream(st):
            h = P.spmv_create(b - a, world * chunk, torch.from_numpy(rr).cuda(), torch.from_numpy(cc).cuda(),
                              torch.from_numpy(vv).to(dtype).cuda(), stream=st)
            P.spmv_convert(h, fmt, **params)
            plan = P.spmv_dist_plan_create(h, comms[r], chunk, flags)
            P.spmv_destroy(h)
            infos[r] = P.spmv_dist_plan_info(plan)
            out = {}
            for E in steps_list:
                b0 = torch.zeros(world * chunk, dtype=dtype, device="cuda")
                b1 = torch.zeros_like(b0)
                sums = torch.zeros(E + 1, 2, dtype=torch.float64, device="cuda")
                fb, _, _ = P.spmv_dist_plan_iterate(plan, xp, b0, b1, E, sums)
                st.synchronize()
                z = (b0 if fb == 0 else b1)[r * chunk: r * chunk + (b - a)].double().cpu().numpy()
                out[E] = (z, sums.cpu().numpy())
            P.spmv_dist_plan_destroy(plan)
        st.synchronize()
        return out

    try:
        with ThreadPoolExecutor(world) as ex:
            per_rank = list(ex.map(rank_main, range(world)))
    finally:
        for c in comms:
            P.spmv_dist_destroy(c)
    for E in steps_list:
        z = np.concatenate([per_rank[r][E][0] for r in range(world)])
        sums = per_rank[0][E][1]
        for r in range(1, world):  # the all-reduce gives every rank the same sums
            assert np.array_equal(per_rank[r][E][1], sums)
        results[E] = (z, sums)
    return infos, results, x0


def check_vs_oracle(coo, results, x0, E, tau=1e-12):
    n = coo.rows
    rp, R, C, V = oracle_csr(coo)
    x_prev = x0.double().cpu().numpy()
    s_prev = float(np.dot(x_prev, x_prev))
    for k in range(1, E + 1):
        z, sums = results[k]
        assert sums[k - 1, 0] == pytest.approx(s_prev, rel=1e-13)
        xo = x_prev / np.sqrt(s_prev)
        y_ref, _, lam_ref, s_ref = oracle.power_step(n, rp, C, V, xo)
        _, a_ref = oracle.spmv_csr(n, rp, C, V, xo)
        ok, worst, bad = oracle.parity_check(z, y_ref, a_ref, 1.0, 0.0, None, tau)
        assert ok, (k, worst, bad[:5] if bad is not None else None)
        lam = sums[k, 1] / np.sqrt(sums[k - 1, 0])
        # λ = x·z: its error bound follows O9 row by row (Σ |x_i|·a_i), plus O11's 1e-10 relative
        lam_tol = 1e-10 * abs(lam_ref) + tau * float(np.dot(np.abs(xo), a_ref))
        assert abs(lam - lam_ref) <= lam_tol, (k, lam, lam_ref)
        assert sums[k, 0] == pytest.approx(float(np.dot(z, z)), rel=1e-12)
        # the longer runs reproduce the shorter ones exactly (deterministic schedule)
        if k < E:
            assert np.array_equal(results[E][1][: k + 1], sums)
        x_prev, s_prev = z, sums[k, 0]


FLAGS = [0, P.PLAN_OVERLAP, P.PLAN_HALO, P.PLAN_OVERLAP | P.PLAN_HALO]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("flags", FLAGS)
@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_plan_stencil_sell(world, flags):
    coo = si.lap2d(40, random_values=True)
    infos, res, x0 = run_plan(coo, world, flags, [1, 2, 3], P.FMT_SELL)
    check_vs_oracle(coo, res, x0, 3)
    for r, inf in enumerate(infos):
        assert inf["world"] == world and inf["rank"] == r
        assert sum(inf["part_rows"]) == inf["rows"]
        if world > 1:
            assert 0 < inf["h0"] <= inf["h1"] or r == 0
            assert inf["part_rows"][0] > 0          # a 2-D stencil slab has interior rows
            assert inf["halo"] == (1 if flags & P.PLAN_HALO else 0)
            if inf["halo"]:
                # 5-point stencil: at most one grid row from each neighbour
                assert 0 < inf["recv_elems"] <= 2 * 40
                assert inf["recv_elems"] < (world - 1) * inf["chunk"]
        else:
            assert inf["part_rows"] == [coo.rows, 0, 0] and inf["recv_elems"] == 0


@pytest.mark.timeout(600)
@pytest.mark.parametrize("fmt,params", [(P.FMT_CSR, {"csr_alg": P.CSR_VECTOR}), (P.FMT_CSR, {"csr_alg": P.CSR_MERGE}),
                                        (P.FMT_ELL, {}), (P.FMT_HYB, {}), (P.FMT_COO, {}),
                                        (P.FMT_SELL, {"sell_C": 32, "sell_sigma": 64}),
                                        (P.FMT_CSR, {"csr_alg": P.CSR_STREAM})])
def test_plan_formats_stencil27(fmt, params):
    coo = si.stencil27(14, random_values=True)
    infos, res, x0 = run_plan(coo, 3, P.PLAN_OVERLAP | P.PLAN_HALO, [1, 2], fmt, params)
    check_vs_oracle(coo, res, x0, 2)
    assert all(i["halo"] == 1 for i in infos)


@pytest.mark.timeout(600)
def test_plan_bell_block_matrix():
    coo = si.block27(8, 3, random_values=True)
    infos, res, x0 = run_plan(coo, 2, P.PLAN_OVERLAP | P.PLAN_HALO, [1, 2], P.FMT_BELL, {"bell_b": 3})
    check_vs_oracle(coo, res, x0, 2)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("flags", [P.PLAN_OVERLAP, P.PLAN_OVERLAP | P.PLAN_HALO])
def test_plan_general_graph(flags):
    # RMAT: columns everywhere -> interior may be empty and the halo lists
    # would move about as much as the all-gather (the plan keeps the all-gather)
    coo = si.rmat(10, 8)
    infos, res, x0 = run_plan(coo, 3, flags, [1, 2], P.FMT_CSR, {"csr_alg": P.CSR_VECTOR})
    check_vs_oracle(coo, res, x0, 2)
    for inf in infos:
        assert sum(inf["part_rows"]) == inf["rows"]


@pytest.mark.timeout(600)
def test_plan_staged_halo(monkeypatch):
    monkeypatch.setenv("SPMV_PLAN_FORCE_STAGED", "1")
    coo = si.stencil27(12, random_values=True)
    infos, res, x0 = run_plan(coo, 4, P.PLAN_OVERLAP | P.PLAN_HALO, [1, 2, 3], P.FMT_SELL)
    check_vs_oracle(coo, res, x0, 3)
    assert all(i["halo"] == 1 and i["direct_recv"] == 0 and i["direct_send"] == 0 for i in infos)


@pytest.mark.timeout(600)
def test_plan_fp32():
    coo = si.lap2d(32, random_values=True)
    infos, res, x0 = run_plan(coo, 2, P.PLAN_OVERLAP | P.PLAN_HALO, [1, 2], P.FMT_SELL, dtype=torch.float32)
    # fp32 storage of z: compare with the fp32 tolerance
    check_vs_oracle(coo, res, x0, 2, tau=1e-5)


@pytest.mark.timeout(600)
def test_plan_matches_single_handle_loop():
    """The plan at world 1 runs the same kernels as spmv_power_iterate: the
    iterate agrees to rounding of the (differently ordered) norm sums."""
    coo = si.stencil27(16, random_values=True)
    n = coo.rows
    E = 6
    infos, res, x0 = run_plan(coo, 1, P.PLAN_OVERLAP, [E], P.FMT_SELL)
    h = P.spmv_create(n, n, torch.from_numpy(coo.row).cuda(), torch.from_numpy(coo.col).cuda(),
                      torch.from_numpy(coo.val).cuda())
    P.spmv_convert(h, P.FMT_SELL)
    b0 = torch.zeros(n, dtype=torch.float64, device="cuda")
    b1 = torch.zeros_like(b0)
    sums = torch.zeros(E + 1, 2, dtype=torch.float64, device="cuda")
    fb, _, _ = P.spmv_power_iterate(h, x0, b0, b1, E, sums)
    torch.cuda.synchronize()
    z1 = (b0 if fb == 0 else b1).cpu().numpy()
    P.spmv_destroy(h)
    zp, sp = res[E]
    assert np.allclose(zp, z1, rtol=1e-12, atol=0)
    assert np.allclose(sp, sums.cpu().numpy(), rtol=1e-12, atol=0)


def test_row_slice_bit_exact():
    coo = si.rmat(9, 8)
    n = coo.rows
    h = P.spmv_create(n, coo.cols, torch.from_numpy(coo.row).cuda(), torch.from_numpy(coo.col).cuda(),
                      torch.from_numpy(coo.val).cuda())
    rp = torch.zeros(n + 1, dtype=torch.int32)
    P.spmv_copy_array(h, P.ARR_CSR_ROW_PTR, rp)
    for (a, b) in [(0, n), (0, 0), (3, 3), (5, n // 2), (n // 3, n)]:
        s = P.spmv_create_row_slice(h, a, b)
        rps = torch.zeros(b - a + 1, dtype=torch.int32)
        P.spmv_copy_array(s, P.ARR_CSR_ROW_PTR, rps)
        assert torch.equal(rps, (rp[a:b + 1] - rp[a]).to(torch.int32))
        nnz = int(rp[b] - rp[a])
        if nnz:
            c = torch.zeros(nnz, dtype=torch.int32)
            P.spmv_copy_array(s, P.ARR_CSR_COL, c)
            assert np.array_equal(c.numpy(), coo.col[int(rp[a]):int(rp[b])])
        P.spmv_destroy(s)
    with pytest.raises(P.SpmvError):
        P.spmv_create_row_slice(h, 5, 3)
    with pytest.raises(P.SpmvError):
        P.spmv_create_row_slice(h, 0, n + 1)
    P.spmv_destroy(h)


def test_plan_errors():
    coo = si.lap2d(8)
    n = coo.rows
    h = P.spmv_create(n, n, torch.from_numpy(coo.row).cuda(), torch.from_numpy(coo.col).cuda(),
                      torch.from_numpy(coo.val).cuda())
    with pytest.raises(P.SpmvError):
        P.spmv_dist_plan_create(h, None, 0, 8)         # unknown flag
    comms = P.spmv_dist_local_group(1, [0])
    with pytest.raises(P.SpmvError):
        P.spmv_dist_plan_create(h, comms[0], n - 1, 0)  # chunk < local rows
    plan = P.spmv_dist_plan_create(h, comms[0], n, P.PLAN_OVERLAP | P.PLAN_HALO)
    info = P.spmv_dist_plan_info(plan)
    assert info["world"] == 1 and info["halo"] == 0 and info["part_rows"] == [n, 0, 0]
    assert P.spmv_dist_plan_part(plan, 1) is None and P.spmv_dist_plan_part(plan, 0) is not None
    P.spmv_dist_plan_destroy(plan)
    P.spmv_dist_destroy(comms[0])
    P.spmv_destroy(h)


GRAPH_VARIANTS = [(P.FMT_CSR, dict(csr_alg=P.CSR_VECTOR), None), (P.FMT_CSR, dict(csr_alg=P.CSR_STREAM), None),
                  (P.FMT_CSR, dict(csr_alg=P.CSR_MERGE), None), (P.FMT_CSR, dict(csr_alg=P.CSR_MERGE), 0x408),
                  (P.FMT_ELL, {}, None), (P.FMT_ELL, dict(index16=2), None), (P.FMT_SELL, {}, None),
                  (P.FMT_HYB, dict(hyb_K=3), None), (P.FMT_COO, {}, None), (P.FMT_BELL, dict(bell_b=2), None)]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("fmt,params,knob", GRAPH_VARIANTS)
def test_power_iterate_graph(fmt, params, knob):
    """spmv_power_iterate_graph (the single-GPU loop as a CUDA graph, SURVEY
    c1): the first call runs eagerly then captures; replays are bitwise equal
    to the eager loop (same kernels, same order) and count their kernels in
    spmv_launch_count; a launch change re-captures; the result matches the
    oracle's power iteration (O11) step by step through the eager loop."""
    coo = si.lap2d(64, random_values=True)   # c1: launch-bound
    n = coo.rows
    E = 20
    h = P.spmv_create(n, n, torch.from_numpy(coo.row).cuda(), torch.from_numpy(coo.col).cuda(),
                      torch.from_numpy(coo.val).cuda())
    try:
        P.spmv_convert(h, fmt, **params)
        if knob is not None:
            P.spmv_set_launch(h, fmt, 128, 64, -1, knob)
        x0 = torch.from_numpy(vec(n, 5, "f64")).cuda()
        b0, b1 = torch.zeros(n, dtype=torch.float64, device="cuda"), torch.zeros(n, dtype=torch.float64, device="cuda")
        s_e = torch.zeros(E + 1, 2, dtype=torch.float64, device="cuda")
        fb, _, _ = P.spmv_power_iterate(h, x0, b0, b1, E, s_e)
        torch.cuda.synchronize()
        z_e = (b0 if fb == 0 else b1).clone()
        l0 = P.launch_count()
        P.spmv_power_iterate(h, x0, b0, b1, E, s_e)
        torch.cuda.synchronize()
        per_loop = P.launch_count() - l0
        g0, g1 = torch.zeros_like(b0), torch.zeros_like(b0)
        s_g = torch.zeros_like(s_e)
        for rep in range(3):
            g0.fill_(float("nan")), g1.fill_(float("nan")), s_g.fill_(float("nan"))
            c0 = P.launch_count()
            fg = P.spmv_power_iterate_graph(h, x0, g0, g1, E, s_g)
            torch.cuda.synchronize()
            assert fg == fb
            assert torch.equal((g0 if fg == 0 else g1), z_e), rep
            assert torch.equal(s_g, s_e), rep
            assert P.launch_count() - c0 == per_loop, (rep, P.launch_count() - c0, per_loop)
        P.spmv_set_launch(h, fmt, *P.spmv_get_launch(h, fmt))     # invalidates: re-captured, same result
        fg = P.spmv_power_iterate_graph(h, x0, g0, g1, E, s_g)
        fg = P.spmv_power_iterate_graph(h, x0, g0, g1, E, s_g)
        torch.cuda.synchronize()
        assert torch.equal((g0 if fg == 0 else g1), z_e) and torch.equal(s_g, s_e)
        res = {}
        zz0, zz1 = torch.zeros_like(b0), torch.zeros_like(b0)
        for k in (1, 2, 3):
            sk = torch.zeros(k + 1, 2, dtype=torch.float64, device="cuda")
            f = P.spmv_power_iterate_graph(h, x0, zz0, zz1, k, sk)
            torch.cuda.synchronize()
            res[k] = ((zz0 if f == 0 else zz1).cpu().numpy().copy(), sk.cpu().numpy())
        check_vs_oracle(coo, res, x0, 3)
    finally:
        P.spmv_destroy(h)
