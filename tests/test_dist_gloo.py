"""N>1 path on CPU: world_size-2 gloo run of the row-partitioned power
iteration driver (paper_2302_05662_b200/dist.py) with the product's host
partition + column remap (C ABI), and the oracle as the per-rank local SpMV.
Result must match a single-process oracle power iteration (O11) step by step."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2302_05662_b200 as P
import spmv_inputs as si
from paper_2302_05662_b200.dist import HaloExchange, Layout, PowerIteration

STEPS = 6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p



def _worker(rank, world, port, q, kind, halo=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        coo = si.rmat(9, ef=8, dtype=np.float64) if kind == "rmat" else si.lap2d(24, random_values=True)
        n = coo.rows
        lengths = np.bincount(coo.row, minlength=n)
        bounds = P.spmv_dist_partition_lengths(lengths, world)
        L = Layout.from_bounds(bounds)
        a, b = L.rows_of(rank)
        sel = (coo.row >= a) & (coo.row < b)
        r_loc = (coo.row[sel] - a).astype(np.int32)
        c_loc = coo.col[sel].copy()
        P.spmv_dist_remap_columns(c_loc, bounds)          # product host logic (C ABI)
        st, R, C, V = oracle.canonicalize(b - a, L.padded_n, r_loc, c_loc, coo.val[sel])
        assert st == oracle.OK
        rp = oracle.csr(b - a, R)

        def local_step(x_full, y_local, sums_prev, sums_out, off):
            alpha = 1.0 / np.sqrt(float(sums_prev[0]))
            xf = x_full.numpy()
            y, _ = oracle.spmv_csr(b - a, rp, C, V, xf, alpha, 0.0, None)
            y_local.copy_(torch.from_numpy(y))
            sums_out[0] = float(np.dot(y, y))
            sums_out[1] = float(np.dot(xf[off: off + (b - a)], y))

        def local_norm2(xl, so):
            v = xl.numpy()
            so[0] = float(np.dot(v, v))
            so[1] = 0.0

        hx = HaloExchange(L, rank, C) if halo else None
        pi = PowerIteration(L, rank, local_step, local_norm2, halo=hx)
        x0 = L.to_padded(si.vector(n))
        z, sums = pi.run(torch.from_numpy(x0), STEPS)
        # own chunk of the final iterate from every rank (halo mode keeps only own + halo entries)
        a0, b0 = L.rows_of(rank)
        own = z[rank * L.chunk: rank * L.chunk + (b0 - a0)].clone()
        parts = [torch.zeros(L.chunk, dtype=own.dtype) for _ in range(world)]
        padded = torch.zeros(L.chunk, dtype=own.dtype)
        padded[: b0 - a0] = own
        dist.all_gather(parts, padded)
        if rank == 0:
            zf = torch.cat(parts).numpy()
            q.put((L.from_padded(zf), PowerIteration.lambdas(sums), hx.recv_elems if hx else None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,halo", [("lap2d", False), ("rmat", False), ("lap2d", True), ("rmat", True)])
def test_power_iteration_gloo_world2(kind, halo):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, kind, halo)) for r in range(world)]
    for p in procs:
        p.start()
    z_dist, lam_dist, recv = q.get(timeout=240)
    if halo and kind == "lap2d":
        assert recv == 24   # one grid row of the 24x24 Laplacian from the neighbour
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process oracle power iteration (O11)
    coo = si.rmat(9, ef=8, dtype=np.float64) if kind == "rmat" else si.lap2d(24, random_values=True)
    st, R, C, V = oracle.canonicalize(coo.rows, coo.cols, coo.row, coo.col, coo.val)
    rp = oracle.csr(coo.rows, R)
    x = si.vector(coo.rows)
    x = x / np.linalg.norm(x)
    lams = []
    for k in range(STEPS):
        y, x, lam, s = oracle.power_step(coo.rows, rp, C, V, x)
        lams.append(lam)
    assert np.allclose(lam_dist, lams, rtol=1e-10, atol=0)
    # z_dist is the unnormalised last iterate; compare directions
    zn = z_dist / np.linalg.norm(z_dist)
    assert np.abs(zn - x).max() < 1e-10
