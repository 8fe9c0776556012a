"""The bench's N > 1 branch executed on the hardware this run has.

* `bench.py --gpus W --virtual` (W = 2, 4) runs the exact multi-rank code of
  bench.py — nnz-balanced partition (O12), per-rank slab generation with the
  column remap into the padded all-gather layout, spmv_dist_plan_create /
  _iterate with overlap and halo exchange — as W threads on one GPU joined by
  the in-process communicator group. Its λ_1..λ_E must match the oracle's
  power iteration (O11) on c2 from the same x0, and the one-rank run.
* With two or more visible GPUs, `torchrun --nproc-per-node 2 bench.py` runs
  the same branch over NCCL (plan with and without halo exchange), checked
  the same way. Collected everywhere; skipped on one-GPU boxes.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import spmv_inputs as si

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
E = 5


def _bench(args, launcher=None, timeout=900):
    cmd = (launcher or [sys.executable]) + [os.path.join(ROOT, "bench.py"), "--config", "c2", "--steps", "2",
                                            "--warmup", "1", "--iters", str(E), "--no-cpu-baseline",
                                            "--per-config", "none", "--no-e2e", "--energy-window", "0"] + args
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.fixture(scope="module")
def oracle_lambdas():
    """O11 on c2 (27-point 128³, random values) from the bench's x0."""
    coo = si.config_host("c2")
    st, R, C, V = oracle.canonicalize(coo.rows, coo.cols, coo.row, coo.col, coo.val)
    rp = oracle.csr(coo.rows, R)
    x = si.vector(coo.cols)
    x = x / np.linalg.norm(x)
    lams = []
    for _ in range(E):
        y, x, lam, s = oracle.power_step(coo.rows, rp, C, V, x, all_cores=True)
        lams.append(lam)
    return np.array(lams)


def _check(line, lam_ref, world, virtual):
    assert line["config"]["workload"] == "c2"
    assert line["config"]["partition"] == ("row, nnz-balanced" if world > 1 else "none")
    if world > 1:
        plan = line["config"]["plan"]
        assert plan is not None and len(plan["part_rows"]) == 3
    if virtual:
        assert line["config"]["virtual_ranks"] == world
    assert line["value"] > 0 and line["gpu_launches"] > 0
    lam = np.array(line["lambdas"][:E])
    # O11: λ to 1e-10 relative (the GPU's iterates drift from the oracle's by
    # O9-sized amounts per step; power iteration does not amplify them)
    assert np.all(np.abs(lam - lam_ref) <= 1e-10 * np.abs(lam_ref)), (lam, lam_ref)


@pytest.mark.timeout(1800)
@pytest.mark.parametrize("world", [1, 2, 4])
def test_bench_virtual_ranks_c2(world, oracle_lambdas):
    args = ["--gpus", str(world)] + (["--virtual"] if world > 1 else [])
    line = _bench(args)
    _check(line, oracle_lambdas, world, world > 1)


@pytest.mark.timeout(1800)
@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two GPUs for a real two-rank NCCL run")
@pytest.mark.parametrize("plan", ["none", "overlap", "overlap,halo"])
def test_bench_two_rank_nccl_c2(plan, oracle_lambdas):
    launcher = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                "--master-addr", "127.0.0.1", "--master-port", "29517"]
    line = _bench(["--gpus", "2", "--plan", plan], launcher=launcher)
    assert line["n_gpus"] == 2
    _check(line, oracle_lambdas, 2, False)
