"""CPU-side checks of the C ABI: the library loads, exports every symbol
include/spmv.h declares, rejects bad arguments before touching a device, and
its host-only multi-GPU logic (partition, column remap) matches the oracle's
definition (O12). No GPU needed; no compute calls."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import paper_2302_05662_b200 as P
import spmv_inputs as si

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "spmv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spmv_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = P.lib()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", P.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (spmv_[a-z0-9_]+)\b", out))
    assert set(syms) <= exported, set(syms) - exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_counter():
    for s in range(9):
        assert P.status_string(s).startswith("SPMV_")
    assert isinstance(P.launch_count(), int)


def test_create_rejects_bad_arguments_without_device():
    L = P.lib()
    h = ctypes.c_void_p()
    assert L.spmv_create(None, 1, 1, 0, None, None, None, 1, 1, 0, None) == P.ERR_INVALID_ARG
    assert L.spmv_create(ctypes.byref(h), -1, 1, 0, None, None, None, 1, 1, 0, None) == P.ERR_INVALID_ARG
    assert L.spmv_create(ctypes.byref(h), 1, 1, 3, None, None, None, 1, 1, 0, None) == P.ERR_INVALID_ARG
    assert L.spmv_create(ctypes.byref(h), 1, 1, 0, None, None, None, 7, 1, 0, None) == P.ERR_INVALID_ARG
    assert L.spmv_create(ctypes.byref(h), 2 ** 31, 1, 0, None, None, None, 1, 1, 0, None) == P.ERR_UNSUPPORTED
    assert h.value is None
    assert L.spmv_destroy(None) == P.OK
    assert L.spmv_run(None, 1.0, None, 0.0, None) == P.ERR_INVALID_ARG
    assert L.spmv_tune(None, 3, 1, None) == P.ERR_INVALID_ARG
    assert L.spmv_release_csr(None) == P.ERR_INVALID_ARG


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_partition_matches_oracle_definition(world):
    rng = np.random.default_rng(world)
    for trial in range(5):
        lengths = rng.integers(0, 40, int(rng.integers(1, 500))) * (rng.random() < 0.9)
        rp = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
        b = P.spmv_dist_partition(rp, world)
        assert b.tolist() == oracle.partition(len(lengths), rp, world).tolist()
        assert P.spmv_dist_partition_lengths(lengths, world).tolist() == b.tolist()


def test_partition_rmat_skew():
    coo = si.rmat(14)
    rp = np.concatenate([[0], np.cumsum(np.bincount(coo.row, minlength=coo.rows))]).astype(np.int64)
    for world in (2, 4, 8):
        b = P.spmv_dist_partition(rp, world)
        assert b.tolist() == oracle.partition(coo.rows, rp, world).tolist()
        per = np.diff(rp[b])
        assert per.max() - per.min() <= 2 * np.diff(rp).max()


def test_remap_columns_host():
    bounds = np.array([0, 3, 4, 10], np.int64)
    col = np.arange(10, dtype=np.int32)
    P.spmv_dist_remap_columns(col, bounds)
    chunk = 6
    expect = [0, 1, 2, chunk + 0, 2 * chunk + 0, 2 * chunk + 1, 2 * chunk + 2, 2 * chunk + 3, 2 * chunk + 4,
              2 * chunk + 5]
    assert col.tolist() == expect
