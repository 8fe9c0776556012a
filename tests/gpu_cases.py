"""Shared corpus + helpers for the GPU parity tests (seeded, synthetic).

Every expected value comes from oracle/ (or is a closed form); nothing is
read back from the CUDA path to build an expectation."""
import numpy as np

import oracle
import spmv_inputs as si


def _lengths(seed, rows, hi, p_empty):
    rng = np.random.default_rng(seed)
    L = rng.integers(1, hi + 1, rows)
    L[rng.random(rows) < p_empty] = 0
    return L


def corpus():
    """name -> host COO (sorted, unique). Sizes span several tiles/slices and
    end in a ragged tail; includes the degenerate shapes of SPEC S:262."""
    g = []
    t = np.array([[3, 5, -1], [0, 5, 2], [4, 4, -3], [0, 0, 4], [3, 0, -2], [0, 2, -1], [4, 2, 0.5],
                  [2, 3, 3], [3, 4, 5], [3, 1, 1]], dtype=np.float64)
    o = np.lexsort((t[:, 1], t[:, 0]))
    g.append(("appendix_d", si.COO(5, 6, t[o, 0].astype(np.int32), t[o, 1].astype(np.int32), t[o, 2].copy())))
    g.append(("empty_7x5", si.COO(7, 5, np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0))))
    g.append(("row_1x300", si.random_coo(1, 300, 120, 1)))
    g.append(("col_300x1", si.random_coo(300, 1, 200, 2)))
    g.append(("uniform_rand", si.random_coo(300, 250, 3000, 3)))
    g.append(("ragged_empty", si.random_coo(1000, 700, 0, 4, lengths=_lengths(4, 1000, 40, 0.3))))
    g.append(("long_rows", si.random_coo(70, 6000, 0, 5, lengths=np.array(
        [5000, 0, 3, 4500, 0, 0, 1] + list(_lengths(5, 63, 30, 0.2))))))
    g.append(("rmat10", si.rmat(10, dtype=np.float64)))
    g.append(("lap2d_20", si.lap2d(20, random_values=True)))
    g.append(("stencil27_9", si.stencil27(9, random_values=True)))
    # staged and overflowing tiles of the TMA kernels side by side (a 3000-entry
    # row every 700 rows), segment starts at every 16-byte residue
    Lm = _lengths(7, 3000, 20, 0.15)
    Lm[::700] = 3000
    g.append(("mixed_tiles", si.random_coo(3000, 5000, 0, 7, lengths=Lm)))
    g.append(("wide_3x70000", si.random_coo(3, 70000, 0, 6, lengths=np.array([66000, 0, 65536]))))
    return g


def small_corpus():
    return [c for c in corpus() if c[0] not in ("wide_3x70000",)]


def oracle_csr(coo):
    st, R, C, V = oracle.canonicalize(coo.rows, coo.cols, coo.row, coo.col, coo.val)
    assert st == oracle.OK
    return oracle.csr(coo.rows, R), R, C, V


def to_device(coo, dtype):
    import torch
    tdt = torch.float64 if dtype == "f64" else torch.float32
    return (torch.from_numpy(np.ascontiguousarray(coo.row)).cuda(),
            torch.from_numpy(np.ascontiguousarray(coo.col)).cuda(),
            torch.from_numpy(np.ascontiguousarray(coo.val)).to(tdt).cuda())


def vec(n, seed, dtype):
    x = si.vector(max(n, 1), seed=seed)[:n]
    return x.astype(np.float32 if dtype == "f32" else np.float64)
