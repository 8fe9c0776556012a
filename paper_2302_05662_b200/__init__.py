"""paper_2302_05662_b200 — B200-native SpMV (Auto-SpMV, arXiv 2302.05662).

Thin ctypes binding over libspmv.so (include/spmv.h). Argument marshalling
only: every step of the path (ingest, CSR build, features, format builds,
SpMV kernels, tuner, selector, power step) runs in the library's sm_100a
CUDA kernels. There is no CPU fallback: importing this package without the
built library, or calling it without a CUDA device, raises.

torch is used for device memory and streams only. Function names follow the
C ABI: spmv_create / spmv_convert / spmv_features / spmv_run / spmv_tune ...
"""
from __future__ import annotations

import ctypes
import json
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libspmv.so")

# ---------------------------------------------------------------- enums (spmv.h)
OK, ERR_INVALID_ARG, ERR_INDEX_OUT_OF_RANGE, ERR_DUPLICATE, ERR_INFEASIBLE, ERR_OUT_OF_MEMORY, \
    ERR_UNSUPPORTED, ERR_CUDA, ERR_NOT_CONVERTED, ERR_NCCL, ERR_NVML = range(11)
R32F, R64F = 0, 1
MEM_HOST, MEM_DEVICE = 0, 1
FMT_COO, FMT_CSR, FMT_ELL, FMT_HYB, FMT_SELL, FMT_BELL = 0, 1, 2, 3, 4, 5
FORMATS = {"COO": FMT_COO, "CSR": FMT_CSR, "ELL": FMT_ELL, "HYB": FMT_HYB, "SELL": FMT_SELL, "BELL": FMT_BELL}
FORMAT_NAMES = {v: k for k, v in FORMATS.items()}
CSR_AUTO, CSR_SCALAR, CSR_VECTOR, CSR_MERGE, CSR_STREAM = 0, 1, 2, 3, 4
TUNE_LAUNCH, TUNE_FORMAT, TUNE_ALL = 1, 2, 3
TUNE_PREDICT = 4  # with TUNE_FORMAT: learned selector + overhead estimators instead of measuring candidates
TUNE_DECIDE_ONLY = 8  # with TUNE_FORMAT | TUNE_PREDICT: report the verdict, leave the handle unconverted
SELECTOR_CLASSES = ["CSR-vector", "CSR-merge", "ELL", "SELL", "HYB", "COO", "BELL-2", "BELL-3", "CSR-stream"]
OBJECTIVES = {"latency": 0, "energy": 1, "power": 2, "efficiency": 3}   # OR-ed into flags as value << 4
(ARR_CSR_ROW_PTR, ARR_CSR_COL, ARR_CSR_VAL, ARR_COO_ROW, ARR_ELL_COL, ARR_ELL_VAL, ARR_SELL_PERM,
 ARR_SELL_SLICE_PTR, ARR_SELL_COL, ARR_SELL_VAL, ARR_HYB_ELL_COL, ARR_HYB_ELL_VAL, ARR_HYB_TAIL_ROW,
 ARR_HYB_TAIL_COL, ARR_HYB_TAIL_VAL, ARR_COO_EMPTY_ROWS, ARR_BELL_COL, ARR_BELL_VAL, ARR_ELL_COL16,
 ARR_SELL_COL16, ARR_ELL_COL8, ARR_SELL_COL8, ARR_DICT8_TAB) = range(23)


class SpmvError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{status_string(status)}: {msg}")
        self.status = status


class FormatParams(ctypes.Structure):
    _fields_ = [("csr_alg", ctypes.c_int32), ("csr_T", ctypes.c_int32), ("sell_C", ctypes.c_int32),
                ("sell_sigma", ctypes.c_int32), ("hyb_K", ctypes.c_int64), ("bell_b", ctypes.c_int32),
                ("index16", ctypes.c_int32)]


class Features(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in
                ("n_rows", "n_cols", "nnz", "max_len", "min_len", "n_empty", "mode", "bw_lower",
                 "bw_upper", "bandwidth")] + \
               [(n, ctypes.c_double) for n in ("mean", "var", "std", "ell_ratio", "median")]

    def as_dict(self):
        return {f[0]: getattr(self, f[0]) for f in self._fields_}


class Launch(ctypes.Structure):
    _fields_ = [("block", ctypes.c_int32), ("maxreg", ctypes.c_int32), ("carveout_pct", ctypes.c_int32),
                ("knob", ctypes.c_int32)]

    def as_tuple(self):
        return (self.block, self.maxreg, self.carveout_pct, self.knob)


class TuneReport(ctypes.Structure):
    _fields_ = [("format", ctypes.c_int32), ("params", FormatParams), ("launch", Launch),
                ("t_csr_s", ctypes.c_double), ("t_best_s", ctypes.c_double),
                ("f_latency_s", ctypes.c_double), ("c_latency_s", ctypes.c_double),
                ("expected_iterations", ctypes.c_int64), ("converted", ctypes.c_int32),
                ("n_candidates", ctypes.c_int32), ("n_variants", ctypes.c_int32),
                ("objective", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("energy_j", ctypes.c_double), ("power_w", ctypes.c_double), ("mflops_per_w", ctypes.c_double)]


class FormatInfo(ctypes.Structure):
    _fields_ = [("present", ctypes.c_int32), ("row_ptr_is64", ctypes.c_int32)] + \
               [(n, ctypes.c_int64) for n in ("K", "n_pad", "C", "sigma", "n_slices", "slots", "tail_nnz",
                                              "n_empty_rows", "stored_bytes", "block", "index_bytes")]


class Prediction(ctypes.Structure):
    _fields_ = [("cls", ctypes.c_int32), ("format", ctypes.c_int32), ("params", FormatParams),
                ("speed_ratio", ctypes.c_double), ("c_latency_s", ctypes.c_double), ("f_latency_s", ctypes.c_double)]


class PlanInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("rank", "world", "overlap", "halo")] + \
               [(n, ctypes.c_int64) for n in ("rows", "chunk", "h0", "h1")] + \
               [("part_rows", ctypes.c_int64 * 3), ("part_nnz", ctypes.c_int64 * 3)] + \
               [(n, ctypes.c_int64) for n in ("recv_elems", "send_elems", "recv_bytes_per_step")] + \
               [(n, ctypes.c_int32) for n in ("direct_recv", "direct_send")]

    def as_dict(self):
        d = {}
        for f in self._fields_:
            v = getattr(self, f[0])
            d[f[0]] = list(v) if f[0] in ("part_rows", "part_nnz") else v
        return d


PLAN_OVERLAP, PLAN_HALO = 1, 2

_lib = None


def lib():
    """Load libspmv.so. Raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, d, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_uint32
    H = ctypes.c_void_p
    sigs = {
        "spmv_create": ([ctypes.POINTER(H), i64, i64, i64, vp, vp, vp, i32, i32, i32, vp], i32),
        "spmv_convert": ([H, i32, ctypes.POINTER(FormatParams)], i32),
        "spmv_set_format": ([H, i32], i32),
        "spmv_get_format": ([H, ctypes.POINTER(ctypes.c_int)], i32),
        "spmv_features": ([H, ctypes.POINTER(Features)], i32),
        "spmv_run": ([H, d, vp, d, vp], i32),
        "spmv_run_format": ([H, i32, d, vp, d, vp], i32),
        "spmv_set_launch": ([H, i32, ctypes.POINTER(Launch)], i32),
        "spmv_get_launch": ([H, i32, ctypes.POINTER(Launch)], i32),
        "spmv_tune": ([H, u32, i64, ctypes.POINTER(TuneReport)], i32),
        "spmv_power_step": ([H, vp, vp, vp, vp, i64], i32),
        "spmv_norm2": ([H, vp, i64, vp], i32),
        "spmv_format_info": ([H, i32, ctypes.POINTER(FormatInfo)], i32),
        "spmv_copy_array": ([H, i32, vp, i64, i32], i32),
        "spmv_set_stream": ([H, vp], i32),
        "spmv_destroy": ([H], i32),
        "spmv_status_string": ([i32], ctypes.c_char_p),
        "spmv_last_error": ([H], ctypes.c_char_p),
        "spmv_decision_log": ([H, ctypes.c_char_p, ctypes.c_size_t], ctypes.c_size_t),
        "spmv_overheads": ([H, ctypes.POINTER(d), ctypes.POINTER(d)], i32),
        "spmv_launch_count": ([], ctypes.c_uint64),
        "spmv_trim_pool": ([i32], i32),
        "spmv_release_csr": ([H], i32),
        "spmv_power_iterate_graph": ([H, vp, vp, vp, i64, i64, vp, ctypes.POINTER(ctypes.c_int)], i32),
        "spmv_power_iterate": ([H, vp, vp, vp, i64, i64, vp, vp, i64, vp, ctypes.POINTER(ctypes.c_float),
                                ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int)], i32),
        "spmv_predict": ([ctypes.POINTER(Features), i32, ctypes.POINTER(Prediction)], i32),
        "spmv_dist_plan_create": ([ctypes.POINTER(vp), H, vp, i64, u32], i32),
        "spmv_dist_plan_info": ([vp, ctypes.POINTER(PlanInfo)], i32),
        "spmv_dist_plan_part": ([vp, i32, ctypes.POINTER(H)], i32),
        "spmv_dist_plan_iterate": ([vp, vp, vp, vp, i64, vp, ctypes.POINTER(ctypes.c_float),
                                    ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int)], i32),
        "spmv_dist_plan_destroy": ([vp], i32),
        "spmv_dist_local_group": ([i32, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(vp)], i32),
        "spmv_create_row_slice": ([ctypes.POINTER(H), H, i64, i64], i32),
        "spmv_dist_unique_id": ([ctypes.c_char_p], i32),
        "spmv_dist_init": ([ctypes.POINTER(vp), ctypes.c_char_p, i32, i32, i32], i32),
        "spmv_dist_destroy": ([vp], i32),
        "spmv_dist_partition": ([i64, vp, i32, vp], i32),
        "spmv_dist_partition_lengths": ([i64, vp, i32, vp], i32),
        "spmv_dist_remap_columns": ([vp, i64, vp, i32, i32, vp], i32),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def status_string(s: int) -> str:
    return lib().spmv_status_string(s).decode()


def _check(st: int, h=None):
    if st != OK:
        msg = (lib().spmv_last_error(h) or b"").decode()
        raise SpmvError(st, msg)


def _ptr(t) -> int | None:
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data  # numpy (host memory)


def _stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def launch_count() -> int:
    return int(lib().spmv_launch_count())


# ---------------------------------------------------------------- C-ABI wrappers (same names)

def spmv_create(rows, cols, row_idx, col_idx, vals, device: int = 0, stream=None):
    """row_idx/col_idx int32, vals float32/float64 — torch CUDA tensors (device
    memory) or numpy arrays / CPU tensors (host memory). Returns a handle."""
    import numpy as np
    import torch
    nnz = int(row_idx.shape[0])
    if isinstance(vals, torch.Tensor):
        dt = R64F if vals.dtype == torch.float64 else (R32F if vals.dtype == torch.float32 else None)
        where = MEM_DEVICE if vals.is_cuda else MEM_HOST
        for t in (row_idx, col_idx):
            assert t.dtype == torch.int32 and t.is_contiguous() and t.is_cuda == vals.is_cuda
        assert vals.is_contiguous()
    else:
        dt = R64F if vals.dtype == np.float64 else (R32F if vals.dtype == np.float32 else None)
        where = MEM_HOST
        for t in (row_idx, col_idx):
            assert t.dtype == np.int32 and t.flags["C_CONTIGUOUS"]
        assert vals.flags["C_CONTIGUOUS"]
    if dt is None:
        raise TypeError("values must be float32 or float64")
    h = ctypes.c_void_p()
    st = lib().spmv_create(ctypes.byref(h), int(rows), int(cols), nnz, _ptr(row_idx), _ptr(col_idx),
                           _ptr(vals), dt, where, device, _stream_ptr(stream))
    _check(st, None)
    return h


def spmv_release_csr(h):
    """Free the CSR/COO arrays after conversion (include/spmv.h)."""
    _check(lib().spmv_release_csr(h), h)


def spmv_convert(h, fmt, csr_alg=0, csr_T=0, sell_C=0, sell_sigma=0, hyb_K=-1, bell_b=0, index16=0):
    p = FormatParams(csr_alg, csr_T, sell_C, sell_sigma, hyb_K, bell_b, index16)
    _check(lib().spmv_convert(h, fmt, ctypes.byref(p)), h)


def spmv_set_format(h, fmt):
    _check(lib().spmv_set_format(h, fmt), h)


def spmv_get_format(h) -> int:
    f = ctypes.c_int()
    _check(lib().spmv_get_format(h, ctypes.byref(f)), h)
    return f.value


def spmv_features(h) -> dict:
    f = Features()
    _check(lib().spmv_features(h, ctypes.byref(f)), h)
    return f.as_dict()


def spmv_run(h, alpha, x, beta, y, fmt=None):
    if fmt is None:
        _check(lib().spmv_run(h, float(alpha), _ptr(x), float(beta), _ptr(y)), h)
    else:
        _check(lib().spmv_run_format(h, fmt, float(alpha), _ptr(x), float(beta), _ptr(y)), h)


def spmv_set_launch(h, fmt, block=0, maxreg=0, carveout_pct=-1, knob=0):
    L = Launch(block, maxreg, carveout_pct, knob)
    _check(lib().spmv_set_launch(h, fmt, ctypes.byref(L)), h)


def spmv_get_launch(h, fmt):
    L = Launch()
    _check(lib().spmv_get_launch(h, fmt, ctypes.byref(L)), h)
    return L.as_tuple()


def spmv_tune(h, flags=TUNE_ALL, expected_iterations=100, objective="latency"):
    """objective: latency | energy | power | efficiency (the paper's four)."""
    r = TuneReport()
    fl = int(flags) | (OBJECTIVES[objective] << 4)
    _check(lib().spmv_tune(h, fl, int(expected_iterations), ctypes.byref(r)), h)
    return r


def spmv_power_step(h, x, y, sums_prev, sums_out, row_offset=0):
    _check(lib().spmv_power_step(h, _ptr(x), _ptr(y), _ptr(sums_prev), _ptr(sums_out), int(row_offset)), h)


def spmv_power_iterate_graph(h, x0, buf0, buf1, steps, sums):
    """The single-GPU power loop replayed as a CUDA graph (see spmv.h).
    Returns the index (0/1) of the buffer holding z_E."""
    fb = ctypes.c_int(0)
    _check(lib().spmv_power_iterate_graph(h, _ptr(x0), _ptr(buf0), _ptr(buf1), int(buf0.numel()), int(steps),
                                          _ptr(sums), ctypes.byref(fb)), h)
    return fb.value


def spmv_power_iterate(h, x0, buf0, buf1, steps, sums, comm=None, chunk=0, chunk_buf=None,
                       time_kernels=False, time_loop=False):
    """Native E-step power iteration (see spmv.h). Returns (final_buf_index,
    per-launch kernel ms list or None, loop ms or None)."""
    km = (ctypes.c_float * max(int(steps), 1))() if time_kernels else None
    lm = ctypes.c_float(0.0)
    fb = ctypes.c_int(0)
    _check(lib().spmv_power_iterate(h, _ptr(x0), _ptr(buf0), _ptr(buf1), int(buf0.numel()), int(steps),
                                    _ptr(sums), comm, int(chunk), _ptr(chunk_buf), km,
                                    ctypes.byref(lm) if time_loop else None, ctypes.byref(fb)), h)
    return fb.value, (list(km)[:int(steps)] if km is not None else None), (lm.value if time_loop else None)


def spmv_predict(features: dict, dtype="f64") -> dict:
    """Learned selector on a features dict (spmv_features output); host only."""
    f = Features()
    for k, v in features.items():
        setattr(f, k, v)
    o = Prediction()
    _check(lib().spmv_predict(ctypes.byref(f), R32F if dtype == "f32" else R64F, ctypes.byref(o)))
    return {"cls": o.cls, "class": SELECTOR_CLASSES[o.cls], "format": o.format,
            "params": {k[0]: getattr(o.params, k[0]) for k in FormatParams._fields_},
            "speed_ratio": o.speed_ratio, "c_latency_s": o.c_latency_s, "f_latency_s": o.f_latency_s}


def spmv_create_row_slice(h, row_begin, row_end):
    out = ctypes.c_void_p()
    _check(lib().spmv_create_row_slice(ctypes.byref(out), h, int(row_begin), int(row_end)), h)
    return out


def spmv_dist_local_group(world: int, devices=None):
    """`world` in-process communicators (rank r on devices[r]); drive each
    rank from its own host thread (ctypes releases the GIL during calls)."""
    devs = list(devices) if devices is not None else [0] * world
    arr = (ctypes.c_int * world)(*devs)
    out = (ctypes.c_void_p * world)()
    _check(lib().spmv_dist_local_group(int(world), arr, out))
    return [ctypes.c_void_p(out[r]) for r in range(world)]


def spmv_dist_plan_create(h, comm, chunk, flags=PLAN_OVERLAP):
    out = ctypes.c_void_p()
    _check(lib().spmv_dist_plan_create(ctypes.byref(out), h, comm, int(chunk), int(flags)), h)
    return out


def spmv_dist_plan_info(plan) -> dict:
    o = PlanInfo()
    _check(lib().spmv_dist_plan_info(plan, ctypes.byref(o)))
    return o.as_dict()


def spmv_dist_plan_part(plan, part):
    out = ctypes.c_void_p()
    _check(lib().spmv_dist_plan_part(plan, int(part), ctypes.byref(out)))
    return out if out.value else None


def spmv_dist_plan_iterate(plan, x0, buf0, buf1, steps, sums, time_loop=False, time_interior=False):
    """Returns (final_buf_index, loop_ms or None, interior kernel ms list or None)."""
    lm = ctypes.c_float(0.0)
    im = (ctypes.c_float * max(int(steps), 1))() if time_interior else None
    fb = ctypes.c_int(0)
    _check(lib().spmv_dist_plan_iterate(plan, _ptr(x0), _ptr(buf0), _ptr(buf1), int(steps), _ptr(sums),
                                        ctypes.byref(lm) if time_loop else None, im, ctypes.byref(fb)))
    return fb.value, (lm.value if time_loop else None), (list(im)[:int(steps)] if im is not None else None)


def spmv_dist_plan_destroy(plan):
    if plan is not None:
        _check(lib().spmv_dist_plan_destroy(plan))


def spmv_dist_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().spmv_dist_unique_id(buf))
    return buf.raw[:128]


def spmv_dist_init(uid: bytes, rank: int, world: int, device: int):
    c = ctypes.c_void_p()
    _check(lib().spmv_dist_init(ctypes.byref(c), uid, rank, world, device))
    return c


def spmv_dist_destroy(comm):
    if comm is not None:
        lib().spmv_dist_destroy(comm)


def spmv_norm2(h, x, sums_out):
    _check(lib().spmv_norm2(h, _ptr(x), int(x.shape[0]), _ptr(sums_out)), h)


def spmv_format_info(h, fmt) -> dict:
    o = FormatInfo()
    _check(lib().spmv_format_info(h, fmt, ctypes.byref(o)), h)
    return {f[0]: getattr(o, f[0]) for f in o._fields_}


def spmv_copy_array(h, which, dst):
    where = MEM_DEVICE if (hasattr(dst, "is_cuda") and dst.is_cuda) else MEM_HOST
    nbytes = dst.numel() * dst.element_size() if hasattr(dst, "element_size") else dst.nbytes
    _check(lib().spmv_copy_array(h, which, _ptr(dst), nbytes, where), h)


def spmv_set_stream(h, stream):
    _check(lib().spmv_set_stream(h, ctypes.c_void_p(stream.cuda_stream)), h)


def spmv_destroy(h):
    if h is not None:
        lib().spmv_destroy(h)


def spmv_decision_log(h) -> list:
    n = lib().spmv_decision_log(h, None, 0)
    buf = ctypes.create_string_buffer(n)
    lib().spmv_decision_log(h, buf, n)
    return json.loads(buf.value.decode() or "[]")


def spmv_overheads(h):
    f = ctypes.c_double()
    c = (ctypes.c_double * 6)()
    _check(lib().spmv_overheads(h, ctypes.byref(f), c), h)
    return f.value, {FORMAT_NAMES[i]: c[i] for i in range(6)}


def spmv_dist_partition(row_ptr, world):
    import numpy as np
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    b = np.empty(world + 1, np.int64)
    _check(lib().spmv_dist_partition(rp.shape[0] - 1, rp.ctypes.data, world, b.ctypes.data))
    return b


def spmv_dist_partition_lengths(lengths, world):
    import numpy as np
    L = np.ascontiguousarray(lengths, dtype=np.int64)
    b = np.empty(world + 1, np.int64)
    _check(lib().spmv_dist_partition_lengths(L.shape[0], L.ctypes.data, world, b.ctypes.data))
    return b


def spmv_dist_remap_columns(col, bounds, stream=None):
    """In-place remap of global columns into the padded all-gather layout."""
    import numpy as np
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    world = b.shape[0] - 1
    if hasattr(col, "is_cuda") and col.is_cuda:
        _check(lib().spmv_dist_remap_columns(col.data_ptr(), col.numel(), b.ctypes.data, world, MEM_DEVICE,
                                             _stream_ptr(stream)))
    else:
        arr = col if isinstance(col, np.ndarray) else col.numpy()
        _check(lib().spmv_dist_remap_columns(arr.ctypes.data, arr.shape[0], b.ctypes.data, world, MEM_HOST,
                                             None))


# ---------------------------------------------------------------- convenience object

@dataclass
class Matrix:
    """Owning wrapper of a handle (torch tensors in, torch tensors out)."""
    handle: object
    rows: int
    cols: int
    nnz: int
    dtype: object

    @classmethod
    def from_coo(cls, rows, cols, row_idx, col_idx, vals, device=0, stream=None):
        h = spmv_create(rows, cols, row_idx, col_idx, vals, device=device, stream=stream)
        return cls(h, int(rows), int(cols), int(row_idx.shape[0]), vals.dtype)

    def convert(self, fmt, **params):
        if isinstance(fmt, str):
            fmt = FORMATS[fmt]
        spmv_convert(self.handle, fmt, **params)
        return self

    def features(self):
        return spmv_features(self.handle)

    def run(self, x, y, alpha=1.0, beta=0.0, fmt=None):
        spmv_run(self.handle, alpha, x, beta, y, fmt=fmt)
        return y

    def tune(self, flags=TUNE_ALL, expected_iterations=100):
        return spmv_tune(self.handle, flags, expected_iterations)

    @property
    def format(self) -> str:
        return FORMAT_NAMES[spmv_get_format(self.handle)]

    def close(self):
        if self.handle is not None:
            spmv_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
