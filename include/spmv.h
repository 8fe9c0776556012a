/* include/spmv.h — C ABI of the B200-native SpMV library (libspmv.so).
 *
 * The operation is the paper's problem statement: "finds the dense vector
 * product Y of a sparse matrix A and a dense vector X such that Y = A × X"
 * (PAPER.md P:145), extended to the BLAS form y <- alpha·A·x + beta·y
 * (reading R1). Input arrives as COO, "the default sparse format
 * ... in SuiteSparse". The library converts it on the device to the
 * paper's formats — CSR, ELL, SELL (generalised to
 * SELL-C-sigma), plus COO and HYB from the north star — extracts the Table 2
 * sparsity features on the device, runs a hand-written sm_100a
 * kernel per format, and implements the paper's two optimisation modes
 * as a launch-configuration tuner and a feature-driven format
 * selector with an overhead gate.
 *
 * Conventions (all entry points):
 *  - Every call returns spmv_status_t. Nothing throws, nothing aborts, no
 *    call ever falls back to the CPU: compute runs only in this library's
 *    CUDA kernels.
 *  - Indices are 0-based int32 (rows, cols <= 2^31-1); nnz is int64.
 *  - Device pointers are plain CUDA device addresses on the handle's device;
 *    host pointers are ordinary (pageable or pinned) host memory.
 *  - On any error, `*out` handles stay NULL and nothing leaks; the handle's
 *    spmv_last_error() holds the detail (incl. CUDA error text).
 *  - Calls on one handle must be externally serialised; distinct handles are
 *    independent and may be driven from different host threads on different
 *    streams at the same time (tests/test_gpu_concurrent.py). Host uploads in
 *    spmv_create go in 64 MB pieces, and small results are read back through
 *    a per-thread pinned buffer, so one handle's work does not wait for
 *    another handle's copies.
 */
#ifndef SPMV_H
#define SPMV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct spmv_matrix* spmv_handle_t;

typedef enum {
  SPMV_OK = 0,
  SPMV_ERR_INVALID_ARG = 1,        /* null pointer, negative size, bad enum, x == y */
  SPMV_ERR_INDEX_OUT_OF_RANGE = 2, /* a triplet outside [0,rows) x [0,cols) */
  SPMV_ERR_DUPLICATE = 3,          /* a repeated (row, col) — SPEC.md S:70 */
  SPMV_ERR_INFEASIBLE = 4,         /* ELL/SELL slot guard exceeded; handle unchanged */
  SPMV_ERR_OUT_OF_MEMORY = 5,
  SPMV_ERR_UNSUPPORTED = 6,        /* rows/cols > 2^31-1, SELL C not in {32,64,128,256}, ... */
  SPMV_ERR_CUDA = 7,               /* CUDA runtime error (sticky device faults surface here) */
  SPMV_ERR_NOT_CONVERTED = 8,      /* requested format has not been built on this handle */
  SPMV_ERR_NCCL = 9,               /* NCCL missing or a collective failed */
  SPMV_ERR_NVML = 10               /* NVML missing (energy/power objectives) */
} spmv_status_t;

typedef enum { SPMV_R32F = 0, SPMV_R64F = 1 } spmv_dtype_t;
typedef enum { SPMV_MEM_HOST = 0, SPMV_MEM_DEVICE = 1 } spmv_mem_t;

/* Storage formats: COO, CSR, ELL, HYB (ELL + COO
 * tail; not in the paper, north star), SELL-C-sigma (P:165 generalised),
 * BELL (ELL over dense b×b blocks, Fig. 2(d) b = 2). */
typedef enum {
  SPMV_FMT_COO = 0,
  SPMV_FMT_CSR = 1,
  SPMV_FMT_ELL = 2,
  SPMV_FMT_HYB = 3,
  SPMV_FMT_SELL = 4,
  SPMV_FMT_BELL = 5
} spmv_format_t;
#define SPMV_NUM_FORMATS 6

/* CSR kernel algorithms: scalar (thread per row), vector (T lanes per row,
 * the "coordination among threads within a warp" of P:159), merge-path, and
 * stream (tiles of consecutive rows: a producer warp bulk-copies each tile's
 * contiguous col/val segment into a two-stage shared-memory ring with TMA
 * (cp.async.bulk + mbarrier), then a thread per row gathers x — consecutive
 * rows gather together, as in ELL, without ELL's padding and without a
 * conversion; tiles whose segment does not fit a stage fall back to
 * warp-per-row; meant for regular rows — the selector measures it only when
 * rows are not skewed; launch knob = entries per row slot, 16/32/64; block
 * 1024 is refused since the producer warp makes it 1056 threads). */
typedef enum {
  SPMV_CSR_AUTO = 0,
  SPMV_CSR_SCALAR = 1,
  SPMV_CSR_VECTOR = 2,
  SPMV_CSR_MERGE = 3,
  SPMV_CSR_STREAM = 4
} spmv_csr_alg_t;

/* Format parameters (NULL = defaults). */
typedef struct {
  int32_t csr_alg;    /* spmv_csr_alg_t; AUTO = vector, T from the mean row length */
  int32_t csr_T;      /* CSR-vector lanes per row in {2,4,8,16,32}; 0 = clamp(next_pow2(ceil(mean)),2,32) */
  int32_t sell_C;     /* SELL slice height in {32,64,128,256}; 0 = 32·(16 B / sizeof(value)) */
  int32_t sell_sigma; /* sorting window: 1 (no sort) or a multiple of sell_C; 0 = 1 */
  int64_t hyb_K;      /* HYB ELL width; -1 = automatic (CUSP/Bell–Garland rule, R12) */
  int32_t bell_b;     /* BELL square block dimension in {2,3,4}; 0 = 2 (the paper's 2×2) */
  int32_t index16;    /* ELL/SELL column storage: 0 = int32 columns (default); 1 = 16-bit offsets
                         d = col − row (10 instead of 12 B per fp64 slot; SPMV_ERR_UNSUPPORTED unless
                         every |col − row| <= 32767); 2 = 8-bit codes of d into a per-matrix
                         dictionary of its distinct offsets (9 B per fp64 slot + a 1 KB table;
                         SPMV_ERR_UNSUPPORTED unless the matrix has at most 255 distinct col − row,
                         as banded / stencil matrices do: 27 for the 27-point stencil); -1 = the
                         narrowest that fits: 8-bit, then 16-bit, else int32 */
} spmv_format_params_t;

/* Table 2 features + the north star's max and bandwidth.
 * Definitions (R5/R6): L_i = row length; population variance;
 * even-n median = mean of the two middle order statistics; mode = smallest
 * most frequent L; ell_ratio = nnz / (n_rows · max_len), 1 if max_len = 0;
 * bw_lower = max(0, max_ij (i − j)), bw_upper = max(0, max_ij (j − i)). */
typedef struct {
  int64_t n_rows, n_cols, nnz, max_len, min_len, n_empty, mode, bw_lower, bw_upper, bandwidth;
  double mean, var, std, ell_ratio, median;
} spmv_features_t;

/* One launch variant: the compile-time-mode knobs of P:376-400 recast for
 * B200 — thread-block size, register cap (__maxnreg__) and the L1/shared
 * carveout (percent shared) — plus a per-kernel knob (CSR-vector T,
 * merge-path items per thread, ELL/SELL rows per warp). 0 = default. */
typedef struct {
  int32_t block;        /* 64, 128, 256, 512, 1024 */
  int32_t maxreg;       /* 32, 64, 128, 255 */
  int32_t carveout_pct; /* -1 = driver default, else 0..100 */
  int32_t knob;         /* CSR-vector: lanes per row; merge-path: items per thread (4/8/16: per-warp
                           merge walk; 0x100 | IPT (IPT 4/8/16/32): row-interleaved tiles of block·IPT items;
                           0x200 | IPT: the same tiles fed by a TMA producer warp, block + 32 threads); COO/HYB: entries
                           per lane (2/4/8: warp chunks of 32·knob entries) or 0x100 | EPT (EPT =
                           4/8/16/32: row-interleaved tiles of block·EPT entries staged in shared memory,
                           thread per row); ELL: rows per warp (32/64/128/256) in the low 16 bits; ELL
                           and SELL: bit 16 (65536) selects the carried-batch loop (see kern_sliced.cuh) */
} spmv_launch_t;

/* spmv_tune flags */
#define SPMV_TUNE_LAUNCH 1u /* compile-time-mode analog: sweep launch variants of the active format */
#define SPMV_TUNE_FORMAT 2u /* run-time-mode analog: select a format from features, measure, gate */
#define SPMV_TUNE_ALL 3u
/* Optimisation objective (the paper's four), OR-ed into the
 * flags. Non-latency objectives measure each candidate's energy with NVML
 * over >= 0.4 s of back-to-back SpMVs (SPMV_ERR_NVML if NVML is missing):
 *  LATENCY    min seconds per SpMV (default)
 *  ENERGY     min joules per SpMV
 *  POWER      min average watts while running
 *  EFFICIENCY max MFLOPS/W (= MFLOP per joule) */
#define SPMV_TUNE_OBJ_LATENCY (0u << 4)
#define SPMV_TUNE_OBJ_ENERGY (1u << 4)
#define SPMV_TUNE_OBJ_POWER (2u << 4)
#define SPMV_TUNE_OBJ_EFFICIENCY (3u << 4)
#define SPMV_TUNE_OBJ_MASK (3u << 4)
/* With SPMV_TUNE_FORMAT: the paper's run-time mode with LEARNED models
 * instead of measuring every
 * candidate: features -> decision-tree class (best format) -> predicted speed
 * ratio vs CSR-vector and predicted conversion latency -> convert iff
 * expected_iterations·(t_csr − ratio·t_csr) > f_latency + c_latency_pred.
 * Only t_csr is measured: the default CSR-vector kernel timed on a row
 * prefix of about 2^25 entries (the whole matrix when nnz <= 2^26), scaled to
 * nnz. Latency objective only (SPMV_ERR_UNSUPPORTED with another objective):
 * the models are trained on latency. */
#define SPMV_TUNE_PREDICT 4u
/* With SPMV_TUNE_FORMAT | SPMV_TUNE_PREDICT only: decide, do not convert.
 * The report carries the verdict (format, params, converted = 1 iff the gate
 * accepts the conversion; format = SPMV_FMT_CSR otherwise) and the handle's
 * active format is left unchanged, so the caller converts with spmv_convert
 * (the bench times selection and conversion as separate phases).
 * SPMV_ERR_INVALID_ARG without PREDICT or together with SPMV_TUNE_LAUNCH. */
#define SPMV_TUNE_DECIDE_ONLY 8u

typedef struct {
  int32_t format;                /* chosen spmv_format_t (active after the call) */
  spmv_format_params_t params;   /* its parameters */
  spmv_launch_t launch;          /* its chosen launch variant */
  double t_csr_s;                /* measured default (CSR) SpMV time */
  double t_best_s;               /* measured time of the chosen format/variant */
  double f_latency_s;            /* feature-extraction time (on device) */
  double c_latency_s;            /* conversion time of the chosen format (on device) */
  int64_t expected_iterations;   /* gate input */
  int32_t converted;             /* 1 iff the gate accepted the conversion */
  int32_t n_candidates;          /* formats measured */
  int32_t n_variants;            /* launch variants measured */
  int32_t objective;             /* 0 latency, 1 energy, 2 power, 3 efficiency */
  int32_t reserved;
  double energy_j;               /* chosen: joules per SpMV (NaN if not measured) */
  double power_w;                /* chosen: average watts while running (NaN if not measured) */
  double mflops_per_w;           /* chosen: MFLOPS/W (NaN if not measured) */
} spmv_tune_report_t;

/* Format introspection (sizes of what spmv_copy_array can export). */
typedef struct {
  int32_t present;       /* 1 if the format is built on this handle */
  int32_t row_ptr_is64;  /* CSR row_ptr element width: 0 = int32, 1 = int64 */
  int64_t K;             /* ELL width / HYB ELL width */
  int64_t n_pad;         /* ELL / HYB row padding (multiple of 128) */
  int64_t C, sigma;      /* SELL */
  int64_t n_slices;      /* SELL */
  int64_t slots;         /* ELL/SELL/HYB-ELL stored slots (incl. padding) */
  int64_t tail_nnz;      /* HYB COO tail */
  int64_t n_empty_rows;  /* COO: rows without entries */
  int64_t stored_bytes;  /* bytes of the format's arrays (padding included) */
  int64_t block;         /* BELL block dimension b (K = blocks per block row, n_pad = padded block rows) */
  int64_t index_bytes;   /* bytes per stored column index (1 / 2 with ELL/SELL index16 = 2 / 1, else 4; 0 = CSR/COO arrays) */
} spmv_format_info_t;

typedef enum {
  SPMV_ARR_CSR_ROW_PTR = 0,  /* int32 or int64 [rows+1] */
  SPMV_ARR_CSR_COL = 1,      /* int32 [nnz] (also the COO column array) */
  SPMV_ARR_CSR_VAL = 2,      /* value [nnz] (also the COO value array) */
  SPMV_ARR_COO_ROW = 3,      /* int32 [nnz] */
  SPMV_ARR_ELL_COL = 4,      /* int32 [K·n_pad], column-major: (i,k) at k·n_pad + i, pad −1 */
  SPMV_ARR_ELL_VAL = 5,      /* value [K·n_pad], pad +0.0 */
  SPMV_ARR_SELL_PERM = 6,    /* int32 [rows] (identity when sigma = 1) */
  SPMV_ARR_SELL_SLICE_PTR = 7, /* int64 [n_slices+1] */
  SPMV_ARR_SELL_COL = 8,     /* int32 [slots]: (s,j,k) at slice_ptr[s] + k·C + j */
  SPMV_ARR_SELL_VAL = 9,
  SPMV_ARR_HYB_ELL_COL = 10,
  SPMV_ARR_HYB_ELL_VAL = 11,
  SPMV_ARR_HYB_TAIL_ROW = 12, /* int32 [tail_nnz], (row, col) order */
  SPMV_ARR_HYB_TAIL_COL = 13,
  SPMV_ARR_HYB_TAIL_VAL = 14,
  SPMV_ARR_COO_EMPTY_ROWS = 15, /* int32 [n_empty_rows], ascending */
  SPMV_ARR_BELL_COL = 16,     /* int32 [K·n_pad]: block column of slot (I, k) at k·n_pad + I, pad −1 */
  SPMV_ARR_BELL_VAL = 17,     /* value [K·b·b·n_pad]: entry (r, c) of slot (I, k) at (k·b·b + r·b + c)·n_pad + I */
  SPMV_ARR_ELL_COL16 = 18,    /* int16 [K·n_pad] when index16: d = col − row, pad −32768 (ELL_COL is then absent) */
  SPMV_ARR_SELL_COL16 = 19,   /* int16 [slots] when index16: d = col − row of the slot's (permuted) row, pad −32768 */
  SPMV_ARR_ELL_COL8 = 20,     /* uint8 [K·n_pad] when index16 = 2: code of d = col − row, pad 255 */
  SPMV_ARR_SELL_COL8 = 21,    /* uint8 [slots] when index16 = 2: code of d for the slot's (permuted) row, pad 255 */
  SPMV_ARR_DICT8_TAB = 22     /* int32 [256]: the offset d of each 8-bit code (after an index16 = 2 build) */
} spmv_array_t;

/* ---------------------------------------------------------------- core API */

/* Ingest + validate + canonicalise COO and build CSR on the device
 * (SURVEY.md §8(a) rows a1–a2). Copies the triplets (host or device memory,
 * per `where`) so the caller may free them on return; synchronous.
 * Unsorted input is radix-sorted by (row, col) on the device; explicit
 * zeros are kept. Errors: INVALID_ARG (nulls with nnz > 0, negative sizes,
 * bad dtype/where), UNSUPPORTED (rows/cols > 2^31-1), INDEX_OUT_OF_RANGE,
 * DUPLICATE, OUT_OF_MEMORY, CUDA. `cuda_stream` (cudaStream_t, may be NULL
 * = legacy default stream) becomes the handle's stream. Active format: CSR
 * (the paper's default). */
spmv_status_t spmv_create(spmv_handle_t* out, int64_t rows, int64_t cols, int64_t nnz,
                          const int32_t* row_idx, const int32_t* col_idx, const void* vals,
                          spmv_dtype_t dtype, spmv_mem_t where, int device, void* cuda_stream);

/* Build (or re-activate, if cached) `fmt` on the device and make it the
 * active format (§8(a) row a4). p = NULL uses defaults. Stream-ordered: the
 * build is enqueued on the handle's stream (later calls on the handle see
 * it); it synchronises only when a host decision needs a device-computed size
 * (HYB tail, COO empty rows, strongly skewed SELL). Its device time is
 * reported by spmv_overheads.
 * INFEASIBLE if ELL/SELL/HYB padding would not fit the device-memory guard
 * (the handle is unchanged); UNSUPPORTED for SELL C outside {32,64,128,256}. */
spmv_status_t spmv_convert(spmv_handle_t h, spmv_format_t fmt, const spmv_format_params_t* p);

/* Make an already-built format active without rebuilding. NOT_CONVERTED if absent. */
spmv_status_t spmv_set_format(spmv_handle_t h, spmv_format_t fmt);

/* Device feature extraction (§8(a) row a3): integer moments, histogram
 * order statistics and bandwidth on the device; exact-integer -> fp64
 * formulas on the host. Synchronous; result cached on the handle. */
spmv_status_t spmv_features(spmv_handle_t h, spmv_features_t* out);

/* y <- alpha·A·x + beta·y with the active format's kernel (§8(a) row a5).
 * x: device, n_cols values; y: device, n_rows values; dtype = handle dtype;
 * x and y must not alias (exact equality -> INVALID_ARG). beta == 0: y is
 * not read (NaN in y cannot propagate); alpha == 0: A is not read.
 * Asynchronous on the handle's stream; fp32 data accumulates in fp64. */
spmv_status_t spmv_run(spmv_handle_t h, double alpha, const void* x, double beta, void* y);

/* Same with an explicit format (must be built) — used by tests and bench. */
spmv_status_t spmv_run_format(spmv_handle_t h, spmv_format_t fmt, double alpha, const void* x,
                              double beta, void* y);

/* Override the launch variant used for `fmt` (block/maxreg/carveout/knob). */
spmv_status_t spmv_set_launch(spmv_handle_t h, spmv_format_t fmt, const spmv_launch_t* v);
spmv_status_t spmv_get_launch(spmv_handle_t h, spmv_format_t fmt, spmv_launch_t* v);

/* The paper's two optimisation modes on B200 (§8(a) a6–a7).
 * LAUNCH: time every launch variant of the active format, keep the fastest.
 * FORMAT: features -> candidate formats -> convert + measure each -> gate:
 *   switch away from CSR iff expected_iterations·(t_csr − t_best) >
 *   f_latency + c_latency(best) (strict >). With an energy /
 *   efficiency objective the gate compares energy (conversion energy =
 *   CSR's average power × (f + c)); with the power objective the format with
 *   the lower average power wins. Uses scratch x/y (never the caller's).
 *   Synchronous. Decisions appended to the JSON log. */
spmv_status_t spmv_tune(spmv_handle_t h, uint32_t flags, int64_t expected_iterations,
                        spmv_tune_report_t* out);

/* The learned selector alone (host-only, no device work): class index into
 * {CSR-vector, CSR-merge, ELL, SELL, HYB, COO, BELL-2, BELL-3}, the format and
 * parameters it maps to, the predicted t_format / t_CSR-vector, and the
 * predicted conversion and feature-extraction latencies in seconds. The
 * model (tools/train_selector.py, profiles/selector_model.json) is compiled
 * into the library. */
typedef struct {
  int32_t cls;
  int32_t format;
  spmv_format_params_t params;
  double speed_ratio;
  double c_latency_s;
  double f_latency_s;
} spmv_prediction_t;
spmv_status_t spmv_predict(const spmv_features_t* features, spmv_dtype_t dtype, spmv_prediction_t* out);

/* ---------------------------------------------------------------- power iteration
 * Power iteration (not in the paper):
 *   z_k = alpha_k · A · z_{k−1},  alpha_k = 1/‖z_{k−1}‖,  x_k = z_{k−1}/‖z_{k−1}‖,
 *   lambda_k = x_k · z_k.
 * spmv_power_step launches ONE SpMV of the active format whose epilogue
 * reads alpha from sums_prev (device, 2 doubles: [Σz², Σ x·z] of the
 * previous step; alpha = 1/sqrt(sums_prev[0])) and writes this step's
 * rank-local [Σz_i², Σ z_{k−1,row_offset+i}·z_i] to sums_out (device) —
 * deterministic order. For a row slab of a larger matrix, `row_offset` is
 * the slab's first global row (x is the full replicated vector). */
spmv_status_t spmv_power_step(spmv_handle_t h, const void* x, void* y, const double* sums_prev,
                              double* sums_out, int64_t row_offset);
/* sums_out[0] = Σ x_i², sums_out[1] = 0 over n values of x (device). */
spmv_status_t spmv_norm2(spmv_handle_t h, const void* x, int64_t n, double* sums_out);

/* The whole E-step power iteration on the handle's stream (no host round
 * trips): buf0 <- x0 (n_full values, may alias buf0), S_0 = Σ over ranks of
 * ||own rows of buf0||², then per step k: one spmv_power_step into the next
 * buffer — at this rank's chunk (rank·chunk) when comm != NULL, followed by
 * the all-reduce of sums[k+1] and an in-place all-gather of the chunks
 * (chunk values per rank). chunk_buf is unused (may be NULL).
 * sums: device double[(steps+1)·2] (row k = [S_k, D_k]); lambda_k =
 * D_k / sqrt(S_{k-1}). buf0/buf1: device, n_full values (n_full = rows for a
 * single rank, world·chunk in the padded multi-GPU layout). kernel_ms: host
 * float[steps] (optional) receives each SpMV launch's CUDA-event time (events
 * between launches: slightly perturbing). loop_ms: host float (optional)
 * receives the CUDA-event time of the whole E-step loop (unperturbed). Either
 * timing output makes the call synchronise. *final_buf (optional) = 0/1:
 * which buffer holds z_E. */
spmv_status_t spmv_power_iterate(spmv_handle_t h, const void* x0, void* buf0, void* buf1, int64_t n_full,
                                 int64_t steps, double* sums, void* comm, int64_t chunk, void* chunk_buf,
                                 float* kernel_ms, float* loop_ms, int* final_buf);

/* ---------------------------------------------------------------- distributed plan
 * Interior/halo overlap and halo exchange (SURVEY.md §8(e) (i)–(iv), §8(f) f4).
 * spmv_dist_plan_create splits the rank's slab h (rows = local rows, columns
 * in the padded layout: rank r owns positions [r·chunk, r·chunk + rows_r))
 * into three row blocks, each a new handle converted to h's active format,
 * parameters and launch variant:
 *   part 0 interior [h0, h1): every column inside the own chunk;
 *   part 1 lo halo  [0, h0):  h0 = 1 + the last row with a column below it;
 *   part 2 hi halo  [h1, n):  h1 = the first row with a column above it.
 * Exact for any matrix (a general graph may have an empty interior). h may
 * be destroyed after the call (the plan owns copies). comm = NULL: one rank,
 * a single interior part, no exchange (chunk ignored).
 * flags: SPMV_PLAN_OVERLAP — the interior SpMV of step k waits only for the
 *   all-reduce of step k−1 and overlaps the exchange of z_{k−1} on a second
 *   stream; the halo SpMVs wait for the exchange. Without it every kernel of
 *   the step waits for the exchange.
 * SPMV_PLAN_HALO — exchange only the remote entries the halo rows reference
 *   (NCCL send/recv, lists built here with the communicator) instead of the
 *   all-gather of whole chunks; kept only if every rank then receives less
 *   than half of what the all-gather moves (collective decision).
 * Collective: every rank of comm must call it. Synchronous. */
/* The single-GPU power iteration of spmv_power_iterate (comm = NULL) as a
 * CUDA graph: the first call with a given (x0, buf0, buf1, n_full, steps,
 * sums) runs the loop eagerly — its result is that call's result, and lazily
 * built scratch, partitions and kernel attributes are set up outside any
 * capture — then captures the same launches (on a private stream) and
 * instantiates them; later calls with the same arguments replay the graph on
 * the handle's stream with one cudaGraphLaunch (the E·(1..3) kernel launches
 * of a loop cost one host call: what matters for small, launch-bound
 * matrices). Any spmv_convert / set_format / set_launch / tune /
 * set_stream / release_csr invalidates the graph (re-captured on the next
 * call). The graph lives with the handle (freed by spmv_destroy). No timing
 * outputs; *final_buf as in spmv_power_iterate. Errors as spmv_power_iterate;
 * SPMV_ERR_CUDA if capture or instantiation fails. */
spmv_status_t spmv_power_iterate_graph(spmv_handle_t h, const void* x0, void* buf0, void* buf1, int64_t n_full,
                                       int64_t steps, double* sums, int* final_buf);

#define SPMV_PLAN_OVERLAP 1u
#define SPMV_PLAN_HALO 2u
typedef struct spmv_dist_plan* spmv_dist_plan_t;
typedef struct {
  int32_t rank, world, overlap, halo;   /* halo: 1 = list exchange in use, 0 = all-gather */
  int64_t rows, chunk, h0, h1;
  int64_t part_rows[3], part_nnz[3];
  int64_t recv_elems, send_elems;       /* per step, per rank */
  int64_t recv_bytes_per_step;
  int32_t direct_recv, direct_send;     /* halo segments move without pack/unpack kernels */
} spmv_dist_plan_info_t;
spmv_status_t spmv_dist_plan_create(spmv_dist_plan_t* out, spmv_handle_t h, void* comm, int64_t chunk,
                                    uint32_t flags);
spmv_status_t spmv_dist_plan_info(spmv_dist_plan_t plan, spmv_dist_plan_info_t* out);
/* Borrowed handle of part p (0..2) or NULL when that block is empty; it may
 * be re-converted or re-tuned (the plan uses its active format). */
spmv_status_t spmv_dist_plan_part(spmv_dist_plan_t plan, int part, spmv_handle_t* out);
/* E power steps with the plan's schedule (same mathematics and sums layout
 * as spmv_power_iterate; buf0/buf1 hold world·chunk values; in halo mode only
 * the own chunk and the received halo entries of the final buffer are
 * current). loop_ms (optional): CUDA-event time of the loop on the compute
 * stream; interior_ms (optional, host float[steps]): each step's interior
 * kernel time. Collective. */
spmv_status_t spmv_dist_plan_iterate(spmv_dist_plan_t plan, const void* x0, void* buf0, void* buf1,
                                     int64_t steps, double* sums, float* loop_ms, float* interior_ms,
                                     int* final_buf);
spmv_status_t spmv_dist_plan_destroy(spmv_dist_plan_t plan); /* NULL is a no-op */

/* W communicators of ONE process (rank r on devices[r]; devices may repeat):
 * collectives are stream-ordered device copies plus a host barrier, so W host
 * threads — one per rank, each calling the collective entry points with its
 * own communicator — run exactly the multi-rank schedule of the NCCL path.
 * comms: host void*[world], each released with spmv_dist_destroy. A rank that
 * fails releases the others from the barrier (they return SPMV_ERR_NCCL). */
spmv_status_t spmv_dist_local_group(int world, const int* devices, void** comms);

/* Rows [row_begin, row_end) of h's CSR as a new handle (same columns, dtype,
 * device and stream; active format CSR). Copies the slice. */
spmv_status_t spmv_create_row_slice(spmv_handle_t* out, spmv_handle_t h, int64_t row_begin, int64_t row_end);

/* ---------------------------------------------------------------- introspection */
spmv_status_t spmv_format_info(spmv_handle_t h, spmv_format_t fmt, spmv_format_info_t* out);
/* Copy a format array into dst (`where` = host or device), dst_bytes >= array bytes. */
spmv_status_t spmv_copy_array(spmv_handle_t h, spmv_array_t which, void* dst, int64_t dst_bytes,
                              spmv_mem_t where);
spmv_status_t spmv_get_format(spmv_handle_t h, spmv_format_t* fmt);
spmv_status_t spmv_set_stream(spmv_handle_t h, void* cuda_stream);
spmv_status_t spmv_destroy(spmv_handle_t h); /* NULL is a no-op */
const char* spmv_status_string(spmv_status_t s);
const char* spmv_last_error(spmv_handle_t h);
/* JSON decision log of spmv_tune (array of records); returns the needed
 * length incl. the terminating NUL; copies min(len, needed) bytes. */
size_t spmv_decision_log(spmv_handle_t h, char* buf, size_t len);
/* Conversion timings measured on the device by the last spmv_create /
 * spmv_convert / spmv_features calls, seconds (c_latency per format, f_latency). */
spmv_status_t spmv_overheads(spmv_handle_t h, double* f_latency_s, double* c_latency_s /*[SPMV_NUM_FORMATS]*/);

/* Free the handle's CSR arrays (row_ptr, col, val) and the COO arrays that
 * share them, keeping the active format (ELL, SELL, HYB or BELL: formats
 * with their own arrays) and the computed features: after conversion the
 * SpMV and the power iteration read only the active format (P:145 — the
 * format is the kernel's input), so a pipeline that converts once and then
 * iterates can hold one copy of the matrix instead of two. Afterwards every
 * call that reads CSR (spmv_convert, spmv_tune, spmv_features if not yet
 * computed, spmv_create_row_slice, spmv_dist_plan_create, runs/copies of CSR
 * or COO) returns SPMV_ERR_NOT_CONVERTED. Stream-ordered frees, no host
 * synchronisation. Errors: SPMV_ERR_INVALID_ARG if h is NULL or the active
 * format is CSR or COO; releasing twice is a no-op. */
spmv_status_t spmv_release_csr(spmv_handle_t h);

/* Number of CUDA kernels this library has launched in this process. */
uint64_t spmv_launch_count(void);
/* Release memory cached by the library's stream-ordered pool. */
spmv_status_t spmv_trim_pool(int device);

/* ---------------------------------------------------------------- multi-GPU (NCCL)
 * One process per GPU. Rank 0 creates the 128-byte NCCL unique id; the caller
 * broadcasts it (e.g. torch.distributed); every rank then calls
 * spmv_dist_init. libnccl.so.2 is loaded on first use (dlopen). */
spmv_status_t spmv_dist_unique_id(uint8_t out[128]);
spmv_status_t spmv_dist_init(void** comm, const uint8_t unique_id[128], int rank, int world, int device);
spmv_status_t spmv_dist_destroy(void* comm); /* NULL is a no-op */

/* ---------------------------------------------------------------- multi-GPU host logic
 * nnz-balanced row partition: bounds[0] = 0,
 * bounds[world] = rows, bounds[k] = first row i with row_ptr[i] >=
 * ceil(k·nnz/world). row_ptr is HOST int64 [rows+1]. Pure host integer code. */
spmv_status_t spmv_dist_partition(int64_t rows, const int64_t* row_ptr, int world,
                                  int64_t* bounds);
/* Same partition computed from per-row lengths given as a host int64 array. */
spmv_status_t spmv_dist_partition_lengths(int64_t rows, const int64_t* lengths, int world,
                                          int64_t* bounds);
/* Remap global column indices of a row slab (host or device int32 array,
 * in place) into the padded all-gather layout: column c owned by rank
 * r (bounds[r] <= c < bounds[r+1]) maps to r·chunk + (c − bounds[r]),
 * chunk = max_r (bounds[r+1] − bounds[r]). */
spmv_status_t spmv_dist_remap_columns(int32_t* col, int64_t nnz, const int64_t* bounds, int world,
                                      spmv_mem_t where, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif
