// handle.cuh — the spmv_matrix handle and the internal entry points shared
// by the translation units of libspmv.so.
#pragma once
#include <functional>
#include <mutex>
#include <string>

#include "common.cuh"

struct spmv_matrix {
  int device = 0;
  cudaStream_t stream = nullptr;
  spmv_dtype_t dtype = SPMV_R64F;
  int vbytes = 8;
  int64_t rows = 0, cols = 0, nnz = 0;

  // CSR (canonical COO columns/values in (row, col) order + row pointers).
  bool rp64 = false;        // row_ptr element type: int64 iff nnz >= 2^31
  void* row_ptr = nullptr;  // [rows+1]
  int32_t* col = nullptr;   // [nnz]
  void* val = nullptr;      // [nnz]

  // COO (rows expanded; columns/values shared with CSR).
  bool coo_built = false;
  int32_t* coo_row = nullptr;
  int32_t* coo_empty = nullptr;  // rows without entries, ascending
  int64_t coo_n_empty = 0;

  // ELL: column-major [K][n_pad].
  bool ell_built = false;
  int64_t ell_K = 0, ell_npad = 0;
  int32_t* ell_col = nullptr;
  void* ell_val = nullptr;
  int16_t* ell_col16 = nullptr;  // 16-bit column offsets (ell_col == nullptr then)
  uint8_t* ell_col8 = nullptr;   // 8-bit dictionary codes (ell_col == nullptr then)

  // SELL-C-sigma.
  bool sell_built = false;
  int64_t sell_C = 0, sell_sigma = 1, sell_ns = 0, sell_slots = 0;
  int32_t* sell_perm = nullptr;  // nullptr when sigma == 1
  int64_t* sell_sp = nullptr;    // [ns+1]
  int32_t* sell_col = nullptr;
  void* sell_val = nullptr;
  int16_t* sell_col16 = nullptr;  // 16-bit column offsets (sell_col == nullptr then)
  uint8_t* sell_col8 = nullptr;   // 8-bit dictionary codes (sell_col == nullptr then)
  // 8-bit dictionary of the distinct offsets d = col − col_origin − row of
  // the matrix (banded / stencil matrices have a few dozen: c5 has 27):
  // column = col_origin + row + dict8_tab[code], pad code 255. Built once per
  // handle (dict8_count = -1 until computed; > 255 = not encodable).
  int dict8_count = -1;
  int64_t dict8_m = 0;           // map covers d in [-m, m]
  uint8_t* dict8_map = nullptr;  // [2m+1]: code of d + m
  int32_t* dict8_tab = nullptr;  // [256]: d of each code
  // 16-bit ELL/SELL column offsets: column = col_origin + row + d, d in
  // [-32767, 32767], pad -32768 (row slices of the distributed plan set the
  // origin to their first global column position).
  int64_t col_origin = 0;

  // HYB: ELL part [K][n_pad] + COO tail.
  bool hyb_built = false;
  int64_t hyb_K = 0, hyb_npad = 0, hyb_tail = 0;
  int32_t* hyb_ecol = nullptr;
  void* hyb_eval = nullptr;
  int32_t* hyb_trow = nullptr;
  int32_t* hyb_tcol = nullptr;
  void* hyb_tval = nullptr;

  // BELL: ELL over dense b×b blocks (value planes, column-major over block rows).
  bool bell_built = false;
  int64_t bell_b = 2, bell_kb = 0, bell_nbr = 0, bell_nbr_pad = 0;
  int32_t* bell_col = nullptr;
  void* bell_val = nullptr;

  // CSR kernel choice.
  int csr_alg = SPMV_CSR_AUTO;
  int csr_T = 0;

  spmv_launch_t launch[SPMV_NUM_FORMATS];
  int active = SPMV_FMT_CSR;

  bool have_features = false;
  spmv_features_t feat{};
  int64_t hyb_auto_K = -1;  // from the feature histogram

  double f_latency = 0.0;
  double c_latency[SPMV_NUM_FORMATS] = {0, 0, 0, 0, 0, 0};
  // conversion timings are recorded as CUDA events and resolved lazily (no sync in convert)
  cudaEvent_t lat_ev[SPMV_NUM_FORMATS][2] = {};
  bool lat_pending[SPMV_NUM_FORMATS] = {false, false, false, false, false, false};
  bool sell_slots_pending = false;  // sell_slots still on the device (sell_sp[ns])

  // Scratch (grow-only) for segmented-reduction chunk records and for the
  // power-step block partials.
  void* seg_scratch = nullptr;
  size_t seg_scratch_bytes = 0;
  void* fix_scratch = nullptr;
  size_t fix_scratch_bytes = 0;
  // merge-path partition (chunk start coordinates) cached per items-per-thread:
  // the CSR arrays never change after create, so it is computed once
  int64_t* merge_coords = nullptr;
  int64_t merge_coords_n = 0;
  int merge_coords_ipt = 0;  // merge items per chunk the cached coordinates were computed for
                             // (negative: entries per chunk of the nnz-split partition)
  // rows without entries, ascending (CSR; the nnz-split merge variant writes
  // them in a separate pass), built on first use (csr_n_empty = -1 until then)
  int32_t* csr_empty = nullptr;
  int64_t csr_n_empty = -1;
  // row map of the nnz-split kernel with a cached row map (knob 0x800): a bit
  // per entry (1 = first entry of its row), the ids of the non-empty rows in
  // order, and per 256-entry chunk the number of row starts before it
  uint32_t* rm_bits = nullptr;
  int32_t* rm_rows = nullptr;
  int64_t* rm_ord0 = nullptr;
  int64_t rm_nchunks = -1;
  // spmv_release_csr: the CSR (and COO) arrays were freed after conversion to
  // a format with its own arrays; everything that reads them now fails
  bool csr_released = false;
  // CUDA-graph replay of the single-GPU power loop (spmv_power_iterate_graph):
  // the instantiated graph and its key; gen counts every change that can
  // alter the launched kernels (convert, set_format, set_launch, tune, ...)
  void* power_graph = nullptr;
  uint64_t gen = 0;
  double* pi_partials = nullptr;
  unsigned* pi_counter = nullptr;
  size_t pi_partials_n = 0;

  std::string last_error;
  std::string log;  // JSON records, comma separated (wrapped in [] on export)
};

namespace spmv {

// ingest.cu
// New handle holding rows [r0, r1) of parent's CSR (same columns, same dtype,
// stream and device; features not computed, active format CSR).
spmv_matrix* make_row_slice(spmv_matrix* parent, int64_t r0, int64_t r1);
void ingest(spmv_matrix* h, const int32_t* row_idx, const int32_t* col_idx, const void* vals,
            spmv_mem_t where);

// features.cu
void compute_features(spmv_matrix* h);

// convert.cu
void build_coo(spmv_matrix* h);
// h->csr_empty / csr_n_empty (rows of the CSR without entries); once per handle.
void build_csr_empty(spmv_matrix* h);
// h->rm_* (row map of the nnz-split kernel, 256-entry chunks); once per handle.
void build_csr_rowmap(spmv_matrix* h);
// index16 (column encoding): 0 = int32 columns, 1 = 16-bit offsets, 2 = 8-bit
// codes into the offset dictionary (SPMV_ERR_UNSUPPORTED if the encoding does
// not fit), -1 = the narrowest that fits (8-bit, then 16-bit, then int32).
void build_ell(spmv_matrix* h, int index16 = 0);
void build_sell(spmv_matrix* h, int64_t C, int64_t sigma, int index16 = 0);
// True iff every column lies within ±32767 of col_origin + its row.
bool offsets16_fit(spmv_matrix* h);
// Distinct offsets d = col − col_origin − row (builds the dictionary once);
// > 255 means the 8-bit encoding does not fit.
int dict8_codes(spmv_matrix* h);
// The encoding index16 = -1 resolves to on this handle (0, 1 or 2).
int resolve_index_auto(spmv_matrix* h);
void build_hyb(spmv_matrix* h, int64_t K);
void build_bell(spmv_matrix* h, int64_t b);
void free_format(spmv_matrix* h, int fmt);
int64_t format_stored_bytes(spmv_matrix* h, int fmt);
// Conversion latency of fmt in seconds (waits for its stop event if needed).
double format_latency(spmv_matrix* h, int fmt);
// SELL stored slot count (reads it back from the device if still pending).
int64_t sell_slots(spmv_matrix* h);

// Epilogue parameters shared by every SpMV kernel.
struct Epilogue {
  double alpha = 1.0, beta = 0.0;
  int mode = 0;  // 0: y = alpha·Ax + beta·y; 1: power step; 2: y += alpha·Ax; 3: y += alpha_dev·Ax
  const double* sums_prev = nullptr;   // mode 1: alpha = 1/sqrt(sums_prev[0])
  double* sums_out = nullptr;          // mode 1: [Σy², Σ x_own·y]
  double* partials = nullptr;          // mode 1: per-block partials (2 per block)
  unsigned* counter = nullptr;         // mode 1: last-block counter (zero at rest)
  int64_t row_offset = 0;              // mode 1: x_own = x[row_offset + i]
  int sums_parts = 1;                  // modes 1/3: alpha = 1/sqrt(Σ_p sums_prev[2p]) (row-block parts)
  bool pdl = true;                     // mode 1: programmatic dependent launch after the previous kernel
};

// spmv kernels (launchers). All asynchronous on h->stream.
void run_csr(spmv_matrix* h, const Epilogue& e, const void* x, void* y, const spmv_launch_t& L);
void run_ell(spmv_matrix* h, const Epilogue& e, const void* x, void* y, const spmv_launch_t& L);
void run_ell_arrays(spmv_matrix* h, const int32_t* col, const void* val, int64_t K, int64_t n_pad,
                    const Epilogue& e, const void* x, void* y, const spmv_launch_t& L,
                    const int16_t* col16 = nullptr, const uint8_t* col8 = nullptr,
                    const int32_t* tab8 = nullptr);
// y <- beta·y over all rows (alpha == 0: A is not read).
void run_scale(spmv_matrix* h, void* y, double beta);
void run_sell(spmv_matrix* h, const Epilogue& e, const void* x, void* y, const spmv_launch_t& L);
void run_coo(spmv_matrix* h, const Epilogue& e, const void* x, void* y, const spmv_launch_t& L);
void run_hyb(spmv_matrix* h, const Epilogue& e, const void* x, void* y, const spmv_launch_t& L);
void run_bell(spmv_matrix* h, const Epilogue& e, const void* x, void* y, const spmv_launch_t& L);
// Σ y_i², Σ x_own_i·y_i over rows (power mode for formats without a fused epilogue).
void run_norms(spmv_matrix* h, const Epilogue& e, const void* x, const void* y, int64_t n);

// Power step / norm (api.cu) and the native loop + NCCL (dist.cu).
void power_step_internal(spmv_matrix* h, const void* x, void* y, const double* sums_prev, double* sums_out,
                         int64_t row_offset, int sums_parts = 1, bool pdl = true);
void spmv_norm2_internal(spmv_matrix* h, const void* x, int64_t n, double* sums_out);
void power_iterate(spmv_matrix* h, const void* x0, void* buf0, void* buf1, int64_t n_full, int64_t steps,
                   double* sums, void* comm, int64_t chunk, void* chunk_buf, float* kernel_ms, float* loop_ms,
                   int* final_buf);
void* dist_init(const uint8_t id[128], int rank, int world, int device);
// plan.cu: the distributed plan (interior/halo split, overlap, halo exchange).
spmv_dist_plan* plan_create(spmv_matrix* h, void* comm, int64_t chunk, uint32_t flags);
void plan_destroy(spmv_dist_plan* P);
void plan_iterate(spmv_dist_plan* P, const void* x0, void* buf0, void* buf1, int64_t steps, double* sums,
                  float* loop_ms, float* interior_ms, int* final_buf);
void plan_info(const spmv_dist_plan* P, spmv_dist_plan_info_t* o);
spmv_matrix* plan_part(spmv_dist_plan* P, int p);
int plan_device(const spmv_dist_plan* P);
void dist_unique_id(uint8_t out[128]);
void dist_destroy(void* comm);

// energy.cu: NVML energy over a window of back-to-back launches.
struct EnergySample {
  double seconds = 0, joules = 0, watts = 0;
  int64_t reps = 0;
};
EnergySample measure_energy(spmv_matrix* h, const std::function<void()>& launch, double min_seconds);
bool nvml_available();

// Make sure the power-step partial buffers hold >= nblocks entries.
void ensure_pi_scratch(spmv_matrix* h, size_t nblocks);
void* ensure_seg_scratch(spmv_matrix* h, size_t bytes);
// device->host copy of a small result through pinned memory; synchronises s
void d2h_sync(void* host_dst, const void* dev_src, size_t bytes, cudaStream_t s);
void* ensure_fixup_scratch(spmv_matrix* h, size_t bytes);

// Resolve a launch variant to the defaults of its kernel.
spmv_launch_t resolve_launch(const spmv_matrix* h, int fmt, const spmv_launch_t& L);
// Grid for a persistent (grid-stride) kernel: min(needed, SMs × resident blocks per SM),
// minus g_sm_reserve SMs' worth of residency (left free for concurrent NCCL kernels).
extern thread_local int g_sm_reserve;
int64_t persistent_grid(const void* func, int block, int64_t needed_blocks, size_t dyn_smem = 0);
// Function attributes of one launch, applied on the CURRENT device (CUDA
// function attributes are per device): the preferred shared-memory carveout
// (pct < 0 = driver default, restored if an earlier launch changed it) and
// the dynamic shared-memory opt-in. The object holds the process-wide
// launch-attribute lock until it is destroyed, so the attributes cannot be
// changed by another thread between the set and the launch: construct it
// right before computing the grid and keep it in scope through the launch.
class LaunchAttrs {
 public:
  LaunchAttrs(const void* fn, int carveout_pct, size_t dyn_smem = 0);
 private:
  std::unique_lock<std::recursive_mutex> lk_;
};

}  // namespace spmv
