// api.cu — the extern "C" boundary of libspmv.so (include/spmv.h).
// Argument validation, handle lifecycle, format dispatch, the launch tuner
// (compile-time mode analog), the format selector with its
// overhead gate (run-time mode analog), the power step, and the
// multi-GPU host logic (partition, column remap).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <sstream>
#include <unordered_map>
#include <vector>

#include "dist.cuh"
#include "kern_coo_decl.cuh"
#include "kern_csr_decl.cuh"
#include "kern_sliced_decl.cuh"
#include "selector.cuh"
#include "spmv_common.cuh"

namespace spmv {

std::atomic<uint64_t> g_launches{0};
thread_local int g_sm_reserve = 0;

namespace {
std::mutex g_mu;
bool g_pool_ready[64] = {};
// launch attributes per (device, function): carveout in effect (-1 = driver
// default) and the dynamic shared memory opted in
std::recursive_mutex g_attr_mu;
std::map<std::pair<int, const void*>, int> g_carveout;
std::map<std::pair<int, const void*>, size_t> g_dyn_smem;
thread_local std::string g_err;
}  // namespace

void* dalloc(size_t bytes, cudaStream_t s) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (dev >= 0 && dev < 64 && !g_pool_ready[dev]) {
    std::lock_guard<std::mutex> lk(g_mu);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    g_pool_ready[dev] = true;
  }
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, bytes, s);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    // give cached pool memory back and retry once
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      cudaStreamSynchronize(s);
      cudaMemPoolTrimTo(pool, 0);
    }
    e = cudaMallocAsync(&p, bytes, s);
  }
  cuda_check(e, "cudaMallocAsync");
  return p;
}

// Small device->host read-backs go through a per-thread pinned buffer: a copy
// into pageable memory is staged by the driver and was measured waiting for
// another stream's bulk host upload (two handles in flight, bench e2e).
void d2h_sync(void* host_dst, const void* dev_src, size_t bytes, cudaStream_t s) {
  thread_local void* pin = nullptr;
  thread_local size_t pin_bytes = 0;
  if (bytes == 0) return;
  if (pin_bytes < bytes) {
    if (pin) cudaFreeHost(pin);
    pin = nullptr;
    pin_bytes = 0;
    const size_t want = std::max<size_t>(bytes, 64 << 10);
    CK(cudaMallocHost(&pin, want));
    pin_bytes = want;
  }
  CK(cudaMemcpyAsync(pin, dev_src, bytes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  std::memcpy(host_dst, pin, bytes);
}

void dfree(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}

int64_t persistent_grid(const void* func, int block, int64_t needed_blocks, size_t dyn_smem) {
  static std::unordered_map<uint64_t, int> occ;
  static int sms = 0;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  int per_sm;
  // the carveout in effect for func on this device changes the
  // shared-memory-limited occupancy (lock order: g_attr_mu, then g_mu)
  std::lock_guard<std::recursive_mutex> alk(g_attr_mu);
  auto cv = g_carveout.find({dev, func});
  const uint64_t carve = cv == g_carveout.end() || cv->second < 0 ? 127 : (uint64_t)cv->second;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (sms == 0) CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const uint64_t key = (uint64_t)(uintptr_t)func ^ ((uint64_t)block << 48) ^ ((uint64_t)dyn_smem << 20) ^
                         (carve << 56) ^ ((uint64_t)dev << 40);
    auto it = occ.find(key);
    if (it == occ.end()) {
      int nb = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, func, block, dyn_smem));
      it = occ.emplace(key, std::max(nb, 1)).first;
    }
    per_sm = it->second;
  }
  const int64_t cap = (int64_t)std::max(sms - std::max(g_sm_reserve, 0), 1) * per_sm;
  return needed_blocks < cap ? needed_blocks : cap;
}

LaunchAttrs::LaunchAttrs(const void* fn, int pct, size_t dyn_smem) : lk_(g_attr_mu) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  const std::pair<int, const void*> key{dev, fn};
  if (dyn_smem > 0) {
    auto it = g_dyn_smem.find(key);
    if (it == g_dyn_smem.end() || it->second < dyn_smem) {
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_smem));
      g_dyn_smem[key] = dyn_smem;
    }
  }
  const int want = pct < 0 ? -1 : pct;
  auto it = g_carveout.find(key);
  const int have = it == g_carveout.end() ? -1 : it->second;
  if (have != want) {
    // -1 is cudaSharedmemCarveoutDefault: restores the driver's choice
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                            want < 0 ? (int)cudaSharedmemCarveoutDefault : want));
    g_carveout[key] = want;
  }
}

void ensure_pi_scratch(spmv_matrix* h, size_t nblocks) {
  if (h->pi_partials && h->pi_partials_n >= nblocks) return;
  CK(cudaStreamSynchronize(h->stream));
  dfree(h->pi_partials, h->stream);
  size_t n = std::max<size_t>(nblocks, 4096);
  h->pi_partials = dalloc_n<double>(2 * (int64_t)n, h->stream);
  h->pi_partials_n = n;
  if (!h->pi_counter) {
    h->pi_counter = dalloc_n<unsigned>(1, h->stream);
    CK(cudaMemsetAsync(h->pi_counter, 0, sizeof(unsigned), h->stream));
  }
}

void* ensure_seg_scratch(spmv_matrix* h, size_t bytes) {
  if (h->seg_scratch && h->seg_scratch_bytes >= bytes) return h->seg_scratch;
  CK(cudaStreamSynchronize(h->stream));
  dfree(h->seg_scratch, h->stream);
  h->seg_scratch = dalloc(bytes, h->stream);
  h->seg_scratch_bytes = bytes;
  return h->seg_scratch;
}

void* ensure_fixup_scratch(spmv_matrix* h, size_t bytes) {
  if (h->fix_scratch && h->fix_scratch_bytes >= bytes) return h->fix_scratch;
  CK(cudaStreamSynchronize(h->stream));
  dfree(h->fix_scratch, h->stream);
  h->fix_scratch = dalloc(bytes, h->stream);
  h->fix_scratch_bytes = bytes;
  return h->fix_scratch;
}

static int csr_default_lanes(const spmv_matrix* h) {
  if (h->csr_T > 0) return h->csr_T;
  double mean = h->rows > 0 ? (double)h->nnz / (double)h->rows : 0.0;
  int t = 1;
  while (t < (int)std::ceil(mean) && t < 32) t <<= 1;
  return std::min(32, std::max(2, t));
}

spmv_launch_t resolve_launch(const spmv_matrix* h, int fmt, const spmv_launch_t& L) {
  spmv_launch_t r = L;
  if (r.block == 0) r.block = 256;
  if (r.maxreg == 0) r.maxreg = 255;
  if (r.knob == 0) {
    switch (fmt) {
      case SPMV_FMT_CSR:
        if (h->csr_alg == SPMV_CSR_MERGE) r.knob = 8;
        else if (h->csr_alg == SPMV_CSR_STREAM) r.knob = 32;
        else if (h->csr_alg == SPMV_CSR_SCALAR) r.knob = 1;
        else r.knob = csr_default_lanes(h);
        break;
      case SPMV_FMT_ELL: r.knob = (h->dtype == SPMV_R64F ? 64 : 128) | kern::kSlicedCarry; break;
      case SPMV_FMT_SELL: r.knob = (int)h->sell_C | kern::kSlicedCarry; break;
      case SPMV_FMT_COO: r.knob = 4; break;
      case SPMV_FMT_HYB: r.knob = 4; break;
      case SPMV_FMT_BELL: r.knob = (int)h->bell_b; break;
    }
  }
  return r;
}

static bool built(const spmv_matrix* h, int fmt) {
  switch (fmt) {
    case SPMV_FMT_CSR: return !h->csr_released;
    case SPMV_FMT_COO: return h->coo_built && !h->csr_released;
    case SPMV_FMT_ELL: return h->ell_built;
    case SPMV_FMT_SELL: return h->sell_built;
    case SPMV_FMT_HYB: return h->hyb_built;
    case SPMV_FMT_BELL: return h->bell_built;
  }
  return false;
}

// Entry points that read the CSR arrays (conversions, features, tuning, row slices).
static void need_csr(const spmv_matrix* h, const char* what) {
  if (h->csr_released)
    fail(SPMV_ERR_NOT_CONVERTED, std::string(what) + ": the CSR arrays were released (spmv_release_csr)");
}

// Launch one SpMV of format fmt (no validation).
static void dispatch(spmv_matrix* h, int fmt, const Epilogue& e, const void* x, void* y, const spmv_launch_t& L0) {
  spmv_launch_t L = resolve_launch(h, fmt, L0);
  if (e.mode == 0 && e.alpha == 0.0) {  // A is not read
    run_scale(h, y, e.beta);
    return;
  }
  switch (fmt) {
    case SPMV_FMT_CSR: run_csr(h, e, x, y, L); break;
    case SPMV_FMT_ELL: run_ell(h, e, x, y, L); break;
    case SPMV_FMT_SELL: run_sell(h, e, x, y, L); break;
    case SPMV_FMT_COO: run_coo(h, e, x, y, L); break;
    case SPMV_FMT_HYB: run_hyb(h, e, x, y, L); break;
    case SPMV_FMT_BELL: run_bell(h, e, x, y, L); break;
    default: fail(SPMV_ERR_INVALID_ARG, "bad format");
  }
}

static bool fused_norms(const spmv_matrix* h, int fmt) {
  return fmt == SPMV_FMT_ELL || fmt == SPMV_FMT_SELL || fmt == SPMV_FMT_BELL ||
         (fmt == SPMV_FMT_CSR && h->csr_alg != SPMV_CSR_MERGE);  // vector, scalar and stream fuse the norms
}

void power_step_internal(spmv_matrix* h, const void* x, void* y, const double* sums_prev, double* sums_out,
                         int64_t row_offset, int sums_parts, bool pdl) {
  const int fmt = h->active;
  Epilogue e;
  e.mode = 1;
  e.sums_prev = sums_prev;
  e.sums_out = sums_out;
  e.row_offset = row_offset;
  e.sums_parts = sums_parts;
  e.pdl = pdl;
  if (h->rows == 0) {
    CK(cudaMemsetAsync(sums_out, 0, 2 * sizeof(double), h->stream));
    return;
  }
  ensure_pi_scratch(h, 4096);
  e.partials = h->pi_partials;
  e.counter = h->pi_counter;
  dispatch(h, fmt, e, x, y, h->launch[fmt]);
  if (!fused_norms(h, fmt)) run_norms(h, e, x, y, h->rows);
}

void spmv_norm2_internal(spmv_matrix* h, const void* x, int64_t n, double* sums_out) {
  if (n == 0) {
    CK(cudaMemsetAsync(sums_out, 0, 2 * sizeof(double), h->stream));
    return;
  }
  Epilogue e;
  e.mode = 1;
  e.sums_out = sums_out;
  run_norms(h, e, nullptr, x, n);
}

// ------------------------------------------------------------------ timing
struct Events {
  cudaEvent_t a, b;
  Events() {
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
  }
  ~Events() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

// Median-of-3 time per SpMV (seconds) for one (format, launch) on scratch x/y.
static double time_variant(spmv_matrix* h, int fmt, const spmv_launch_t& L, const void* x, void* y) {
  Epilogue e;
  e.alpha = 1.0;
  e.beta = 0.0;
  Events ev;
  for (int w = 0; w < 2; ++w) dispatch(h, fmt, e, x, y, L);
  CK(cudaEventRecord(ev.a, h->stream));
  dispatch(h, fmt, e, x, y, L);
  CK(cudaEventRecord(ev.b, h->stream));
  CK(cudaEventSynchronize(ev.b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, ev.a, ev.b));
  int reps = (int)std::min(200.0, std::max(3.0, std::ceil(2.0 / std::max(ms, 1e-3f))));
  double t[3];
  for (int trial = 0; trial < 3; ++trial) {
    CK(cudaEventRecord(ev.a, h->stream));
    for (int r = 0; r < reps; ++r) dispatch(h, fmt, e, x, y, L);
    CK(cudaEventRecord(ev.b, h->stream));
    CK(cudaEventSynchronize(ev.b));
    CK(cudaEventElapsedTime(&ms, ev.a, ev.b));
    t[trial] = ms * 1e-3 / reps;
  }
  std::sort(t, t + 3);
  return t[1];
}

// The run-time mode's own t_CSR (it is paid on every matrix, so it
// is kept short): one warm-up launch, then the median of three individually
// timed launches — on the 2^25-entry sample each is ≈ 0.25 ms of HBM-bound
// streaming, long against event resolution.
static double time_variant_quick(spmv_matrix* h, int fmt, const spmv_launch_t& L, const void* x, void* y) {
  Epilogue e;
  e.alpha = 1.0;
  e.beta = 0.0;
  Events ev[3];
  dispatch(h, fmt, e, x, y, L);
  for (auto& q : ev) {
    CK(cudaEventRecord(q.a, h->stream));
    dispatch(h, fmt, e, x, y, L);
    CK(cudaEventRecord(q.b, h->stream));
  }
  CK(cudaEventSynchronize(ev[2].b));
  double t[3];
  for (int i = 0; i < 3; ++i) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ev[i].a, ev[i].b));
    t[i] = ms * 1e-3;
  }
  std::sort(t, t + 3);
  return t[1];
}

template <class T>
__global__ void k_fill_one(T* p, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) p[i] = T(1);
}

struct TuneScratch {
  spmv_matrix* h;
  void* x = nullptr;
  void* y = nullptr;
  explicit TuneScratch(spmv_matrix* hh) : h(hh) {
    x = dalloc((size_t)std::max<int64_t>(h->cols, 1) * h->vbytes, h->stream);
    y = dalloc((size_t)std::max<int64_t>(h->rows, 1) * h->vbytes, h->stream);
    if (h->dtype == SPMV_R64F) LAUNCH(k_fill_one<double>, grid_for(h->cols, 256), 256, 0, h->stream, (double*)x, h->cols);
    else LAUNCH(k_fill_one<float>, grid_for(h->cols, 256), 256, 0, h->stream, (float*)x, h->cols);
  }
  ~TuneScratch() {
    dfree(x, h->stream);
    dfree(y, h->stream);
  }
};

// Objective-aware measurement.
struct Objective {
  int obj = 0;  // 0 latency, 1 energy, 2 power, 3 efficiency
  static const char* name(int o) {
    static const char* n[] = {"latency", "energy", "power", "efficiency"};
    return (o >= 0 && o < 4) ? n[o] : "?";
  }
};

struct Measured {
  double t = 0;                           // seconds per SpMV (latency sweep)
  double ej = std::nan(""), w = std::nan(""), eff = std::nan("");  // J per SpMV, W, MFLOPS/W
};

static void measure_objective(spmv_matrix* h, int fmt, const spmv_launch_t& L, const void* x, void* y,
                              Measured& m) {
  Epilogue e;
  EnergySample s = measure_energy(h, [&] { dispatch(h, fmt, e, x, y, L); }, 0.4);
  m.ej = s.reps > 0 ? s.joules / (double)s.reps : std::nan("");
  m.w = s.watts;
  m.eff = s.joules > 0 ? 2.0 * (double)h->nnz * (double)s.reps / 1e6 / s.joules : std::nan("");
}

// Smaller is better for every objective (efficiency is negated).
static double objective_value(int obj, const Measured& m) {
  switch (obj) {
    case 1: return m.ej;
    case 2: return m.w;
    case 3: return -m.eff;
    default: return m.t;
  }
}

// Column encoding of a built ELL/SELL layout: 0 int32, 1 16-bit offsets, 2 8-bit dictionary codes.
static int index_encoding(const spmv_matrix* h, int fmt) {
  if (fmt == SPMV_FMT_ELL) return h->ell_col8 ? 2 : (h->ell_col16 ? 1 : 0);
  if (fmt == SPMV_FMT_SELL) return h->sell_col8 ? 2 : (h->sell_col16 ? 1 : 0);
  return 0;
}

static const char* fmt_name(int f) {
  static const char* n[] = {"COO", "CSR", "ELL", "HYB", "SELL", "BELL"};
  return (f >= 0 && f < 6) ? n[f] : "?";
}

static void log_append(spmv_matrix* h, const std::string& rec) {
  if (!h->log.empty()) h->log += ",";
  h->log += rec;
}

// Knob values tried per format by the launch sweep.
static std::vector<int> knob_set(const spmv_matrix* h, int fmt) {
  switch (fmt) {
    case SPMV_FMT_CSR:
      if (h->csr_alg == SPMV_CSR_MERGE)  // per-warp merge walk, or row-interleaved tiles of block·IPT items
        return {4, 8, 16, kern::kMergeTile | 4, kern::kMergeTile | 8, kern::kMergeTile | 16, kern::kMergeTile | 32,
                kern::kMergeStream | 4, kern::kMergeStream | 8, kern::kMergeStream | 16, kern::kMergeStream | 32,
                kern::kMergeNnz | 4, kern::kMergeNnz | 8, kern::kMergeRowmap | 8};
      if (h->csr_alg == SPMV_CSR_STREAM) return {16, 32, 64};
      {
        int t = csr_default_lanes(h);
        std::vector<int> v{t};
        if (t / 2 >= 1) v.push_back(t / 2);
        if (t * 2 <= 32) v.push_back(t * 2);
        for (int q : {t / 2, t})  // quad (128-bit) loads: a lane covers 4 entries per step
          if (q >= 4) v.push_back(kern::kCsrQuad | q);
        return v;
      }
    case SPMV_FMT_ELL:  // rows per warp × batch loop (kern::kSlicedCarry)
      return {32, 64, 128, 32 | kern::kSlicedCarry, 64 | kern::kSlicedCarry, 128 | kern::kSlicedCarry};
    case SPMV_FMT_SELL: return {(int)h->sell_C, (int)h->sell_C | kern::kSlicedCarry};
    case SPMV_FMT_COO:  // warp chunks of 32·W entries, or row-interleaved tiles of block·EPT entries
    case SPMV_FMT_HYB:
      return {2, 4, 8, kern::kCooTile | 4, kern::kCooTile | 8, kern::kCooTile | 16, kern::kCooTile | 32};
    case SPMV_FMT_BELL: return {(int)h->bell_b};
  }
  return {0};
}

// Compile-time mode analog: sweep block × maxreg × carveout × knob
// for the active format; keep the argmin of the median time.
// Compile-time mode analog: sweep block × maxreg × carveout × knob
// for the active format; keep the argmin of the median time. With a
// non-latency objective the 6 fastest variants are re-measured with NVML and
// the objective decides among them.
static void tune_launch(spmv_matrix* h, int fmt, TuneScratch& ts, spmv_tune_report_t* rep, int obj) {
  static const int blocks[] = {64, 128, 256, 512, 1024};
  static const int regs[] = {32, 64, 128, 255};
  static const int carve[] = {0, 25, 50, 100};
  spmv_launch_t best = resolve_launch(h, fmt, h->launch[fmt]);
  double tbest;
  try {
    tbest = time_variant(h, fmt, best, ts.x, ts.y);
  } catch (const SpmvError&) {  // the current variant is invalid for this kernel: start from defaults
    cudaGetLastError();
    best = resolve_launch(h, fmt, spmv_launch_t{0, 0, -1, 0});
    tbest = time_variant(h, fmt, best, ts.x, ts.y);
  }
  std::vector<std::pair<double, spmv_launch_t>> all{{tbest, best}};
  int n = 1;
  std::ostringstream os;
  os.precision(9);
  os << "{\"kind\":\"launch_sweep\",\"format\":\"" << fmt_name(fmt) << "\",\"objective\":\""
     << Objective::name(obj) << "\",\"variants\":[";
  bool first = true;
  for (int knob : knob_set(h, fmt))
    for (int b : blocks)
      for (int r : regs)
        for (int c : carve) {
          spmv_launch_t L{b, r, c, knob};
          double t;
          try {
            t = time_variant(h, fmt, L, ts.x, ts.y);
          } catch (const SpmvError&) {
            cudaGetLastError();
            continue;
          }
          ++n;
          all.push_back({t, L});
          os << (first ? "" : ",") << "[" << b << "," << r << "," << c << "," << knob << "," << t << "]";
          first = false;
          if (t < tbest) {
            tbest = t;
            best = L;
          }
        }
  os << "],\"best\":[" << best.block << "," << best.maxreg << "," << best.carveout_pct << "," << best.knob
     << "],\"t_best_s\":" << tbest;
  Measured chosen;
  chosen.t = tbest;
  if (obj != 0) {
    std::sort(all.begin(), all.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    const size_t top = std::min<size_t>(6, all.size());
    double vbest = 0;
    os << ",\"objective_top\":[";
    for (size_t i = 0; i < top; ++i) {
      Measured m;
      m.t = all[i].first;
      measure_objective(h, fmt, all[i].second, ts.x, ts.y, m);
      const double v = objective_value(obj, m);
      const spmv_launch_t& L = all[i].second;
      os << (i ? "," : "") << "{\"launch\":[" << L.block << "," << L.maxreg << "," << L.carveout_pct << ","
         << L.knob << "],\"t_s\":" << m.t << ",\"j_per_spmv\":" << m.ej << ",\"w\":" << m.w
         << ",\"mflops_per_w\":" << m.eff << "}";
      if (i == 0 || v < vbest) {
        vbest = v;
        best = L;
        chosen = m;
      }
    }
    os << "],\"objective_best\":[" << best.block << "," << best.maxreg << "," << best.carveout_pct << ","
       << best.knob << "]";
  }
  os << "}";
  log_append(h, os.str());
  h->launch[fmt] = best;
  if (rep) {
    rep->launch = best;
    rep->t_best_s = chosen.t;
    rep->n_variants += n;
    rep->energy_j = chosen.ej;
    rep->power_w = chosen.w;
    rep->mflops_per_w = chosen.eff;
  }
}

static double sell_padding(spmv_matrix* h) {
  const int64_t sl = sell_slots(h);
  return sl > 0 ? 1.0 - (double)h->nnz / (double)sl : 0.0;
}

// Run-time mode analog: features -> candidates -> measure -> gate.
// With tune_each (spmv_tune LAUNCH|FORMAT) every candidate is launch-tuned
// before the comparison, so the gate compares the end states it would
// produce (the compile-time mode inside the run-time mode); conversion
// latencies are measured on a warm rebuild (the first build of a process
// also pays lazy module loading, which a later conversion does not).
static void tune_format(spmv_matrix* h, int64_t iters, TuneScratch& ts, spmv_tune_report_t* rep, int obj,
                        bool tune_each) {
  if (!h->have_features) compute_features(h);
  const spmv_features_t& f = h->feat;
  const int orig_alg = h->csr_alg;
  std::ostringstream os;
  os.precision(9);
  os << "{\"kind\":\"format_select\",\"features\":{\"n\":" << f.n_rows << ",\"nnz\":" << f.nnz
     << ",\"mean\":" << f.mean << ",\"var\":" << f.var << ",\"std\":" << f.std << ",\"max\":" << f.max_len
     << ",\"ell_ratio\":" << f.ell_ratio << ",\"median\":" << f.median << ",\"mode\":" << f.mode
     << ",\"bandwidth\":" << f.bandwidth << "},\"tuned_candidates\":" << (tune_each ? "true" : "false")
     << ",\"candidates\":[";
  struct Cand {
    int fmt;
    int alg;
    double t, c;
    std::string why;
    Measured m;
    spmv_launch_t L;
  };
  std::vector<Cand> cands;
  // time one candidate (format fmt, the active CSR algorithm for CSR) from launch L
  auto measure = [&](int fmt, spmv_launch_t L) -> std::pair<double, spmv_launch_t> {
    L = resolve_launch(h, fmt, L);
    if (tune_each) {
      h->launch[fmt] = L;
      tune_launch(h, fmt, ts, rep, obj);
      L = resolve_launch(h, fmt, h->launch[fmt]);
    }
    return {time_variant(h, fmt, L, ts.x, ts.y), L};
  };
  const spmv_launch_t csr_launch0 = h->launch[SPMV_FMT_CSR];
  const spmv_launch_t dflt{0, 0, -1, 0};
  // CSR (paper default): CSR-vector with T from the mean.
  h->csr_alg = SPMV_CSR_VECTOR;
  auto mc = measure(SPMV_FMT_CSR, dflt);
  double t_csr = mc.first;
  cands.push_back({SPMV_FMT_CSR, SPMV_CSR_VECTOR, t_csr, 0.0, "default", Measured{}, mc.second});
  const bool skewed = (f.mean > 0 && f.std / f.mean > 1.0) || (double)f.max_len > 32.0 * f.mean;
  if (skewed) {
    h->csr_alg = SPMV_CSR_MERGE;
    auto m = measure(SPMV_FMT_CSR, dflt);
    cands.push_back({SPMV_FMT_CSR, SPMV_CSR_MERGE, m.first, 0.0, "std/mean>1 or max>32*mean", Measured{}, m.second});
  } else {
    // CSR-stream (TMA-staged tiles, thread per row): no conversion at all
    h->csr_alg = SPMV_CSR_STREAM;
    try {
      auto m = measure(SPMV_FMT_CSR, dflt);
      cands.push_back({SPMV_FMT_CSR, SPMV_CSR_STREAM, m.first, 0.0, "regular rows (no conversion)", Measured{},
                       m.second});
    } catch (const SpmvError& e) {
      cudaGetLastError();
      os << "{\"format\":\"CSR\",\"alg\":\"stream\",\"rejected\":\"" << e.msg << "\"},";
    }
  }
  h->csr_alg = orig_alg;
  h->launch[SPMV_FMT_CSR] = csr_launch0;
  int64_t bell_b_try = 2;
  auto do_build = [&](int fmt) {
    switch (fmt) {
      case SPMV_FMT_BELL: build_bell(h, bell_b_try); break;
      case SPMV_FMT_ELL: build_ell(h, -1); break;
      case SPMV_FMT_SELL: build_sell(h, h->dtype == SPMV_R64F ? 64 : 128, 1, -1); break;
      case SPMV_FMT_HYB: build_hyb(h, -1); break;
      case SPMV_FMT_COO: build_coo(h); break;
    }
  };
  std::vector<int> built_here;  // candidates this call converted (the caller's own builds are kept)
  auto try_build = [&](int fmt, const char* why) {
    bool was = built(h, fmt);
    try {
      if (!was) do_build(fmt);
    } catch (const SpmvError& e) {
      cudaGetLastError();
      os << "{\"format\":\"" << fmt_name(fmt) << "\",\"rejected\":\"" << e.msg << "\"},";
      return;
    }
    if (fmt == SPMV_FMT_SELL && sell_padding(h) > 0.10) {
      os << "{\"format\":\"SELL\",\"rejected\":\"padding " << sell_padding(h) << " > 0.10\"},";
      if (!was) free_format(h, fmt);
      return;
    }
    if (fmt == SPMV_FMT_BELL) {
      const double slots = (double)h->bell_kb * (double)h->bell_nbr * (double)(h->bell_b * h->bell_b);
      const double pad = slots > 0 ? 1.0 - (double)h->nnz / slots : 1.0;
      if (pad > 0.10) {
        os << "{\"format\":\"BELL\",\"b\":" << h->bell_b << ",\"rejected\":\"block padding " << pad
           << " > 0.10\"},";
        if (!was) free_format(h, fmt);
        return;
      }
    }
    if (!was) {  // warm conversion latency: rebuild once the kernels are loaded
      free_format(h, fmt);
      do_build(fmt);
      built_here.push_back(fmt);
    }
    auto m = measure(fmt, h->launch[fmt]);
    cands.push_back({fmt, 0, m.first, format_latency(h, fmt), why, Measured{}, m.second});
  };
  if (f.ell_ratio >= 0.9) try_build(SPMV_FMT_ELL, "ell_ratio>=0.9");
  if (!skewed) try_build(SPMV_FMT_SELL, "SELL padding<=10%");
  // BELL: only block-structured matrices keep block padding <= 10%
  if (!skewed && f.mean >= 4.0) {
    if (built(h, SPMV_FMT_BELL)) {
      bell_b_try = h->bell_b;
      try_build(SPMV_FMT_BELL, "block padding<=10% (pre-built)");
    } else {
      for (int64_t b : {int64_t(3), int64_t(2)}) {
        bell_b_try = b;
        try_build(SPMV_FMT_BELL, b == 2 ? "2x2 block padding<=10%" : "3x3 block padding<=10%");
        if (built(h, SPMV_FMT_BELL)) break;  // accepted (rejections free the build)
      }
    }
  }
  if (skewed) {
    try_build(SPMV_FMT_HYB, "skewed rows");
    try_build(SPMV_FMT_COO, "skewed rows");
  }
  for (Cand& c : cands) {
    c.m.t = c.t;
    if (obj != 0) {  // energy / power / efficiency: NVML window per candidate
      if (c.fmt == SPMV_FMT_CSR) h->csr_alg = c.alg;
      measure_objective(h, c.fmt, c.L, ts.x, ts.y, c.m);
      h->csr_alg = orig_alg;
    }
  }
  size_t bi = 0;
  for (size_t i = 0; i < cands.size(); ++i) {
    const Cand& c = cands[i];
    os << "{\"format\":\"" << fmt_name(c.fmt) << "\""
       << (c.alg == SPMV_CSR_MERGE ? ",\"alg\":\"merge\"" : (c.alg == SPMV_CSR_STREAM ? ",\"alg\":\"stream\"" : ""))
       << ",\"t_s\":" << c.t << ",\"c_latency_s\":" << c.c << ",\"why\":\"" << c.why << "\"";
    if (obj != 0)
      os << ",\"j_per_spmv\":" << c.m.ej << ",\"w\":" << c.m.w << ",\"mflops_per_w\":" << c.m.eff;
    os << "}" << (i + 1 < cands.size() ? "," : "");
  }
  const Cand& csr = cands[0];
  // Gate (strict >): a candidate's gain over the default
  // CSR minus its overhead. Among several candidates the one with the largest
  // net benefit wins (reading R31): with a short run a conversion-free
  // candidate can beat a slightly faster one that needs a conversion.
  auto gain_of = [&](const Cand& c) {
    if (obj == 0) return (double)iters * (t_csr - c.t);
    if (obj == 2) return csr.m.w - c.m.w;  // average power: no amortisation, the lower draw wins
    return (double)iters * (csr.m.ej - c.m.ej);  // energy / efficiency: joules
  };
  auto overhead_of = [&](const Cand& c) {
    if (obj == 0) return h->f_latency + c.c;
    if (obj == 2) return 0.0;
    return csr.m.w * (h->f_latency + c.c);  // conversion energy at CSR's average power
  };
  for (size_t i = 1; i < cands.size(); ++i)
    if (bi == 0 || gain_of(cands[i]) - overhead_of(cands[i]) > gain_of(cands[bi]) - overhead_of(cands[bi])) bi = i;
  const Cand& best = cands[bi];
  const double gain = bi ? gain_of(best) : 0.0, overhead = bi ? overhead_of(best) : 0.0;
  const bool convert = bi != 0 && gain > overhead;
  const int chosen = convert ? best.fmt : SPMV_FMT_CSR;
  const int chosen_alg = convert ? best.alg : SPMV_CSR_VECTOR;
  os << "],\"objective\":\"" << Objective::name(obj) << "\",\"gate\":{\"expected_iterations\":" << iters
     << ",\"t_csr_s\":" << t_csr << ",\"t_best_s\":" << best.t << ",\"gain_s\":" << gain
     << ",\"gain\":" << gain << ",\"overhead\":" << overhead
     << ",\"f_latency_s\":" << h->f_latency << ",\"c_latency_s\":" << best.c
     << ",\"convert\":" << (convert ? "true" : "false") << "},\"chosen\":\"" << fmt_name(chosen)
     << (chosen == SPMV_FMT_CSR && chosen_alg == SPMV_CSR_MERGE ? "-merge" : "")
     << (chosen == SPMV_FMT_CSR && chosen_alg == SPMV_CSR_STREAM ? "-stream" : "") << "\"}";
  log_append(h, os.str());
  // release candidates that were built here and not chosen
  for (int fmt : built_here)
    if (fmt != chosen) free_format(h, fmt);
  h->active = chosen;
  if (chosen == SPMV_FMT_CSR) h->csr_alg = chosen_alg;
  if (tune_each) {  // the chosen end state keeps its tuned launch
    const Cand& kept = convert ? best : csr;
    h->launch[kept.fmt] = kept.L;
  } else if (chosen == SPMV_FMT_CSR && chosen_alg != orig_alg) {
    h->launch[SPMV_FMT_CSR] = spmv_launch_t{0, 0, -1, 0};  // another kernel: defaults
  }
  if (rep) {
    rep->format = chosen;
    rep->t_csr_s = t_csr;
    rep->t_best_s = convert ? best.t : t_csr;
    rep->f_latency_s = h->f_latency;
    rep->c_latency_s = best.c;
    rep->expected_iterations = iters;
    rep->converted = convert ? 1 : 0;
    rep->n_candidates = (int32_t)cands.size();
    const Measured& cm = convert ? best.m : csr.m;
    rep->energy_j = cm.ej;
    rep->power_w = cm.w;
    rep->mflops_per_w = cm.eff;
    rep->params.csr_alg = h->csr_alg;
    rep->params.csr_T = h->csr_T;
    rep->params.sell_C = (int32_t)h->sell_C;
    rep->params.sell_sigma = (int32_t)h->sell_sigma;
    rep->params.hyb_K = h->hyb_K;
    rep->params.bell_b = (int32_t)h->bell_b;
    rep->params.index16 = index_encoding(h, h->active);
  }
}

// Run-time mode with the learned models (SPMV_TUNE_PREDICT):
// features -> predicted format -> estimated overhead -> gate.
// t_CSR for the run-time mode: the default CSR-vector kernel timed on a row
// prefix holding about kPredictSampleNnz entries (the whole matrix when it is
// smaller), scaled to the full nnz. The kernel's time is linear in the
// entries it streams, and a per-matrix selection must not cost a sizeable
// share of the SpMVs it is choosing for (c5: 3.6e9 entries, 13 ms per CSR
// SpMV, twelve timed launches otherwise).
constexpr int64_t kPredictSampleNnz = 1LL << 25;
static double predict_t_csr(spmv_matrix* h, TuneScratch& ts, int64_t* sample_nnz) {
  const spmv_launch_t L = resolve_launch(h, SPMV_FMT_CSR, spmv_launch_t{0, 0, -1, 0});
  if (h->nnz <= 2 * kPredictSampleNnz || h->rows < 2) {
    *sample_nnz = h->nnz;
    return time_variant_quick(h, SPMV_FMT_CSR, L, ts.x, ts.y);
  }
  int64_t R = (int64_t)((double)h->rows * (double)kPredictSampleNnz / (double)h->nnz);
  R = std::max<int64_t>(1, std::min(R, h->rows));
  int64_t nnzR = 0;
  if (h->rp64) {
    d2h_sync(&nnzR, static_cast<const int64_t*>(h->row_ptr) + R, sizeof(int64_t), h->stream);
  } else {
    int32_t v = 0;
    d2h_sync(&v, static_cast<const int32_t*>(h->row_ptr) + R, sizeof(int32_t), h->stream);
    nnzR = v;
  }
  if (nnzR <= 0) {
    *sample_nnz = h->nnz;
    return time_variant_quick(h, SPMV_FMT_CSR, L, ts.x, ts.y);
  }
  const int64_t rows0 = h->rows;
  h->rows = R;  // CSR-vector reads rows [0, R) only
  double t;
  try {
    t = time_variant_quick(h, SPMV_FMT_CSR, L, ts.x, ts.y);
  } catch (...) {
    h->rows = rows0;
    throw;
  }
  h->rows = rows0;
  *sample_nnz = nnzR;
  return t * (double)h->nnz / (double)nnzR;
}

static void tune_predict(spmv_matrix* h, int64_t iters, TuneScratch& ts, spmv_tune_report_t* rep,
                         bool decide_only) {
  if (!h->have_features) compute_features(h);
  const spmv_features_t& f = h->feat;
  double x[kSelectorFeatures];
  selector_features(f, h->vbytes, x);
  const int cls = selector_class(x);
  int fmt;
  spmv_format_params_t q;
  selector_class_format(cls, &fmt, &q);
  const int orig_alg = h->csr_alg;
  h->csr_alg = SPMV_CSR_VECTOR;
  int64_t sample_nnz = 0;
  double t_csr;
  try {
    t_csr = predict_t_csr(h, ts, &sample_nnz);
  } catch (...) {
    h->csr_alg = orig_alg;
    throw;
  }
  h->csr_alg = orig_alg;
  const double ratio = selector_speed_ratio(cls, x);
  const double t_pred = t_csr * ratio;
  const double c_pred = (fmt == SPMV_FMT_CSR) ? 0.0 : selector_c_latency(cls, f);
  const double gain = (double)iters * (t_csr - t_pred);
  const double overhead = h->f_latency + c_pred;
  bool convert = cls != 0 && gain > overhead;
  std::ostringstream os;
  os.precision(9);
  os << "{\"kind\":\"format_predict\",\"x\":[";
  for (int i = 0; i < kSelectorFeatures; ++i) os << x[i] << (i + 1 < kSelectorFeatures ? "," : "");
  os << "],\"class\":\"" << selector_class_name(cls) << "\",\"speed_ratio\":" << ratio << ",\"t_csr_s\":" << t_csr
     << ",\"t_csr_sample_nnz\":" << sample_nnz << ",\"t_pred_s\":" << t_pred << ",\"gate\":{\"expected_iterations\":" << iters << ",\"gain_s\":" << gain
     << ",\"f_latency_s\":" << h->f_latency << ",\"c_latency_pred_s\":" << c_pred << ",\"overhead\":" << overhead
     << ",\"convert\":" << (convert ? "true" : "false") << "}";
  if (convert && decide_only) {
    // SPMV_TUNE_DECIDE_ONLY: report the verdict, leave the handle as it is
    os << ",\"decide_only\":true,\"chosen\":\"" << selector_class_name(cls) << "\"}";
    log_append(h, os.str());
    if (rep) {
      rep->format = fmt;
      rep->params = q;
      rep->t_csr_s = t_csr;
      rep->t_best_s = t_pred;
      rep->f_latency_s = h->f_latency;
      rep->c_latency_s = c_pred;
      rep->expected_iterations = iters;
      rep->converted = 1;
      rep->n_candidates = 1;
    }
    return;
  }
  if (convert) {
    try {
      switch (fmt) {
        case SPMV_FMT_CSR: h->csr_alg = q.csr_alg; break;
        case SPMV_FMT_ELL: if (!built(h, fmt)) build_ell(h, -1); break;
        case SPMV_FMT_SELL: if (!built(h, fmt)) build_sell(h, h->dtype == SPMV_R64F ? 64 : 128, 1, -1); break;
        case SPMV_FMT_HYB: if (!built(h, fmt)) build_hyb(h, -1); break;
        case SPMV_FMT_COO: if (!built(h, fmt)) build_coo(h); break;
        case SPMV_FMT_BELL:
          if (built(h, fmt) && h->bell_b != q.bell_b) free_format(h, fmt);
          if (!built(h, fmt)) build_bell(h, q.bell_b);
          break;
      }
      h->active = fmt;
    } catch (const SpmvError& e) {
      cudaGetLastError();
      convert = false;
      os << ",\"build_failed\":\"" << e.msg << "\"";
    }
  }
  if (!convert && !decide_only) {
    h->active = SPMV_FMT_CSR;
    h->csr_alg = SPMV_CSR_VECTOR;
  }
  os << ",\"chosen\":\"" << (convert ? selector_class_name(cls) : "CSR-vector") << "\"}";
  log_append(h, os.str());
  if (rep) {
    rep->format = convert || !decide_only ? h->active : SPMV_FMT_CSR;
    rep->t_csr_s = t_csr;
    rep->t_best_s = convert ? t_pred : t_csr;
    rep->f_latency_s = h->f_latency;
    rep->c_latency_s = c_pred;
    rep->expected_iterations = iters;
    rep->converted = convert ? 1 : 0;
    rep->n_candidates = 1;
    rep->params.csr_alg = h->csr_alg;
    rep->params.csr_T = h->csr_T;
    rep->params.sell_C = (int32_t)h->sell_C;
    rep->params.sell_sigma = (int32_t)h->sell_sigma;
    rep->params.hyb_K = h->hyb_K;
    rep->params.bell_b = (int32_t)h->bell_b;
    rep->params.index16 = index_encoding(h, h->active);
  }
}

// ---------------------------------------------------------------- CUDA-graph power loop
namespace {
struct PowerGraph {
  cudaGraphExec_t exec = nullptr;
  uint64_t gen = 0;
  const void* x0 = nullptr;
  void* b0 = nullptr;
  void* b1 = nullptr;
  int64_t n = 0, steps = 0;
  double* sums = nullptr;
  int final_buf = 0;
  uint64_t kernels = 0;  // kernel nodes (library launches) per replay
};
}  // namespace

void destroy_power_graph(spmv_matrix* h) {
  auto* g = static_cast<PowerGraph*>(h->power_graph);
  if (!g) return;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  delete g;
  h->power_graph = nullptr;
}

static void destroy_handle(spmv_matrix* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  destroy_power_graph(h);
  for (int f = 0; f < SPMV_NUM_FORMATS; ++f) free_format(h, f);
  dfree(h->seg_scratch, h->stream);
  dfree(h->fix_scratch, h->stream);
  dfree(h->merge_coords, h->stream);
  dfree(h->csr_empty, h->stream);
  dfree(h->rm_bits, h->stream);
  dfree(h->rm_rows, h->stream);
  dfree(h->rm_ord0, h->stream);
  dfree(h->dict8_map, h->stream);
  dfree(h->dict8_tab, h->stream);
  dfree(h->pi_partials, h->stream);
  dfree(h->pi_counter, h->stream);  // stream-ordered frees: no host synchronisation
  for (auto& evs : h->lat_ev)
    for (auto& ev : evs)
      if (ev) cudaEventDestroy(ev);
  delete h;
}

struct DeviceGuard {
  explicit DeviceGuard(int dev) {
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != dev) CK(cudaSetDevice(dev));
  }
};

}  // namespace spmv

namespace spmv {
__global__ void k_remap(int32_t* col, int64_t nnz, const int64_t* bounds, int world, int64_t chunk) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride) {
    const int64_t c = col[i];
    int lo = 0, hi = world - 1;  // owner: last r with bounds[r] <= c
    while (lo < hi) {
      int mid = (lo + hi + 1) / 2;
      if (bounds[mid] <= c) lo = mid;
      else hi = mid - 1;
    }
    col[i] = (int32_t)(lo * chunk + (c - bounds[lo]));
  }
}
}  // namespace spmv

using namespace spmv;

#define API_TRY try {
#define API_CATCH(h)                                          \
  }                                                           \
  catch (const SpmvError& e) {                                \
    g_err = e.msg;                                            \
    if (h) (h)->last_error = e.msg;                           \
    return e.status;                                          \
  }                                                           \
  catch (const std::bad_alloc&) {                             \
    g_err = "host allocation failed";                         \
    return SPMV_ERR_OUT_OF_MEMORY;                            \
  }                                                           \
  return SPMV_OK;

static spmv_matrix* const kNoHandle = nullptr;

extern "C" {

spmv_status_t spmv_create(spmv_handle_t* out, int64_t rows, int64_t cols, int64_t nnz, const int32_t* row_idx,
                          const int32_t* col_idx, const void* vals, spmv_dtype_t dtype, spmv_mem_t where,
                          int device, void* cuda_stream) {
  const NvtxRange nvtx_range("spmv_create");
  if (!out) return SPMV_ERR_INVALID_ARG;
  *out = nullptr;
  if (rows < 0 || cols < 0 || nnz < 0) return SPMV_ERR_INVALID_ARG;
  if (dtype != SPMV_R32F && dtype != SPMV_R64F) return SPMV_ERR_INVALID_ARG;
  if (where != SPMV_MEM_HOST && where != SPMV_MEM_DEVICE) return SPMV_ERR_INVALID_ARG;
  if (nnz > 0 && (!row_idx || !col_idx || !vals)) return SPMV_ERR_INVALID_ARG;
  if (rows > INT32_MAX || cols > INT32_MAX) return SPMV_ERR_UNSUPPORTED;
  if (nnz > 0 && (rows == 0 || cols == 0)) return SPMV_ERR_INDEX_OUT_OF_RANGE;
  spmv_matrix* h = nullptr;
  API_TRY
  DeviceGuard g(device);
  h = new spmv_matrix();
  h->device = device;
  h->stream = static_cast<cudaStream_t>(cuda_stream);
  h->dtype = dtype;
  h->vbytes = dtype == SPMV_R64F ? 8 : 4;
  h->rows = rows;
  h->cols = cols;
  h->nnz = nnz;
  for (auto& L : h->launch) L = spmv_launch_t{0, 0, -1, 0};
  try {
    ingest(h, row_idx, col_idx, vals, where);
  } catch (...) {
    destroy_handle(h);
    h = nullptr;
    throw;
  }
  *out = h;
  API_CATCH(kNoHandle)
}

spmv_status_t spmv_convert(spmv_handle_t h, spmv_format_t fmt, const spmv_format_params_t* p) {
  const NvtxRange nvtx_range("spmv_convert");
  if (!h) return SPMV_ERR_INVALID_ARG;
  if (fmt < 0 || fmt >= SPMV_NUM_FORMATS) return SPMV_ERR_INVALID_ARG;
  API_TRY
  DeviceGuard g(h->device);
  need_csr(h, "spmv_convert");
  spmv_format_params_t q{};
  q.hyb_K = -1;
  if (p) q = *p;
  switch (fmt) {
    case SPMV_FMT_CSR:
      if (q.csr_alg < 0 || q.csr_alg > SPMV_CSR_STREAM) fail(SPMV_ERR_INVALID_ARG, "bad csr_alg");
      if (q.csr_T != 0 && (q.csr_T < 1 || q.csr_T > 32 || (q.csr_T & (q.csr_T - 1))))
        fail(SPMV_ERR_INVALID_ARG, "csr_T must be a power of two in [1, 32]");
      if (h->csr_alg != q.csr_alg) h->launch[SPMV_FMT_CSR] = spmv_launch_t{0, 0, -1, 0};  // other kernel
      h->csr_alg = q.csr_alg;
      h->csr_T = q.csr_T;
      h->launch[SPMV_FMT_CSR].knob = 0;
      break;
    case SPMV_FMT_COO:
      if (!h->coo_built) build_coo(h);
      break;
    case SPMV_FMT_ELL: {
      if (q.index16 < -1 || q.index16 > 2) fail(SPMV_ERR_INVALID_ARG, "index16 must be -1, 0, 1 or 2");
      if (!h->have_features) compute_features(h);
      const int want = q.index16 == -1 ? resolve_index_auto(h) : q.index16;
      if (h->ell_built && want == index_encoding(h, SPMV_FMT_ELL)) break;
      if (h->ell_built) free_format(h, SPMV_FMT_ELL);
      build_ell(h, want);
      break;
    }
    case SPMV_FMT_SELL: {
      int64_t C = q.sell_C ? q.sell_C : (h->dtype == SPMV_R64F ? 64 : 128);
      int64_t sigma = q.sell_sigma ? q.sell_sigma : 1;
      if (C != 32 && C != 64 && C != 128 && C != 256) fail(SPMV_ERR_UNSUPPORTED, "SELL C must be 32, 64, 128 or 256");
      if (sigma < 1 || (sigma != 1 && sigma % C != 0)) fail(SPMV_ERR_INVALID_ARG, "SELL sigma must be 1 or a multiple of C");
      if (q.index16 < -1 || q.index16 > 2) fail(SPMV_ERR_INVALID_ARG, "index16 must be -1, 0, 1 or 2");
      if (!h->have_features) compute_features(h);
      const int want = q.index16 == -1 ? resolve_index_auto(h) : q.index16;
      if (!h->sell_built || h->sell_C != C || h->sell_sigma != sigma || want != index_encoding(h, SPMV_FMT_SELL)) {
        if (h->sell_built) free_format(h, SPMV_FMT_SELL);
        build_sell(h, C, sigma, want);
      }
      break;
    }
    case SPMV_FMT_BELL: {
      const int64_t b = q.bell_b ? q.bell_b : 2;
      if (b < 2 || b > 4) fail(SPMV_ERR_UNSUPPORTED, "BELL block dimension must be 2, 3 or 4");
      if (!h->bell_built || h->bell_b != b) {
        if (h->bell_built) free_format(h, SPMV_FMT_BELL);
        build_bell(h, b);
      }
      break;
    }
    case SPMV_FMT_HYB: {
      int64_t K = q.hyb_K;
      if (K < -1) fail(SPMV_ERR_INVALID_ARG, "hyb_K must be >= -1");
      if (!h->have_features) compute_features(h);
      int64_t want = K < 0 ? h->hyb_auto_K : K;
      if (!h->hyb_built || h->hyb_K != want) {
        if (h->hyb_built) free_format(h, SPMV_FMT_HYB);
        build_hyb(h, want);
      }
      break;
    }
  }
  h->active = fmt;  // builds are stream-ordered: no synchronisation here
  ++h->gen;
  API_CATCH(h)
}

spmv_status_t spmv_set_format(spmv_handle_t h, spmv_format_t fmt) {
  if (!h || fmt < 0 || fmt >= SPMV_NUM_FORMATS) return SPMV_ERR_INVALID_ARG;
  if (!built(h, fmt)) return SPMV_ERR_NOT_CONVERTED;
  h->active = fmt;
  ++h->gen;
  return SPMV_OK;
}

spmv_status_t spmv_get_format(spmv_handle_t h, spmv_format_t* fmt) {
  if (!h || !fmt) return SPMV_ERR_INVALID_ARG;
  *fmt = (spmv_format_t)h->active;
  return SPMV_OK;
}

spmv_status_t spmv_features(spmv_handle_t h, spmv_features_t* out) {
  const NvtxRange nvtx_range("spmv_features");
  if (!h || !out) return SPMV_ERR_INVALID_ARG;
  API_TRY
  DeviceGuard g(h->device);
  if (!h->have_features) need_csr(h, "spmv_features");
  if (!h->csr_released) compute_features(h);
  *out = h->feat;
  API_CATCH(h)
}

spmv_status_t spmv_release_csr(spmv_handle_t h) {
  if (!h) return SPMV_ERR_INVALID_ARG;
  if (h->active == SPMV_FMT_CSR || h->active == SPMV_FMT_COO) return SPMV_ERR_INVALID_ARG;
  if (h->csr_released) return SPMV_OK;
  API_TRY
  DeviceGuard g(h->device);
  free_format(h, SPMV_FMT_COO);  // shares col/val with CSR
  for (void** q : {&h->row_ptr, (void**)&h->col, &h->val, (void**)&h->merge_coords, (void**)&h->csr_empty,
                   (void**)&h->rm_bits, (void**)&h->rm_rows, (void**)&h->rm_ord0}) {
    dfree(*q, h->stream);
    *q = nullptr;
  }
  h->merge_coords_n = 0;
  h->merge_coords_ipt = 0;
  h->csr_n_empty = -1;
  h->rm_nchunks = -1;
  h->csr_released = true;
  ++h->gen;
  API_CATCH(h)
}

static spmv_status_t run_common(spmv_handle_t h, int fmt, double alpha, const void* x, double beta, void* y) {
  if (!h) return SPMV_ERR_INVALID_ARG;
  if (fmt < 0 || fmt >= SPMV_NUM_FORMATS) return SPMV_ERR_INVALID_ARG;
  if ((!x && h->cols > 0 && alpha != 0.0) || (!y && h->rows > 0)) return SPMV_ERR_INVALID_ARG;
  if (x && x == y) return SPMV_ERR_INVALID_ARG;
  if (!built(h, fmt)) return SPMV_ERR_NOT_CONVERTED;
  if (h->rows == 0) return SPMV_OK;
  API_TRY
  DeviceGuard g(h->device);
  Epilogue e;
  e.alpha = alpha;
  e.beta = beta;
  dispatch(h, fmt, e, x, y, h->launch[fmt]);
  API_CATCH(h)
}

spmv_status_t spmv_run(spmv_handle_t h, double alpha, const void* x, double beta, void* y) {
  if (!h) return SPMV_ERR_INVALID_ARG;
  return run_common(h, h->active, alpha, x, beta, y);
}

spmv_status_t spmv_run_format(spmv_handle_t h, spmv_format_t fmt, double alpha, const void* x, double beta, void* y) {
  return run_common(h, fmt, alpha, x, beta, y);
}

spmv_status_t spmv_set_launch(spmv_handle_t h, spmv_format_t fmt, const spmv_launch_t* v) {
  if (!h || !v || fmt < 0 || fmt >= SPMV_NUM_FORMATS) return SPMV_ERR_INVALID_ARG;
  API_TRY
  spmv_launch_t L = *v;
  if (L.block) block_index(L.block);
  if (L.maxreg) reg_index(L.maxreg);
  if (L.carveout_pct > 100) fail(SPMV_ERR_INVALID_ARG, "carveout must be -1 or 0..100");
  h->launch[fmt] = L;
  ++h->gen;
  API_CATCH(h)
}

spmv_status_t spmv_get_launch(spmv_handle_t h, spmv_format_t fmt, spmv_launch_t* v) {
  if (!h || !v || fmt < 0 || fmt >= SPMV_NUM_FORMATS) return SPMV_ERR_INVALID_ARG;
  API_TRY
  *v = resolve_launch(h, fmt, h->launch[fmt]);
  API_CATCH(h)
}

spmv_status_t spmv_tune(spmv_handle_t h, uint32_t flags, int64_t expected_iterations, spmv_tune_report_t* out) {
  const NvtxRange nvtx_range("spmv_tune");
  const uint32_t what = flags & SPMV_TUNE_ALL;
  const int obj = (int)((flags & SPMV_TUNE_OBJ_MASK) >> 4);
  if (!h || (flags & ~(SPMV_TUNE_ALL | SPMV_TUNE_OBJ_MASK | SPMV_TUNE_PREDICT | SPMV_TUNE_DECIDE_ONLY)) ||
      what == 0 || expected_iterations < 0)
    return SPMV_ERR_INVALID_ARG;
  const bool predict = (flags & SPMV_TUNE_PREDICT) != 0;
  const bool decide_only = (flags & SPMV_TUNE_DECIDE_ONLY) != 0;
  if (predict && !(what & SPMV_TUNE_FORMAT)) return SPMV_ERR_INVALID_ARG;
  if (decide_only && (!predict || (what & SPMV_TUNE_LAUNCH))) return SPMV_ERR_INVALID_ARG;
  if (predict && obj != 0) return SPMV_ERR_UNSUPPORTED;
  if (h->rows == 0 || h->nnz == 0) return SPMV_ERR_INVALID_ARG;
  API_TRY
  DeviceGuard g(h->device);
  need_csr(h, "spmv_tune");
  ++h->gen;  // format and launch choices may change
  if (obj != 0 && !nvml_available()) fail(SPMV_ERR_NVML, "energy/power objectives need libnvidia-ml");
  spmv_tune_report_t rep{};
  rep.format = h->active;
  rep.expected_iterations = expected_iterations;
  rep.objective = obj;
  rep.energy_j = rep.power_w = rep.mflops_per_w = std::nan("");
  TuneScratch ts(h);
  if (what & SPMV_TUNE_FORMAT) {
    if (predict) tune_predict(h, expected_iterations, ts, &rep, decide_only);
    else tune_format(h, expected_iterations, ts, &rep, obj, (what & SPMV_TUNE_LAUNCH) != 0);
  }
  // after a measured format selection with LAUNCH the chosen launch is already tuned
  if ((what & SPMV_TUNE_LAUNCH) && (predict || !(what & SPMV_TUNE_FORMAT))) tune_launch(h, h->active, ts, &rep, obj);
  if (!decide_only) {
    rep.format = h->active;
    rep.launch = resolve_launch(h, h->active, h->launch[h->active]);
  }
  CK(cudaStreamSynchronize(h->stream));
  if (out) *out = rep;
  API_CATCH(h)
}

spmv_status_t spmv_predict(const spmv_features_t* f, spmv_dtype_t dtype, spmv_prediction_t* out) {
  if (!f || !out || (dtype != SPMV_R32F && dtype != SPMV_R64F) || f->n_rows < 0 || f->nnz < 0)
    return SPMV_ERR_INVALID_ARG;
  double x[kSelectorFeatures];
  selector_features(*f, dtype == SPMV_R64F ? 8 : 4, x);
  out->cls = selector_class(x);
  int fmt;
  selector_class_format(out->cls, &fmt, &out->params);
  out->format = fmt;
  out->speed_ratio = selector_speed_ratio(out->cls, x);
  out->c_latency_s = fmt == SPMV_FMT_CSR ? 0.0 : selector_c_latency(out->cls, *f);
  out->f_latency_s = selector_f_latency(*f);
  return SPMV_OK;
}

spmv_status_t spmv_power_step(spmv_handle_t h, const void* x, void* y, const double* sums_prev, double* sums_out,
                              int64_t row_offset) {
  if (!h || !x || !y || !sums_prev || !sums_out || x == y || row_offset < 0) return SPMV_ERR_INVALID_ARG;
  if (!built(h, h->active)) return SPMV_ERR_NOT_CONVERTED;
  API_TRY
  DeviceGuard g(h->device);
  power_step_internal(h, x, y, sums_prev, sums_out, row_offset);
  API_CATCH(h)
}

spmv_status_t spmv_norm2(spmv_handle_t h, const void* x, int64_t n, double* sums_out) {
  if (!h || !sums_out || n < 0 || (n > 0 && !x)) return SPMV_ERR_INVALID_ARG;
  API_TRY
  DeviceGuard g(h->device);
  spmv_norm2_internal(h, x, n, sums_out);
  API_CATCH(h)
}

spmv_status_t spmv_power_iterate(spmv_handle_t h, const void* x0, void* buf0, void* buf1, int64_t n_full,
                                 int64_t steps, double* sums, void* comm, int64_t chunk, void* chunk_buf,
                                 float* kernel_ms, float* loop_ms, int* final_buf) {
  const NvtxRange nvtx_range("spmv_power_iterate");
  if (!h || !x0 || !buf0 || !buf1 || !sums || steps < 0 || n_full < h->rows || buf0 == buf1) return SPMV_ERR_INVALID_ARG;
  if (comm && (!chunk_buf || chunk < h->rows)) return SPMV_ERR_INVALID_ARG;
  if (!built(h, h->active)) return SPMV_ERR_NOT_CONVERTED;
  API_TRY
  DeviceGuard g(h->device);
  power_iterate(h, x0, buf0, buf1, n_full, steps, sums, comm, chunk, chunk_buf, kernel_ms, loop_ms, final_buf);
  API_CATCH(h)
}

spmv_status_t spmv_power_iterate_graph(spmv_handle_t h, const void* x0, void* buf0, void* buf1, int64_t n_full,
                                       int64_t steps, double* sums, int* final_buf) {
  const NvtxRange nvtx_range("spmv_power_iterate_graph");
  if (!h || !x0 || !buf0 || !buf1 || !sums || steps < 0 || n_full < h->rows || buf0 == buf1) return SPMV_ERR_INVALID_ARG;
  if (!built(h, h->active)) return SPMV_ERR_NOT_CONVERTED;
  API_TRY
  DeviceGuard g(h->device);
  auto* pg = static_cast<PowerGraph*>(h->power_graph);
  if (pg && pg->exec && pg->gen == h->gen && pg->x0 == x0 && pg->b0 == buf0 && pg->b1 == buf1 && pg->n == n_full &&
      pg->steps == steps && pg->sums == sums) {
    CK(cudaGraphLaunch(pg->exec, h->stream));
    g_launches.fetch_add(pg->kernels, std::memory_order_relaxed);
    if (final_buf) *final_buf = pg->final_buf;
    return SPMV_OK;
  }
  destroy_power_graph(h);
  // first call with these arguments: run the loop eagerly (its result is this
  // call's result; lazily built scratch, partitions and kernel attributes are
  // set up outside the capture), then capture the same loop for the replays
  int fb = 0;
  power_iterate(h, x0, buf0, buf1, n_full, steps, sums, nullptr, 0, nullptr, nullptr, nullptr, &fb);
  cudaStream_t cs = nullptr;  // capture on a private stream (the legacy stream cannot be captured)
  CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  cudaStream_t saved = h->stream;
  h->stream = cs;
  const uint64_t l0 = g_launches.load();
  cudaGraph_t graph = nullptr;
  try {
    CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    int fb2 = 0;
    try {
      power_iterate(h, x0, buf0, buf1, n_full, steps, sums, nullptr, 0, nullptr, nullptr, nullptr, &fb2);
    } catch (...) {
      cudaStreamEndCapture(cs, &graph);
      throw;
    }
    CK(cudaStreamEndCapture(cs, &graph));
  } catch (...) {
    if (graph) cudaGraphDestroy(graph);
    h->stream = saved;
    g_launches.fetch_sub(g_launches.load() - l0);
    cudaStreamDestroy(cs);
    throw;
  }
  h->stream = saved;
  const uint64_t nk = g_launches.load() - l0;
  g_launches.fetch_sub(nk);  // captured, not launched: counted at each replay
  cudaGraphExec_t exec = nullptr;
  cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  cudaStreamDestroy(cs);
  cuda_check(e, "cudaGraphInstantiate");
  pg = new PowerGraph{exec, h->gen, x0, buf0, buf1, n_full, steps, sums, fb, nk};
  h->power_graph = pg;
  if (final_buf) *final_buf = fb;
  API_CATCH(h)
}

spmv_status_t spmv_dist_plan_create(spmv_dist_plan_t* out, spmv_handle_t h, void* comm, int64_t chunk,
                                    uint32_t flags) {
  const NvtxRange nvtx_range("spmv_dist_plan_create");
  if (!out) return SPMV_ERR_INVALID_ARG;
  *out = nullptr;
  if (!h || (comm && chunk < 1) || (flags & ~(SPMV_PLAN_OVERLAP | SPMV_PLAN_HALO))) return SPMV_ERR_INVALID_ARG;
  if (!built(h, h->active)) return SPMV_ERR_NOT_CONVERTED;
  API_TRY
  DeviceGuard g(h->device);
  need_csr(h, "spmv_dist_plan_create");
  *out = plan_create(h, comm, chunk, flags);
  API_CATCH(h)
}

spmv_status_t spmv_dist_plan_info(spmv_dist_plan_t plan, spmv_dist_plan_info_t* out) {
  if (!plan || !out) return SPMV_ERR_INVALID_ARG;
  plan_info(plan, out);
  return SPMV_OK;
}

spmv_status_t spmv_dist_plan_part(spmv_dist_plan_t plan, int part, spmv_handle_t* out) {
  if (!plan || !out || part < 0 || part > 2) return SPMV_ERR_INVALID_ARG;
  *out = plan_part(plan, part);
  return SPMV_OK;
}

spmv_status_t spmv_dist_plan_iterate(spmv_dist_plan_t plan, const void* x0, void* buf0, void* buf1, int64_t steps,
                                     double* sums, float* loop_ms, float* interior_ms, int* final_buf) {
  const NvtxRange nvtx_range("spmv_dist_plan_iterate");
  if (!plan || !x0 || !buf0 || !buf1 || !sums || steps < 0 || buf0 == buf1) return SPMV_ERR_INVALID_ARG;
  API_TRY
  DeviceGuard g(plan_device(plan));
  plan_iterate(plan, x0, buf0, buf1, steps, sums, loop_ms, interior_ms, final_buf);
  API_CATCH(kNoHandle)
}

spmv_status_t spmv_dist_plan_destroy(spmv_dist_plan_t plan) {
  API_TRY
  plan_destroy(plan);
  API_CATCH(kNoHandle)
}

spmv_status_t spmv_dist_local_group(int world, const int* devices, void** comms) {
  if (world < 1 || !devices || !comms) return SPMV_ERR_INVALID_ARG;
  for (int r = 0; r < world; ++r) comms[r] = nullptr;
  API_TRY
  std::vector<CommBase*> v = local_group(world, devices);
  for (int r = 0; r < world; ++r) comms[r] = v[r];
  API_CATCH(kNoHandle)
}

spmv_status_t spmv_create_row_slice(spmv_handle_t* out, spmv_handle_t h, int64_t row_begin, int64_t row_end) {
  const NvtxRange nvtx_range("spmv_create_row_slice");
  if (!out) return SPMV_ERR_INVALID_ARG;
  *out = nullptr;
  if (!h || row_begin < 0 || row_end < row_begin || row_end > h->rows) return SPMV_ERR_INVALID_ARG;
  API_TRY
  DeviceGuard g(h->device);
  need_csr(h, "spmv_create_row_slice");
  *out = make_row_slice(h, row_begin, row_end);
  API_CATCH(h)
}

spmv_status_t spmv_dist_unique_id(uint8_t out[128]) {
  if (!out) return SPMV_ERR_INVALID_ARG;
  API_TRY
  dist_unique_id(out);
  API_CATCH(kNoHandle)
}

spmv_status_t spmv_dist_init(void** comm, const uint8_t unique_id[128], int rank, int world, int device) {
  if (!comm || !unique_id || world < 1 || rank < 0 || rank >= world) return SPMV_ERR_INVALID_ARG;
  *comm = nullptr;
  API_TRY
  *comm = dist_init(unique_id, rank, world, device);
  API_CATCH(kNoHandle)
}

spmv_status_t spmv_dist_destroy(void* comm) {
  API_TRY
  dist_destroy(comm);
  API_CATCH(kNoHandle)
}

spmv_status_t spmv_format_info(spmv_handle_t h, spmv_format_t fmt, spmv_format_info_t* o) {
  if (!h || !o || fmt < 0 || fmt >= SPMV_NUM_FORMATS) return SPMV_ERR_INVALID_ARG;
  std::memset(o, 0, sizeof(*o));
  o->present = built(h, fmt) ? 1 : 0;
  o->row_ptr_is64 = h->rp64 ? 1 : 0;
  switch (fmt) {
    case SPMV_FMT_ELL: o->K = h->ell_K; o->n_pad = h->ell_npad; o->slots = h->ell_K * h->ell_npad; break;
    case SPMV_FMT_SELL:
      o->C = h->sell_C; o->sigma = h->sell_sigma; o->n_slices = h->sell_ns;
      try {
        o->slots = h->sell_built ? sell_slots(h) : 0;
      } catch (const SpmvError& e) {
        h->last_error = e.msg;
        return e.status;
      }
      break;
    case SPMV_FMT_HYB:
      o->K = h->hyb_K; o->n_pad = h->hyb_npad; o->slots = h->hyb_K * h->hyb_npad; o->tail_nnz = h->hyb_tail;
      break;
    case SPMV_FMT_COO: o->n_empty_rows = h->coo_n_empty; break;
    case SPMV_FMT_BELL:
      o->K = h->bell_kb; o->n_pad = h->bell_nbr_pad; o->block = h->bell_b;
      o->slots = h->bell_kb * h->bell_nbr * h->bell_b * h->bell_b;
      break;
    default: break;
  }
  o->stored_bytes = o->present ? format_stored_bytes(h, fmt) : 0;
  if (o->present && (fmt == SPMV_FMT_ELL || fmt == SPMV_FMT_SELL || fmt == SPMV_FMT_HYB || fmt == SPMV_FMT_BELL))
    o->index_bytes = index_encoding(h, fmt) == 2 ? 1 : (index_encoding(h, fmt) == 1 ? 2 : 4);
  return SPMV_OK;
}

spmv_status_t spmv_copy_array(spmv_handle_t h, spmv_array_t which, void* dst, int64_t dst_bytes, spmv_mem_t where) {
  if (!h || (!dst && dst_bytes > 0) || (where != SPMV_MEM_HOST && where != SPMV_MEM_DEVICE)) return SPMV_ERR_INVALID_ARG;
  const void* src = nullptr;
  int64_t bytes = 0;
  const int64_t vb = h->vbytes;
  bool need = true;
  switch (which) {
    case SPMV_ARR_CSR_ROW_PTR: need = !h->csr_released; src = h->row_ptr; bytes = (h->rows + 1) * (h->rp64 ? 8 : 4); break;
    case SPMV_ARR_CSR_COL: need = !h->csr_released; src = h->col; bytes = h->nnz * 4; break;
    case SPMV_ARR_CSR_VAL: need = !h->csr_released; src = h->val; bytes = h->nnz * vb; break;
    case SPMV_ARR_COO_ROW: need = h->coo_built; src = h->coo_row; bytes = h->nnz * 4; break;
    case SPMV_ARR_COO_EMPTY_ROWS: need = h->coo_built; src = h->coo_empty; bytes = h->coo_n_empty * 4; break;
    case SPMV_ARR_ELL_COL: need = h->ell_built && h->ell_col; src = h->ell_col; bytes = h->ell_K * h->ell_npad * 4; break;
    case SPMV_ARR_ELL_COL16: need = h->ell_built && h->ell_col16; src = h->ell_col16; bytes = h->ell_K * h->ell_npad * 2; break;
    case SPMV_ARR_SELL_COL16:
      need = h->sell_built && h->sell_col16;
      src = h->sell_col16;
      bytes = (need ? sell_slots(h) : 0) * 2;
      break;
    case SPMV_ARR_ELL_COL8: need = h->ell_built && h->ell_col8; src = h->ell_col8; bytes = h->ell_K * h->ell_npad; break;
    case SPMV_ARR_SELL_COL8:
      need = h->sell_built && h->sell_col8;
      src = h->sell_col8;
      bytes = need ? sell_slots(h) : 0;
      break;
    case SPMV_ARR_DICT8_TAB: need = h->dict8_tab != nullptr; src = h->dict8_tab; bytes = 256 * 4; break;
    case SPMV_ARR_ELL_VAL: need = h->ell_built; src = h->ell_val; bytes = h->ell_K * h->ell_npad * vb; break;
    case SPMV_ARR_SELL_PERM: need = h->sell_built; src = h->sell_perm; bytes = h->rows * 4; break;
    case SPMV_ARR_SELL_SLICE_PTR: need = h->sell_built; src = h->sell_sp; bytes = (h->sell_ns + 1) * 8; break;
    case SPMV_ARR_SELL_COL: need = h->sell_built && h->sell_col; src = h->sell_col; bytes = (need ? sell_slots(h) : 0) * 4; break;
    case SPMV_ARR_SELL_VAL: need = h->sell_built; src = h->sell_val; bytes = (h->sell_built ? sell_slots(h) : 0) * vb; break;
    case SPMV_ARR_HYB_ELL_COL: need = h->hyb_built; src = h->hyb_ecol; bytes = h->hyb_K * h->hyb_npad * 4; break;
    case SPMV_ARR_HYB_ELL_VAL: need = h->hyb_built; src = h->hyb_eval; bytes = h->hyb_K * h->hyb_npad * vb; break;
    case SPMV_ARR_HYB_TAIL_ROW: need = h->hyb_built; src = h->hyb_trow; bytes = h->hyb_tail * 4; break;
    case SPMV_ARR_HYB_TAIL_COL: need = h->hyb_built; src = h->hyb_tcol; bytes = h->hyb_tail * 4; break;
    case SPMV_ARR_HYB_TAIL_VAL: need = h->hyb_built; src = h->hyb_tval; bytes = h->hyb_tail * vb; break;
    case SPMV_ARR_BELL_COL: need = h->bell_built; src = h->bell_col; bytes = h->bell_kb * h->bell_nbr_pad * 4; break;
    case SPMV_ARR_BELL_VAL:
      need = h->bell_built;
      src = h->bell_val;
      bytes = h->bell_kb * h->bell_b * h->bell_b * h->bell_nbr_pad * vb;
      break;
    default: return SPMV_ERR_INVALID_ARG;
  }
  if (!need) return SPMV_ERR_NOT_CONVERTED;
  if (dst_bytes < bytes) return SPMV_ERR_INVALID_ARG;
  API_TRY
  DeviceGuard g(h->device);
  if (which == SPMV_ARR_SELL_PERM && !h->sell_perm) {
    // sigma == 1: identity permutation
    std::vector<int32_t> id((size_t)h->rows);
    for (int64_t i = 0; i < h->rows; ++i) id[(size_t)i] = (int32_t)i;
    CK(cudaMemcpyAsync(dst, id.data(), bytes, where == SPMV_MEM_HOST ? cudaMemcpyHostToHost : cudaMemcpyHostToDevice,
                       h->stream));
  } else if (bytes > 0) {
    CK(cudaMemcpyAsync(dst, src, bytes, where == SPMV_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                       h->stream));
  }
  CK(cudaStreamSynchronize(h->stream));
  API_CATCH(h)
}

spmv_status_t spmv_set_stream(spmv_handle_t h, void* s) {
  if (!h) return SPMV_ERR_INVALID_ARG;
  API_TRY
  DeviceGuard g(h->device);
  CK(cudaStreamSynchronize(h->stream));
  h->stream = static_cast<cudaStream_t>(s);
  ++h->gen;
  API_CATCH(h)
}

spmv_status_t spmv_destroy(spmv_handle_t h) {
  const NvtxRange nvtx_range("spmv_destroy");
  if (!h) return SPMV_OK;
  destroy_handle(h);
  return SPMV_OK;
}

const char* spmv_status_string(spmv_status_t s) {
  switch (s) {
    case SPMV_OK: return "SPMV_OK";
    case SPMV_ERR_INVALID_ARG: return "SPMV_ERR_INVALID_ARG";
    case SPMV_ERR_INDEX_OUT_OF_RANGE: return "SPMV_ERR_INDEX_OUT_OF_RANGE";
    case SPMV_ERR_DUPLICATE: return "SPMV_ERR_DUPLICATE";
    case SPMV_ERR_INFEASIBLE: return "SPMV_ERR_INFEASIBLE";
    case SPMV_ERR_OUT_OF_MEMORY: return "SPMV_ERR_OUT_OF_MEMORY";
    case SPMV_ERR_UNSUPPORTED: return "SPMV_ERR_UNSUPPORTED";
    case SPMV_ERR_CUDA: return "SPMV_ERR_CUDA";
    case SPMV_ERR_NOT_CONVERTED: return "SPMV_ERR_NOT_CONVERTED";
    case SPMV_ERR_NCCL: return "SPMV_ERR_NCCL";
    case SPMV_ERR_NVML: return "SPMV_ERR_NVML";
  }
  return "SPMV_ERR_UNKNOWN";
}

const char* spmv_last_error(spmv_handle_t h) { return h ? h->last_error.c_str() : g_err.c_str(); }

size_t spmv_decision_log(spmv_handle_t h, char* buf, size_t len) {
  if (!h) return 0;
  std::string s = "[" + h->log + "]";
  size_t need = s.size() + 1;
  if (buf && len > 0) {
    size_t n = std::min(len - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return need;
}

spmv_status_t spmv_overheads(spmv_handle_t h, double* f_latency_s, double* c_latency_s) {
  if (!h) return SPMV_ERR_INVALID_ARG;
  if (f_latency_s) *f_latency_s = h->f_latency;
  API_TRY
  if (c_latency_s)
    for (int i = 0; i < SPMV_NUM_FORMATS; ++i) c_latency_s[i] = format_latency(h, i);
  API_CATCH(h)
}

uint64_t spmv_launch_count(void) { return g_launches.load(); }

spmv_status_t spmv_trim_pool(int device) {
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return SPMV_ERR_CUDA;
  cudaDeviceSynchronize();
  if (cudaMemPoolTrimTo(pool, 0) != cudaSuccess) return SPMV_ERR_CUDA;
  return SPMV_OK;
}

// ------------------------------------------------------------------ multi-GPU host logic
spmv_status_t spmv_dist_partition(int64_t rows, const int64_t* row_ptr, int world, int64_t* bounds) {
  if (rows < 0 || !row_ptr || world < 1 || !bounds) return SPMV_ERR_INVALID_ARG;
  const int64_t nnz = row_ptr[rows];
  bounds[0] = 0;
  bounds[world] = rows;
  for (int k = 1; k < world; ++k) {
    const unsigned __int128 num = (unsigned __int128)k * (unsigned __int128)(nnz < 0 ? 0 : nnz);
    const int64_t target = (int64_t)((num + (unsigned)world - 1) / (unsigned)world);
    bounds[k] = std::lower_bound(row_ptr, row_ptr + rows + 1, target) - row_ptr;
  }
  return SPMV_OK;
}

spmv_status_t spmv_dist_partition_lengths(int64_t rows, const int64_t* lengths, int world, int64_t* bounds) {
  if (rows < 0 || !lengths || world < 1 || !bounds) return SPMV_ERR_INVALID_ARG;
  try {
    std::vector<int64_t> rp((size_t)rows + 1);
    rp[0] = 0;
    for (int64_t i = 0; i < rows; ++i) rp[(size_t)i + 1] = rp[(size_t)i] + lengths[i];
    return spmv_dist_partition(rows, rp.data(), world, bounds);
  } catch (const std::bad_alloc&) {
    return SPMV_ERR_OUT_OF_MEMORY;
  }
}


spmv_status_t spmv_dist_remap_columns(int32_t* col, int64_t nnz, const int64_t* bounds, int world, spmv_mem_t where,
                                      void* cuda_stream) {
  if ((!col && nnz > 0) || !bounds || world < 1 || nnz < 0) return SPMV_ERR_INVALID_ARG;
  int64_t chunk = 0;
  for (int r = 0; r < world; ++r) chunk = std::max(chunk, bounds[r + 1] - bounds[r]);
  if (chunk * world > INT32_MAX) return SPMV_ERR_UNSUPPORTED;
  if (where == SPMV_MEM_HOST) {
    for (int64_t i = 0; i < nnz; ++i) {
      const int64_t c = col[i];
      const int r = (int)(std::upper_bound(bounds, bounds + world, c) - bounds) - 1;
      col[i] = (int32_t)(r * chunk + (c - bounds[r]));
    }
    return SPMV_OK;
  }
  API_TRY
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  int64_t* db = dalloc_n<int64_t>(world + 1, s);
  CK(cudaMemcpyAsync(db, bounds, (world + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  if (nnz > 0) LAUNCH(k_remap, grid_for(nnz, 256), 256, 0, s, col, nnz, (const int64_t*)db, world, chunk);
  dfree(db, s);
  CK(cudaStreamSynchronize(s));
  API_CATCH(kNoHandle)
}

}  // extern "C"
