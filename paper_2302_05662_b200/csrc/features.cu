// features.cu — device feature extraction, spmv_features (SURVEY.md §8(a)
// row a3): the Table 2 sparsity features (n, nnz,
// Avg_nnz, Var_nnz, ELL_ratio, Median, Mode, Std_nnz) plus max/min/#empty
// and the bandwidth the north star adds. The paper computes them on the CPU
// in NumPy (f_latency); here two kernels do the integer work:
//   k_row_stats: one pass over row_ptr (and the first/last column of each
//     row): Σ L², max, min, #empty, bandwidth, and a row-length histogram
//     (shared-memory privatised bins < 4096, global bins < 65536, a list of
//     the rare longer rows);
//   k_select: one block finds order statistics (median ranks, the HYB
//     threshold rank) and the mode from the histogram.
// The host turns the exact integers into fp64 with the formulas of
// DESIGN.md reading R6 (population variance from 128-bit moments).
#include <algorithm>
#include <climits>
#include <cmath>
#include <vector>

#include "handle.cuh"

namespace spmv {
namespace {

constexpr int kStatThreads = 256;
constexpr int kSmemBins = 4096;
constexpr int kBins = 65536;
constexpr int kChunk = 1024;
constexpr int kChunks = kBins / kChunk;

struct StatPartial {
  unsigned long long s2_lo, s2_hi;
  long long max_len, min_len, n_empty, bw_lo, bw_hi;
};

__device__ __forceinline__ void add_u128(unsigned long long& lo, unsigned long long& hi,
                                         unsigned long long a_lo, unsigned long long a_hi) {
  unsigned long long r = lo + a_lo;
  hi += a_hi + (r < lo ? 1ull : 0ull);
  lo = r;
}

template <class RP>
__global__ void __launch_bounds__(kStatThreads) k_row_stats(const RP* __restrict__ rp,
                                                            const int32_t* __restrict__ col, int64_t rows,
                                                            StatPartial* __restrict__ part,
                                                            unsigned* __restrict__ hist,
                                                            long long* __restrict__ big,
                                                            unsigned long long* __restrict__ nbig) {
  __shared__ unsigned s_hist[kSmemBins];
  __shared__ StatPartial s_w[kStatThreads / 32];
  for (int b = threadIdx.x; b < kSmemBins; b += blockDim.x) s_hist[b] = 0;
  __syncthreads();
  unsigned long long lo = 0, hi = 0;
  long long mx = 0, mn = LLONG_MAX, empty = 0, bl = LLONG_MIN, bu = LLONG_MIN;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += stride) {
    int64_t a = rp[i], b = rp[i + 1];
    long long L = (long long)(b - a);
    unsigned long long L2 = (unsigned long long)L * (unsigned long long)L;  // L < 2^32
    add_u128(lo, hi, L2, 0ull);
    mx = L > mx ? L : mx;
    mn = L < mn ? L : mn;
    if (L == 0) {
      ++empty;
    } else {
      long long f = (long long)i - (long long)col[a];
      long long g = (long long)col[b - 1] - (long long)i;
      bl = f > bl ? f : bl;
      bu = g > bu ? g : bu;
    }
    if (L < kSmemBins) atomicAdd(&s_hist[L], 1u);
    else if (L < kBins) atomicAdd(&hist[L], 1u);
    else big[atomicAdd(nbig, 1ull)] = L;
  }
  // warp reduce
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long olo = __shfl_xor_sync(0xffffffffu, lo, o);
    unsigned long long ohi = __shfl_xor_sync(0xffffffffu, hi, o);
    add_u128(lo, hi, olo, ohi);
    long long v;
    v = __shfl_xor_sync(0xffffffffu, mx, o); mx = v > mx ? v : mx;
    v = __shfl_xor_sync(0xffffffffu, mn, o); mn = v < mn ? v : mn;
    empty += __shfl_xor_sync(0xffffffffu, empty, o);
    v = __shfl_xor_sync(0xffffffffu, bl, o); bl = v > bl ? v : bl;
    v = __shfl_xor_sync(0xffffffffu, bu, o); bu = v > bu ? v : bu;
  }
  if (lane == 0) s_w[warp] = StatPartial{lo, hi, mx, mn, empty, bl, bu};
  __syncthreads();
  if (threadIdx.x == 0) {
    StatPartial p = s_w[0];
    for (int w = 1; w < kStatThreads / 32; ++w) {
      const StatPartial& q = s_w[w];
      add_u128(p.s2_lo, p.s2_hi, q.s2_lo, q.s2_hi);
      p.max_len = q.max_len > p.max_len ? q.max_len : p.max_len;
      p.min_len = q.min_len < p.min_len ? q.min_len : p.min_len;
      p.n_empty += q.n_empty;
      p.bw_lo = q.bw_lo > p.bw_lo ? q.bw_lo : p.bw_lo;
      p.bw_hi = q.bw_hi > p.bw_hi ? q.bw_hi : p.bw_hi;
    }
    part[blockIdx.x] = p;
  }
  for (int b = threadIdx.x; b < kSmemBins; b += blockDim.x) {
    unsigned c = s_hist[b];
    if (c) atomicAdd(&hist[b], c);
  }
}

// Order-statistic ranks, passed by value (no host->device copy that could
// queue behind another stream's bulk upload on the copy engine).
struct SelectTargets {
  long long v[4];
};

// One block of 1024 threads. out[t] = the targets[t]-th smallest row length
// (0-based, targets[t] < rows), t < 3; out[3] = mode (smallest most frequent).
__global__ void __launch_bounds__(1024) k_select(const unsigned* __restrict__ hist,
                                                 const long long* __restrict__ big,
                                                 const unsigned long long* __restrict__ nbig_p,
                                                 const SelectTargets targets,
                                                 const StatPartial* __restrict__ part, int nparts,
                                                 long long* __restrict__ out) {
  __shared__ long long s_chunk[kChunks + 1];
  __shared__ long long s_scan[1024];
  __shared__ unsigned long long s_best[32];
  __shared__ long long s_max[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const long long nbig = (long long)*nbig_p;
  // largest row length (from the row-stats partials) bounds the bins to scan
  {
    long long m = 0;
    for (int i = t; i < nparts; i += blockDim.x) m = part[i].max_len > m ? part[i].max_len : m;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const long long v = __shfl_xor_sync(0xffffffffu, m, o);
      m = v > m ? v : m;
    }
    if (lane == 0) s_max[warp] = m;
  }
  __syncthreads();
  long long maxlen = 0;
  for (int w = 0; w < 32; ++w) maxlen = s_max[w] > maxlen ? s_max[w] : maxlen;
  const int maxbin = (int)(maxlen < kBins - 1 ? maxlen : kBins - 1);
  const int nchunk = maxbin / kChunk + 1;
  // chunk sums over the used chunks: a warp per chunk, coalesced loads
  for (int c = warp; c < kChunks; c += 32) {
    long long sum = 0;
    if (c < nchunk)
      for (int b = lane; b < kChunk; b += 32) sum += hist[c * kChunk + b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) s_chunk[c + 1] = sum;
  }
  __syncthreads();
  if (t == 0) {
    s_chunk[0] = 0;
    for (int c = 0; c < kChunks; ++c) s_chunk[c + 1] += s_chunk[c];
  }
  __syncthreads();
  const long long small_total = s_chunk[kChunks];
  for (int q = 0; q < 3; ++q) {
    long long r = targets.v[q];
    if (r < 0) {
      if (t == 0) out[q] = -1;
      continue;
    }
    if (r < small_total) {
      int c = 0;
      while (s_chunk[c + 1] <= r) ++c;  // uniform across threads
      long long v = hist[c * kChunk + t];
      s_scan[t] = v;
      __syncthreads();
      for (int o = 1; o < 1024; o <<= 1) {  // Hillis–Steele inclusive scan
        long long add = t >= o ? s_scan[t - o] : 0;
        __syncthreads();
        s_scan[t] += add;
        __syncthreads();
      }
      long long incl = s_chunk[c] + s_scan[t];
      long long excl = incl - v;
      if (excl <= r && r < incl) out[q] = (long long)(c * kChunk + t);
      __syncthreads();
    } else {
      long long rr = r - small_total;  // rank among the long rows
      for (long long j = t; j < nbig; j += blockDim.x) {
        long long less = 0, eq = 0, vj = big[j];
        for (long long i = 0; i < nbig; ++i) {
          less += big[i] < vj;
          eq += big[i] == vj;
        }
        if (less <= rr && rr < less + eq) out[q] = vj;  // equal writers write equal values
      }
      __syncthreads();
    }
  }
  // mode: max count, smallest length on ties. Pack (count, ~bin) into u64.
  unsigned long long best = 0;
  for (int b = t; b <= maxbin; b += blockDim.x) {
    unsigned long long key = ((unsigned long long)hist[b] << 32) | (unsigned long long)(0xFFFFFFFFu - (unsigned)b);
    if (hist[b] && key > best) best = key;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long v = __shfl_xor_sync(0xffffffffu, best, o);
    best = v > best ? v : best;
  }
  if (lane == 0) s_best[warp] = best;
  __syncthreads();
  if (t == 0) {
    unsigned long long b = 0;
    for (int w = 0; w < 32; ++w) b = s_best[w] > b ? s_best[w] : b;
    long long mode = (long long)(0xFFFFFFFFu - (unsigned)(b & 0xFFFFFFFFull));
    long long mcount = (long long)(b >> 32);
    for (long long j = 0; j < nbig; ++j) {  // long rows (rare): count equal lengths
      long long vj = big[j], c = 0;
      for (long long i = 0; i < nbig; ++i) c += big[i] == vj;
      if (c > mcount || (c == mcount && vj < mode)) {
        mcount = c;
        mode = vj;
      }
    }
    out[3] = mode;
  }
}

template <class RP>
void features_typed(spmv_matrix* h) {
  cudaStream_t s = h->stream;
  const int64_t n = h->rows;
  Scratch sc(s);
  const unsigned grid = grid_for(n, kStatThreads, (int64_t)kNumSMs * 8);
  StatPartial* part = sc.get<StatPartial>(grid);
  unsigned* hist = sc.get<unsigned>(kBins);
  const int64_t big_cap = h->nnz / kBins + 1;
  long long* big = sc.get<long long>(big_cap);
  unsigned long long* nbig = sc.get<unsigned long long>(1);
  long long* d_out = sc.get<long long>(4);

  // Order-statistic ranks: median lo/hi, and the HYB rule's rank (R12):
  // K_h = L_(q-1) with q = rows − max(floor((rows−1)/3), 4095), or 0 if q <= 0.
  long long targets[4] = {(n - 1) / 2, n / 2, -1, 0};
  long long T = std::max<long long>((n - 1) / 3, 4095);
  long long q = n - T;
  if (q >= 1) targets[2] = q - 1;

  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, s));
  CK(cudaMemsetAsync(hist, 0, kBins * sizeof(unsigned), s));
  CK(cudaMemsetAsync(nbig, 0, sizeof(unsigned long long), s));
  LAUNCH(k_row_stats<RP>, grid, kStatThreads, 0, s, static_cast<const RP*>(h->row_ptr), h->col, n, part,
         hist, big, nbig);
  SelectTargets tg;
  for (int i = 0; i < 4; ++i) tg.v[i] = targets[i];
  LAUNCH(k_select, 1, 1024, 0, s, (const unsigned*)hist, (const long long*)big,
         (const unsigned long long*)nbig, tg, (const StatPartial*)part, (int)grid, d_out);
  std::vector<StatPartial> hp(grid);
  long long res[4];
  CK(cudaEventRecord(e1, s));
  d2h_sync(hp.data(), part, grid * sizeof(StatPartial), s);
  d2h_sync(res, d_out, sizeof(res), s);
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);

  unsigned __int128 S2 = 0;
  long long mx = 0, mn = LLONG_MAX, empty = 0, bl = LLONG_MIN, bu = LLONG_MIN;
  for (const StatPartial& p : hp) {
    S2 += ((unsigned __int128)p.s2_hi << 64) | (unsigned __int128)p.s2_lo;
    mx = std::max(mx, p.max_len);
    mn = std::min(mn, p.min_len);
    empty += p.n_empty;
    bl = std::max(bl, p.bw_lo);
    bu = std::max(bu, p.bw_hi);
  }
  const unsigned __int128 S1 = (unsigned __int128)h->nnz;
  const unsigned __int128 nn = (unsigned __int128)n;
  spmv_features_t& f = h->feat;
  f.n_rows = n;
  f.n_cols = h->cols;
  f.nnz = h->nnz;
  f.max_len = mx;
  f.min_len = mn;
  f.n_empty = empty;
  f.mode = res[3];
  f.bw_lower = bl > 0 ? bl : 0;
  f.bw_upper = bu > 0 ? bu : 0;
  f.bandwidth = std::max(f.bw_lower, f.bw_upper);
  f.mean = (double)h->nnz / (double)n;
  f.var = (double)(nn * S2 - S1 * S1) / (double)n / (double)n;
  f.std = std::sqrt(f.var);
  f.ell_ratio = (mx == 0) ? 1.0 : (double)h->nnz / (double)(n * mx);
  f.median = ((double)res[0] + (double)res[1]) / 2.0;
  h->hyb_auto_K = (targets[2] < 0) ? 0 : res[2];
  h->have_features = true;
  h->f_latency = ms * 1e-3;
}

}  // namespace

void compute_features(spmv_matrix* h) {
  if (h->rows <= 0) fail(SPMV_ERR_INVALID_ARG, "spmv_features: matrix has no rows (S:302)");
  if (h->rp64)
    features_typed<int64_t>(h);
  else
    features_typed<int32_t>(h);
}

}  // namespace spmv
