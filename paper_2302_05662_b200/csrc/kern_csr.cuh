// kern_csr.cuh — CSR SpMV kernels on sm_100a ("This format requires
// coordination among threads within a warp to accumulate per-thread results
// together").
//   k_csr_vector<LANES>: LANES ∈ {1 (scalar), 2, 4, 8, 16, 32} consecutive
//     lanes per row, strided coalesced loads of col/val, shuffle reduction;
//     LANES picked from the mean row length (reading R13).
//   k_csr_merge<IPT>: merge-path CSR (Merrill & Garland) for skewed rows:
//     every lane consumes exactly IPT items of the merged (row-end, nnz)
//     sequence, so one 150K-entry row and 4M empty rows cost the same per
//     item; rows crossing lanes are combined with a warp segmented scan, rows
//     crossing warps through chunk records + k_seg_fixup (deterministic).
#include "spmv_common.cuh"

#pragma once
#include "kern_csr_decl.cuh"

namespace spmv {
namespace kern {



// A group of LANES lanes owns UR consecutive rows per iteration and issues
// the loads of all UR rows before any gather, so a warp keeps
// (32/LANES)·UR rows of col/val traffic in flight; groups walk the rows
// grid-stride (persistent grid).
template <int B, int R, class T, int LANES, class RP>
__global__ void __launch_bounds__(B) __maxnreg__(regcap(B, R)) k_csr_vector(const CsrParams p) {
  constexpr int UR = LANES >= 16 ? 4 : (LANES >= 4 ? 2 : 1);
  const RP* __restrict__ rp = static_cast<const RP*>(p.rp);
  const T* __restrict__ val = static_cast<const T*>(p.val);
  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ y = static_cast<T*>(p.y);
  const int64_t g0 = ((int64_t)blockIdx.x * B + threadIdx.x) / LANES;
  const int64_t ngroups = (int64_t)gridDim.x * (B / LANES);
  const int li = (int)(threadIdx.x & (LANES - 1));
  const double alpha = epi_alpha(p.e);
  double yy = 0.0, xy = 0.0;
  // warp-uniform trip count: groups of one warp leave the loop together so the
  // shuffle reductions below always run with the full warp.
  const int64_t gw0 = g0 - (int64_t)((threadIdx.x & 31) / LANES);
  for (int64_t it = 0;; ++it) {
    if ((gw0 + it * ngroups) * UR >= p.rows) break;
    const int64_t row0 = (g0 + it * ngroups) * UR;
    int64_t a[UR], b[UR];
    int64_t m = 0;
#pragma unroll
    for (int j = 0; j < UR; ++j) {
      const bool ok = row0 + j < p.rows;
      a[j] = ok ? (int64_t)rp[row0 + j] : 0;
      b[j] = ok ? (int64_t)rp[row0 + j + 1] : 0;
      m = max(m, b[j] - a[j]);
    }
    double acc[UR];
#pragma unroll
    for (int j = 0; j < UR; ++j) acc[j] = 0.0;
    for (int64_t off = li; off < m; off += LANES) {
      int c[UR];
      T v[UR];
#pragma unroll
      for (int j = 0; j < UR; ++j) {
        const int64_t k = a[j] + off;
        const bool ok = k < b[j];
        c[j] = ok ? ld_stream(p.col + k) : -1;
        v[j] = ok ? ld_stream(val + k) : T(0);
      }
      T xv[UR];
#pragma unroll
      for (int j = 0; j < UR; ++j) xv[j] = c[j] >= 0 ? ld_x(x + c[j]) : T(0);
#pragma unroll
      for (int j = 0; j < UR; ++j) acc[j] = fma((double)v[j], (double)xv[j], acc[j]);
    }
#pragma unroll
    for (int j = 0; j < UR; ++j)
#pragma unroll
      for (int o = LANES / 2; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
    if (li == 0) {
#pragma unroll
      for (int j = 0; j < UR; ++j) {
        const int64_t row = row0 + j;
        if (row < p.rows) {
          const T out = epi_value<T>(p.e, alpha, acc[j], y, row);
          y[row] = out;
          if (p.e.mode == 1) {
            yy += (double)out * (double)out;
            xy += (double)x[p.e.row_offset + row] * (double)out;
          }
        }
      }
    }
  }
  if (p.e.mode == 1) power_reduce(p.e, yy, xy);
}

// ------------------------------------------------------------------ merge-path
template <class RP>
__device__ __forceinline__ void merge_search(const RP* rp, int64_t rows, int64_t nnz, int64_t d, int64_t& x,
                                             int64_t& yk) {
  int64_t lo = d - nnz > 0 ? d - nnz : 0;
  int64_t hi = d < rows ? d : rows;
  while (lo < hi) {
    int64_t pivot = (lo + hi) >> 1;
    if ((int64_t)rp[pivot + 1] <= d - pivot - 1) lo = pivot + 1;
    else hi = pivot;
  }
  x = lo < rows ? lo : rows;
  yk = d - lo;
}

template <int B, int R, class T, int IPT, class RP>
__global__ void __launch_bounds__(B) __maxnreg__(regcap(B, R)) k_csr_merge(const CsrParams p) {
  const RP* __restrict__ rp = static_cast<const RP*>(p.rp);
  const T* __restrict__ val = static_cast<const T*>(p.val);
  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ y = static_cast<T*>(p.y);
  const int lane = threadIdx.x & 31;
  const int64_t chunk = ((int64_t)blockIdx.x * B + threadIdx.x) >> 5;
  const int64_t total = p.rows + p.nnz;
  const int64_t d0 = chunk * 32 * IPT;
  if (d0 >= total) return;  // whole warp exits together
  const double alpha = epi_alpha(p.e);
  const int64_t d = d0 + (int64_t)lane * IPT;
  int64_t xr, yk;
  merge_search(rp, p.rows, p.nnz, d < total ? d : total, xr, yk);
  // chunk start coordinate (lane 0's) and whether its first row began earlier
  const int64_t x0 = __shfl_sync(0xffffffffu, xr, 0);
  const int64_t y0 = __shfl_sync(0xffffffffu, yk, 0);
  const bool cont_in = x0 < p.rows && y0 > (int64_t)rp[x0];
  const int64_t xs = xr;  // this lane's start row
  double acc = 0.0, first_part = 0.0;
  int64_t first_row = -1;  // first row completed by this lane
  int64_t row_end = xr < p.rows ? (int64_t)rp[xr + 1] : 0;
#pragma unroll 4
  for (int i = 0; i < IPT; ++i) {
    if (d + i >= total) break;
    if (yk < row_end) {
      acc = fma((double)ld_stream(val + yk), (double)ld_x(x + ld_stream(p.col + yk)), acc);
      ++yk;
    } else {
      if (first_row < 0) {
        first_row = xr;
        first_part = acc;
      } else {
        y[xr] = epi_value<T>(p.e, alpha, acc, y, xr);
      }
      acc = 0.0;
      ++xr;
      row_end = xr < p.rows ? (int64_t)rp[xr + 1] : 0;
    }
  }
  // lane carry-out: (row xr in progress, acc). Warp inclusive segmented scan.
  double s = acc;
  const int64_t key = xr;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double su = __shfl_up_sync(0xffffffffu, s, o);
    int64_t ku = __shfl_up_sync(0xffffffffu, key, o);
    if (lane >= o && ku == key) s += su;
  }
  const double s_prev = __shfl_up_sync(0xffffffffu, s, 1);
  const int64_t k_prev = __shfl_up_sync(0xffffffffu, key, 1);
  const double carry_in = (lane > 0 && k_prev == xs) ? s_prev : 0.0;
  if (first_row >= 0) {
    const double tot = carry_in + first_part;
    if (cont_in && first_row == x0) p.recs[chunk].head = tot;
    else y[first_row] = epi_value<T>(p.e, alpha, tot, y, first_row);
  }
  if (lane == 31) {
    ChunkRec& rec = p.recs[chunk];
    rec.first_row = (int32_t)x0;
    rec.cont_in = cont_in;
    const bool cont_out = xr < p.rows && yk > (int64_t)rp[xr];
    rec.last_row = (int32_t)(xr < p.rows ? xr : p.rows - 1);
    rec.cont_out = cont_out;
    if (cont_out) {
      rec.tail = s;
      if (cont_in && xr == x0) rec.head = s;
    }
  }
}


#define CSRV_ROW(B, L) {&k_csr_vector<B, 32, T, L, RP>, &k_csr_vector<B, 64, T, L, RP>, \
                        &k_csr_vector<B, 128, T, L, RP>, &k_csr_vector<B, 255, T, L, RP>}
#define CSRV_TAB(L) {CSRV_ROW(64, L), CSRV_ROW(128, L), CSRV_ROW(256, L), CSRV_ROW(512, L), CSRV_ROW(1024, L)}
template <class T, class RP, int L>
CsrFn csr_vector_fn(int bi, int ri) {
  static const CsrFn tab[5][4] = CSRV_TAB(L);
  return tab[bi][ri];
}
#undef CSRV_TAB
#undef CSRV_ROW

#define CSRM_ROW(B, I) {&k_csr_merge<B, 32, T, I, RP>, &k_csr_merge<B, 64, T, I, RP>, \
                        &k_csr_merge<B, 128, T, I, RP>, &k_csr_merge<B, 255, T, I, RP>}
#define CSRM_TAB(I) {CSRM_ROW(64, I), CSRM_ROW(128, I), CSRM_ROW(256, I), CSRM_ROW(512, I), CSRM_ROW(1024, I)}
template <class T, class RP, int I>
CsrFn csr_merge_fn(int bi, int ri) {
  static const CsrFn tab[5][4] = CSRM_TAB(I);
  return tab[bi][ri];
}
#undef CSRM_TAB
#undef CSRM_ROW

}  // namespace kern
}  // namespace spmv
