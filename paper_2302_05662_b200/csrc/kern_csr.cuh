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

// ------------------------------------------------------------------ CSR-stream
// A block owns B consecutive rows per step (persistent grid-stride). If their
// nnz fits the block's shared-memory segment (B·EPT entries), the block copies
// the contiguous CSR segment into shared memory with coalesced 128-bit loads
// and then thread t accumulates row r0+t from shared memory: at every step k
// the 32 lanes of a warp gather the k-th entry of 32 consecutive rows, which
// for banded/stencil matrices are adjacent x values (4 lines per instruction,
// like ELL) instead of one row's scattered neighbours. Blocks with longer
// rows fall back to warp-per-row accumulation over global memory.
template <int B, int R, class T, int EPT, class RP>
__global__ void __launch_bounds__(B) __maxnreg__(regcap(B, R)) k_csr_stream(const CsrParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* s_val = reinterpret_cast<T*>(smem_raw);
  int32_t* s_col = reinterpret_cast<int32_t*>(smem_raw + (size_t)B * EPT * sizeof(T));
  constexpr int CAP = B * EPT;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const RP* __restrict__ rp = static_cast<const RP*>(p.rp);
  const T* __restrict__ val = static_cast<const T*>(p.val);
  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ y = static_cast<T*>(p.y);
  const double alpha = epi_alpha(p.e);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  double yy = 0.0, xy = 0.0;
  for (int64_t r0 = (int64_t)blockIdx.x * B; r0 < p.rows; r0 += (int64_t)gridDim.x * B) {
    const int64_t r1 = r0 + B < p.rows ? r0 + B : p.rows;
    const int64_t s0 = rp[r0], s1 = rp[r1];
    const int64_t seg = s1 - s0;
    if (seg <= CAP) {
      // coalesced staging: align the copy to 16 B so the bulk uses vector loads
      for (int64_t j = t; j < seg; j += B) {
        s_col[j] = ld_stream(p.col + s0 + j);
        s_val[j] = ld_stream(val + s0 + j);
      }
      __syncthreads();
      const int64_t row = r0 + t;
      if (row < r1) {
        const int a = (int)(rp[row] - s0), b = (int)(rp[row + 1] - s0);
        double acc = 0.0;
        int k = a;
        for (; k + 3 < b; k += 4) {
          const int c0 = s_col[k], c1 = s_col[k + 1], c2 = s_col[k + 2], c3 = s_col[k + 3];
          const T x0 = ld_x(x + c0), x1 = ld_x(x + c1), x2 = ld_x(x + c2), x3 = ld_x(x + c3);
          acc = fma((double)s_val[k], (double)x0, acc);
          acc = fma((double)s_val[k + 1], (double)x1, acc);
          acc = fma((double)s_val[k + 2], (double)x2, acc);
          acc = fma((double)s_val[k + 3], (double)x3, acc);
        }
        for (; k < b; ++k) acc = fma((double)s_val[k], (double)ld_x(x + s_col[k]), acc);
        const T out = epi_value<T>(p.e, alpha, acc, y, row);
        y[row] = out;
        if (p.e.mode == 1) {
          yy += (double)out * (double)out;
          xy += (double)x[p.e.row_offset + row] * (double)out;
        }
      }
      __syncthreads();
    } else {
      // long rows: warp per row over global memory, shuffle reduction
      for (int64_t row = r0 + warp; row < r1; row += B / 32) {
        const int64_t a = rp[row], b = rp[row + 1];
        double acc = 0.0;
        for (int64_t k = a + lane; k < b; k += 32)
          acc = fma((double)ld_stream(val + k), (double)ld_x(x + ld_stream(p.col + k)), acc);
        acc = warp_sum(acc);
        if (lane == 0) {
          const T out = epi_value<T>(p.e, alpha, acc, y, row);
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

// Merge-path CSR (Merrill & Garland). A warp owns a chunk of 32·IPT items of
// the merged (row ends, nnz indices) sequence; its start/end coordinates come
// from the partition pre-pass. The warp stages the chunk's row ends in shared
// memory and computes the chunk's products a·x cooperatively (consecutive
// lanes, coalesced col/val loads, independent x gathers), then each lane
// walks IPT items of the merge path summing staged products. Rows crossing lanes are combined by
// a warp segmented scan; rows crossing chunks go through chunk records and
// k_seg_fixup (deterministic, no float atomics).
template <int B, int R, class T, int IPT, class RP>
__global__ void __launch_bounds__(B) __maxnreg__(regcap(B, R)) k_csr_merge(const CsrParams p) {
  constexpr int ITEMS = 32 * IPT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t chunk = ((int64_t)blockIdx.x * B + threadIdx.x) >> 5;
  if (chunk >= p.nchunks) return;  // whole warp exits together
  unsigned char* base = smem_raw + (size_t)wib * merge_warp_smem(IPT);
  double* s_prod = reinterpret_cast<double*>(base);                         // ITEMS products a·x (fp64)
  int32_t* s_end = reinterpret_cast<int32_t*>(base + (size_t)ITEMS * 8);    // ITEMS+1 row ends
  const RP* __restrict__ rp = static_cast<const RP*>(p.rp);
  const T* __restrict__ val = static_cast<const T*>(p.val);
  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ y = static_cast<T*>(p.y);
  const double alpha = epi_alpha(p.e);
  const int64_t x0 = p.coords[2 * chunk], y0 = p.coords[2 * chunk + 1];
  const int64_t x1 = p.coords[2 * chunk + 2], y1 = p.coords[2 * chunk + 3];
  const int nrow = (int)(x1 - x0), nnzc = (int)(y1 - y0);
  // stage row ends (relative to y0, clamped) and the chunk's products; the
  // trip counts are bounded by IPT(+1), so both loops are fully unrolled and
  // every lane has IPT column loads, then IPT x gathers, in flight together.
#pragma unroll
  for (int q = 0; q <= IPT; ++q) {
    const int i = lane + 32 * q;
    if (i <= nrow) {
      const int64_t r = x0 + i;
      const int64_t e = r < p.rows ? (int64_t)rp[r + 1] - y0 : (int64_t)ITEMS + 1;
      s_end[i] = (int32_t)(e > ITEMS + 1 ? ITEMS + 1 : e);
    }
  }
  {
    int c[IPT];
    T v[IPT];
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      const int j = lane + 32 * q;
      const bool ok = j < nnzc;
      c[q] = ok ? ld_stream(p.col + y0 + j) : -1;
      v[q] = ok ? ld_stream(val + y0 + j) : T(0);
    }
    T xv[IPT];
#pragma unroll
    for (int q = 0; q < IPT; ++q) xv[q] = c[q] >= 0 ? ld_x(x + c[q]) : T(0);
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      const int j = lane + 32 * q;
      if (j < nnzc) s_prod[j] = (double)v[q] * (double)xv[q];
    }
  }
  const bool cont_in = x0 < p.rows && y0 > (int64_t)rp[x0];
  __syncwarp();
  // this lane's start on the chunk-local merge path (diagonal d)
  const int d = lane * IPT;
  int lo = d - nnzc > 0 ? d - nnzc : 0, hi = d < nrow ? d : nrow;
  while (lo < hi) {
    const int pivot = (lo + hi) >> 1;
    if (s_end[pivot] <= d - pivot - 1) lo = pivot + 1;
    else hi = pivot;
  }
  int xr = lo, yk = d - lo;
  const int total = nrow + nnzc;
  const int xs = xr;
  double acc = 0.0, first_part = 0.0;
  int first_row = -1;
  int row_end = s_end[xr];
#pragma unroll 4
  for (int i = 0; i < IPT; ++i) {
    if (d + i >= total) break;
    if (yk < row_end) {
      acc += s_prod[yk];
      ++yk;
    } else {
      if (first_row < 0) {
        first_row = xr;
        first_part = acc;
      } else {
        const int64_t gr = x0 + xr;
        y[gr] = epi_value<T>(p.e, alpha, acc, y, gr);
      }
      acc = 0.0;
      ++xr;
      row_end = s_end[xr];
    }
  }
  // lane carry-out: (row xr in progress, acc). Warp inclusive segmented scan.
  double s = acc;
  const int key = xr;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double su = __shfl_up_sync(0xffffffffu, s, o);
    const int ku = __shfl_up_sync(0xffffffffu, key, o);
    if (lane >= o && ku == key) s += su;
  }
  const double s_prev = __shfl_up_sync(0xffffffffu, s, 1);
  const int k_prev = __shfl_up_sync(0xffffffffu, key, 1);
  const double carry_in = (lane > 0 && k_prev == xs) ? s_prev : 0.0;
  if (first_row >= 0) {
    const double tot = carry_in + first_part;
    const int64_t gr = x0 + first_row;
    if (cont_in && first_row == 0) p.recs[chunk].head = tot;
    else y[gr] = epi_value<T>(p.e, alpha, tot, y, gr);
  }
  if (lane == 31) {
    ChunkRec& rec = p.recs[chunk];
    rec.first_row = (int32_t)x0;
    rec.cont_in = cont_in;
    const int64_t gx = x0 + xr;  // == x1 for a full chunk
    const bool cont_out = gx < p.rows && y0 + yk > (int64_t)rp[gx];
    rec.last_row = (int32_t)(gx < p.rows ? gx : p.rows - 1);
    rec.cont_out = cont_out;
    if (cont_out) {
      rec.tail = s;
      if (cont_in && xr == 0) rec.head = s;
    }
  }
}

template <class RP>
__global__ void k_merge_partition(const RP* __restrict__ rp, int64_t rows, int64_t nnz, int64_t items,
                                  int64_t nchunks, int64_t* __restrict__ coords) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t total = rows + nnz;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c <= nchunks; c += stride) {
    int64_t d = c * items;
    if (d > total) d = total;
    int64_t xx, yy;
    merge_search(rp, rows, nnz, d, xx, yy);
    coords[2 * c] = xx;
    coords[2 * c + 1] = yy;
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

#define CSRS_ROW(B, E) {&k_csr_stream<B, 32, T, E, RP>, &k_csr_stream<B, 64, T, E, RP>, \
                        &k_csr_stream<B, 128, T, E, RP>, &k_csr_stream<B, 255, T, E, RP>}
#define CSRS_TAB(E) {CSRS_ROW(64, E), CSRS_ROW(128, E), CSRS_ROW(256, E), CSRS_ROW(512, E), CSRS_ROW(1024, E)}
template <class T, class RP, int E>
CsrFn csr_stream_fn(int bi, int ri) {
  static const CsrFn tab[5][4] = CSRS_TAB(E);
  return tab[bi][ri];
}
#undef CSRS_TAB
#undef CSRS_ROW

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
