// kern_coo.cuh — COO SpMV via warp-shuffle segmented reduction (north star),
// the HYB tail (same kernel in accumulate mode), the chunk fixup shared
// with merge-path CSR, and small helper kernels (row scaling, norms).
//
// COO: a warp owns a chunk of 32·W consecutive entries sorted by
// (row, col); lane l loads W of them with vector loads (row/col as int2/int4,
// values as double2/float4), reduces its own runs, then a 5-step warp
// segmented scan keyed by row combines runs that cross lanes. Rows entirely
// inside the chunk are written by the chunk; rows crossing chunk boundaries
// leave head/tail partials that k_seg_fixup combines in chunk order.
#include "spmv_common.cuh"

#pragma once
#include "kern_coo_decl.cuh"

namespace spmv {
namespace kern {



template <class T, int W>
__device__ __forceinline__ void load_w(const T* p, T (&v)[W]) {
  if constexpr (W == 2 && sizeof(T) == 8) {
    double2 a = ld_stream(reinterpret_cast<const double2*>(p));
    v[0] = a.x; v[1] = a.y;
  } else if constexpr (W == 4 && sizeof(T) == 8) {
    double2 a = ld_stream(reinterpret_cast<const double2*>(p));
    double2 b = ld_stream(reinterpret_cast<const double2*>(p + 2));
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  } else if constexpr (W == 2) {
    float2 a = ld_stream(reinterpret_cast<const float2*>(p));
    v[0] = a.x; v[1] = a.y;
  } else if constexpr (W == 4) {
    float4 a = ld_stream(reinterpret_cast<const float4*>(p));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  } else {
#pragma unroll
    for (int q = 0; q < W; q += 4) load_w<T, 4>(p + q, *reinterpret_cast<T(*)[4]>(&v[q]));
  }
}
template <int W>
__device__ __forceinline__ void load_wi(const int* p, int (&v)[W]) {
  if constexpr (W == 2) {
    int2 a = ld_stream(reinterpret_cast<const int2*>(p));
    v[0] = a.x; v[1] = a.y;
  } else {
#pragma unroll
    for (int q = 0; q < W; q += 4) {
      int4 a = ld_stream(reinterpret_cast<const int4*>(p + q));
      v[q] = a.x; v[q + 1] = a.y; v[q + 2] = a.z; v[q + 3] = a.w;
    }
  }
}

template <int B, int R, class T, int W>
__global__ void __launch_bounds__(B) __maxnreg__(regcap(B, R)) k_coo(const CooParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t chunk = ((int64_t)blockIdx.x * B + threadIdx.x) >> 5;
  const int64_t base = chunk * 32 * W;
  if (base >= p.nnz) return;  // warp-uniform
  const T* __restrict__ val = static_cast<const T*>(p.val);
  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ y = static_cast<T*>(p.y);
  const double alpha = epi_alpha(p.e);
  const int64_t k0 = base + (int64_t)lane * W;
  int r[W], c[W];
  T v[W];
  if (k0 + W <= p.nnz) {
    load_wi<W>(p.row + k0, r);
    load_wi<W>(p.col + k0, c);
    load_w<T, W>(val + k0, v);
  } else {
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const bool ok = k0 + q < p.nnz;
      r[q] = ok ? p.row[k0 + q] : INT_MAX;  // sentinel row after the last entry
      c[q] = ok ? p.col[k0 + q] : 0;
      v[q] = ok ? val[k0 + q] : T(0);
    }
  }
  double prod[W];
#pragma unroll
  for (int q = 0; q < W; ++q) prod[q] = r[q] != INT_MAX ? (double)v[q] * (double)ld_x(x + c[q]) : 0.0;
  const int64_t end = base + 32 * W;
  const int chunk_first = __shfl_sync(0xffffffffu, r[0], 0);
  const bool cont_in = base > 0 && p.row[base - 1] == chunk_first;
  // lane-local runs: rows strictly inside the lane are complete here
  const int first = r[0];
  double first_sum = 0.0, run = 0.0;
  bool first_closed = false;
  int cur = r[0];
#pragma unroll
  for (int q = 0; q < W; ++q) {
    if (r[q] != cur) {
      if (!first_closed) {
        first_sum = run;
        first_closed = true;
      } else {
        y[cur] = epi_value<T>(p.e, alpha, run, y, cur);
      }
      cur = r[q];
      run = 0.0;
    }
    run += prod[q];
  }
  const int last = cur;
  if (!first_closed) first_sum = run;  // single-run lane
  // warp inclusive segmented scan of the last run (key = row)
  double s = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double su = __shfl_up_sync(0xffffffffu, s, o);
    int ku = __shfl_up_sync(0xffffffffu, last, o);
    if (lane >= o && ku == last) s += su;
  }
  const double s_prev = __shfl_up_sync(0xffffffffu, s, 1);
  const int k_prev = __shfl_up_sync(0xffffffffu, last, 1);
  const double carry_in = (lane > 0 && k_prev == first) ? s_prev : 0.0;
  int next_first = __shfl_down_sync(0xffffffffu, r[0], 1);
  if (lane == 31) next_first = end < p.nnz ? p.row[end] : INT_MAX;
  // first run closed inside this lane
  if (first_closed && first != INT_MAX) {
    const double tot = carry_in + first_sum;
    if (cont_in && first == chunk_first) p.recs[chunk].head = tot;
    else y[first] = epi_value<T>(p.e, alpha, tot, y, first);
  }
  // last run: closes at the lane end if the next entry starts another row
  if (last != INT_MAX) {
    if (next_first != last) {
      if (cont_in && last == chunk_first) p.recs[chunk].head = s;
      else y[last] = epi_value<T>(p.e, alpha, s, y, last);
    } else if (lane == 31) {
      p.recs[chunk].tail = s;
      if (cont_in && last == chunk_first) p.recs[chunk].head = s;
    }
  }
  // chunk record: the last valid row of the chunk
  int chunk_last = last;
  {
    unsigned valid = __ballot_sync(0xffffffffu, r[0] != INT_MAX);
    int src = 31 - __clz((int)valid);
    int lastv = __shfl_sync(0xffffffffu, last, src);
    chunk_last = lastv;
  }
  if (lane == 31) {
    ChunkRec& rec = p.recs[chunk];
    rec.first_row = chunk_first;
    rec.cont_in = cont_in;
    rec.last_row = chunk_last;
    rec.cont_out = (next_first == last) && last != INT_MAX;
  }
}

#define COO_ROW(B, W) {&k_coo<B, 32, T, W>, &k_coo<B, 64, T, W>, &k_coo<B, 128, T, W>, &k_coo<B, 255, T, W>}
#define COO_TAB(W) {COO_ROW(64, W), COO_ROW(128, W), COO_ROW(256, W), COO_ROW(512, W), COO_ROW(1024, W)}
template <class T, int W>
CooFn coo_fn(int bi, int ri) {
  static const CooFn tab[5][4] = COO_TAB(W);
  return tab[bi][ri];
}
#undef COO_TAB
#undef COO_ROW

}  // namespace kern
}  // namespace spmv
