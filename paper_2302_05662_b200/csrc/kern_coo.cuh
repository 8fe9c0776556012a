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
  // W = 8 on 32-byte aligned arrays: one 256-bit load per array (two for
  // fp64 values) instead of two 128-bit loads (warp-uniform choice)
  const bool v256 = W == 8 && ((((uintptr_t)p.row | (uintptr_t)p.col | (uintptr_t)p.val) & 31) == 0);
  if (k0 + W <= p.nnz && v256) {
    if constexpr (W == 8) {
      ld_stream256_w<W>(p.row + k0, r);
      ld_stream256_w<W>(p.col + k0, c);
      ld_stream256_w<W>(val + k0, v);
    }
  } else if (k0 + W <= p.nnz) {
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

// ------------------------------------------------------------------ row-interleaved tiles
// The warp-chunk kernel above gathers, in one instruction, entries of the
// same few rows (lane l holds W consecutive entries): on a stencil the 27
// neighbours of a point span ~12 x lines, so each gather instruction costs
// ~24 L1TEX wavefronts and COO is L1TEX-bound at ~0.55 of the HBM roofline
// (profiles/README.md). k_coo_tile applies CSR-stream's remedy to COO: a
// block stages a tile of B·EPT consecutive entries (row, col, val) in shared
// memory with coalesced 128-bit loads, finds the row segments of the tile
// (ballot + block scan of row changes), and walks them thread-per-segment, so
// at step k the lanes of a warp gather the k-th entry of 32 consecutive rows
// (adjacent x on banded matrices, as in ELL). Segments longer than kLong
// entries (hub rows of power-law graphs) are summed warp-cooperatively after
// the thread pass. The tile is a chunk for the deterministic fixup: its first
// segment, if the row began in the previous tile, goes to rec.head; its last,
// if the row continues, to rec.tail; every other row is finished here.
template <int B, int R, class T, int EPT>
__global__ void __launch_bounds__(B) __maxnreg__(regcap(B, R)) k_coo_tile(const CooParams p) {
  constexpr int TILE = B * EPT;
  constexpr int NW = B / 32;
  constexpr int kLong = 64;
  constexpr int U = 8;  // gathers in flight per thread
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* s_val = reinterpret_cast<T*>(smem_raw);
  int32_t* s_row = reinterpret_cast<int32_t*>(smem_raw + (size_t)TILE * sizeof(T));
  int32_t* s_col = s_row + TILE;
  int32_t* s_seg = s_col + TILE;          // TILE + 1 segment starts
  int32_t* s_cnt = s_seg + TILE + 1;      // EPT·NW head counts, then their exclusive scan
  __shared__ int s_nseg, s_nlong;
  __shared__ int s_long[TILE / kLong + 1];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t tile = blockIdx.x;
  const int64_t t0 = tile * TILE;
  const int n = (int)(p.nnz - t0 < TILE ? p.nnz - t0 : TILE);
  const T* __restrict__ val = static_cast<const T*>(p.val);
  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ y = static_cast<T*>(p.y);
  // ---- stage the tile (16-byte vector loads; the ragged last tile by elements)
  if (n == TILE) {
    constexpr int VI = TILE / 4;                      // int4 vectors per index array
    constexpr int VV = TILE * (int)sizeof(T) / 16;    // 16-byte vectors of values
#pragma unroll
    for (int q = t; q < VI; q += B) {
      reinterpret_cast<int4*>(s_row)[q] = ld_stream(reinterpret_cast<const int4*>(p.row + t0) + q);
      reinterpret_cast<int4*>(s_col)[q] = ld_stream(reinterpret_cast<const int4*>(p.col + t0) + q);
    }
#pragma unroll
    for (int q = t; q < VV; q += B) {
      if constexpr (sizeof(T) == 8)
        reinterpret_cast<double2*>(s_val)[q] = ld_stream(reinterpret_cast<const double2*>(val + t0) + q);
      else
        reinterpret_cast<float4*>(s_val)[q] = ld_stream(reinterpret_cast<const float4*>(val + t0) + q);
    }
  } else {
    for (int i = t; i < n; i += B) {
      s_row[i] = ld_stream(p.row + t0 + i);
      s_col[i] = ld_stream(p.col + t0 + i);
      s_val[i] = ld_stream(val + t0 + i);
    }
  }
  if (t == 0) s_nlong = 0;
  __syncthreads();
  // ---- segment heads in entry order i = pass·B + t (ballot counts, one scan)
#pragma unroll
  for (int ps = 0; ps < EPT; ++ps) {
    const int i = ps * B + t;
    const bool f = i < n && (i == 0 || s_row[i] != s_row[i - 1]);
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) s_cnt[ps * NW + w] = __popc(bal);
  }
  __syncthreads();
  if (w == 0) {  // exclusive scan of the EPT·NW counts, in (pass, warp) order
    int carry = 0;
    for (int base = 0; base < EPT * NW; base += 32) {
      const int v = base + lane < EPT * NW ? s_cnt[base + lane] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (base + lane < EPT * NW) s_cnt[base + lane] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_nseg = carry;
  }
  __syncthreads();
#pragma unroll
  for (int ps = 0; ps < EPT; ++ps) {
    const int i = ps * B + t;
    const bool f = i < n && (i == 0 || s_row[i] != s_row[i - 1]);
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (f) s_seg[s_cnt[ps * NW + w] + __popc(bal & ((1u << lane) - 1u))] = i;
  }
  const int nseg = s_nseg;
  if (t == 0) s_seg[nseg] = n;
  __syncthreads();
  const bool cont_in = t0 > 0 && p.row[t0 - 1] == s_row[0];
  const bool cont_out = t0 + n < p.nnz && p.row[t0 + n] == s_row[n - 1];
  const double alpha = epi_alpha(p.e);
  auto finish = [&](int sg, double acc) {
    const int row = s_row[s_seg[sg]];
    const bool first = sg == 0 && cont_in, last = sg == nseg - 1 && cont_out;
    if (first || last) {
      ChunkRec& rec = p.recs[tile];
      if (first) rec.head = acc;
      if (last) rec.tail = acc;
    } else {
      y[row] = epi_value<T>(p.e, alpha, acc, y, row);
    }
  };
  // ---- thread per segment (row-interleaved gathers)
  for (int sg = t; sg < nseg; sg += B) {
    const int a = s_seg[sg], len = s_seg[sg + 1] - a;
    if (len > kLong) {
      s_long[atomicAdd(&s_nlong, 1)] = sg;
      continue;
    }
    // lengths ≡ 0 mod 8 put a warp's lanes on the same banks: walk from a lane rotation
    int rot = (len & 7) == 0 && len > 0 ? lane : 0;
    if (len > 0 && rot >= len) rot %= len;
    double acc = 0.0;
    for (int k = 0; k < len; k += U) {
      int c[U];
      T v[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        int q = k + j + rot;
        q = q >= len ? q - len : q;
        const bool ok = k + j < len;
        c[j] = ok ? s_col[a + q] : 0;
        v[j] = ok ? s_val[a + q] : T(0);
      }
      T xv[U];
#pragma unroll
      for (int j = 0; j < U; ++j) xv[j] = k + j < len ? ld_x(x + c[j]) : T(0);
#pragma unroll
      for (int j = 0; j < U; ++j) acc = fma((double)v[j], (double)xv[j], acc);
    }
    finish(sg, acc);
  }
  __syncthreads();
  // ---- long segments: warp per segment, lanes stride the entries
  const int nlong = s_nlong;
  for (int q = w; q < nlong; q += NW) {
    const int sg = s_long[q];
    const int a = s_seg[sg], b = s_seg[sg + 1];
    double acc = 0.0;
    for (int k = a + lane; k < b; k += 32) acc = fma((double)s_val[k], (double)ld_x(x + s_col[k]), acc);
    acc = warp_sum(acc);
    if (lane == 0) finish(sg, acc);
  }
  if (t == 0) {
    ChunkRec& rec = p.recs[tile];
    rec.first_row = s_row[0];
    rec.last_row = s_row[n - 1];
    rec.cont_in = cont_in;
    rec.cont_out = cont_out;
  }
}

template <int B, int R, class T, int EPT>
constexpr CooFn coo_tile_ptr() {
  if constexpr (coo_tile_smem<T>(B, EPT) > 200 * 1024) return nullptr;
  else return &k_coo_tile<B, R, T, EPT>;
}
#define COOT_ROW(B, E) {coo_tile_ptr<B, 32, T, E>(), coo_tile_ptr<B, 64, T, E>(), coo_tile_ptr<B, 128, T, E>(), \
                        coo_tile_ptr<B, 255, T, E>()}
template <class T, int EPT>
CooFn coo_tile_fn(int bi, int ri) {
  static const CooFn tab[5][4] = {COOT_ROW(64, EPT), COOT_ROW(128, EPT), COOT_ROW(256, EPT), COOT_ROW(512, EPT),
                                  COOT_ROW(1024, EPT)};
  return tab[bi][ri];
}
#undef COOT_ROW

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
