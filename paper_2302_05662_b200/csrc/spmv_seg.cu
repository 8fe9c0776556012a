// spmv_seg.cu — COO SpMV via warp-shuffle segmented reduction (north star),
// the HYB tail (same kernel in accumulate mode), the chunk fixup shared
// with merge-path CSR, and small helper kernels (row scaling, norms).
//
// COO: a warp owns a chunk of 32·W consecutive entries sorted by
// (row, col); lane l loads W of them with vector loads (row/col as int2/int4,
// values as double2/float4), reduces its own runs, then a 5-step warp
// segmented scan keyed by row combines runs that cross lanes. Rows entirely
// inside the chunk are written by the chunk; rows crossing chunk boundaries
// leave head/tail partials that k_seg_fixup combines in chunk order.
#include "kern_coo_decl.cuh"
#include "kern_sliced_decl.cuh"

namespace spmv {
namespace {
// Rows crossing chunk boundaries: the chunk where such a row starts (cont_out
// and not a single-row continuation chunk) owns it.
//  k_seg_fixup: thread per chunk; a row that ends in the next chunk (the usual
//    case) is finished directly; longer runs are appended to a list.
//  k_seg_fixup_long: one warp per listed run reads the following chunk records
//    32 at a time, finds where the row ends (ballot) and sums the heads with a
//    fixed-shape reduction — a 150K-entry row spanning hundreds of chunks costs
//    a few warp steps. Both orders are fixed by the data: deterministic.
__device__ __forceinline__ bool rec_mid(const ChunkRec& r) {
  return r.cont_out && r.cont_in && r.first_row == r.last_row;
}

template <class T>
__global__ void k_seg_fixup(const ChunkRec* __restrict__ recs, int64_t n, Epilogue e, T* __restrict__ y,
                            int64_t* __restrict__ longs, unsigned long long* __restrict__ nlong) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const double alpha = epi_alpha(e);
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += stride) {
    const ChunkRec rc = recs[c];
    if (!rc.cont_out || rec_mid(rc) || c + 1 >= n) continue;
    const ChunkRec rn = recs[c + 1];
    if (rec_mid(rn)) {
      longs[atomicAdd(nlong, 1ull)] = c;
      continue;
    }
    const int r = rc.last_row;
    y[r] = epi_value<T>(e, alpha, rc.tail + rn.head, y, r);
  }
}

template <class T>
__global__ void k_seg_fixup_long(const ChunkRec* __restrict__ recs, int64_t n, Epilogue e, T* __restrict__ y,
                                 const int64_t* __restrict__ longs, const unsigned long long* __restrict__ nlong) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t count = (int64_t)*nlong;
  const double alpha = epi_alpha(e);
  for (int64_t w = warp0; w < count; w += nwarps) {
    const int64_t c = longs[w];
    const ChunkRec rc = recs[c];
    double part = 0.0;
    for (int64_t q0 = c + 1; q0 < n; q0 += 32) {
      const int64_t q = q0 + lane;
      const bool valid = q < n;
      bool mid = false;
      if (valid) mid = rec_mid(recs[q]);  // flags are always written; head only when cont_in
      const unsigned endm = __ballot_sync(0xffffffffu, valid && !mid);
      const int last = endm ? __ffs(endm) - 1 : 31;
      if (valid && lane <= last) part += recs[q].head;
      if (endm || !__ballot_sync(0xffffffffu, valid)) break;
    }
    part = warp_sum(part);
    if (lane == 0) {
      const int r = rc.last_row;
      y[r] = epi_value<T>(e, alpha, rc.tail + part, y, r);
    }
  }
}

template <class T>
__global__ void k_rows_scale(const int32_t* __restrict__ rows, int64_t n, Epilogue e, T* __restrict__ y) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const double alpha = epi_alpha(e);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int r = rows[i];
    y[r] = epi_value<T>(e, alpha, 0.0, y, r);
  }
}

template <class T>
__global__ void k_norms(const T* __restrict__ x, const T* __restrict__ y, int64_t n, Epilogue e) {
  double yy = 0.0, xy = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double v = (double)y[i];
    yy += v * v;
    if (x) xy += (double)x[e.row_offset + i] * v;
  }
  power_reduce(e, yy, xy);
}

template <class T>
__global__ void k_scale(T* __restrict__ y, int64_t n, double beta) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = beta == 0.0 ? T(0) : (T)(beta * (double)y[i]);
}


template <class T>
void coo_launch(spmv_matrix* h, const int32_t* row, const int32_t* col, const void* val, int64_t nnz,
                const Epilogue& e, const void* x, void* y, const spmv_launch_t& L) {
  if (nnz <= 0) return;
  const int W = L.knob;
  const int bi = block_index(L.block), ri = reg_index(L.maxreg);
  const void* fn;
  const bool tile = (W & kern::kCooTile) != 0;
  const int ept = W & 0xff;
  size_t smem = 0;
  int64_t per_chunk = 32LL * W;
  if (tile) {
    switch (ept) {
      case 4: fn = (const void*)kern::coo_tile_fn<T, 4>(bi, ri); break;
      case 8: fn = (const void*)kern::coo_tile_fn<T, 8>(bi, ri); break;
      case 16: fn = (const void*)kern::coo_tile_fn<T, 16>(bi, ri); break;
      case 32: fn = (const void*)kern::coo_tile_fn<T, 32>(bi, ri); break;
      default: fail(SPMV_ERR_INVALID_ARG, "COO tile entries per thread must be 4, 8, 16 or 32");
    }
    if (!fn) fail(SPMV_ERR_UNSUPPORTED, "COO tile: block × entries per thread exceeds shared memory");
    if (((uintptr_t)row | (uintptr_t)col | (uintptr_t)val) & 15)
      fail(SPMV_ERR_UNSUPPORTED, "COO tile: row/col/val must be 16-byte aligned for vector staging");
    smem = kern::coo_tile_smem<T>(L.block, ept);
    per_chunk = (int64_t)L.block * ept;
  } else {
    switch (W) {
      case 2: fn = (const void*)kern::coo_fn<T, 2>(bi, ri); break;
      case 4: fn = (const void*)kern::coo_fn<T, 4>(bi, ri); break;
      case 8: fn = (const void*)kern::coo_fn<T, 8>(bi, ri); break;
      default: fail(SPMV_ERR_INVALID_ARG, "COO entries per lane must be 2, 4 or 8, or kCooTile | 4, 8, 16, 32");
    }
  }
  const LaunchAttrs attrs(fn, L.carveout_pct, smem);
  const int64_t nchunks = (nnz + per_chunk - 1) / per_chunk;
  kern::CooParams p{};
  p.row = row;
  p.col = col;
  p.val = val;
  p.nnz = nnz;
  p.x = x;
  p.y = y;
  p.e = e;
  p.recs = static_cast<ChunkRec*>(ensure_seg_scratch(h, (size_t)nchunks * sizeof(ChunkRec)));
  const int64_t grid = tile ? nchunks : (nchunks * 32 + L.block - 1) / L.block;
  void* args[] = {&p};
  launch_checked(fn, dim3((unsigned)grid), dim3(L.block), args, smem, h->stream);
  run_seg_fixup(h, p.recs, nchunks, e, y);
}

}  // namespace

void run_seg_fixup(spmv_matrix* h, const ChunkRec* recs, int64_t nchunks, const Epilogue& e, void* y) {
  if (nchunks <= 1) return;
  // scratch for the long-run list lives after the records (same grow-only buffer)
  const size_t rec_bytes = ((size_t)nchunks * sizeof(ChunkRec) + 255) / 256 * 256;
  (void)rec_bytes;
  int64_t* longs = static_cast<int64_t*>(ensure_fixup_scratch(h, (size_t)nchunks * sizeof(int64_t) + 256));
  unsigned long long* nlong = reinterpret_cast<unsigned long long*>(longs + nchunks);
  CK(cudaMemsetAsync(nlong, 0, sizeof(unsigned long long), h->stream));
  const unsigned g = grid_for(nchunks, 256);
  const unsigned gl = (unsigned)(kNumSMs * 8);
  if (h->dtype == SPMV_R64F) {
    LAUNCH(k_seg_fixup<double>, g, 256, 0, h->stream, recs, nchunks, e, (double*)y, longs, nlong);
    LAUNCH(k_seg_fixup_long<double>, gl, 256, 0, h->stream, recs, nchunks, e, (double*)y, (const int64_t*)longs,
           (const unsigned long long*)nlong);
  } else {
    LAUNCH(k_seg_fixup<float>, g, 256, 0, h->stream, recs, nchunks, e, (float*)y, longs, nlong);
    LAUNCH(k_seg_fixup_long<float>, gl, 256, 0, h->stream, recs, nchunks, e, (float*)y, (const int64_t*)longs,
           (const unsigned long long*)nlong);
  }
}

void run_rows_scale(spmv_matrix* h, const int32_t* rows_list, int64_t n, const Epilogue& e, void* y) {
  if (n <= 0) return;
  const unsigned g = grid_for(n, 256);
  if (h->dtype == SPMV_R64F) LAUNCH(k_rows_scale<double>, g, 256, 0, h->stream, rows_list, n, e, (double*)y);
  else LAUNCH(k_rows_scale<float>, g, 256, 0, h->stream, rows_list, n, e, (float*)y);
}

void run_norms(spmv_matrix* h, const Epilogue& e0, const void* x, const void* y, int64_t n) {
  Epilogue e = e0;
  const unsigned g = grid_for(n, 256, (int64_t)kNumSMs * 4);
  ensure_pi_scratch(h, g);
  e.partials = h->pi_partials;
  e.counter = h->pi_counter;
  if (h->dtype == SPMV_R64F)
    LAUNCH(k_norms<double>, g, 256, 0, h->stream, (const double*)x, (const double*)y, n, e);
  else
    LAUNCH(k_norms<float>, g, 256, 0, h->stream, (const float*)x, (const float*)y, n, e);
}

void run_scale(spmv_matrix* h, void* y, double beta) {
  if (h->rows <= 0) return;
  const unsigned g = grid_for(h->rows, 256);
  if (h->dtype == SPMV_R64F) LAUNCH(k_scale<double>, g, 256, 0, h->stream, (double*)y, h->rows, beta);
  else LAUNCH(k_scale<float>, g, 256, 0, h->stream, (float*)y, h->rows, beta);
}

void run_coo(spmv_matrix* h, const Epilogue& e, const void* x, void* y, const spmv_launch_t& L) {
  // empty rows first (they are disjoint from every row the chunks write)
  run_rows_scale(h, h->coo_empty, h->coo_n_empty, e, y);
  if (h->dtype == SPMV_R64F) coo_launch<double>(h, h->coo_row, h->col, h->val, h->nnz, e, x, y, L);
  else coo_launch<float>(h, h->coo_row, h->col, h->val, h->nnz, e, x, y, L);
}

void run_hyb(spmv_matrix* h, const Epilogue& e, const void* x, void* y, const spmv_launch_t& L) {
  // ELL part writes every row (alpha·s_ell + beta·y); the COO tail then adds
  // alpha·s_tail to the rows that have one (mode 2, or 3 with device alpha).
  spmv_launch_t le = L;
  le.knob = (h->dtype == SPMV_R64F ? 64 : 128) | kern::kSlicedCarry;
  run_ell_arrays(h, h->hyb_ecol, h->hyb_eval, h->hyb_K, h->hyb_npad, e, x, y, le);
  Epilogue et = e;
  et.mode = (e.mode == 1) ? 3 : 2;
  spmv_launch_t lt = L;
  if (h->dtype == SPMV_R64F) coo_launch<double>(h, h->hyb_trow, h->hyb_tcol, h->hyb_tval, h->hyb_tail, et, x, y, lt);
  else coo_launch<float>(h, h->hyb_trow, h->hyb_tcol, h->hyb_tval, h->hyb_tail, et, x, y, lt);
}

}  // namespace spmv
