// spmv_sliced.cu — ELL and SELL-C-sigma SpMV on sm_100a.
// One kernel serves both layouts: a warp owns a slice of C rows; lane l owns
// rows l·(C/32) .. l·(C/32)+C/32−1 of the slice, so each step k of the slice
// width reads C consecutive values and C consecutive column indices —
// 128-bit coalesced loads (double2/int2 for fp64 C=64, float4/int4 for fp32
// C=128) — then gathers x through L1/L2 and accumulates in fp64.
//   ELL : element (i, k) at k·n_pad + i     -> base = s·C,        stride = n_pad, width = K
//   SELL: element (s,j,k) at sp[s] + k·C + j -> base = sp[s],      stride = C,     width = (sp[s+1]−sp[s])/C
// Padding slots carry col −1 and are skipped (never multiply x, reading R9).
// The power-step epilogue (mode 1) fuses Σy² and Σx·y into the same pass.
#include "spmv_common.cuh"

namespace spmv {
namespace {

struct SlicedParams {
  const int32_t* col;
  const void* val;
  const int64_t* sp;    // SELL slice pointers (nullptr for ELL)
  const int32_t* perm;  // SELL row permutation (nullptr = identity)
  int64_t rows;
  int64_t nslices;
  int64_t ell_K, ell_stride;
  const void* x;
  void* y;
  Epilogue e;
};

template <int B, int R, class T, int C>
__global__ void __launch_bounds__(B) __maxnreg__(regcap(B, R)) k_sliced(const SlicedParams p) {
  constexpr int RPL = C / 32;                                       // rows per lane
  constexpr int VW = (int)(16 / sizeof(T)) < RPL ? (int)(16 / sizeof(T)) : RPL;  // elems per vector load
  constexpr int NV = RPL / VW;
  constexpr int U = RPL >= 8 ? 1 : 8 / RPL;                         // k-unroll
  const int lane = threadIdx.x & 31;
  const int64_t slice = ((int64_t)blockIdx.x * B + threadIdx.x) >> 5;
  const T* __restrict__ val = static_cast<const T*>(p.val);
  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ y = static_cast<T*>(p.y);
  double yy = 0.0, xy = 0.0;
  if (slice < p.nslices) {
    const double alpha = epi_alpha(p.e);
    int64_t base, stride, width;
    if (p.sp) {
      base = p.sp[slice];
      width = (p.sp[slice + 1] - base) / C;
      stride = C;
    } else {
      base = slice * C;
      width = p.ell_K;
      stride = p.ell_stride;
    }
    const int32_t* __restrict__ cp = p.col + base + lane * RPL;
    const T* __restrict__ vp = val + base + lane * RPL;
    double acc[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) acc[r] = 0.0;
    int64_t k = 0;
    for (; k + U <= width; k += U) {
      T v[U][RPL];
      int c[U][RPL];
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          T tv[VW];
          int tc[VW];
          load_vals<T, VW>(vp + (k + u) * stride + q * VW, tv);
          load_cols<VW>(cp + (k + u) * stride + q * VW, tc);
#pragma unroll
          for (int w = 0; w < VW; ++w) {
            v[u][q * VW + w] = tv[w];
            c[u][q * VW + w] = tc[w];
          }
        }
      }
      T xv[U][RPL];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < RPL; ++r) xv[u][r] = c[u][r] >= 0 ? ld_x(x + c[u][r]) : T(0);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < RPL; ++r) acc[r] = fma((double)v[u][r], (double)xv[u][r], acc[r]);
    }
    for (; k < width; ++k) {
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        T tv[VW];
        int tc[VW];
        load_vals<T, VW>(vp + k * stride + q * VW, tv);
        load_cols<VW>(cp + k * stride + q * VW, tc);
#pragma unroll
        for (int w = 0; w < VW; ++w)
          if (tc[w] >= 0) acc[q * VW + w] = fma((double)tv[w], (double)ld_x(x + tc[w]), acc[q * VW + w]);
      }
    }
    const int64_t r0 = slice * C + lane * RPL;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int64_t ri = r0 + r;
      if (ri < p.rows) {
        const int64_t row = p.perm ? (int64_t)p.perm[ri] : ri;
        const T out = epi_value<T>(p.e, alpha, acc[r], y, row);
        y[row] = out;
        if (p.e.mode == 1) {
          yy += (double)out * (double)out;
          xy += (double)x[p.e.row_offset + row] * (double)out;
        }
      }
    }
  }
  if (p.e.mode == 1) power_reduce(p.e, yy, xy);
}

template <class T, int C>
using SlicedFn = void (*)(const SlicedParams);

#define SL_ROW(B) {&k_sliced<B, 32, T, C>, &k_sliced<B, 64, T, C>, &k_sliced<B, 128, T, C>, &k_sliced<B, 255, T, C>}
template <class T, int C>
SlicedFn<T, C> sliced_fn(int bi, int ri) {
  static const SlicedFn<T, C> tab[5][4] = {SL_ROW(64), SL_ROW(128), SL_ROW(256), SL_ROW(512), SL_ROW(1024)};
  return tab[bi][ri];
}
#undef SL_ROW

template <class T>
void launch_sliced(spmv_matrix* h, SlicedParams& p, int C, const spmv_launch_t& L) {
  const int bi = block_index(L.block), ri = reg_index(L.maxreg);
  const void* fn;
  switch (C) {
    case 32: fn = (const void*)sliced_fn<T, 32>(bi, ri); break;
    case 64: fn = (const void*)sliced_fn<T, 64>(bi, ri); break;
    case 128: fn = (const void*)sliced_fn<T, 128>(bi, ri); break;
    case 256: fn = (const void*)sliced_fn<T, 256>(bi, ri); break;
    default: fail(SPMV_ERR_UNSUPPORTED, "slice height C must be 32, 64, 128 or 256");
  }
  set_carveout(fn, L.carveout_pct);
  const int64_t warps_per_block = L.block / 32;
  const int64_t grid = (p.nslices + warps_per_block - 1) / warps_per_block;
  if (grid <= 0) return;
  if (p.e.mode == 1) {
    ensure_pi_scratch(h, (size_t)grid);
    p.e.partials = h->pi_partials;
    p.e.counter = h->pi_counter;
  }
  void* args[] = {&p};
  launch_checked(fn, dim3((unsigned)grid), dim3(L.block), args, 0, h->stream);
}

}  // namespace

void run_ell_arrays(spmv_matrix* h, const int32_t* col, const void* val, int64_t K, int64_t n_pad,
                    const Epilogue& e, const void* x, void* y, const spmv_launch_t& L) {
  SlicedParams p{};
  const int C = L.knob;
  if (n_pad % C != 0) fail(SPMV_ERR_UNSUPPORTED, "ELL rows-per-warp must divide n_pad (a multiple of 128)");
  p.col = col;
  p.val = val;
  p.sp = nullptr;
  p.perm = nullptr;
  p.rows = h->rows;
  p.nslices = n_pad / C;
  p.ell_K = K;
  p.ell_stride = n_pad;
  p.x = x;
  p.y = y;
  p.e = e;
  if (h->dtype == SPMV_R64F) launch_sliced<double>(h, p, C, L);
  else launch_sliced<float>(h, p, C, L);
}

void run_ell(spmv_matrix* h, const Epilogue& e, const void* x, void* y, const spmv_launch_t& L) {
  run_ell_arrays(h, h->ell_col, h->ell_val, h->ell_K, h->ell_npad, e, x, y, L);
}

void run_sell(spmv_matrix* h, const Epilogue& e, const void* x, void* y, const spmv_launch_t& L) {
  SlicedParams p{};
  p.col = h->sell_col;
  p.val = h->sell_val;
  p.sp = h->sell_sp;
  p.perm = h->sell_perm;
  p.rows = h->rows;
  p.nslices = h->sell_ns;
  p.x = x;
  p.y = y;
  p.e = e;
  if (h->dtype == SPMV_R64F) launch_sliced<double>(h, p, (int)h->sell_C, L);
  else launch_sliced<float>(h, p, (int)h->sell_C, L);
}

}  // namespace spmv
