// kern_bell.cuh — BELL SpMV ("a block of non-zero elements is
// considered as an element of the ELL format", Fig. 2(d) 2×2 blocks).
// Thread per block row (persistent grid-stride): for each block slot k it
// loads the block column (one int per b×b block: 9 B/nnz for 2×2 fp64 instead
// of ELL's 12) and the b² value planes — each plane read is coalesced across
// consecutive block rows — gathers the b adjacent x values of the block
// column and accumulates b row sums in fp64. Power-step epilogue as in ELL/SELL.
#pragma once
#include "kern_bell_decl.cuh"

namespace spmv {
namespace kern {

template <int B, int R, class T, int BS>
__global__ void __launch_bounds__(B) __maxnreg__(regcap(B, R)) k_bell(const BellParams p) {
  constexpr int BE = BS * BS;
  constexpr int U = BS >= 3 ? 1 : 2;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const T* __restrict__ val = static_cast<const T*>(p.bval);
  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ y = static_cast<T*>(p.y);
  const double alpha = epi_alpha(p.e);
  double yy = 0.0, xy = 0.0;
  const int64_t stride = (int64_t)gridDim.x * B;
  const int64_t plane = p.nbr_pad;
  for (int64_t I = (int64_t)blockIdx.x * B + threadIdx.x; I < p.nbr; I += stride) {
    double acc[BS];
#pragma unroll
    for (int r = 0; r < BS; ++r) acc[r] = 0.0;
    for (int64_t k = 0; k < p.kb; k += U) {
      int J[U];
      T v[U][BE];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool ok = k + u < p.kb;
        J[u] = ok ? ld_stream(p.bcol + (k + u) * plane + I) : -1;
#pragma unroll
        for (int e = 0; e < BE; ++e) v[u][e] = ok ? ld_stream(val + ((k + u) * BE + e) * plane + I) : T(0);
      }
      T xv[U][BS];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int c = 0; c < BS; ++c) {
          const int64_t cc = (int64_t)J[u] * BS + c;
          xv[u][c] = (J[u] >= 0 && cc < p.cols) ? ld_x(x + cc) : T(0);
        }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < BS; ++r)
#pragma unroll
          for (int c = 0; c < BS; ++c) acc[r] = fma((double)v[u][r * BS + c], (double)xv[u][c], acc[r]);
    }
#pragma unroll
    for (int r = 0; r < BS; ++r) {
      const int64_t row = I * BS + r;
      if (row < p.rows) {
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

#define BELL_ROW(Bk) {&k_bell<Bk, 32, T, BS>, &k_bell<Bk, 64, T, BS>, &k_bell<Bk, 128, T, BS>, &k_bell<Bk, 255, T, BS>}
template <class T, int BS>
BellFn bell_fn(int bi, int ri) {
  static const BellFn tab[5][4] = {BELL_ROW(64), BELL_ROW(128), BELL_ROW(256), BELL_ROW(512), BELL_ROW(1024)};
  return tab[bi][ri];
}
#undef BELL_ROW

}  // namespace kern
}  // namespace spmv
