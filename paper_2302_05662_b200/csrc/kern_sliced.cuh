// kern_sliced.cuh — ELL and SELL-C-sigma SpMV on sm_100a.
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

#pragma once
#include "kern_sliced_decl.cuh"
#include <climits>

namespace spmv {
namespace kern {



// N 16-bit column offsets of one lane (N·2 bytes, aligned): one load.
template <int N>
__device__ __forceinline__ void load_d16(const int16_t* p, int (&d)[N]) {
  if constexpr (N == 1) {
    unsigned short v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(l2_evict_first()));
    d[0] = (int)(int16_t)v;
  } else {
    constexpr int W = N / 2;  // 32-bit words
    int w[W];
    if constexpr (W == 1) {
      w[0] = ld_stream(reinterpret_cast<const int*>(p));
    } else if constexpr (W == 2) {
      int2 t = ld_stream(reinterpret_cast<const int2*>(p));
      w[0] = t.x; w[1] = t.y;
    } else {
      int4 t = ld_stream(reinterpret_cast<const int4*>(p));
      w[0] = t.x; w[1] = t.y; w[2] = t.z; w[3] = t.w;
    }
#pragma unroll
    for (int i = 0; i < W; ++i) {
      d[2 * i] = (int)(int16_t)(w[i] & 0xffff);
      d[2 * i + 1] = (int)(int16_t)((unsigned)w[i] >> 16);
    }
  }
}

// N 8-bit dictionary codes of one lane (N bytes, aligned): one load.
template <int N>
__device__ __forceinline__ void load_c8(const uint8_t* p, int (&d)[N]) {
  if constexpr (N == 1) {
    unsigned short v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(l2_evict_first()));
    d[0] = (int)(v & 0xff);
  } else if constexpr (N == 2) {
    unsigned short v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(l2_evict_first()));
    d[0] = (int)(v & 0xff);
    d[1] = (int)(v >> 8);
  } else if constexpr (N == 4) {
    const unsigned v = (unsigned)ld_stream(reinterpret_cast<const int*>(p));
#pragma unroll
    for (int i = 0; i < 4; ++i) d[i] = (int)((v >> (8 * i)) & 0xff);
  } else {
    const int2 v = ld_stream(reinterpret_cast<const int2*>(p));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      d[i] = (int)(((unsigned)v.x >> (8 * i)) & 0xff);
      d[4 + i] = (int)(((unsigned)v.y >> (8 * i)) & 0xff);
    }
  }
}

// N (<= 4) 8-bit codes of one lane as one 32-bit word (code r in byte r).
template <int N>
__device__ __forceinline__ uint32_t load_c8_word(const uint8_t* p) {
  if constexpr (N == 1) {
    unsigned short v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(l2_evict_first()));
    return 0xffffff00u | (uint32_t)(v & 0xff);
  } else if constexpr (N == 2) {
    unsigned short v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(l2_evict_first()));
    return 0xffff0000u | (uint32_t)v;
  } else {
    return (uint32_t)ld_stream(reinterpret_cast<const int*>(p));
  }
}

// ENC selects the stored column encoding: 0 int32 columns (pad −1); 1 16-bit
// offsets d = col − origin − row (pad −32768); 2 8-bit codes into the
// matrix's offset dictionary (pad 255), decoded through a 256-entry table in
// shared memory (a stencil's k-th slot holds the same code on most lanes:
// the lookup is a broadcast). 12 / 10 / 9 bytes per fp64 slot.
// CARRY selects the batch loop (a launch-tuner knob, SPMV_SLICED_CARRY):
//  CARRY = 1: batch k+U is loaded under a branch after batch k's FMAs and
//             carried in registers (fastest on stencils: c2 ELL-16 96 µs);
//  CARRY = 0: the batch load is unconditional and predicated per k-step
//             (fastest on scattered gathers: c4 ELL 539 vs 564 µs).
template <int B, int R, class T, int C, int ENC, bool CARRY>
__global__ void __launch_bounds__(B) __maxnreg__(regcap(B, R)) k_sliced(const SlicedParams p) {
  constexpr bool D16 = ENC == 1, D8 = ENC == 2, DOFF = ENC != 0;
  // 8-bit codes of up to 4 rows per lane stay packed in one register per
  // k-step until the gather (decoded through the shared table there): the
  // batch holds U words instead of U·RPL columns (register pressure at the
  // 64-register cap of 1024-thread blocks)
  constexpr int RPL = C / 32;                                       // rows per lane
  constexpr int VW = (int)(16 / sizeof(T)) < RPL ? (int)(16 / sizeof(T)) : RPL;  // elems per vector load
  constexpr int NV = RPL / VW;
  constexpr int U = RPL >= 8 ? 1 : 8 / RPL;                         // k-unroll (loads in flight)
  constexpr bool PACK = D8 && RPL <= 4;
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = ((int64_t)blockIdx.x * B + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * (B / 32);
  const T* __restrict__ val = static_cast<const T*>(p.val);
  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ y = static_cast<T*>(p.y);
  // Programmatic dependent launch (power loop): let the next step's grid get
  // resident while this one drains, and wait for the previous step's writes
  // (x, sums_prev) before reading them. No-ops without the launch attribute.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ int s_tab[D8 ? 256 : 1];
  if constexpr (D8) {
    // the pad code's entry makes every padded column negative (origin + row
    // < 2^31, so origin + row + INT_MIN is in [INT_MIN, -1]): the gather's
    // col >= 0 test skips padding without a separate code == 255 test
    for (int i = threadIdx.x; i < 256; i += B) s_tab[i] = i < 255 ? p.tab8[i] : INT_MIN;
    __syncthreads();
  }
  // the power-step partial sums live in shared memory (one slot per warp,
  // filled by a warp reduction at each slice end), not in registers across
  // the slice loop: the loop runs at the 64-register cap of 1024-thread
  // blocks, and every register kept live there is a spill. Per-warp slots
  // keep the block's static shared memory small (a per-thread array would
  // cut the residency of small blocks at carveout 0).
  __shared__ double s_pw[B / 32][2];
  if (lane == 0) {
    s_pw[threadIdx.x >> 5][0] = 0.0;
    s_pw[threadIdx.x >> 5][1] = 0.0;
  }
  // persistent: each warp walks slices warp0, warp0 + nwarps, ... so the
  // per-block epilogue (power-step partial sums) is paid once per block.
  for (int64_t slice = warp0; slice < p.nslices; slice += nwarps) {
    // slot offsets need 64 bits (c5: 3.6·10⁹ slots); a k-step stride (n_pad
    // or C) and a slice width fit 32 (fewer live registers in the loop)
    int64_t base;
    int stride, width;
    if (p.sp) {
      base = p.sp[slice];
      width = (int)((p.sp[slice + 1] - base) / C);
      stride = C;
    } else {
      base = slice * C;
      width = (int)p.ell_K;
      stride = (int)p.ell_stride;
    }
    const int32_t* __restrict__ cp = DOFF ? nullptr : p.col + base + lane * RPL;
    const int16_t* __restrict__ dp = D16 ? p.col16 + base + lane * RPL : nullptr;
    const uint8_t* __restrict__ bp = D8 ? p.col8 + base + lane * RPL : nullptr;
    const T* __restrict__ vp = val + base + lane * RPL;
    double acc[RPL];
    int rowv[DOFF ? RPL : 1];  // 16/8-bit: column origin of each of the lane's rows (< 2^31)
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      acc[r] = 0.0;
      if constexpr (DOFF) {
        const int64_t ri = slice * C + lane * RPL + r;
        rowv[r] = (int)(p.col_origin + (ri < p.rows ? (p.perm ? (int64_t)p.perm[ri] : ri) : 0));
      }
    }
    // One batch = U consecutive k-steps of the lane's RPL rows (values +
    // column indices), predicated past the slice width.
    constexpr int CU = PACK ? 1 : U, CR = PACK ? 1 : RPL;  // unpacked column array (unused when packed)
    auto load_batch = [&](int k, T (&v)[U][RPL], int (&c)[CU][CR], uint32_t (&cw)[U]) {
      // running row pointers (one 64-bit add per k-step) instead of per-step
      // offsets k·stride + u·stride, which the compiler would keep live
      const int64_t ks = (int64_t)k * stride;
      const T* vrow = vp + ks;
      const int32_t* crow = DOFF ? nullptr : cp + ks;
      const int16_t* drow = D16 ? dp + ks : nullptr;
      const uint8_t* brow = D8 ? bp + ks : nullptr;
#pragma unroll
      for (int u = 0; u < U; ++u, vrow += stride) {
        const bool ok = k + u < width;  // predicated tail batch
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          T tv[VW];
          int tc[VW];
          if (ok) {
            load_vals<T, VW>(vrow + q * VW, tv);
            if constexpr (!DOFF) load_cols<VW>(crow + q * VW, tc);
          } else {
#pragma unroll
            for (int w = 0; w < VW; ++w) {
              tv[w] = T(0);
              tc[w] = -1;
            }
          }
#pragma unroll
          for (int w = 0; w < VW; ++w) {
            v[u][q * VW + w] = tv[w];
            if constexpr (!DOFF) c[u][q * VW + w] = tc[w];
          }
        }
        if constexpr (!DOFF) crow += stride;
        if constexpr (D16) {
          int dd[RPL];
          if (ok) {
            load_d16<RPL>(drow, dd);
          } else {
#pragma unroll
            for (int r = 0; r < RPL; ++r) dd[r] = -32768;
          }
#pragma unroll
          for (int r = 0; r < RPL; ++r) c[u][r] = dd[r] == -32768 ? -1 : rowv[r] + dd[r];
          drow += stride;
        }
        if constexpr (PACK) {
          cw[u] = ok ? load_c8_word<RPL>(brow) : 0xffffffffu;
          brow += stride;
        } else if constexpr (D8) {
          int dd[RPL];
          if (ok) {
            load_c8<RPL>(brow, dd);
          } else {
#pragma unroll
            for (int r = 0; r < RPL; ++r) dd[r] = 255;
          }
#pragma unroll
          for (int r = 0; r < RPL; ++r) c[u][r] = rowv[r] + s_tab[dd[r]];  // < 0 for the pad code
          brow += stride;
        }
      }
    };
    // Batch k+U is loaded after batch k's gathers and FMAs (issuing it before
    // them — a software pipeline — doubles the live registers and measured
    // slower on c2 and c4: lower occupancy costs more than it hides).
    // CARRY = 1 guards the reload with a branch, CARRY = 0 predicates it.
    T v[U][RPL];
    int c[CU][CR];
    uint32_t cw[U];
    if (width > 0) load_batch(0, v, c, cw);
    for (int k = 0; k < width; k += U) {
      T vn[U][RPL];
      int cn[CU][CR];
      uint32_t cwn[U];
      T xv[U][RPL];
      if constexpr (PACK) {
        int col[U][RPL];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int r = 0; r < RPL; ++r) {
            const uint32_t code = (cw[u] >> (8 * r)) & 0xffu;
            col[u][r] = rowv[r] + s_tab[code];  // < 0 for the pad code
          }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int r = 0; r < RPL; ++r) xv[u][r] = col[u][r] >= 0 ? ld_x(x + col[u][r]) : T(0);
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int r = 0; r < RPL; ++r) xv[u][r] = c[u][r] >= 0 ? ld_x(x + c[u][r]) : T(0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < RPL; ++r) acc[r] = fma((double)v[u][r], (double)xv[u][r], acc[r]);
      if (!CARRY || k + U < width) {
        load_batch(k + U, vn, cn, cwn);  // predicated: nothing is read past the width
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int r = 0; r < RPL; ++r) v[u][r] = vn[u][r];
          cw[u] = cwn[u];
        }
#pragma unroll
        for (int u = 0; u < CU; ++u)
#pragma unroll
          for (int r = 0; r < CR; ++r) c[u][r] = cn[u][r];
      }
    }
    const int64_t r0 = slice * C + lane * RPL;
    double yy = 0.0, xy = 0.0;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int64_t ri = r0 + r;
      if (ri < p.rows) {
        const int64_t row = p.perm ? (int64_t)p.perm[ri] : ri;
        const T out = epi_value<T>(p.e, epi_alpha(p.e), acc[r], y, row);
        y[row] = out;
        if (p.e.mode == 1) {
          yy += (double)out * (double)out;
          xy += (double)x[p.e.row_offset + row] * (double)out;
        }
      }
    }
    if (p.e.mode == 1) {  // warp-uniform
      yy = warp_sum(yy);
      xy = warp_sum(xy);
      if (lane == 0) {
        s_pw[threadIdx.x >> 5][0] += yy;
        s_pw[threadIdx.x >> 5][1] += xy;
      }
    }
  }
  if (p.e.mode == 1)
    power_reduce(p.e, lane == 0 ? s_pw[threadIdx.x >> 5][0] : 0.0, lane == 0 ? s_pw[threadIdx.x >> 5][1] : 0.0);
}


#define SL_ROW(B) {&k_sliced<B, 32, T, C, ENC, CARRY>, &k_sliced<B, 64, T, C, ENC, CARRY>, \
                   &k_sliced<B, 128, T, C, ENC, CARRY>, &k_sliced<B, 255, T, C, ENC, CARRY>}
template <class T, int C, int ENC, bool CARRY>
SlicedFn sliced_fn(int bi, int ri) {
  static const SlicedFn tab[5][4] = {SL_ROW(64), SL_ROW(128), SL_ROW(256), SL_ROW(512), SL_ROW(1024)};
  return tab[bi][ri];
}
#undef SL_ROW

}  // namespace kern
}  // namespace spmv
