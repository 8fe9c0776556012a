// spmv_common.cuh — epilogue and vector-load helpers shared by every SpMV
// kernel. y_i <- alpha·(Σ_k a_ik·x_k) + beta·y_i (P:145 + reading R1),
// accumulated in fp64 for both value types (reading R3).
#pragma once
#include "handle.cuh"

namespace spmv {

constexpr int kBlocks[5] = {64, 128, 256, 512, 1024};
// Register cap actually compiled for a (block, maxreg) variant: never more
// than the 64K-register file allows for one block of B threads.
constexpr int regcap(int B, int R) { return R < ((65536 / B) & ~7) ? R : ((65536 / B) & ~7); }
constexpr int kRegs[4] = {32, 64, 128, 255};

inline int block_index(int b) {
  for (int i = 0; i < 5; ++i)
    if (kBlocks[i] == b) return i;
  fail(SPMV_ERR_INVALID_ARG, "launch block must be one of 64,128,256,512,1024");
}
inline int reg_index(int r) {
  for (int i = 0; i < 4; ++i)
    if (kRegs[i] == r) return i;
  fail(SPMV_ERR_INVALID_ARG, "launch maxreg must be one of 32,64,128,255");
}

// Vector types for 128-bit loads.
template <class T, int N> struct VecT;
template <> struct VecT<double, 1> { using type = double; };
template <> struct VecT<double, 2> { using type = double2; };
template <> struct VecT<float, 1> { using type = float; };
template <> struct VecT<float, 2> { using type = float2; };
template <> struct VecT<float, 4> { using type = float4; };
template <int N> struct IVecT;
template <> struct IVecT<1> { using type = int; };
template <> struct IVecT<2> { using type = int2; };
template <> struct IVecT<4> { using type = int4; };

template <class T, int N>
__device__ __forceinline__ void load_vals(const T* p, T (&out)[N]) {
  using V = typename VecT<T, N>::type;
  V v = ld_stream(reinterpret_cast<const V*>(p));
  if constexpr (N == 1) {
    out[0] = v;
  } else if constexpr (N == 2) {
    out[0] = v.x; out[1] = v.y;
  } else {
    out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
  }
}
template <int N>
__device__ __forceinline__ void load_cols(const int* p, int (&out)[N]) {
  using V = typename IVecT<N>::type;
  V v = ld_stream(reinterpret_cast<const V*>(p));
  if constexpr (N == 1) {
    out[0] = v;
  } else if constexpr (N == 2) {
    out[0] = v.x; out[1] = v.y;
  } else {
    out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
  }
}

// Epilogue modes: 0 y = alpha·s + beta·y; 1 y = alpha_dev·s (power step);
// 2 y += alpha·s (HYB tail); 3 y += alpha_dev·s (HYB tail in a power step).
// alpha_dev = 1/sqrt(sums_prev[0] + sums_prev[2] + ...) over e.sums_parts row-block parts.
__device__ __forceinline__ double epi_alpha(const Epilogue& e) {
  if (e.mode != 1 && e.mode != 3) return e.alpha;
  double s = __ldcg(e.sums_prev);
  for (int p = 1; p < e.sums_parts; ++p) s += __ldcg(e.sums_prev + 2 * p);  // fixed order: same on every rank
  return 1.0 / sqrt(s);
}

// Final value of row r given its accumulated Σ a·x.
template <class T>
__device__ __forceinline__ T epi_value(const Epilogue& e, double alpha, double acc, const T* y, int64_t r) {
  if (e.mode >= 2) return (T)fma(alpha, acc, (double)y[r]);
  double v = alpha * acc;
  if (e.mode == 0 && e.beta != 0.0) v = fma(e.beta, (double)y[r], v);
  return (T)v;
}

// Power-step block reduction of (Σy², Σx·y): every thread of the block must
// call it. Each block writes its partial; the last block to finish sums all
// partials in block order (deterministic) into sums_out and re-arms counter.
__device__ __forceinline__ void power_reduce(const Epilogue& e, double yy, double xy) {
  __shared__ double s_yy[32], s_xy[32];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  yy = warp_sum(yy);
  xy = warp_sum(xy);
  if (lane == 0) {
    s_yy[warp] = yy;
    s_xy[warp] = xy;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0;
    for (int w = 0; w < nw; ++w) {
      a += s_yy[w];
      b += s_xy[w];
    }
    e.partials[2 * blockIdx.x] = a;
    e.partials[2 * blockIdx.x + 1] = b;
    __threadfence();
    unsigned prev = atomicAdd(e.counter, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  double a = 0, b = 0;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
    a += __ldcg(e.partials + 2 * i);
    b += __ldcg(e.partials + 2 * i + 1);
  }
  a = warp_sum(a);
  b = warp_sum(b);
  __syncthreads();
  if (lane == 0) {
    s_yy[warp] = a;
    s_xy[warp] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double A = 0, Bv = 0;
    for (int w = 0; w < nw; ++w) {
      A += s_yy[w];
      Bv += s_xy[w];
    }
    e.sums_out[0] = A;
    e.sums_out[1] = Bv;
    *e.counter = 0u;
    __threadfence();
  }
}

// Chunk record of the segmented-reduction kernels (merge-path CSR, COO, HYB
// tail). A chunk is a contiguous range of work handled by one warp; rows
// entirely inside a chunk are written by the chunk, rows crossing a chunk
// boundary leave partial sums here and are finished by k_seg_fixup in chunk
// order (deterministic, no float atomics).
struct ChunkRec {
  int32_t first_row, last_row;
  int32_t cont_in, cont_out;  // first row began before the chunk / last row continues after it
  double head, tail;          // partial of the first row (if cont_in) / of the last row (if cont_out)
};

// Finish rows that cross chunk boundaries (launch after the chunk kernel).
void run_seg_fixup(spmv_matrix* h, const ChunkRec* recs, int64_t nchunks, const Epilogue& e, void* y);
// y <- beta·y (mode 0) / 0 (mode 1) for the listed rows (COO empty rows).
void run_rows_scale(spmv_matrix* h, const int32_t* rows_list, int64_t n, const Epilogue& e, void* y);

}  // namespace spmv
