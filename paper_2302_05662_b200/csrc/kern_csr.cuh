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
#include "tma.cuh"

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

// CSR-vector with quad loads (knob kCsrQuad | LANES): like k_csr_vector, but
// a lane reads 4 consecutive entries of its row per step with one 128-bit
// column load and 128-bit value loads, aligned to the array's 4-entry quads
// (entries of the quad outside the row are masked, never gathered): 4× fewer
// load instructions for long rows, the same bytes. A quad reaching past the
// last nonzero is read entry by entry.
template <int B, int R, class T, int LANES, class RP>
__global__ void __launch_bounds__(B) __maxnreg__(regcap(B, R)) k_csr_vector4(const CsrParams p) {
  constexpr int UR = LANES >= 16 ? 2 : 1;
  const RP* __restrict__ rp = static_cast<const RP*>(p.rp);
  const T* __restrict__ val = static_cast<const T*>(p.val);
  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ y = static_cast<T*>(p.y);
  const int64_t g0 = ((int64_t)blockIdx.x * B + threadIdx.x) / LANES;
  const int64_t ngroups = (int64_t)gridDim.x * (B / LANES);
  const int li = (int)(threadIdx.x & (LANES - 1));
  const double alpha = epi_alpha(p.e);
  double yy = 0.0, xy = 0.0;
  const int64_t gw0 = g0 - (int64_t)((threadIdx.x & 31) / LANES);
  for (int64_t it = 0;; ++it) {
    if ((gw0 + it * ngroups) * UR >= p.rows) break;
    const int64_t row0 = (g0 + it * ngroups) * UR;
    int64_t a[UR], b[UR], q0[UR], nq[UR];
    int64_t m = 0;
#pragma unroll
    for (int j = 0; j < UR; ++j) {
      const bool ok = row0 + j < p.rows;
      a[j] = ok ? (int64_t)rp[row0 + j] : 0;
      b[j] = ok ? (int64_t)rp[row0 + j + 1] : 0;
      q0[j] = a[j] >> 2;
      nq[j] = b[j] > a[j] ? ((b[j] + 3) >> 2) - q0[j] : 0;
      m = max(m, nq[j]);
    }
    double acc[UR];
#pragma unroll
    for (int j = 0; j < UR; ++j) acc[j] = 0.0;
    for (int64_t oq = li; oq < m; oq += LANES) {
      int c[UR][4];
      T v[UR][4];
#pragma unroll
      for (int j = 0; j < UR; ++j) {
        const int64_t e0 = (q0[j] + oq) * 4;
        if (oq < nq[j] && e0 + 4 <= p.nnz) {
          const int4 cc = ld_stream(reinterpret_cast<const int4*>(p.col + e0));
          c[j][0] = cc.x; c[j][1] = cc.y; c[j][2] = cc.z; c[j][3] = cc.w;
          if constexpr (sizeof(T) == 8) {
            const double2 v0 = ld_stream(reinterpret_cast<const double2*>(val + e0));
            const double2 v1 = ld_stream(reinterpret_cast<const double2*>(val + e0 + 2));
            v[j][0] = v0.x; v[j][1] = v0.y; v[j][2] = v1.x; v[j][3] = v1.y;
          } else {
            const float4 v0 = ld_stream(reinterpret_cast<const float4*>(val + e0));
            v[j][0] = v0.x; v[j][1] = v0.y; v[j][2] = v0.z; v[j][3] = v0.w;
          }
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int64_t e = e0 + t;
            const bool ok = oq < nq[j] && e < p.nnz;
            c[j][t] = ok ? ld_stream(p.col + e) : -1;
            v[j][t] = ok ? ld_stream(val + e) : T(0);
          }
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int64_t e = e0 + t;
          if (e < a[j] || e >= b[j]) c[j][t] = -1;  // another row's entry: masked
        }
      }
      T xv[UR][4];
#pragma unroll
      for (int j = 0; j < UR; ++j)
#pragma unroll
        for (int t = 0; t < 4; ++t) xv[j][t] = c[j][t] >= 0 ? ld_x(x + c[j][t]) : T(0);
#pragma unroll
      for (int j = 0; j < UR; ++j)
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (c[j][t] >= 0) acc[j] = fma((double)v[j][t], (double)xv[j][t], acc[j]);
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
// Thread per row over a shared-memory copy of the tile's CSR segment, fed by a
// TMA pipeline. A tile is B consecutive rows; its entries [rp[r0], rp[r0+B])
// are contiguous in col/val, so one producer warp moves them into a ring of
// two shared-memory stages with cp.async.bulk (mbarrier transaction counts,
// L2 evict-first) while the B consumer threads work on the other stage. The
// consumers then read row r0+t from shared memory: at step k the 32 lanes of
// a warp gather the k-th entry of 32 consecutive rows, which for banded /
// stencil matrices are adjacent x values (a few lines per instruction, like
// ELL) instead of one row's scattered neighbours (CSR-vector), and the matrix
// stream never occupies L1TEX. Tiles whose segment exceeds the stage (long
// rows) are handled warp-per-row straight from global memory.
template <int B, int R, class T, int EPT, class RP>
__global__ void __launch_bounds__(B + 32) __maxnreg__(regcap(B + 32, R)) k_csr_stream(const CsrParams p) {
  constexpr int CAP = B * EPT;
  constexpr int NS = kStreamStages;
  constexpr int VP = StreamStage<T>::kValPad;
  constexpr int U = sizeof(T) == 8 ? 16 : 16;  // entries per gather batch (independent loads in flight)
  constexpr size_t STAGE = StreamStage<T>::bytes(CAP);
  constexpr size_t COLB = StreamStage<T>::col_bytes(CAP);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[NS], empty_bar[NS];
  __shared__ int64_t meta_s0[NS];
  __shared__ int meta_staged[NS];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t == 0) {
    for (int s = 0; s < NS; ++s) {
      tma::mbar_init(&full_bar[s], 32);          // the 32 producer lanes arrive (lane 0 also adds the tx)
      tma::mbar_init(&empty_bar[s], B / 32);     // one arrival per consumer warp
    }
    tma::fence_barrier_init();
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const RP* __restrict__ rp = static_cast<const RP*>(p.rp);
  const T* __restrict__ val = static_cast<const T*>(p.val);
  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ y = static_cast<T*>(p.y);
  const int64_t ntiles = (p.rows + B - 1) / B;
  double yy = 0.0, xy = 0.0;
  if (warp == B / 32) {
    // ------------------------------------------------------------ producer
    const uint64_t pol = tma::policy_evict_first();
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t r0 = tile * B, r1 = r0 + B < p.rows ? r0 + B : p.rows;
      const int64_t s0 = (int64_t)rp[r0], s1 = (int64_t)rp[r1];
      const bool staged = s1 - s0 <= CAP;
      tma::mbar_wait(&empty_bar[stage], phase ^ 1);
      unsigned char* st = smem_raw + (size_t)stage * STAGE;
      int32_t* s_col = reinterpret_cast<int32_t*>(st);
      T* s_val = reinterpret_cast<T*>(st + COLB);
      if (lane == 0) {
        meta_s0[stage] = s0;
        meta_staged[stage] = staged;
      }
      if (staged && s1 > s0) {
        // 16-byte aligned inner ranges go by bulk copy; the (< 16 B) head and
        // tail of each array are copied by the lanes.
        const int64_t cb = s0 & ~3LL;
        int64_t ci0 = (s0 + 3) & ~3LL, ci1 = s1 & ~3LL;
        if (ci1 <= ci0) ci0 = ci1 = s1;
        const int64_t vb = s0 & ~(int64_t)(VP - 1);
        int64_t vi0 = (s0 + VP - 1) & ~(int64_t)(VP - 1), vi1 = s1 & ~(int64_t)(VP - 1);
        if (vi1 <= vi0) vi0 = vi1 = s1;
        if (lane == 0) {
          const uint32_t tx = (uint32_t)((ci1 - ci0) * 4 + (vi1 - vi0) * (int64_t)sizeof(T));
          if (tx) tma::mbar_expect_tx(&full_bar[stage], tx);
          if (ci1 > ci0)
            tma::bulk_g2s(s_col + (ci0 - cb), p.col + ci0, (uint32_t)((ci1 - ci0) * 4), &full_bar[stage], pol);
          if (vi1 > vi0)
            tma::bulk_g2s(s_val + (vi0 - vb), val + vi0, (uint32_t)((vi1 - vi0) * sizeof(T)), &full_bar[stage], pol);
        }
        const int ch = (int)(ci0 - s0), ct = (int)(s1 - ci1);
        if (lane < ch) s_col[s0 + lane - cb] = ld_stream(p.col + s0 + lane);
        else if (lane >= 16 && lane - 16 < ct) s_col[ci1 + lane - 16 - cb] = ld_stream(p.col + ci1 + lane - 16);
        const int vh = (int)(vi0 - s0), vt = (int)(s1 - vi1);
        if (lane < vh) s_val[s0 + lane - vb] = ld_stream(val + s0 + lane);
        else if (lane >= 16 && lane - 16 < vt) s_val[vi1 + lane - 16 - vb] = ld_stream(val + vi1 + lane - 16);
      }
      tma::mbar_arrive(&full_bar[stage]);  // releases this lane's plain stores
      if (++stage == NS) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ consumers
    const double alpha = epi_alpha(p.e);
    int stage = 0;
    uint32_t phase = 0;
    int64_t tile = blockIdx.x;
    int64_t a_nx = 0, b_nx = 0;
    if (tile < ntiles) {
      const int64_t row = tile * B + t;
      if (row < p.rows) {
        a_nx = (int64_t)rp[row];
        b_nx = (int64_t)rp[row + 1];
      }
    }
    for (; tile < ntiles; tile += gridDim.x) {
      const int64_t r0 = tile * B, r1 = r0 + B < p.rows ? r0 + B : p.rows;
      const int64_t row = r0 + t;
      const int64_t a_g = a_nx, b_g = b_nx;
      {  // prefetch the next tile's row bounds
        const int64_t nrow = row + (int64_t)gridDim.x * B;
        if (nrow < p.rows) {
          a_nx = (int64_t)rp[nrow];
          b_nx = (int64_t)rp[nrow + 1];
        }
      }
      tma::mbar_wait(&full_bar[stage], phase);
      const unsigned char* st = smem_raw + (size_t)stage * STAGE;
      if (meta_staged[stage]) {
        // local entry j of the tile sits at s_col[j + oc], s_val[j + ov]
        const int64_t s0 = meta_s0[stage];
        const int32_t* s_col = reinterpret_cast<const int32_t*>(st) + (int)(s0 & 3);
        const T* s_val = reinterpret_cast<const T*>(st + COLB) + (int)(s0 & (VP - 1));
        if (row < r1) {
          double acc = 0.0;
          const int ka = (int)(a_g - s0), kb = (int)(b_g - s0), len = kb - ka;
          // Rows whose length is a multiple of 8 would put the lanes of a warp
          // on the same banks (stride len words): such a row is walked from a
          // lane-dependent rotation. Other lengths (the stencil's 27) keep
          // k-aligned lanes, so the gathers of a step stay on adjacent x.
          int rot = (len & 7) == 0 && len > 0 ? lane : 0;
          if (len > 0 && rot >= len) rot %= len;
          for (int k = 0; k < len; k += U) {
            int c[U];
            T v[U];
#pragma unroll
            for (int j = 0; j < U; ++j) {
              const bool ok = k + j < len;
              int q = k + j + rot;
              q = q >= len ? q - len : q;
              c[j] = ok ? s_col[ka + q] : 0;
              v[j] = ok ? s_val[ka + q] : T(0);
            }
            T xv[U];
#pragma unroll
            for (int j = 0; j < U; ++j) xv[j] = k + j < len ? ld_x(x + c[j]) : T(0);
#pragma unroll
            for (int j = 0; j < U; ++j) acc = fma((double)v[j], (double)xv[j], acc);
          }
          const T out = epi_value<T>(p.e, alpha, acc, y, row);
          y[row] = out;
          if (p.e.mode == 1) {
            yy += (double)out * (double)out;
            xy += (double)x[p.e.row_offset + row] * (double)out;
          }
        }
      } else {
        // long rows: warp per row over global memory, shuffle reduction
        for (int64_t rr = r0 + warp; rr < r1; rr += B / 32) {
          const int64_t a = rp[rr], b = rp[rr + 1];
          double acc = 0.0;
          for (int64_t k = a + lane; k < b; k += 32)
            acc = fma((double)ld_stream(val + k), (double)ld_x(x + ld_stream(p.col + k)), acc);
          acc = warp_sum(acc);
          if (lane == 0) {
            const T out = epi_value<T>(p.e, alpha, acc, y, rr);
            y[rr] = out;
            if (p.e.mode == 1) {
              yy += (double)out * (double)out;
              xy += (double)x[p.e.row_offset + rr] * (double)out;
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&empty_bar[stage]);
      if (++stage == NS) {
        stage = 0;
        phase ^= 1;
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

// Merge-path CSR on row-interleaved tiles. A block owns the merge-path chunk
// of B·IPT items [(x0, y0), (x1, y1)) from the partition pre-pass, so one
// 150K-entry row and thousands of empty rows cost the same per item (the
// load balance of merge-path). The block stages the chunk's entries
// (col, val of [y0, y1), coalesced) and the starts of its rows x0 .. x1
// (clamped to the chunk) in shared memory, then walks the rows thread per
// row: at step k the lanes of a warp gather the k-th entry of 32 consecutive
// rows (adjacent x on banded matrices) instead of staging products and
// walking the merge path per lane (k_csr_merge above), and rows longer than
// kLong entries are summed by a warp. Empty rows are written here too. Row
// x0, if it began before y0, leaves its partial in rec.head; row x1, if it
// has entries here and continues past y1, in rec.tail; k_seg_fixup finishes
// both (deterministic). Same chunk-record semantics as k_csr_merge.
template <int B, int R, class T, int IPT, class RP>
__global__ void __launch_bounds__(B) __maxnreg__(regcap(B, R)) k_csr_merge_tile(const CsrParams p) {
  constexpr int ITEMS = B * IPT;
  constexpr int NW = B / 32;
  constexpr int kLong = 64;
  constexpr int U = 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* s_val = reinterpret_cast<T*>(smem_raw);
  int32_t* s_col = reinterpret_cast<int32_t*>(smem_raw + (size_t)ITEMS * sizeof(T));
  int32_t* s_rs = s_col + ITEMS;  // row starts relative to y0, clamped to [0, nnzc]
  __shared__ int s_nlong;
  __shared__ int s_long[ITEMS / kLong + 1];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t chunk = blockIdx.x;
  const RP* __restrict__ rp = static_cast<const RP*>(p.rp);
  const T* __restrict__ val = static_cast<const T*>(p.val);
  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ y = static_cast<T*>(p.y);
  const int64_t x0 = p.coords[2 * chunk], y0 = p.coords[2 * chunk + 1];
  const int64_t x1 = p.coords[2 * chunk + 2], y1 = p.coords[2 * chunk + 3];
  const int nnzc = (int)(y1 - y0);
  const bool cont_in = x0 < p.rows && y0 > (int64_t)rp[x0];
  const bool cont_out = x1 < p.rows && y1 > (int64_t)rp[x1];
  // rows x0 .. x1-1 end in this chunk; row x1 is here iff it has entries here
  const int nseg = (int)(x1 - x0) + (cont_out ? 1 : 0);
  for (int i = t; i < nnzc; i += B) {
    s_col[i] = ld_stream(p.col + y0 + i);
    s_val[i] = ld_stream(val + y0 + i);
  }
  for (int j = t; j <= nseg; j += B) {
    const int64_t r = x0 + j;
    int64_t v = r <= p.rows ? (int64_t)rp[r] : (int64_t)y1;
    v = v < y0 ? y0 : (v > y1 ? y1 : v);
    s_rs[j] = (int)(v - y0);
  }
  if (t == 0) s_nlong = 0;
  __syncthreads();
  const double alpha = epi_alpha(p.e);
  auto finish = [&](int j, double acc) {
    const int64_t row = x0 + j;
    const bool first = j == 0 && cont_in, last = j == nseg - 1 && cont_out;
    if (first || last) {
      ChunkRec& rec = p.recs[chunk];
      if (first) rec.head = acc;
      if (last) rec.tail = acc;
    } else {
      y[row] = epi_value<T>(p.e, alpha, acc, y, row);
    }
  };
  for (int j = t; j < nseg; j += B) {
    const int a = s_rs[j], len = s_rs[j + 1] - a;
    if (len > kLong) {
      s_long[atomicAdd(&s_nlong, 1)] = j;
      continue;
    }
    int rot = (len & 7) == 0 && len > 0 ? lane : 0;
    if (len > 0 && rot >= len) rot %= len;
    double acc = 0.0;
    for (int k = 0; k < len; k += U) {
      int c[U];
      T v[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        int i = k + q + rot;
        i = i >= len ? i - len : i;
        const bool ok = k + q < len;
        c[q] = ok ? s_col[a + i] : 0;
        v[q] = ok ? s_val[a + i] : T(0);
      }
      T xv[U];
#pragma unroll
      for (int q = 0; q < U; ++q) xv[q] = k + q < len ? ld_x(x + c[q]) : T(0);
#pragma unroll
      for (int q = 0; q < U; ++q) acc = fma((double)v[q], (double)xv[q], acc);
    }
    finish(j, acc);
  }
  __syncthreads();
  const int nlong = s_nlong;
  for (int q = w; q < nlong; q += NW) {
    const int j = s_long[q];
    const int a = s_rs[j], b = s_rs[j + 1];
    double acc = 0.0;
    for (int k = a + lane; k < b; k += 32) acc = fma((double)s_val[k], (double)ld_x(x + s_col[k]), acc);
    acc = warp_sum(acc);
    if (lane == 0) finish(j, acc);
  }
  if (t == 0) {
    ChunkRec& rec = p.recs[chunk];
    rec.first_row = (int32_t)x0;
    rec.cont_in = cont_in;
    rec.last_row = (int32_t)(cont_out ? x1 : (x1 - 1 > x0 ? x1 - 1 : x0));
    rec.cont_out = cont_out;
  }
}

// Pipelined merge-path CSR: the merge-path chunks of k_csr_merge_tile, fed
// by CSR-stream's TMA pipeline. The block is persistent over chunks; one
// producer warp moves each chunk's contiguous col/val segment [y0, y1) and
// its row starts rp[x0 .. x1+1] into a two-stage shared-memory ring with
// cp.async.bulk (16-byte aligned interiors; < 16 B heads/tails by the lanes)
// while the B consumer threads walk the other stage thread per row
// (row-interleaved gathers). Rows longer than kLong entries are cut into
// pieces of kPiece entries that the consumer warps sum with kU gathers in
// flight per lane (a 150K-entry hub row fills whole chunks: every warp works
// on it); the pieces of a row are added in piece order (deterministic).
// Chunk records and the fixup are those of the other merge kernels.
template <int B, int R, class T, int IPT, class RP>
__global__ void __launch_bounds__(B + 32) __maxnreg__(regcap(B + 32, R)) k_csr_merge_stream(const CsrParams p) {
  constexpr int ITEMS = B * IPT;
  constexpr int NS = kStreamStages;
  constexpr int NW = B / 32;
  constexpr int VP = StreamStage<T>::kValPad;
  constexpr int RPP = MergeStage<T, RP>::kRpPad;
  constexpr int U = 8;
  constexpr int kLong = 64, kPiece = 256, kU = 4;
  constexpr int kMaxPieces = ITEMS / kPiece + ITEMS / kLong + 1;
  constexpr size_t STAGE = MergeStage<T, RP>::bytes(ITEMS);
  constexpr size_t COLB = StreamStage<T>::col_bytes(ITEMS);
  constexpr size_t RPOFF = MergeStage<T, RP>::rp_off(ITEMS);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[NS], empty_bar[NS];
  __shared__ int64_t m_x0[NS], m_y0[NS], m_rb[NS];
  __shared__ int m_nseg[NS], m_nnz[NS], m_in[NS], m_out[NS];
  __shared__ int s_nlong, s_npiece;
  __shared__ int s_lrow[ITEMS / kLong + 1], s_lfirst[ITEMS / kLong + 2];
  __shared__ int s_pa[kMaxPieces], s_pb[kMaxPieces];
  __shared__ double s_part[kMaxPieces];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t == 0) {
    for (int s = 0; s < NS; ++s) {
      tma::mbar_init(&full_bar[s], 32);
      tma::mbar_init(&empty_bar[s], NW);
    }
    tma::fence_barrier_init();
  }
  __syncthreads();
  const RP* __restrict__ rp = static_cast<const RP*>(p.rp);
  const T* __restrict__ val = static_cast<const T*>(p.val);
  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ y = static_cast<T*>(p.y);
  const int64_t nchunks = p.nchunks;
  if (warp == NW) {
    // ------------------------------------------------------------ producer
    const uint64_t pol = tma::policy_evict_first();
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      const int64_t x0 = p.coords[2 * c], y0 = p.coords[2 * c + 1];
      const int64_t x1 = p.coords[2 * c + 2], y1 = p.coords[2 * c + 3];
      const bool cin = x0 < p.rows && y0 > (int64_t)rp[x0];
      const bool cout = x1 < p.rows && y1 > (int64_t)rp[x1];
      const int nseg = (int)(x1 - x0) + (cout ? 1 : 0);
      // row starts rp[x0 .. x0 + nseg] (nseg + 1 values, all <= rows)
      const int64_t r0 = x0, r1 = x0 + nseg + 1;
      tma::mbar_wait(&empty_bar[stage], phase ^ 1);
      unsigned char* st = smem_raw + (size_t)stage * STAGE;
      int32_t* s_col = reinterpret_cast<int32_t*>(st);
      T* s_val = reinterpret_cast<T*>(st + COLB);
      RP* s_rp = reinterpret_cast<RP*>(st + RPOFF);
      if (lane == 0) {
        m_x0[stage] = x0;
        m_y0[stage] = y0;
        m_rb[stage] = r0 & ~(int64_t)(RPP - 1);
        m_nseg[stage] = nseg;
        m_nnz[stage] = (int)(y1 - y0);
        m_in[stage] = cin;
        m_out[stage] = cout;
      }
      // aligned interiors by bulk copy, heads/tails (< 16 B) by the lanes
      const int64_t cb = y0 & ~3LL;
      int64_t ci0 = (y0 + 3) & ~3LL, ci1 = y1 & ~3LL;
      if (ci1 <= ci0) ci0 = ci1 = y1;
      const int64_t vb = y0 & ~(int64_t)(VP - 1);
      int64_t vi0 = (y0 + VP - 1) & ~(int64_t)(VP - 1), vi1 = y1 & ~(int64_t)(VP - 1);
      if (vi1 <= vi0) vi0 = vi1 = y1;
      const int64_t rb = r0 & ~(int64_t)(RPP - 1);
      int64_t ri0 = (r0 + RPP - 1) & ~(int64_t)(RPP - 1), ri1 = r1 & ~(int64_t)(RPP - 1);
      if (ri1 <= ri0) ri0 = ri1 = r1;
      if (lane == 0) {
        const uint32_t tx = (uint32_t)((ci1 - ci0) * 4 + (vi1 - vi0) * (int64_t)sizeof(T) +
                                       (ri1 - ri0) * (int64_t)sizeof(RP));
        if (tx) tma::mbar_expect_tx(&full_bar[stage], tx);
        if (ci1 > ci0)
          tma::bulk_g2s(s_col + (ci0 - cb), p.col + ci0, (uint32_t)((ci1 - ci0) * 4), &full_bar[stage], pol);
        if (vi1 > vi0)
          tma::bulk_g2s(s_val + (vi0 - vb), val + vi0, (uint32_t)((vi1 - vi0) * sizeof(T)), &full_bar[stage], pol);
        if (ri1 > ri0)
          tma::bulk_g2s(s_rp + (ri0 - rb), rp + ri0, (uint32_t)((ri1 - ri0) * sizeof(RP)), &full_bar[stage], pol);
      }
      const int ch = (int)(ci0 - y0), ct = (int)(y1 - ci1);
      if (lane < ch) s_col[y0 + lane - cb] = ld_stream(p.col + y0 + lane);
      else if (lane >= 16 && lane - 16 < ct) s_col[ci1 + lane - 16 - cb] = ld_stream(p.col + ci1 + lane - 16);
      const int vh = (int)(vi0 - y0), vt = (int)(y1 - vi1);
      if (lane < vh) s_val[y0 + lane - vb] = ld_stream(val + y0 + lane);
      else if (lane >= 16 && lane - 16 < vt) s_val[vi1 + lane - 16 - vb] = ld_stream(val + vi1 + lane - 16);
      const int rh = (int)(ri0 - r0), rt = (int)(r1 - ri1);
      if (lane < rh) s_rp[r0 + lane - rb] = rp[r0 + lane];
      else if (lane >= 16 && lane - 16 < rt) s_rp[ri1 + lane - 16 - rb] = rp[ri1 + lane - 16];
      tma::mbar_arrive(&full_bar[stage]);
      if (++stage == NS) {
        stage = 0;
        phase ^= 1;
      }
    }
    return;
  }
  // ------------------------------------------------------------ consumers
  const double alpha = epi_alpha(p.e);
  int stage = 0;
  uint32_t phase = 0;
  auto cbar = [] { asm volatile("bar.sync 1, %0;" ::"r"(B) : "memory"); };  // consumer warps only
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    tma::mbar_wait(&full_bar[stage], phase);
    const unsigned char* st = smem_raw + (size_t)stage * STAGE;
    const int64_t y0 = m_y0[stage], x0 = m_x0[stage];
    const int nseg = m_nseg[stage], nnzc = m_nnz[stage];
    const bool cin = m_in[stage], cout = m_out[stage];
    const int32_t* s_col = reinterpret_cast<const int32_t*>(st) + (int)(y0 & 3);
    const T* s_val = reinterpret_cast<const T*>(st + COLB) + (int)(y0 & (VP - 1));
    const RP* s_rp = reinterpret_cast<const RP*>(st + RPOFF) + (int)(x0 - m_rb[stage]);
    auto seg_start = [&](int j) {  // row x0 + j's first entry, relative to y0, clamped to the chunk
      int64_t v = (int64_t)s_rp[j] - y0;
      return (int)(v < 0 ? 0 : (v > nnzc ? nnzc : v));
    };
    auto finish = [&](int j, double acc) {
      const int64_t row = x0 + j;
      const bool first = j == 0 && cin, last = j == nseg - 1 && cout;
      if (first || last) {
        ChunkRec& rec = p.recs[c];
        if (first) rec.head = acc;
        if (last) rec.tail = acc;
      } else {
        y[row] = epi_value<T>(p.e, alpha, acc, y, row);
      }
    };
    if (t == 0) s_nlong = 0;
    cbar();
    for (int j = t; j < nseg; j += B) {
      const int a = seg_start(j), len = seg_start(j + 1) - a;
      if (len > kLong) {
        s_lrow[atomicAdd(&s_nlong, 1)] = j;
        continue;
      }
      int rot = (len & 7) == 0 && len > 0 ? lane : 0;
      if (len > 0 && rot >= len) rot %= len;
      double acc = 0.0;
      for (int k = 0; k < len; k += U) {
        int cc[U];
        T v[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          int i = k + q + rot;
          i = i >= len ? i - len : i;
          const bool ok = k + q < len;
          cc[q] = ok ? s_col[a + i] : 0;
          v[q] = ok ? s_val[a + i] : T(0);
        }
        T xv[U];
#pragma unroll
        for (int q = 0; q < U; ++q) xv[q] = k + q < len ? ld_x(x + cc[q]) : T(0);
#pragma unroll
        for (int q = 0; q < U; ++q) acc = fma((double)v[q], (double)xv[q], acc);
      }
      finish(j, acc);
    }
    cbar();
    const int nlong = s_nlong;
    if (nlong > 0) {
      if (t == 0) {  // pieces of kPiece entries, rows in ascending order (deterministic)
        for (int i = 1; i < nlong; ++i) {  // insertion sort of the (few) long rows
          const int v = s_lrow[i];
          int q = i - 1;
          while (q >= 0 && s_lrow[q] > v) {
            s_lrow[q + 1] = s_lrow[q];
            --q;
          }
          s_lrow[q + 1] = v;
        }
        int np = 0;
        for (int i = 0; i < nlong; ++i) {
          const int a = seg_start(s_lrow[i]), b = seg_start(s_lrow[i] + 1);
          s_lfirst[i] = np;
          for (int q = a; q < b; q += kPiece) {
            s_pa[np] = q;
            s_pb[np] = q + kPiece < b ? q + kPiece : b;
            ++np;
          }
        }
        s_lfirst[nlong] = np;
        s_npiece = np;
      }
      cbar();
      const int np = s_npiece;
      for (int q = warp; q < np; q += NW) {
        const int a = s_pa[q], b = s_pb[q];
        double acc = 0.0;
        for (int k = a + lane; k < b; k += 32 * kU) {
          T v[kU], xv[kU];
          int cc[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int i = k + 32 * u;
            cc[u] = i < b ? s_col[i] : 0;
            v[u] = i < b ? s_val[i] : T(0);
          }
#pragma unroll
          for (int u = 0; u < kU; ++u) xv[u] = k + 32 * u < b ? ld_x(x + cc[u]) : T(0);
#pragma unroll
          for (int u = 0; u < kU; ++u) acc = fma((double)v[u], (double)xv[u], acc);
        }
        acc = warp_sum(acc);
        if (lane == 0) s_part[q] = acc;
      }
      cbar();
      for (int i = t; i < nlong; i += B) {
        double acc = 0.0;
        for (int q = s_lfirst[i]; q < s_lfirst[i + 1]; ++q) acc += s_part[q];
        finish(s_lrow[i], acc);
      }
    }
    if (t == 0) {
      ChunkRec& rec = p.recs[c];
      rec.first_row = (int32_t)x0;
      rec.cont_in = cin;
      const int64_t x1 = x0 + nseg - (cout ? 1 : 0);
      rec.last_row = (int32_t)(cout ? x1 : (x1 - 1 > x0 ? x1 - 1 : x0));
      rec.cont_out = cout;
    }
    // every consumer warp is done with this stage (incl. the long pieces)
    __syncwarp();
    if (lane == 0) tma::mbar_arrive(&empty_bar[stage]);
    if (++stage == NS) {
      stage = 0;
      phase ^= 1;
    }
  }
}

template <int B, int R, class T, int I, class RP>
constexpr CsrFn merge_stream_ptr() {
  if constexpr (B + 32 > 1024 || merge_stream_smem<T, RP>(B, I) > 200 * 1024) return nullptr;
  else return &k_csr_merge_stream<B, R, T, I, RP>;
}

// nnz-split CSR (the merge-path family's load balance over the nonzeros:
// knob kMergeNnz | W). A warp owns the 32·W consecutive entries [base, base +
// 32·W) (every warp the same work, however long or short the rows: P:159's
// imbalance is gone); lane l loads its W entries [base + l·W, ...) with
// 128-bit loads of col and val (the vector loads of COO, without COO's row
// array) and gathers x for all W. The row of each entry comes from the row
// pointers: the cached partition gives the row holding the warp's first
// entry and the row holding the entry after its last, the lane binary-searches
// its first row in that window and, when an entry passes the row's end,
// the next row the same way (empty rows in between cost nothing).
// Runs of one row inside the lane are summed there; runs crossing lanes are
// combined by a 5-step warp segmented scan keyed by the row (COO's
// reduction), rows crossing warps by chunk records + k_seg_fixup, rows
// without entries by a separate pass over the handle's empty-row list.
template <int B, int R, class T, int W, class RP>
__global__ void __launch_bounds__(B) __maxnreg__(regcap(B, R)) k_csr_nnz(const CsrParams p) {
  constexpr int VW = (int)(16 / sizeof(T));  // values per 128-bit load
  const int lane = threadIdx.x & 31;
  const int64_t chunk = ((int64_t)blockIdx.x * B + threadIdx.x) >> 5;
  if (chunk >= p.nchunks) return;  // warp-uniform
  const RP* __restrict__ rp = static_cast<const RP*>(p.rp);
  const T* __restrict__ val = static_cast<const T*>(p.val);
  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ y = static_cast<T*>(p.y);
  const double alpha = epi_alpha(p.e);
  const int64_t base = chunk * 32 * W;
  const int64_t end = base + 32 * W;
  const int64_t k0 = base + (int64_t)lane * W;
  const int64_t rlo = p.coords[chunk], rhi = p.coords[chunk + 1];  // rows holding entries base and end
  int c[W];
  T v[W];
  if (k0 + W <= p.nnz) {
#pragma unroll
    for (int q = 0; q < W; q += 4) {
      int t4[4];
      load_cols<4>(p.col + k0 + q, t4);
#pragma unroll
      for (int u = 0; u < 4; ++u) c[q + u] = t4[u];
    }
#pragma unroll
    for (int q = 0; q < W; q += VW) {
      T tv[VW];
      load_vals<T, VW>(val + k0 + q, tv);
#pragma unroll
      for (int u = 0; u < VW; ++u) v[q + u] = tv[u];
    }
  } else {
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const bool ok = k0 + q < p.nnz;
      c[q] = ok ? p.col[k0 + q] : -1;
      v[q] = ok ? val[k0 + q] : T(0);
    }
  }
  double prod[W];
#pragma unroll
  for (int q = 0; q < W; ++q) prod[q] = c[q] >= 0 ? (double)v[q] * (double)ld_x(x + c[q]) : 0.0;
  // rows of the lane's entries (overlaps the gathers): first row by binary
  // search in [rlo, rhi] (rp[lo] <= k0 < rp[hi + 1]), then forward
  int r[W];
  if (k0 < p.nnz) {
    int64_t lo = rlo, hi = rhi;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if ((int64_t)__ldg(rp + mid) <= k0) lo = mid;
      else hi = mid - 1;
    }
    int64_t row = lo, next = (int64_t)__ldg(rp + row + 1);
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const int64_t k = k0 + q;
      if (k < p.nnz) {
        if (k >= next) {  // a later row (empty rows in between are skipped by the search)
          int64_t a = row + 1, b = rhi;
          while (a < b) {
            const int64_t mid = (a + b + 1) >> 1;
            if ((int64_t)__ldg(rp + mid) <= k) a = mid;
            else b = mid - 1;
          }
          row = a;
          next = (int64_t)__ldg(rp + row + 1);
        }
        r[q] = (int)row;
      } else {
        r[q] = INT_MAX;
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < W; ++q) r[q] = INT_MAX;
  }
  const int chunk_first = (int)rlo;
  const bool cont_in = base > 0 && (int64_t)__ldg(rp + rlo) < base;
  // lane-local runs (as k_coo): rows strictly inside the lane are complete here
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
  if (!first_closed) first_sum = run;
  double s = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double su = __shfl_up_sync(0xffffffffu, s, o);
    const int ku = __shfl_up_sync(0xffffffffu, last, o);
    if (lane >= o && ku == last) s += su;
  }
  const double s_prev = __shfl_up_sync(0xffffffffu, s, 1);
  const int k_prev = __shfl_up_sync(0xffffffffu, last, 1);
  const double carry_in = (lane > 0 && k_prev == first) ? s_prev : 0.0;
  int next_first = __shfl_down_sync(0xffffffffu, r[0], 1);
  if (lane == 31) next_first = end < p.nnz ? (int)rhi : INT_MAX;
  if (first_closed && first != INT_MAX) {
    const double tot = carry_in + first_sum;
    if (cont_in && first == chunk_first) p.recs[chunk].head = tot;
    else y[first] = epi_value<T>(p.e, alpha, tot, y, first);
  }
  if (last != INT_MAX) {
    if (next_first != last) {
      if (cont_in && last == chunk_first) p.recs[chunk].head = s;
      else y[last] = epi_value<T>(p.e, alpha, s, y, last);
    } else if (lane == 31) {
      p.recs[chunk].tail = s;
      if (cont_in && last == chunk_first) p.recs[chunk].head = s;
    }
  }
  const unsigned valid = __ballot_sync(0xffffffffu, r[0] != INT_MAX);
  const int lastv = __shfl_sync(0xffffffffu, last, 31 - __clz((int)valid));
  if (lane == 31) {
    ChunkRec& rec = p.recs[chunk];
    rec.first_row = chunk_first;
    rec.cont_in = cont_in;
    rec.last_row = lastv;
    rec.cont_out = (next_first == last) && last != INT_MAX;
  }
}

// nnz-split CSR with a cached row map (knob kMergeRowmap | 8): the chunks of
// k_csr_nnz (W = 8, 256 entries per warp), but the row of each entry comes
// from a map built once per handle from the row pointers instead of a search:
// one bit per entry marks the first entry of each row (a byte per lane), the
// lane's starts before it are a warp prefix sum of popcounts on top of the
// chunk's cached count, and the ordinal of a row start indexes the list of
// non-empty rows. 0.125 B per entry of map against COO's 4 B of row index;
// no dependent searches.
template <int B, int R, class T, class RP>
__global__ void __launch_bounds__(B) __maxnreg__(regcap(B, R)) k_csr_nnz_map(const CsrParams p) {
  constexpr int W = 8;
  constexpr int VW = (int)(16 / sizeof(T));
  const int lane = threadIdx.x & 31;
  const int64_t chunk = ((int64_t)blockIdx.x * B + threadIdx.x) >> 5;
  if (chunk >= p.nchunks) return;  // warp-uniform
  const T* __restrict__ val = static_cast<const T*>(p.val);
  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ y = static_cast<T*>(p.y);
  const double alpha = epi_alpha(p.e);
  const int64_t base = chunk * 32 * W;
  const int64_t end = base + 32 * W;
  const int64_t k0 = base + (int64_t)lane * W;
  // issue order: row-map words, then the matrix loads, then the prefix scan
  // and the row-id loads (they overlap the matrix loads), then the gathers
  const uint32_t bword = __ldg(p.rm_bits + (k0 >> 5));
  const int64_t ord0 = __ldg(p.rm_ord0 + chunk);
  int c[W];
  T v[W];
  const bool v256 = ((((uintptr_t)p.col | (uintptr_t)p.val) & 31) == 0);  // warp-uniform
  if (k0 + W <= p.nnz && v256) {
    ld_stream256_w<W>(p.col + k0, c);
    ld_stream256_w<W>(val + k0, v);
  } else if (k0 + W <= p.nnz) {
#pragma unroll
    for (int q = 0; q < W; q += 4) {
      int t4[4];
      load_cols<4>(p.col + k0 + q, t4);
#pragma unroll
      for (int u = 0; u < 4; ++u) c[q + u] = t4[u];
    }
#pragma unroll
    for (int q = 0; q < W; q += VW) {
      T tv[VW];
      load_vals<T, VW>(val + k0 + q, tv);
#pragma unroll
      for (int u = 0; u < VW; ++u) v[q + u] = tv[u];
    }
  } else {
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const bool ok = k0 + q < p.nnz;
      c[q] = ok ? p.col[k0 + q] : -1;
      v[q] = ok ? val[k0 + q] : T(0);
    }
  }
  // rows of the lane's entries: row starts (bits beyond nnz are 0) before the
  // lane by a warp prefix sum of popcounts, ids from the non-empty row list
  const unsigned byte = (bword >> (k0 & 31)) & 0xffu;
  const int cnt = __popc(byte);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  int r[W];
  {
    int64_t ord = ord0 + (incl - cnt) - 1;  // ordinal of the row holding the entry before the lane's first
    auto row_of = [&](int64_t o) { return p.rm_identity ? (int)o : __ldg(p.rm_rows + o); };
    int row = ord >= 0 ? row_of(ord) : 0;
#pragma unroll
    for (int q = 0; q < W; ++q) {
      if ((byte >> q) & 1u) row = row_of(++ord);
      r[q] = k0 + q < p.nnz ? row : INT_MAX;
    }
  }
  double prod[W];
#pragma unroll
  for (int q = 0; q < W; ++q) prod[q] = c[q] >= 0 ? (double)v[q] * (double)ld_x(x + c[q]) : 0.0;
  const int chunk_first = __shfl_sync(0xffffffffu, r[0], 0);
  const bool cont_in = base > 0 && !(__shfl_sync(0xffffffffu, byte, 0) & 1u);
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
  if (!first_closed) first_sum = run;
  double s = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double su = __shfl_up_sync(0xffffffffu, s, o);
    const int ku = __shfl_up_sync(0xffffffffu, last, o);
    if (lane >= o && ku == last) s += su;
  }
  const double s_prev = __shfl_up_sync(0xffffffffu, s, 1);
  const int k_prev = __shfl_up_sync(0xffffffffu, last, 1);
  const double carry_in = (lane > 0 && k_prev == first) ? s_prev : 0.0;
  int next_first = __shfl_down_sync(0xffffffffu, r[0], 1);
  if (lane == 31) {
    if (end < p.nnz) {  // the row holding entry `end`: a start there, else the row of the last start before it
      const bool st = (__ldg(p.rm_bits + (end >> 5)) >> (end & 31)) & 1u;
      const int64_t o = __ldg(p.rm_ord0 + chunk + 1) - (st ? 0 : 1);
      next_first = p.rm_identity ? (int)o : __ldg(p.rm_rows + o);
    } else {
      next_first = INT_MAX;
    }
  }
  if (first_closed && first != INT_MAX) {
    const double tot = carry_in + first_sum;
    if (cont_in && first == chunk_first) p.recs[chunk].head = tot;
    else y[first] = epi_value<T>(p.e, alpha, tot, y, first);
  }
  if (last != INT_MAX) {
    if (next_first != last) {
      if (cont_in && last == chunk_first) p.recs[chunk].head = s;
      else y[last] = epi_value<T>(p.e, alpha, s, y, last);
    } else if (lane == 31) {
      p.recs[chunk].tail = s;
      if (cont_in && last == chunk_first) p.recs[chunk].head = s;
    }
  }
  const unsigned valid = __ballot_sync(0xffffffffu, r[0] != INT_MAX);
  const int lastv = __shfl_sync(0xffffffffu, last, 31 - __clz((int)valid));
  if (lane == 31) {
    ChunkRec& rec = p.recs[chunk];
    rec.first_row = chunk_first;
    rec.cont_in = cont_in;
    rec.last_row = lastv;
    rec.cont_out = (next_first == last) && last != INT_MAX;
  }
}

// nnz-split partition: coords[c] = the row holding entry c·per (rows when
// c·per >= nnz): the largest r with rp[r] <= c·per.
template <class RP>
__global__ void k_nnz_partition(const RP* __restrict__ rp, int64_t rows, int64_t nnz, int64_t per, int64_t nchunks,
                                int64_t* __restrict__ coords) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c <= nchunks; c += stride) {
    const int64_t k = c * per < nnz ? c * per : nnz;
    int64_t lo = 0, hi = rows;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if ((int64_t)rp[mid] <= k) lo = mid;
      else hi = mid - 1;
    }
    coords[c] = k >= nnz ? rows : lo;
  }
}

template <int B, int R, class T, int I, class RP>
constexpr CsrFn merge_tile_ptr() {
  if constexpr (merge_tile_smem<T>(B, I) > 200 * 1024) return nullptr;
  else return &k_csr_merge_tile<B, R, T, I, RP>;
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

#define CSRV4_ROW(B, L) {&k_csr_vector4<B, 32, T, L, RP>, &k_csr_vector4<B, 64, T, L, RP>, \
                         &k_csr_vector4<B, 128, T, L, RP>, &k_csr_vector4<B, 255, T, L, RP>}
template <class T, class RP, int L>
CsrFn csr_vector4_fn(int bi, int ri) {
  static const CsrFn tab[5][4] = {CSRV4_ROW(64, L), CSRV4_ROW(128, L), CSRV4_ROW(256, L), CSRV4_ROW(512, L),
                                  CSRV4_ROW(1024, L)};
  return tab[bi][ri];
}
#undef CSRV4_ROW

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

// B + 32 threads per block (one producer warp): B = 1024 has no variant.
template <int B, int R, class T, int E, class RP>
constexpr CsrFn stream_ptr() {
  if constexpr (B + 32 > 1024) return nullptr;
  else return &k_csr_stream<B, R, T, E, RP>;
}
#define CSRS_ROW(B, E) {stream_ptr<B, 32, T, E, RP>(), stream_ptr<B, 64, T, E, RP>(), \
                        stream_ptr<B, 128, T, E, RP>(), stream_ptr<B, 255, T, E, RP>()}
#define CSRS_TAB(E) {CSRS_ROW(64, E), CSRS_ROW(128, E), CSRS_ROW(256, E), CSRS_ROW(512, E), CSRS_ROW(1024, E)}
template <class T, class RP, int E>
CsrFn csr_stream_fn(int bi, int ri) {
  static const CsrFn tab[5][4] = CSRS_TAB(E);
  return tab[bi][ri];
}
#undef CSRS_TAB
#undef CSRS_ROW

#define CSRMS_ROW(B, I) {merge_stream_ptr<B, 32, T, I, RP>(), merge_stream_ptr<B, 64, T, I, RP>(), \
                         merge_stream_ptr<B, 128, T, I, RP>(), merge_stream_ptr<B, 255, T, I, RP>()}
template <class T, class RP, int I>
CsrFn csr_merge_stream_fn(int bi, int ri) {
  static const CsrFn tab[5][4] = {CSRMS_ROW(64, I), CSRMS_ROW(128, I), CSRMS_ROW(256, I), CSRMS_ROW(512, I),
                                  CSRMS_ROW(1024, I)};
  return tab[bi][ri];
}
#undef CSRMS_ROW

#define CSRMT_ROW(B, I) {merge_tile_ptr<B, 32, T, I, RP>(), merge_tile_ptr<B, 64, T, I, RP>(), \
                         merge_tile_ptr<B, 128, T, I, RP>(), merge_tile_ptr<B, 255, T, I, RP>()}
template <class T, class RP, int I>
CsrFn csr_merge_tile_fn(int bi, int ri) {
  static const CsrFn tab[5][4] = {CSRMT_ROW(64, I), CSRMT_ROW(128, I), CSRMT_ROW(256, I), CSRMT_ROW(512, I),
                                  CSRMT_ROW(1024, I)};
  return tab[bi][ri];
}
#undef CSRMT_ROW

#define CSRNM_ROW(B) {&k_csr_nnz_map<B, 32, T, RP>, &k_csr_nnz_map<B, 64, T, RP>, \
                     &k_csr_nnz_map<B, 128, T, RP>, &k_csr_nnz_map<B, 255, T, RP>}
template <class T, class RP>
CsrFn csr_nnz_map_fn(int bi, int ri) {
  static const CsrFn tab[5][4] = {CSRNM_ROW(64), CSRNM_ROW(128), CSRNM_ROW(256), CSRNM_ROW(512), CSRNM_ROW(1024)};
  return tab[bi][ri];
}
#undef CSRNM_ROW

#define CSRN_ROW(B, W) {&k_csr_nnz<B, 32, T, W, RP>, &k_csr_nnz<B, 64, T, W, RP>, \
                        &k_csr_nnz<B, 128, T, W, RP>, &k_csr_nnz<B, 255, T, W, RP>}
template <class T, class RP, int W>
CsrFn csr_nnz_fn(int bi, int ri) {
  static const CsrFn tab[5][4] = {CSRN_ROW(64, W), CSRN_ROW(128, W), CSRN_ROW(256, W), CSRN_ROW(512, W),
                                  CSRN_ROW(1024, W)};
  return tab[bi][ri];
}
#undef CSRN_ROW

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
