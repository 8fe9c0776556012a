// convert.cu — on-device format builds, spmv_convert.
// The paper converts COO to each format on the CPU (c_latency);
// here every build is a handful of bandwidth-bound kernels over the CSR:
//   ELL: column-major [K][n_pad], n_pad = ceil(rows/128)·128,
//        padding (col −1, +0.0) so padding never multiplies x (reading R9);
//   SELL (generalised to SELL-C-sigma, reading R10): sigma-window
//        sort of rows by length (descending, ties by row) via the stable
//        radix sort, slice widths, exclusive scan -> int64 slice_ptr, fill;
//   HYB  (north star; Bell–Garland): ELL part of width K_h + COO tail;
//   COO: expanded row array + the list of empty rows.
#include <algorithm>
#include <cstdlib>

#include "handle.cuh"
#include "primitives.cuh"

namespace spmv {
namespace {

// ---------------------------------------------------------------- ELL
// Column index as stored: int32 column (pad -1), a 16-bit offset from
// origin + row (pad -32768), see spmv_matrix::col_origin, or the 8-bit code
// of that offset in the handle's dictionary (pad 255; map[d + m] = code).
struct Dict8View {
  const uint8_t* map = nullptr;
  int64_t m = 0;
};
template <class IDX>
__device__ __forceinline__ IDX enc_col(int32_t c, int64_t row, int64_t origin, Dict8View dv) {
  if constexpr (sizeof(IDX) == 1) return dv.map[(int64_t)c - origin - row + dv.m];
  else if constexpr (sizeof(IDX) == 2) return (IDX)((int64_t)c - origin - row);
  else return (IDX)c;
}
template <class IDX>
__device__ __forceinline__ IDX pad_col() {
  return sizeof(IDX) == 1 ? (IDX)255 : (sizeof(IDX) == 2 ? (IDX)-32768 : (IDX)-1);
}

// Offset dictionary: flag every offset d = col − origin − row that occurs
// (thread per row), scan the flags into codes, then map[d + m] = code and
// tab[code] = d for the first 255 codes.
template <class RP>
__global__ void k_dict_flags(const RP* __restrict__ rp, const int32_t* __restrict__ col, int64_t rows,
                             int64_t origin, int64_t m, int64_t* __restrict__ flags) {
  // thread per row, a warp on 32 consecutive rows: at step k the lanes read
  // the k-th entry of their rows (the warp's rows share cache lines, so the
  // strided column reads hit L1 after the first), four loads in flight. On a
  // banded matrix the lanes of a step carry the same offset: a per-warp cache
  // of seen offsets in shared memory (512 slots, multiplicative hash: no two
  // offsets of the 5-/27-point stencils of any tested size share a slot;
  // with the earlier 32-slot xor hash 20 of c5's 27 offsets collided and the
  // pass ran at 1.1 TB/s) is a broadcast read, and the rare first sighting
  // reads the flag before writing it (no same-address store storm).
  constexpr int kSlots = 512;
  const int lane = threadIdx.x & 31, warp_in_block = threadIdx.x >> 5;
  __shared__ int32_t s_seen[8][kSlots];  // 256-thread blocks; |d| < 2^31, INT_MIN = empty
  for (int i = lane; i < kSlots; i += 32) s_seen[warp_in_block][i] = INT_MIN;
  __syncwarp();
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r0 = w0 * 32; r0 < rows; r0 += nw * 32) {
    const int64_t r = r0 + lane;
    const int64_t a = r < rows ? (int64_t)rp[r] : 0, b = r < rows ? (int64_t)rp[r + 1] : 0;
    const int64_t base = origin + r;
    for (int64_t k = a; __any_sync(0xffffffffu, k < b); k += 4) {
      int cv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) cv[j] = k + j < b ? col[k + j] : 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (k + j < b) {
          const int32_t d = (int32_t)((int64_t)cv[j] - base);
          const int slot = (int)(((uint32_t)d * 0x165667B1u) >> 23);
          if (s_seen[warp_in_block][slot] != d) {
            int64_t* f = flags + ((int64_t)d + m);
            if (*f == 0) *f = 1;
            s_seen[warp_in_block][slot] = d;
          }
        }
      }
    }
  }
}
__global__ void k_dict_build(const int64_t* __restrict__ flags, const int64_t* __restrict__ codes, int64_t bins,
                             int64_t m, uint8_t* __restrict__ map, int32_t* __restrict__ tab) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < bins; b += stride) {
    const int64_t c = codes[b];
    const bool hit = flags[b] != 0 && c < 255;
    map[b] = hit ? (uint8_t)c : (uint8_t)255;
    if (hit) tab[c] = (int32_t)(b - m);
  }
}

template <class RP, class V, class IDX>
__global__ void k_ell_fill(const RP* __restrict__ rp, const int32_t* __restrict__ col,
                           const V* __restrict__ val, int64_t rows, int64_t K, int64_t n_pad,
                           IDX* __restrict__ colE, V* __restrict__ valE, int64_t origin, Dict8View dv) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pad; i += stride) {
    int64_t a = 0, L = 0;
    if (i < rows) {
      a = rp[i];
      L = rp[i + 1] - a;
      if (L > K) L = K;
    }
    for (int64_t k = 0; k < K; ++k) {
      int64_t pos = k * n_pad + i;
      if (k < L) {
        colE[pos] = enc_col<IDX>(col[a + k], i, origin, dv);
        valE[pos] = val[a + k];
      } else {
        colE[pos] = pad_col<IDX>();
        valE[pos] = V(0);
      }
    }
  }
}

// Largest |column − (origin + row)| over the first and last entry of every
// row (columns are sorted within a row, so these bound all of them).
template <class RP>
__global__ void k_offset_range(const RP* __restrict__ rp, const int32_t* __restrict__ col, int64_t rows,
                               int64_t origin, unsigned long long* out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += stride) {
    const int64_t a = rp[i], b = rp[i + 1];
    if (a == b) continue;
    const int64_t d0 = (int64_t)col[a] - origin - i, d1 = (int64_t)col[b - 1] - origin - i;
    const int64_t e = (d0 < 0 ? -d0 : d0) > (d1 < 0 ? -d1 : d1) ? (d0 < 0 ? -d0 : d0) : (d1 < 0 ? -d1 : d1);
    m = (unsigned long long)e > m ? (unsigned long long)e : m;
  }
  if (m) atomicMax(out, m);
}

// ---------------------------------------------------------------- SELL
template <class RP>
__global__ void k_sell_keys(const RP* __restrict__ rp, int64_t rows, int64_t sigma, int lenbits,
                            int64_t maxlen, uint64_t* __restrict__ keys) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += stride) {
    int64_t L = rp[i + 1] - rp[i];
    keys[i] = ((uint64_t)(i / sigma) << lenbits) | (uint64_t)(maxlen - L);
  }
}

template <class RP>
__global__ void k_sell_widths(const RP* __restrict__ rp, const int32_t* __restrict__ perm, int64_t rows,
                              int64_t C, int64_t ns, int64_t* __restrict__ cw) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = w0; s < ns; s += nw) {  // warp per slice, lanes over its rows
    int64_t w = 0;
    for (int64_t j = lane; j < C; j += 32) {
      const int64_t q = s * C + j;
      if (q < rows) {
        const int64_t i = perm ? perm[q] : q;
        const int64_t L = rp[i + 1] - rp[i];
        w = L > w ? L : w;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int64_t v = __shfl_xor_sync(0xffffffffu, w, o);
      w = v > w ? v : w;
    }
    if (lane == 0) cw[s] = C * w;
  }
}

// Thread per (slice, lane): writes of one step k are coalesced across the
// lanes of a slice; each thread walks its own row's entries in order.
template <class RP, class V, class IDX>
__global__ void k_sell_fill(const RP* __restrict__ rp, const int32_t* __restrict__ col,
                            const V* __restrict__ val, const int32_t* __restrict__ perm, int64_t rows,
                            int64_t C, int64_t ns, const int64_t* __restrict__ sp,
                            IDX* __restrict__ colS, V* __restrict__ valS, int64_t origin, Dict8View dv) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t total = ns * C;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
    const int64_t s = t / C, j = t - s * C;
    const int64_t base = sp[s], w = (sp[s + 1] - base) / C;
    int64_t a = 0, L = 0, i = 0;
    if (t < rows) {
      i = perm ? perm[t] : t;
      a = rp[i];
      L = rp[i + 1] - a;
    }
    for (int64_t k = 0; k < w; ++k) {
      const int64_t pos = base + k * C + j;
      if (k < L) {
        colS[pos] = enc_col<IDX>(col[a + k], i, origin, dv);
        valS[pos] = val[a + k];
      } else {
        colS[pos] = pad_col<IDX>();
        valS[pos] = V(0);
      }
    }
  }
}

__global__ void k_u32_to_i32(const uint32_t* __restrict__ in, int32_t* __restrict__ out, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = (int32_t)in[i];
}

// ---------------------------------------------------------------- per-nnz row lookup
// Row containing entry k: the largest i with rp[i] <= k (empty rows skipped).
template <class RP>
__device__ __forceinline__ int64_t row_of(const RP* rp, int64_t lo, int64_t hi, int64_t k) {
  while (lo < hi) {  // invariant: answer in [lo, hi]
    int64_t mid = lo + (hi - lo + 1) / 2;
    if ((int64_t)rp[mid] <= k) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

constexpr int kExpandThreads = 256;
constexpr int kExpandTile = kExpandThreads * 8;

// mode 0: COO row expansion (out_row[k] = row of k).
// mode 1: HYB tail (entries with in-row rank >= K go to toff[row] + rank − K).
template <class RP, class V>
__global__ void __launch_bounds__(kExpandThreads)
    k_expand(const RP* __restrict__ rp, const int32_t* __restrict__ col, const V* __restrict__ val,
             int64_t rows, int64_t nnz, int mode, int64_t K, const int64_t* __restrict__ toff,
             int32_t* __restrict__ out_row, int32_t* __restrict__ out_col, V* __restrict__ out_val) {
  __shared__ int64_t s_r[2];
  const int64_t k0 = (int64_t)blockIdx.x * kExpandTile;
  const int64_t k1 = min(k0 + kExpandTile, nnz);
  if (threadIdx.x < 2) s_r[threadIdx.x] = row_of(rp, 0, rows - 1, threadIdx.x == 0 ? k0 : k1 - 1);
  __syncthreads();
  const int64_t r0 = s_r[0], r1 = s_r[1];
  for (int64_t k = k0 + threadIdx.x; k < k1; k += kExpandThreads) {
    int64_t r = row_of(rp, r0, r1, k);
    if (mode == 0) {
      out_row[k] = (int32_t)r;
    } else {
      int64_t rank = k - (int64_t)rp[r];
      if (rank >= K) {
        int64_t pos = toff[r] + rank - K;
        out_row[pos] = (int32_t)r;
        out_col[pos] = col[k];
        out_val[pos] = val[k];
      }
    }
  }
}

template <class RP>
__global__ void k_row_counts(const RP* __restrict__ rp, int64_t rows, int mode, int64_t K,
                             int64_t* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += stride) {
    int64_t L = rp[i + 1] - rp[i];
    out[i] = mode == 0 ? (L == 0 ? 1 : 0) : (L > K ? L - K : 0);
  }
}

template <class RP>
__global__ void k_compact_empty(const RP* __restrict__ rp, const int64_t* __restrict__ off, int64_t rows,
                                int32_t* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += stride)
    if (rp[i + 1] == rp[i]) out[off[i]] = (int32_t)i;
}

// ---------------------------------------------------------------- BELL
// Block row I merges the column lists of its b rows (each sorted) and walks
// the distinct block columns J = col / b in increasing order.
template <class RP>
__device__ __forceinline__ int64_t bell_next_block(const RP* rp, const int32_t* col, int64_t r0, int nr, int64_t b,
                                                   const int64_t* pos, int64_t last) {
  int64_t best = -1;
  for (int r = 0; r < nr; ++r) {
    const int64_t k = pos[r];
    if (k < (int64_t)rp[r0 + r + 1]) {
      const int64_t J = col[k] / b;
      if (J > last && (best < 0 || J < best)) best = J;
    }
  }
  return best;
}

template <class RP>
__global__ void k_bell_count(const RP* __restrict__ rp, const int32_t* __restrict__ col, int64_t rows, int64_t b,
                             int64_t nbr, unsigned long long* __restrict__ kb_max) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long local = 0;
  for (int64_t I = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; I < nbr; I += stride) {
    const int64_t r0 = I * b;
    const int nr = (int)(rows - r0 < b ? rows - r0 : b);
    int64_t pos[4];
    for (int r = 0; r < nr; ++r) pos[r] = rp[r0 + r];
    int64_t last = -1, count = 0;
    for (;;) {
      const int64_t J = bell_next_block(rp, col, r0, nr, b, pos, last);
      if (J < 0) break;
      for (int r = 0; r < nr; ++r)
        while (pos[r] < (int64_t)rp[r0 + r + 1] && col[pos[r]] / b == J) ++pos[r];
      last = J;
      ++count;
    }
    local = (unsigned long long)count > local ? (unsigned long long)count : local;
  }
  if (local) atomicMax(kb_max, local);
}

template <class RP, class V>
__global__ void k_bell_fill(const RP* __restrict__ rp, const int32_t* __restrict__ col, const V* __restrict__ val,
                            int64_t rows, int64_t b, int64_t nbr_pad, int64_t kb, int32_t* __restrict__ bcol,
                            V* __restrict__ bval) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t be = b * b;
  for (int64_t I = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; I < nbr_pad; I += stride) {
    const int64_t r0 = I * b;
    const int nr = r0 < rows ? (int)(rows - r0 < b ? rows - r0 : b) : 0;
    int64_t pos[4];
    for (int r = 0; r < nr; ++r) pos[r] = rp[r0 + r];
    int64_t last = -1;
    for (int64_t s = 0; s < kb; ++s) {
      const int64_t J = nr > 0 ? bell_next_block(rp, col, r0, nr, b, pos, last) : -1;
      bcol[s * nbr_pad + I] = (int32_t)J;
      for (int64_t e = 0; e < be; ++e) bval[(s * be + e) * nbr_pad + I] = V(0);
      if (J < 0) continue;
      for (int r = 0; r < nr; ++r)
        while (pos[r] < (int64_t)rp[r0 + r + 1] && col[pos[r]] / b == J) {
          const int64_t c = col[pos[r]] - J * b;
          bval[(s * be + r * b + c) * nbr_pad + I] = val[pos[r]];
          ++pos[r];
        }
      last = J;
    }
  }
}

int64_t read_i64(const int64_t* d, cudaStream_t s) {
  int64_t v = 0;
  d2h_sync(&v, d, sizeof(v), s);
  return v;
}

// Device memory a new layout may use: what the library's stream-ordered pool
// holds unused (reused before it grows) plus, only if that is not enough, the
// device's free memory (cudaMemGetInfo is comparatively slow).
void guard_bytes(double bytes, const char* what) {
  double avail = 0.0;
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t reserved = 0, used = 0;
    if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess && reserved > used)
      avail = (double)(reserved - used);
  }
  if (bytes <= avail) return;
  size_t fr = 0, tot = 0;
  CK(cudaMemGetInfo(&fr, &tot));
  avail += (double)fr;
  if (bytes > 0.95 * avail)
    fail(SPMV_ERR_INFEASIBLE, std::string(what) + ": padded layout needs " + std::to_string(bytes / 1e9) +
                                  " GB, more than 95% of the device memory available (" +
                                  std::to_string(avail / 1e9) + " GB)");
}

void lat_begin(spmv_matrix* h, int fmt) {
  for (int i = 0; i < 2; ++i)
    if (!h->lat_ev[fmt][i]) CK(cudaEventCreate(&h->lat_ev[fmt][i]));
  CK(cudaEventRecord(h->lat_ev[fmt][0], h->stream));
}

void lat_end(spmv_matrix* h, int fmt) {
  CK(cudaEventRecord(h->lat_ev[fmt][1], h->stream));
  h->lat_pending[fmt] = true;
}

template <class RP, class V>
void ell_typed(spmv_matrix* h, int enc) {
  cudaStream_t s = h->stream;
  const int64_t K = h->feat.max_len, n_pad = (h->rows + 127) / 128 * 128;
  const double ib = enc == 2 ? 1.0 : (enc == 1 ? 2.0 : 4.0);
  guard_bytes((double)K * n_pad * (ib + sizeof(V)), "ELL");
  Scratch sc(s);
  int32_t* colE = enc == 0 ? sc.get<int32_t>(K * n_pad) : nullptr;
  int16_t* colE16 = enc == 1 ? sc.get<int16_t>(K * n_pad) : nullptr;
  uint8_t* colE8 = enc == 2 ? sc.get<uint8_t>(K * n_pad) : nullptr;
  V* valE = sc.get<V>(K * n_pad);
  const Dict8View dv{h->dict8_map, h->dict8_m};
  const RP* rp = static_cast<const RP*>(h->row_ptr);
  const V* val = static_cast<const V*>(h->val);
  lat_begin(h, SPMV_FMT_ELL);  // c_latency = device time of the conversion kernels (allocation excluded)
  // 3 resident 256-thread blocks per SM: the warps' strided row reads then
  // stay in L1 (c5 ELL-8 fill 17.8 ms vs 20.3 ms with a full grid, 31.4 with 1)
  static const int fill_bps = [] {
    const char* e = getenv("SPMV_ELL_FILL_BPS");  // measurement override
    return e ? atoi(e) : 3;
  }();
  const unsigned g = grid_for(n_pad, 256, (int64_t)kNumSMs * (fill_bps > 0 ? fill_bps : 32));
  if (enc == 2)
    LAUNCH((k_ell_fill<RP, V, uint8_t>), g, 256, 0, s, rp, h->col, val, h->rows, K, n_pad, colE8, valE,
           h->col_origin, dv);
  else if (enc == 1)
    LAUNCH((k_ell_fill<RP, V, int16_t>), g, 256, 0, s, rp, h->col, val, h->rows, K, n_pad, colE16, valE,
           h->col_origin, dv);
  else
    LAUNCH((k_ell_fill<RP, V, int32_t>), g, 256, 0, s, rp, h->col, val, h->rows, K, n_pad, colE, valE, int64_t(0),
           dv);
  lat_end(h, SPMV_FMT_ELL);
  for (void* p : {(void*)colE, (void*)colE16, (void*)colE8, (void*)valE})
    if (p) sc.keep(p);
  h->ell_K = K;
  h->ell_npad = n_pad;
  h->ell_col = colE;
  h->ell_col16 = colE16;
  h->ell_col8 = colE8;
  h->ell_val = valE;
  h->ell_built = true;
}

template <class RP, class V>
void sell_typed(spmv_matrix* h, int64_t C, int64_t sigma, int enc) {
  cudaStream_t s = h->stream;
  const int64_t rows = h->rows, ns = (rows + C - 1) / C;
  Scratch sc(s);
  const RP* rp = static_cast<const RP*>(h->row_ptr);
  // Near-regular matrices: allocate the upper bound ns·C·max_len up front (no
  // host round trip); the exact slot count stays on the device until asked for.
  const int64_t ub = ns * C * h->feat.max_len;
  const bool use_ub = (double)ub <= 1.25 * (double)h->nnz + (double)(64 << 20) / (4.0 + sizeof(V));
  int32_t* perm = nullptr;
  uint64_t *keys = nullptr, *keys_s = nullptr;
  uint32_t* p32 = nullptr;
  if (sigma > 1 && rows > 0) {
    keys = sc.get<uint64_t>(rows);
    keys_s = sc.get<uint64_t>(rows);
    p32 = sc.get<uint32_t>(rows);
    perm = sc.get<int32_t>(rows);
  }
  int64_t* cw = sc.get<int64_t>(ns);
  int64_t* sp = sc.get<int64_t>(ns + 1);
  int32_t* colS = nullptr;
  int16_t* colS16 = nullptr;
  uint8_t* colS8 = nullptr;
  V* valS = nullptr;
  const double ib = enc == 2 ? 1.0 : (enc == 1 ? 2.0 : 4.0);
  auto alloc_cols = [&](int64_t n) {
    if (enc == 2) colS8 = sc.get<uint8_t>(n);
    else if (enc == 1) colS16 = sc.get<int16_t>(n);
    else colS = sc.get<int32_t>(n);
  };
  if (use_ub) {
    guard_bytes((double)ub * (ib + sizeof(V)), "SELL");
    alloc_cols(ub);
    valS = sc.get<V>(ub);
  }
  lat_begin(h, SPMV_FMT_SELL);  // c_latency = device time of the conversion kernels
  if (perm) {
    const int64_t maxlen = h->feat.max_len;
    int lenbits = bits_for((uint64_t)maxlen);
    int winbits = bits_for((uint64_t)((rows - 1) / sigma));
    LAUNCH(k_sell_keys<RP>, grid_for(rows, 256), 256, 0, s, rp, rows, sigma, lenbits, maxlen, keys);
    radix_sort_pairs(keys, nullptr, keys_s, p32, rows, lenbits + winbits, s);
    LAUNCH(k_u32_to_i32, grid_for(rows, 256), 256, 0, s, (const uint32_t*)p32, perm, rows);
  }
  LAUNCH(k_sell_widths<RP>, grid_for(ns * 32, 256, (int64_t)kNumSMs * 16), 256, 0, s, rp, (const int32_t*)perm,
         rows, C, ns, cw);
  exclusive_scan_i64(cw, sp, ns, s);
  const int64_t slots = use_ub ? ub : read_i64(sp + ns, s);
  if (!use_ub) {
    guard_bytes((double)slots * (ib + sizeof(V)), "SELL");
    alloc_cols(slots);
    valS = sc.get<V>(slots);
  }
  const Dict8View dv{h->dict8_map, h->dict8_m};
  const unsigned g = grid_for(ns * C, 256);
  const V* val = static_cast<const V*>(h->val);
  if (enc == 2)
    LAUNCH((k_sell_fill<RP, V, uint8_t>), g, 256, 0, s, rp, h->col, val, (const int32_t*)perm, rows, C, ns,
           (const int64_t*)sp, colS8, valS, h->col_origin, dv);
  else if (enc == 1)
    LAUNCH((k_sell_fill<RP, V, int16_t>), g, 256, 0, s, rp, h->col, val, (const int32_t*)perm, rows, C, ns,
           (const int64_t*)sp, colS16, valS, h->col_origin, dv);
  else
    LAUNCH((k_sell_fill<RP, V, int32_t>), g, 256, 0, s, rp, h->col, val, (const int32_t*)perm, rows, C, ns,
           (const int64_t*)sp, colS, valS, int64_t(0), dv);
  lat_end(h, SPMV_FMT_SELL);
  for (void* p : {(void*)perm, (void*)sp, (void*)colS, (void*)colS16, (void*)colS8, (void*)valS})
    if (p) sc.keep(p);
  h->sell_col16 = colS16;
  h->sell_col8 = colS8;
  h->sell_C = C;
  h->sell_sigma = sigma;
  h->sell_ns = ns;
  h->sell_slots = slots;
  h->sell_slots_pending = use_ub;
  h->sell_perm = perm;
  h->sell_sp = sp;
  h->sell_col = colS;
  h->sell_val = valS;
  h->sell_built = true;
}

template <class RP, class V>
void hyb_typed(spmv_matrix* h, int64_t K) {
  cudaStream_t s = h->stream;
  const int64_t rows = h->rows, n_pad = (rows + 127) / 128 * 128;
  guard_bytes((double)K * n_pad * (4.0 + sizeof(V)), "HYB");
  Scratch sc(s);
  const RP* rp = static_cast<const RP*>(h->row_ptr);
  int32_t* colE = sc.get<int32_t>(K * n_pad);
  V* valE = sc.get<V>(K * n_pad);
  int64_t* cnt = sc.get<int64_t>(rows);
  int64_t* toff = sc.get<int64_t>(rows + 1);
  lat_begin(h, SPMV_FMT_HYB);  // kernels + the tail-size read-back
  LAUNCH((k_ell_fill<RP, V, int32_t>), grid_for(n_pad, 256), 256, 0, s, rp, h->col, static_cast<const V*>(h->val),
         rows, K, n_pad, colE, valE, int64_t(0), Dict8View{});
  LAUNCH(k_row_counts<RP>, grid_for(rows, 256), 256, 0, s, rp, rows, 1, K, cnt);
  exclusive_scan_i64(cnt, toff, rows, s);
  const int64_t tail = read_i64(toff + rows, s);
  int32_t* trow = sc.get<int32_t>(tail);
  int32_t* tcol = sc.get<int32_t>(tail);
  V* tval = sc.get<V>(tail);
  if (h->nnz > 0 && tail > 0)
    LAUNCH((k_expand<RP, V>), (unsigned)((h->nnz + kExpandTile - 1) / kExpandTile), kExpandThreads, 0, s, rp,
           h->col, static_cast<const V*>(h->val), rows, h->nnz, 1, K, (const int64_t*)toff, trow, tcol, tval);
  lat_end(h, SPMV_FMT_HYB);
  for (void* p : {(void*)colE, (void*)valE, (void*)trow, (void*)tcol, (void*)tval}) sc.keep(p);
  h->hyb_K = K;
  h->hyb_npad = n_pad;
  h->hyb_tail = tail;
  h->hyb_ecol = colE;
  h->hyb_eval = valE;
  h->hyb_trow = trow;
  h->hyb_tcol = tcol;
  h->hyb_tval = tval;
  h->hyb_built = true;
}

template <class RP, class V>
void coo_typed(spmv_matrix* h) {
  cudaStream_t s = h->stream;
  const int64_t rows = h->rows;
  Scratch sc(s);
  const RP* rp = static_cast<const RP*>(h->row_ptr);
  int32_t* crow = sc.get<int32_t>(h->nnz);
  int64_t* flag = sc.get<int64_t>(rows);
  int64_t* off = sc.get<int64_t>(rows + 1);
  lat_begin(h, SPMV_FMT_COO);  // kernels + the empty-row count read-back
  if (h->nnz > 0)
    LAUNCH((k_expand<RP, V>), (unsigned)((h->nnz + kExpandTile - 1) / kExpandTile), kExpandThreads, 0, s, rp,
           h->col, static_cast<const V*>(h->val), rows, h->nnz, 0, (int64_t)0, (const int64_t*)nullptr, crow,
           (int32_t*)nullptr, (V*)nullptr);
  LAUNCH(k_row_counts<RP>, grid_for(rows, 256), 256, 0, s, rp, rows, 0, (int64_t)0, flag);
  exclusive_scan_i64(flag, off, rows, s);
  const int64_t n_empty = read_i64(off + rows, s);
  int32_t* empty = sc.get<int32_t>(n_empty);
  if (n_empty > 0)
    LAUNCH(k_compact_empty<RP>, grid_for(rows, 256), 256, 0, s, rp, (const int64_t*)off, rows, empty);
  lat_end(h, SPMV_FMT_COO);
  sc.keep(crow);
  sc.keep(empty);
  h->coo_row = crow;
  h->coo_empty = empty;
  h->coo_n_empty = n_empty;
  h->coo_built = true;
}

template <class RP, class V>
void bell_typed(spmv_matrix* h, int64_t b) {
  cudaStream_t s = h->stream;
  const int64_t rows = h->rows, nbr = (rows + b - 1) / b, nbr_pad = (nbr + 127) / 128 * 128;
  const RP* rp = static_cast<const RP*>(h->row_ptr);
  Scratch sc(s);
  unsigned long long* d_kb = sc.get<unsigned long long>(1);
  lat_begin(h, SPMV_FMT_BELL);  // kernels + the block-width read-back
  CK(cudaMemsetAsync(d_kb, 0, sizeof(unsigned long long), s));
  if (nbr > 0) LAUNCH(k_bell_count<RP>, grid_for(nbr, 256), 256, 0, s, rp, h->col, rows, b, nbr, d_kb);
  unsigned long long kbu = 0;
  d2h_sync(&kbu, d_kb, sizeof(kbu), s);
  const int64_t kb = (int64_t)kbu;
  guard_bytes((double)kb * nbr_pad * (4.0 + b * b * sizeof(V)), "BELL");
  int32_t* bcol = sc.get<int32_t>(kb * nbr_pad);
  V* bval = sc.get<V>(kb * b * b * nbr_pad);
  if (kb > 0)
    LAUNCH((k_bell_fill<RP, V>), grid_for(nbr_pad, 256), 256, 0, s, rp, h->col, static_cast<const V*>(h->val), rows,
           b, nbr_pad, kb, bcol, bval);
  lat_end(h, SPMV_FMT_BELL);
  sc.keep(bcol);
  sc.keep(bval);
  h->bell_b = b;
  h->bell_kb = kb;
  h->bell_nbr = nbr;
  h->bell_nbr_pad = nbr_pad;
  h->bell_col = bcol;
  h->bell_val = bval;
  h->bell_built = true;
}

template <class F>
void dispatch(spmv_matrix* h, F&& f) {
  if (h->dtype == SPMV_R64F) {
    if (h->rp64) f((int64_t*)nullptr, (double*)nullptr);
    else f((int32_t*)nullptr, (double*)nullptr);
  } else {
    if (h->rp64) f((int64_t*)nullptr, (float*)nullptr);
    else f((int32_t*)nullptr, (float*)nullptr);
  }
}

}  // namespace

// Largest |col − col_origin − row| over the matrix (device pass unless the
// features already hold the bandwidth).
static int64_t max_offset(spmv_matrix* h) {
  if (h->col_origin == 0 && h->have_features) return std::max(h->feat.bw_lower, h->feat.bw_upper);
  if (h->rows == 0 || h->nnz == 0) return 0;
  Scratch sc(h->stream);
  unsigned long long* d = sc.get<unsigned long long>(1);
  CK(cudaMemsetAsync(d, 0, sizeof(unsigned long long), h->stream));
  const unsigned g = grid_for(h->rows, 256);
  if (h->rp64)
    LAUNCH(k_offset_range<int64_t>, g, 256, 0, h->stream, static_cast<const int64_t*>(h->row_ptr), h->col, h->rows,
           h->col_origin, d);
  else
    LAUNCH(k_offset_range<int32_t>, g, 256, 0, h->stream, static_cast<const int32_t*>(h->row_ptr), h->col, h->rows,
           h->col_origin, d);
  unsigned long long m = 0;
  d2h_sync(&m, d, sizeof(m), h->stream);
  return (int64_t)m;
}

bool offsets16_fit(spmv_matrix* h) { return max_offset(h) <= 32767; }

// Offsets wider than this are not dictionary-coded (the flag array would
// exceed 2^23 bins); such matrices are not banded anyway.
constexpr int64_t kDictMaxOffset = 1LL << 22;

int dict8_codes(spmv_matrix* h) {
  if (h->dict8_count >= 0) return h->dict8_count;
  const int64_t m = max_offset(h);
  if (m > kDictMaxOffset) {
    h->dict8_count = 256;
    return h->dict8_count;
  }
  cudaStream_t s = h->stream;
  const int64_t bins = 2 * m + 1;
  Scratch sc(s);
  int64_t* flags = sc.get<int64_t>(bins);
  int64_t* codes = sc.get<int64_t>(bins + 1);
  CK(cudaMemsetAsync(flags, 0, (size_t)bins * sizeof(int64_t), s));
  const unsigned g = grid_for((h->rows + 31) / 32 * 32, 256, (int64_t)kNumSMs * 8);
  if (h->rows > 0) {
    if (h->rp64)
      LAUNCH(k_dict_flags<int64_t>, g, 256, 0, s, static_cast<const int64_t*>(h->row_ptr), h->col, h->rows,
             h->col_origin, m, flags);
    else
      LAUNCH(k_dict_flags<int32_t>, g, 256, 0, s, static_cast<const int32_t*>(h->row_ptr), h->col, h->rows,
             h->col_origin, m, flags);
  }
  exclusive_scan_i64(flags, codes, bins, s);
  const int64_t count = read_i64(codes + bins, s);
  h->dict8_count = (int)std::min<int64_t>(count, 256);
  if (count <= 255) {
    uint8_t* map = sc.get<uint8_t>(bins);
    int32_t* tab = sc.get<int32_t>(256);
    CK(cudaMemsetAsync(tab, 0, 256 * sizeof(int32_t), s));
    LAUNCH(k_dict_build, grid_for(bins, 256), 256, 0, s, (const int64_t*)flags, (const int64_t*)codes, bins, m, map,
           tab);
    sc.keep(map);
    sc.keep(tab);
    h->dict8_map = map;
    h->dict8_tab = tab;
    h->dict8_m = m;
  }
  return h->dict8_count;
}

int resolve_index_auto(spmv_matrix* h) {
  if (dict8_codes(h) <= 255) return 2;
  return offsets16_fit(h) ? 1 : 0;
}

static int resolve_enc(spmv_matrix* h, int index16, const char* what) {
  if (index16 == 0) return 0;
  if (index16 < 0) return resolve_index_auto(h);
  if (index16 == 1 && !offsets16_fit(h))
    fail(SPMV_ERR_UNSUPPORTED, std::string(what) + ": 16-bit column offsets need every |col - row| <= 32767");
  if (index16 == 2 && dict8_codes(h) > 255)
    fail(SPMV_ERR_UNSUPPORTED, std::string(what) + ": 8-bit column codes need at most 255 distinct col - row offsets");
  return index16;
}

void build_ell(spmv_matrix* h, int index16) {
  if (!h->have_features) compute_features(h);
  const int enc = resolve_enc(h, index16, "ELL");
  dispatch(h, [&](auto rpt, auto vt) {
    using RP = std::remove_pointer_t<decltype(rpt)>;
    using V = std::remove_pointer_t<decltype(vt)>;
    ell_typed<RP, V>(h, enc);
  });
}

void build_sell(spmv_matrix* h, int64_t C, int64_t sigma, int index16) {
  if (!h->have_features) compute_features(h);
  const int enc = resolve_enc(h, index16, "SELL");
  dispatch(h, [&](auto rpt, auto vt) {
    using RP = std::remove_pointer_t<decltype(rpt)>;
    using V = std::remove_pointer_t<decltype(vt)>;
    sell_typed<RP, V>(h, C, sigma, enc);
  });
}

void build_hyb(spmv_matrix* h, int64_t K) {
  if (!h->have_features) compute_features(h);
  if (K < 0) K = h->hyb_auto_K;  // an explicit K is used as given (O6), even above max_len
  dispatch(h, [&](auto rpt, auto vt) {
    using RP = std::remove_pointer_t<decltype(rpt)>;
    using V = std::remove_pointer_t<decltype(vt)>;
    hyb_typed<RP, V>(h, K);
  });
}

void build_bell(spmv_matrix* h, int64_t b) {
  dispatch(h, [&](auto rpt, auto vt) {
    using RP = std::remove_pointer_t<decltype(rpt)>;
    using V = std::remove_pointer_t<decltype(vt)>;
    bell_typed<RP, V>(h, b);
  });
}

template <class RP>
void csr_empty_typed(spmv_matrix* h) {
  cudaStream_t s = h->stream;
  const int64_t rows = h->rows;
  Scratch sc(s);
  const RP* rp = static_cast<const RP*>(h->row_ptr);
  int64_t* flag = sc.get<int64_t>(rows);
  int64_t* off = sc.get<int64_t>(rows + 1);
  LAUNCH(k_row_counts<RP>, grid_for(rows, 256), 256, 0, s, rp, rows, 0, (int64_t)0, flag);
  exclusive_scan_i64(flag, off, rows, s);
  const int64_t n_empty = read_i64(off + rows, s);
  int32_t* empty = sc.get<int32_t>(n_empty);
  if (n_empty > 0) LAUNCH(k_compact_empty<RP>, grid_for(rows, 256), 256, 0, s, rp, (const int64_t*)off, rows, empty);
  sc.keep(empty);
  h->csr_empty = empty;
  h->csr_n_empty = n_empty;
}

template <class RP>
__global__ void k_rowmap_marks(const RP* __restrict__ rp, const int64_t* __restrict__ off_empty, int64_t rows,
                               uint32_t* __restrict__ bits, int32_t* __restrict__ nz_rows) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += stride) {
    const int64_t a = rp[r];
    if ((int64_t)rp[r + 1] == a) continue;
    atomicOr(bits + (a >> 5), 1u << (a & 31));
    nz_rows[r - off_empty[r]] = (int32_t)r;
  }
}

// starts in chunk c (256 entries = 8 words)
__global__ void k_rowmap_counts(const uint32_t* __restrict__ bits, int64_t nchunks, int64_t* __restrict__ cnt) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += stride) {
    int64_t n = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) n += __popc(bits[c * 8 + j]);
    cnt[c] = n;
  }
}

template <class RP>
void csr_rowmap_typed(spmv_matrix* h) {
  cudaStream_t s = h->stream;
  const int64_t rows = h->rows, nchunks = (h->nnz + 255) / 256;
  Scratch sc(s);
  const RP* rp = static_cast<const RP*>(h->row_ptr);
  int64_t* flag = sc.get<int64_t>(rows);
  int64_t* off = sc.get<int64_t>(rows + 1);
  LAUNCH(k_row_counts<RP>, grid_for(rows, 256), 256, 0, s, rp, rows, 0, (int64_t)0, flag);
  exclusive_scan_i64(flag, off, rows, s);
  uint32_t* bits = sc.get<uint32_t>(nchunks * 8);
  int32_t* nz_rows = sc.get<int32_t>(rows);
  int64_t* cnt = sc.get<int64_t>(nchunks);
  int64_t* ord0 = sc.get<int64_t>(nchunks + 1);
  CK(cudaMemsetAsync(bits, 0, (size_t)nchunks * 8 * sizeof(uint32_t), s));
  LAUNCH(k_rowmap_marks<RP>, grid_for(rows, 256), 256, 0, s, rp, (const int64_t*)off, rows, bits, nz_rows);
  LAUNCH(k_rowmap_counts, grid_for(nchunks, 256), 256, 0, s, (const uint32_t*)bits, nchunks, cnt);
  exclusive_scan_i64(cnt, ord0, nchunks, s);
  for (void* p : {(void*)bits, (void*)nz_rows, (void*)ord0}) sc.keep(p);
  h->rm_bits = bits;
  h->rm_rows = nz_rows;
  h->rm_ord0 = ord0;
  h->rm_nchunks = nchunks;
}

void build_csr_rowmap(spmv_matrix* h) {
  if (h->rm_nchunks >= 0) return;
  if (h->rp64) csr_rowmap_typed<int64_t>(h);
  else csr_rowmap_typed<int32_t>(h);
}

void build_csr_empty(spmv_matrix* h) {
  if (h->csr_n_empty >= 0) return;
  if (h->rp64) csr_empty_typed<int64_t>(h);
  else csr_empty_typed<int32_t>(h);
}

void build_coo(spmv_matrix* h) {
  dispatch(h, [&](auto rpt, auto vt) {
    using RP = std::remove_pointer_t<decltype(rpt)>;
    using V = std::remove_pointer_t<decltype(vt)>;
    coo_typed<RP, V>(h);
  });
}

void free_format(spmv_matrix* h, int fmt) {
  cudaStream_t s = h->stream;
  auto F = [&](auto*& p) {
    if (p) dfree((void*)p, s);
    p = nullptr;
  };
  switch (fmt) {
    case SPMV_FMT_COO:
      F(h->coo_row); F(h->coo_empty);
      h->coo_built = false;
      break;
    case SPMV_FMT_ELL:
      F(h->ell_col); F(h->ell_col16); F(h->ell_col8); F(h->ell_val);
      h->ell_built = false;
      break;
    case SPMV_FMT_SELL:
      F(h->sell_perm); F(h->sell_sp); F(h->sell_col); F(h->sell_col16); F(h->sell_col8); F(h->sell_val);
      h->sell_built = false;
      h->sell_slots_pending = false;
      break;
    case SPMV_FMT_HYB:
      F(h->hyb_ecol); F(h->hyb_eval); F(h->hyb_trow); F(h->hyb_tcol); F(h->hyb_tval);
      h->hyb_built = false;
      break;
    case SPMV_FMT_CSR:
      F(h->row_ptr); F(h->col); F(h->val);
      break;
    case SPMV_FMT_BELL:
      F(h->bell_col); F(h->bell_val);
      h->bell_built = false;
      break;
  }
}

double format_latency(spmv_matrix* h, int fmt) {
  if (h->lat_pending[fmt]) {
    CK(cudaEventSynchronize(h->lat_ev[fmt][1]));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->lat_ev[fmt][0], h->lat_ev[fmt][1]));
    h->c_latency[fmt] = ms * 1e-3;
    h->lat_pending[fmt] = false;
  }
  return h->c_latency[fmt];
}

int64_t sell_slots(spmv_matrix* h) {
  if (h->sell_built && h->sell_slots_pending) {
    int64_t v = 0;
    d2h_sync(&v, h->sell_sp + h->sell_ns, sizeof(v), h->stream);
    h->sell_slots = v;
    h->sell_slots_pending = false;
  }
  return h->sell_slots;
}

int64_t format_stored_bytes(spmv_matrix* h, int fmt) {
  const int64_t vb = h->vbytes, rpb = h->rp64 ? 8 : 4;
  switch (fmt) {
    case SPMV_FMT_CSR: return (h->rows + 1) * rpb + h->nnz * (4 + vb);
    case SPMV_FMT_COO: return h->nnz * (8 + vb) + h->coo_n_empty * 4;
    case SPMV_FMT_ELL:
      return h->ell_K * h->ell_npad * ((h->ell_col8 ? 1 : (h->ell_col16 ? 2 : 4)) + vb) + (h->ell_col8 ? 1024 : 0);
    case SPMV_FMT_SELL:
      return sell_slots(h) * ((h->sell_col8 ? 1 : (h->sell_col16 ? 2 : 4)) + vb) + (h->sell_ns + 1) * 8 +
             (h->sell_perm ? h->rows * 4 : 0) + (h->sell_col8 ? 1024 : 0);
    case SPMV_FMT_HYB: return h->hyb_K * h->hyb_npad * (4 + vb) + h->hyb_tail * (8 + vb);
    case SPMV_FMT_BELL: return h->bell_kb * h->bell_nbr_pad * (4 + h->bell_b * h->bell_b * vb);
  }
  return 0;
}

}  // namespace spmv
