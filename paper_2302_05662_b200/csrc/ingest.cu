// ingest.cu — spmv_create's device path (SURVEY.md §8(a) rows a1–a2):
// copy the COO triplets ("the default sparse format ... in SuiteSparse",
// P:1285) into handle-owned buffers, validate bounds, detect order and
// duplicates, and build CSR row pointers ("The boundaries of each row are
// saved in a third array called Row Index") — fused into ONE pass
// over the triplets when the input is already sorted (28 B/nnz for fp64).
// Unsorted input is radix-sorted by (row, col) first.
#include <algorithm>
#include <cstdlib>

#include "handle.cuh"
#include "primitives.cuh"

namespace spmv {
namespace {

enum : unsigned { F_RANGE = 1u, F_UNSORTED = 2u, F_DUP = 4u };

struct Gap {
  int64_t lo, hi, value;  // row_ptr[lo..hi] = value
};
constexpr int64_t kShortGap = 32;

template <class RP>
__device__ __forceinline__ void fill_rows(RP* row_ptr, int64_t lo, int64_t hi, int64_t value, Gap* gaps,
                                          unsigned long long* ngaps, int64_t cap) {
  if (hi < lo) return;
  if (hi - lo + 1 <= kShortGap) {
    for (int64_t i = lo; i <= hi; ++i) row_ptr[i] = (RP)value;
  } else {
    unsigned long long g = atomicAdd(ngaps, 1ull);
    if ((int64_t)g < cap) gaps[g] = Gap{lo, hi, value};
  }
}

// One pass over the triplets: bounds check, order/duplicate check against the
// predecessor, row-pointer boundary fill, and (copy mode) copy of col/val into
// the handle. Each thread handles 4 consecutive entries (128-bit loads when
// every pointer is 16-byte aligned).
template <class RP, class V, bool VEC>
__global__ void __launch_bounds__(256) k_check(const int32_t* __restrict__ R, const int32_t* __restrict__ Cc,
                                               const V* __restrict__ Vin, int32_t* __restrict__ col_out,
                                               V* __restrict__ val_out, int64_t nnz, int64_t rows,
                                               int64_t cols, RP* __restrict__ row_ptr, unsigned* flags,
                                               Gap* gaps, unsigned long long* ngaps, int64_t gap_cap) {
  unsigned f = 0;
  const int64_t stride = 4LL * gridDim.x * blockDim.x;
  for (int64_t k0 = 4LL * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); k0 < nnz; k0 += stride) {
    int r[4], c[4];
    const bool full = k0 + 3 < nnz;
    if (VEC && full) {
      int4 rr = ld_stream(reinterpret_cast<const int4*>(R + k0));
      int4 cc = ld_stream(reinterpret_cast<const int4*>(Cc + k0));
      r[0] = rr.x; r[1] = rr.y; r[2] = rr.z; r[3] = rr.w;
      c[0] = cc.x; c[1] = cc.y; c[2] = cc.z; c[3] = cc.w;
      if (col_out) {
        *reinterpret_cast<int4*>(col_out + k0) = cc;
        if constexpr (sizeof(V) == 8) {
          double2 a = ld_stream(reinterpret_cast<const double2*>(Vin + k0));
          double2 b = ld_stream(reinterpret_cast<const double2*>(Vin + k0 + 2));
          reinterpret_cast<double2*>(val_out + k0)[0] = a;
          reinterpret_cast<double2*>(val_out + k0)[1] = b;
        } else {
          float4 a = ld_stream(reinterpret_cast<const float4*>(Vin + k0));
          *reinterpret_cast<float4*>(val_out + k0) = a;
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int64_t k = k0 + q;
        r[q] = k < nnz ? R[k] : 0;
        c[q] = k < nnz ? Cc[k] : 0;
        if (col_out && k < nnz) {
          col_out[k] = c[q];
          val_out[k] = Vin[k];
        }
      }
    }
    // the predecessor of entry k0 is the last entry of the previous lane
    // (consecutive lanes own consecutive groups of 4): a shuffle, and only
    // lane 0 reads it from memory (the previous lane's streaming loads did not
    // allocate in L1, so a load would be one more L2 request per thread)
    const int lane = threadIdx.x & 31;
    const int64_t kw = k0 - 4LL * lane;  // the warp's first entry in this iteration
    const int64_t left = (nnz - kw + 3) / 4;  // lanes of the warp still in the loop (a prefix)
    const unsigned am = left >= 32 ? 0xffffffffu : ((1u << left) - 1u);
    int pr = __shfl_up_sync(am, r[3], 1), pc = __shfl_up_sync(am, c[3], 1);
    if (lane == 0) {
      pr = k0 > 0 ? R[k0 - 1] : -1;
      pc = k0 > 0 ? Cc[k0 - 1] : -1;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int64_t k = k0 + q;
      if (k >= nnz) break;
      bool ok = r[q] >= 0 && r[q] < rows && c[q] >= 0 && c[q] < cols;
      if (!ok) f |= F_RANGE;
      if (k > 0) {
        if (r[q] < pr || (r[q] == pr && c[q] < pc)) f |= F_UNSORTED;
        else if (r[q] == pr && c[q] == pc) f |= F_DUP;
      }
      bool pok = (k == 0) || (pr >= 0 && pr < rows);
      if (ok && pok) fill_rows(row_ptr, k == 0 ? 0 : (int64_t)pr + 1, (int64_t)r[q], k, gaps, ngaps, gap_cap);
      if (ok && k == nnz - 1) fill_rows(row_ptr, (int64_t)r[q] + 1, rows, nnz, gaps, ngaps, gap_cap);
      pr = r[q];
      pc = c[q];
    }
  }
  if (f) atomicOr(flags, f);
}

template <class RP>
__global__ void k_fill_gaps(RP* __restrict__ row_ptr, const Gap* __restrict__ gaps,
                            const unsigned long long* ngaps, int64_t cap) {
  int64_t n = (int64_t)*ngaps;
  if (n > cap) n = cap;
  for (int64_t g = blockIdx.x; g < n; g += gridDim.x) {
    Gap q = gaps[g];
    for (int64_t i = q.lo + threadIdx.x; i <= q.hi; i += blockDim.x) row_ptr[i] = (RP)q.value;
  }
}

template <class RP>
__global__ void k_zero_rp(RP* row_ptr, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) row_ptr[i] = 0;
}

__global__ void k_make_keys(const int32_t* __restrict__ R, const int32_t* __restrict__ Cc,
                            uint64_t* __restrict__ keys, int64_t nnz, int colbits) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < nnz; i += stride) keys[i] = ((uint64_t)(uint32_t)R[i] << colbits) | (uint64_t)(uint32_t)Cc[i];
}

template <class V>
__global__ void k_unpack(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ perm,
                         const V* __restrict__ vsrc, int32_t* __restrict__ R, int32_t* __restrict__ Cc,
                         V* __restrict__ vdst, int64_t nnz, int colbits) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t mask = colbits >= 64 ? ~0ull : ((1ull << colbits) - 1);
  for (; i < nnz; i += stride) {
    uint64_t k = keys[i];
    R[i] = (int32_t)(k >> colbits);
    Cc[i] = (int32_t)(k & mask);
    vdst[i] = vsrc[perm[i]];
  }
}

inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

template <class RP, class V>
unsigned run_check(spmv_matrix* h, const int32_t* R, const int32_t* Cc, const V* Vin, int32_t* col_out,
                   V* val_out, unsigned* d_flags, Gap* gaps, unsigned long long* ngaps, int64_t cap) {
  cudaStream_t s = h->stream;
  CK(cudaMemsetAsync(d_flags, 0, sizeof(unsigned), s));
  CK(cudaMemsetAsync(ngaps, 0, sizeof(unsigned long long), s));
  RP* rp = static_cast<RP*>(h->row_ptr);
  bool vec = aligned16(R) && aligned16(Cc) && (!col_out || (aligned16(Vin) && aligned16(col_out) &&
                                                             aligned16(val_out)));
  unsigned grid = grid_for((h->nnz + 3) / 4, 256, (int64_t)kNumSMs * 16);
  if (vec)
    LAUNCH((k_check<RP, V, true>), grid, 256, 0, s, R, Cc, Vin, col_out, val_out, h->nnz, h->rows,
           h->cols, rp, d_flags, gaps, ngaps, cap);
  else
    LAUNCH((k_check<RP, V, false>), grid, 256, 0, s, R, Cc, Vin, col_out, val_out, h->nnz, h->rows,
           h->cols, rp, d_flags, gaps, ngaps, cap);
  LAUNCH(k_fill_gaps<RP>, kNumSMs * 4, 256, 0, s, rp, (const Gap*)gaps, (const unsigned long long*)ngaps, cap);
  unsigned flags = 0;
  d2h_sync(&flags, d_flags, sizeof(unsigned), s);
  return flags;
}

template <class RP, class V>
void ingest_typed(spmv_matrix* h, const int32_t* row_idx, const int32_t* col_idx, const V* vals,
                  spmv_mem_t where) {
  cudaStream_t s = h->stream;
  const int64_t nnz = h->nnz;
  h->row_ptr = dalloc_n<RP>(h->rows + 1, s);
  h->col = dalloc_n<int32_t>(nnz, s);
  h->val = dalloc_n<V>(nnz, s);
  if (nnz == 0) {
    LAUNCH(k_zero_rp<RP>, grid_for(h->rows + 1, 256), 256, 0, s, static_cast<RP*>(h->row_ptr), h->rows + 1);
    CK(cudaStreamSynchronize(s));
    return;
  }
  Scratch sc(s);
  V* hval = static_cast<V*>(h->val);
  const int32_t* R;
  const int32_t* Cc;
  const V* Vsrc;
  int32_t* r_tmp = nullptr;
  bool copy_mode;
  if (where == SPMV_MEM_HOST) {
    r_tmp = sc.get<int32_t>(nnz);
    // 64 MB pieces: another stream's copies (e.g. the next handle's vector
    // upload) interleave instead of queueing behind a whole-matrix upload
    auto upload = [&](void* dst, const void* src, size_t bytes) {
      constexpr size_t kPiece = (size_t)64 << 20;
      for (size_t off = 0; off < bytes; off += kPiece)
        CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off,
                           std::min(kPiece, bytes - off), cudaMemcpyHostToDevice, s));
    };
    upload(r_tmp, row_idx, nnz * sizeof(int32_t));
    upload(h->col, col_idx, nnz * sizeof(int32_t));
    upload(hval, vals, nnz * sizeof(V));
    R = r_tmp;
    Cc = h->col;
    Vsrc = hval;
    copy_mode = false;
  } else {
    R = row_idx;
    Cc = col_idx;
    Vsrc = vals;
    copy_mode = true;
  }
  const int64_t cap = (h->rows + 1) / (kShortGap + 1) + 2;
  unsigned* d_flags = sc.get<unsigned>(1);
  unsigned long long* ngaps = sc.get<unsigned long long>(1);
  Gap* gaps = sc.get<Gap>(cap);

  unsigned flags = run_check<RP, V>(h, R, Cc, Vsrc, copy_mode ? h->col : nullptr,
                                    copy_mode ? hval : nullptr, d_flags, gaps, ngaps, cap);
  if (flags & F_RANGE) fail(SPMV_ERR_INDEX_OUT_OF_RANGE, "spmv_create: a triplet lies outside [0,rows)x[0,cols)");
  if (!(flags & F_UNSORTED)) {
    if (flags & F_DUP) fail(SPMV_ERR_DUPLICATE, "spmv_create: repeated (row, col) coordinate");
    return;
  }
  // Unsorted: sort (row, col) keys on the device, then re-run the fused pass.
  if (nnz >= (int64_t)1 << 32) fail(SPMV_ERR_UNSUPPORTED, "spmv_create: unsorted input with nnz >= 2^32");
  int colbits = bits_for((uint64_t)(h->cols > 0 ? h->cols - 1 : 0));
  int rowbits = bits_for((uint64_t)(h->rows > 0 ? h->rows - 1 : 0));
  uint64_t* keys = sc.get<uint64_t>(nnz);
  uint64_t* keys_s = sc.get<uint64_t>(nnz);
  uint32_t* perm = sc.get<uint32_t>(nnz);
  int32_t* r_sorted = sc.get<int32_t>(nnz);
  V* v_new = sc.get<V>(nnz);
  LAUNCH(k_make_keys, grid_for(nnz, 256), 256, 0, s, R, Cc, keys, nnz, colbits);
  radix_sort_pairs(keys, nullptr, keys_s, perm, nnz, rowbits + colbits, s);
  LAUNCH(k_unpack<V>, grid_for(nnz, 256), 256, 0, s, (const uint64_t*)keys_s, (const uint32_t*)perm, Vsrc,
         r_sorted, h->col, v_new, nnz, colbits);
  CK(cudaStreamSynchronize(s));
  dfree(h->val, s);
  h->val = v_new;
  sc.keep(v_new);
  flags = run_check<RP, V>(h, r_sorted, h->col, v_new, nullptr, nullptr, d_flags, gaps, ngaps, cap);
  if (flags & F_DUP) fail(SPMV_ERR_DUPLICATE, "spmv_create: repeated (row, col) coordinate");
  if (flags & (F_UNSORTED | F_RANGE)) fail(SPMV_ERR_CUDA, "spmv_create: internal sort failure");
}

}  // namespace

namespace {
template <class RI, class RO>
__global__ void k_slice_rp(const RI* __restrict__ in, int64_t r0, int64_t n, RO* __restrict__ out) {
  const int64_t base = (int64_t)in[r0];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = (RO)((int64_t)in[r0 + i] - base);
}

template <class RI>
void slice_rp(const spmv_matrix* p, spmv_matrix* h, int64_t r0) {
  const unsigned g = grid_for(h->rows + 1, 256);
  if (h->rp64)
    LAUNCH((k_slice_rp<RI, int64_t>), g, 256, 0, h->stream, static_cast<const RI*>(p->row_ptr), r0, h->rows + 1,
           static_cast<int64_t*>(h->row_ptr));
  else
    LAUNCH((k_slice_rp<RI, int32_t>), g, 256, 0, h->stream, static_cast<const RI*>(p->row_ptr), r0, h->rows + 1,
           static_cast<int32_t*>(h->row_ptr));
}
}  // namespace

// Row block [r0, r1) of the parent's CSR as a new handle (the interior/halo
// split of the distributed power iteration). The row
// pointers are rebased to 0; col/val are copied (the slice owns its memory).
spmv_matrix* make_row_slice(spmv_matrix* p, int64_t r0, int64_t r1) {
  cudaStream_t s = p->stream;
  int64_t lohi[2] = {0, 0};
  if (p->rp64) {
    CK(cudaMemcpyAsync(&lohi[0], static_cast<int64_t*>(p->row_ptr) + r0, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&lohi[1], static_cast<int64_t*>(p->row_ptr) + r1, 8, cudaMemcpyDeviceToHost, s));
  } else {
    int32_t t[2];
    CK(cudaMemcpyAsync(&t[0], static_cast<int32_t*>(p->row_ptr) + r0, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&t[1], static_cast<int32_t*>(p->row_ptr) + r1, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    lohi[0] = t[0];
    lohi[1] = t[1];
  }
  CK(cudaStreamSynchronize(s));
  spmv_matrix* h = new spmv_matrix();
  h->device = p->device;
  h->stream = s;
  h->dtype = p->dtype;
  h->vbytes = p->vbytes;
  h->rows = r1 - r0;
  h->cols = p->cols;
  h->nnz = lohi[1] - lohi[0];
  for (auto& L : h->launch) L = spmv_launch_t{0, 0, -1, 0};
  try {
    h->rp64 = p->rp64 && h->nnz > 0 && (h->nnz > (int64_t)INT32_MAX || (getenv("SPMV_FORCE_RP64") && getenv("SPMV_FORCE_RP64")[0] == '1'));
    h->row_ptr = h->rp64 ? (void*)dalloc_n<int64_t>(h->rows + 1, s) : (void*)dalloc_n<int32_t>(h->rows + 1, s);
    h->col = dalloc_n<int32_t>(h->nnz, s);
    h->val = dalloc((size_t)std::max<int64_t>(h->nnz, 1) * h->vbytes, s);
    if (p->rp64) slice_rp<int64_t>(p, h, r0);
    else slice_rp<int32_t>(p, h, r0);
    if (h->nnz > 0) {
      CK(cudaMemcpyAsync(h->col, p->col + lohi[0], (size_t)h->nnz * 4, cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(h->val, static_cast<const char*>(p->val) + lohi[0] * p->vbytes,
                         (size_t)h->nnz * p->vbytes, cudaMemcpyDeviceToDevice, s));
    }
  } catch (...) {
    dfree(h->row_ptr, s);
    dfree(h->col, s);
    dfree(h->val, s);
    delete h;
    throw;
  }
  return h;
}

void ingest(spmv_matrix* h, const int32_t* row_idx, const int32_t* col_idx, const void* vals,
            spmv_mem_t where) {
  // int64 row pointers iff nnz >= 2^31; SPMV_FORCE_RP64=1 forces them (testing the int64 paths)
  static const bool force64 = [] {
    const char* e = getenv("SPMV_FORCE_RP64");
    return e && e[0] == '1';
  }();
  h->rp64 = force64 || h->nnz > (int64_t)INT32_MAX;
  if (h->dtype == SPMV_R64F) {
    if (h->rp64)
      ingest_typed<int64_t, double>(h, row_idx, col_idx, static_cast<const double*>(vals), where);
    else
      ingest_typed<int32_t, double>(h, row_idx, col_idx, static_cast<const double*>(vals), where);
  } else {
    if (h->rp64)
      ingest_typed<int64_t, float>(h, row_idx, col_idx, static_cast<const float*>(vals), where);
    else
      ingest_typed<int32_t, float>(h, row_idx, col_idx, static_cast<const float*>(vals), where);
  }
}

}  // namespace spmv
