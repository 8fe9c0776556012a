// spmv_inputs/gen_dev.cu — device twin of gen_host.c (INPUTS ONLY).
// Emits the same triplets and vectors bit-for-bit on the GPU, so large
// configs (SURVEY.md §8(d) c2–c5) can be generated in HBM without a host
// round-trip. Tests check host/device identity on small sizes.
#include <cuda_runtime.h>
#include <stdint.h>
#include "gen_common.h"

#define EXPORT extern "C" __attribute__((visibility("default")))

namespace {

template <class V>
__device__ __forceinline__ void store_val(void* base, int64_t k, double v) {
  static_cast<V*>(base)[k] = (V)v;
}

__global__ void k_stencil_len(int kind, int64_t N, int64_t r0, int64_t r1, int64_t* out) {
  int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < r1) out[r - r0] = gen_stencil_row_len(kind, N, r);
}

template <class V>
__global__ void k_stencil_fill(int kind, int64_t N, int64_t r0, int64_t r1, int64_t row_base,
                               const int64_t* __restrict__ offsets, int32_t* row, int32_t* col,
                               void* val, int random_vals, uint64_t seed) {
  int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= r1) return;
  int32_t c[GEN_MAX_ROW];
  double v[GEN_MAX_ROW];
  int n = gen_stencil_row(kind, N, r, random_vals, seed, c, v);
  int64_t off = offsets[r - r0];
  for (int t = 0; t < n; ++t) {
    row[off + t] = (int32_t)(r - row_base);
    col[off + t] = c[t];
    store_val<V>(val, off + t, v[t]);
  }
}

template <class V>
__global__ void k_uniform(int64_t n, int k, uint64_t seed, int64_t r0, int64_t r1,
                          int64_t row_base, int32_t* row, int32_t* col, void* val) {
  int64_t i = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r1) return;
  int32_t c[64];
  double v[64];
  gen_uniform_row(n, k, seed, i, c, v);
  int64_t off = (i - r0) * (int64_t)k;
  for (int t = 0; t < k; ++t) {
    row[off + t] = (int32_t)(i - row_base);
    col[off + t] = c[t];
    store_val<V>(val, off + t, v[t]);
  }
}

__global__ void k_rmat_keys(int scale, uint64_t seed, uint64_t t1, uint64_t t2, uint64_t t3,
                            int64_t m, uint64_t* keys) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; e < m; e += stride) keys[e] = gen_rmat_edge(scale, seed, (uint64_t)e, t1, t2, t3);
}

template <class V>
__global__ void k_pair_values(int64_t nnz, const int32_t* row, const int32_t* col, uint64_t seed,
                              void* val) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; q < nnz; q += stride)
    store_val<V>(val, q, gen_value(gen_hash3(seed, (uint64_t)row[q], (uint64_t)col[q])));
}

template <class V>
__global__ void k_vector(uint64_t seed, int64_t n, void* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) store_val<V>(out, i, gen_value(gen_hash3(seed, (uint64_t)i, 0)));
}

inline unsigned blocks_for(int64_t n, int b) {
  int64_t g = (n + b - 1) / b;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace

EXPORT int gen_dev_stencil_rowlen(int kind, int64_t N, int64_t r0, int64_t r1, int64_t* out,
                                  void* stream) {
  if (r1 <= r0) return 0;
  k_stencil_len<<<blocks_for(r1 - r0, 256), 256, 0, (cudaStream_t)stream>>>(kind, N, r0, r1, out);
  return (int)cudaGetLastError();
}

EXPORT int gen_dev_stencil_fill(int kind, int64_t N, int64_t r0, int64_t r1, int64_t row_base,
                                const int64_t* offsets, int32_t* row, int32_t* col, void* val,
                                int val_is_f32, int random_vals, uint64_t seed, void* stream) {
  if (r1 <= r0) return 0;
  unsigned g = blocks_for(r1 - r0, 128);
  if (val_is_f32)
    k_stencil_fill<float><<<g, 128, 0, (cudaStream_t)stream>>>(kind, N, r0, r1, row_base, offsets,
                                                               row, col, val, random_vals, seed);
  else
    k_stencil_fill<double><<<g, 128, 0, (cudaStream_t)stream>>>(kind, N, r0, r1, row_base, offsets,
                                                                row, col, val, random_vals, seed);
  return (int)cudaGetLastError();
}

EXPORT int gen_dev_uniform(int64_t n, int k, uint64_t seed, int64_t r0, int64_t r1,
                           int64_t row_base, int32_t* row, int32_t* col, void* val,
                           int val_is_f32, void* stream) {
  if (r1 <= r0) return 0;
  if (k > 64) return -1;
  unsigned g = blocks_for(r1 - r0, 128);
  if (val_is_f32)
    k_uniform<float><<<g, 128, 0, (cudaStream_t)stream>>>(n, k, seed, r0, r1, row_base, row, col, val);
  else
    k_uniform<double><<<g, 128, 0, (cudaStream_t)stream>>>(n, k, seed, r0, r1, row_base, row, col, val);
  return (int)cudaGetLastError();
}

EXPORT int gen_dev_rmat_keys(int scale, int ef, uint64_t seed, uint64_t t1, uint64_t t2,
                             uint64_t t3, uint64_t* keys, void* stream) {
  int64_t m = (int64_t)ef << scale;
  if (m <= 0) return 0;
  unsigned g = blocks_for(m, 256);
  if (g > 148u * 64u) g = 148u * 64u;
  k_rmat_keys<<<g, 256, 0, (cudaStream_t)stream>>>(scale, seed, t1, t2, t3, m, keys);
  return (int)cudaGetLastError();
}

EXPORT int gen_dev_pair_values(int64_t nnz, const int32_t* row, const int32_t* col,
                               uint64_t seed, void* val, int val_is_f32, void* stream) {
  if (nnz <= 0) return 0;
  unsigned g = blocks_for(nnz, 256);
  if (g > 148u * 64u) g = 148u * 64u;
  if (val_is_f32)
    k_pair_values<float><<<g, 256, 0, (cudaStream_t)stream>>>(nnz, row, col, seed, val);
  else
    k_pair_values<double><<<g, 256, 0, (cudaStream_t)stream>>>(nnz, row, col, seed, val);
  return (int)cudaGetLastError();
}

EXPORT int gen_dev_vector(uint64_t seed, int64_t n, void* out, int val_is_f32, void* stream) {
  if (n <= 0) return 0;
  unsigned g = blocks_for(n, 256);
  if (g > 148u * 64u) g = 148u * 64u;
  if (val_is_f32)
    k_vector<float><<<g, 256, 0, (cudaStream_t)stream>>>(seed, n, out);
  else
    k_vector<double><<<g, 256, 0, (cudaStream_t)stream>>>(seed, n, out);
  return (int)cudaGetLastError();
}
