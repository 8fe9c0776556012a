/* spmv_inputs/gen_host.c — host generators for the synthetic inputs of
 * SURVEY.md §8(d) (INPUTS ONLY: no arithmetic of the SpMV method lives here).
 * Every matrix is emitted as COO triplets sorted by (row, col) with unique
 * coordinates; rows are written relative to `row_base` so a caller can cut a
 * row slab [r0, r1) out of a larger matrix. Values are always written as
 * double (they are exact in fp32 too, see gen_common.h). */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include "gen_common.h"

#define EXPORT __attribute__((visibility("default")))

EXPORT int64_t gen_stencil_nnz(int kind, int64_t N, int64_t r0, int64_t r1) {
  int64_t s = 0;
  for (int64_t r = r0; r < r1; ++r) s += gen_stencil_row_len(kind, N, r);
  return s;
}

EXPORT void gen_stencil(int kind, int64_t N, int64_t r0, int64_t r1, int64_t row_base,
                        int random_vals, uint64_t seed, int32_t* row, int32_t* col,
                        double* val) {
  int64_t k = 0;
  for (int64_t r = r0; r < r1; ++r) {
    int n = gen_stencil_row(kind, N, r, random_vals, seed, col + k, val + k);
    for (int t = 0; t < n; ++t) row[k + t] = (int32_t)(r - row_base);
    k += n;
  }
}

EXPORT void gen_uniform(int64_t n, int k, uint64_t seed, int64_t r0, int64_t r1,
                        int64_t row_base, int32_t* row, int32_t* col, double* val) {
#pragma omp parallel for schedule(static)
  for (int64_t i = r0; i < r1; ++i) {
    int64_t off = (i - r0) * (int64_t)k;
    gen_uniform_row(n, k, seed, i, col + off, val + off);
    for (int t = 0; t < k; ++t) row[off + t] = (int32_t)(i - row_base);
  }
}

EXPORT void gen_vector(uint64_t seed, int64_t n, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = gen_value(gen_hash3(seed, (uint64_t)i, 0));
}

/* LSD radix sort of 64-bit keys, 16-bit digits (generator-private). */
static void gen_sort_u64(uint64_t* a, int64_t n) {
  uint64_t* tmp = (uint64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(uint64_t));
  int64_t* cnt = (int64_t*)malloc(65536 * sizeof(int64_t));
  for (int pass = 0; pass < 4; ++pass) {
    int sh = 16 * pass;
    memset(cnt, 0, 65536 * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) cnt[(a[i] >> sh) & 0xFFFF]++;
    int64_t s = 0;
    for (int d = 0; d < 65536; ++d) { int64_t c = cnt[d]; cnt[d] = s; s += c; }
    for (int64_t i = 0; i < n; ++i) tmp[cnt[(a[i] >> sh) & 0xFFFF]++] = a[i];
    uint64_t* t = a; a = tmp; tmp = t;
  }
  /* four passes: data is back in the original buffer */
  free(tmp);
  free(cnt);
}

/* RMAT(scale, edgefactor): generate ef·2^scale edges, sort, drop duplicates.
 * Self-loops are kept. Writes at most ef·2^scale triplets; returns the count.
 * Values: gen_value(h(seed + 1, r, c)). */
EXPORT int64_t gen_rmat(int scale, int ef, uint64_t seed, uint64_t t1, uint64_t t2, uint64_t t3,
                        int32_t* row, int32_t* col, double* val) {
  int64_t m = (int64_t)ef << scale;
  uint64_t* keys = (uint64_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(uint64_t));
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < m; ++e) keys[e] = gen_rmat_edge(scale, seed, (uint64_t)e, t1, t2, t3);
  gen_sort_u64(keys, m);
  int64_t k = 0;
  for (int64_t e = 0; e < m; ++e) {
    if (e > 0 && keys[e] == keys[e - 1]) continue;
    row[k] = (int32_t)(keys[e] >> 32);
    col[k] = (int32_t)(keys[e] & 0xFFFFFFFFull);
    ++k;
  }
  free(keys);
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < k; ++q)
    val[q] = gen_value(gen_hash3(seed + 1, (uint64_t)row[q], (uint64_t)col[q]));
  return k;
}
