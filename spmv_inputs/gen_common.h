/* spmv_inputs/gen_common.h — seeded synthetic-input generators (INPUTS ONLY).
 *
 * This header holds no arithmetic of the SpMV method: only the counter-based
 * hash and the closed-form stencil/uniform/RMAT structure rules that produce
 * the synthetic matrices and vectors of SURVEY.md §8(d) ("Synthetic inputs").
 * It is shared by the host generator (gen_host.c) and its device twin
 * (gen_dev.cu) so that both emit bit-identical triplets; neither the oracle
 * (oracle/) nor the product library (paper_2302_05662_b200/csrc) includes it.
 *
 * Value rule: h(seed,i,j) = splitmix64(seed ^ splitmix64(i ^ splitmix64(j)));
 * a value is s·(1 + m·2^-20) with s the hash's top bit and m its low 20 bits,
 * so every value lies in ±[1,2), is never zero, and is exact in fp32 and fp64.
 */
#ifndef SPMV_INPUTS_GEN_COMMON_H
#define SPMV_INPUTS_GEN_COMMON_H
#include <stdint.h>

#ifdef __CUDACC__
#define GEN_HD __host__ __device__ __forceinline__
#else
#define GEN_HD static inline
#endif

GEN_HD uint64_t gen_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

GEN_HD uint64_t gen_hash3(uint64_t seed, uint64_t i, uint64_t j) {
  return gen_splitmix64(seed ^ gen_splitmix64(i ^ gen_splitmix64(j)));
}

GEN_HD double gen_value(uint64_t h) {
  double v = 1.0 + (double)(h & 0xFFFFFull) * (1.0 / 1048576.0);
  return (h >> 63) ? -v : v;
}

/* Stencil kinds. 5-point 2-D Laplacian on an N×N grid (row r = y·N + x) and
 * the 27-point 3-D stencil on an N³ grid (row r = (z·N + y)·N + x, HPCG
 * convention). Neighbours are emitted in increasing column order.
 * GEN_BLOCK27 + B (B = 2..4): the 27-point stencil with B unknowns per grid
 * point and dense B×B couplings (row r = p·B + a, columns q·B + b for every
 * neighbour q of p and b < B) — a block-structured matrix (BELL's case). */
enum { GEN_LAP2D = 0, GEN_STENCIL27 = 1, GEN_BLOCK27 = 100 };
#define GEN_MAX_ROW 108

/* Number of entries in row r of the stencil. */
GEN_HD int gen_stencil_row_len(int kind, int64_t N, int64_t r) {
  if (kind > GEN_BLOCK27) {
    const int B = kind - GEN_BLOCK27;
    return B * gen_stencil_row_len(GEN_STENCIL27, N, r / B);
  }
  if (kind == GEN_LAP2D) {
    int64_t y = r / N, x = r % N;
    return 1 + (y > 0) + (y < N - 1) + (x > 0) + (x < N - 1);
  } else {
    int64_t x = r % N, y = (r / N) % N, z = r / (N * N);
    int cx = 1 + (x > 0) + (x < N - 1);
    int cy = 1 + (y > 0) + (y < N - 1);
    int cz = 1 + (z > 0) + (z < N - 1);
    return cx * cy * cz;
  }
}

/* Write row r's entries (columns ascending). Returns the count written.
 * random_vals = 0: Laplacian values (diagonal 4 or 26, neighbours -1).
 * random_vals = 1: values gen_value(h(seed, r, c)) on the same pattern. */
GEN_HD int gen_stencil_row(int kind, int64_t N, int64_t r, int random_vals, uint64_t seed,
                           int32_t* cols, double* vals) {
  int n = 0;
  if (kind > GEN_BLOCK27) {  /* no recursion: device stacks are small */
    const int B = kind - GEN_BLOCK27;
    const int64_t pt = r / B;
    const int64_t x = pt % N, y = (pt / N) % N, z = pt / (N * N);
    for (int dz = -1; dz <= 1; ++dz) {
      const int64_t zz = z + dz;
      if (zz < 0 || zz >= N) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        const int64_t yy = y + dy;
        if (yy < 0 || yy >= N) continue;
        for (int dx = -1; dx <= 1; ++dx) {
          const int64_t xx = x + dx;
          if (xx < 0 || xx >= N) continue;
          const int64_t q = (zz * N + yy) * N + xx;
          for (int b = 0; b < B; ++b) {
            const int64_t c = q * B + b;
            cols[n] = (int32_t)c;
            vals[n] = random_vals ? gen_value(gen_hash3(seed, (uint64_t)r, (uint64_t)c)) : (c == r ? 26.0 * B : -1.0);
            ++n;
          }
        }
      }
    }
    return n;
  }
  if (kind == GEN_LAP2D) {
    int64_t y = r / N, x = r % N;
    int64_t cand[5];
    int ok[5];
    cand[0] = r - N; ok[0] = (y > 0);
    cand[1] = r - 1; ok[1] = (x > 0);
    cand[2] = r;     ok[2] = 1;
    cand[3] = r + 1; ok[3] = (x < N - 1);
    cand[4] = r + N; ok[4] = (y < N - 1);
    for (int t = 0; t < 5; ++t) {
      if (!ok[t]) continue;
      int64_t c = cand[t];
      cols[n] = (int32_t)c;
      vals[n] = random_vals ? gen_value(gen_hash3(seed, (uint64_t)r, (uint64_t)c))
                            : (c == r ? 4.0 : -1.0);
      ++n;
    }
  } else {
    int64_t x = r % N, y = (r / N) % N, z = r / (N * N);
    for (int dz = -1; dz <= 1; ++dz) {
      int64_t zz = z + dz;
      if (zz < 0 || zz >= N) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        int64_t yy = y + dy;
        if (yy < 0 || yy >= N) continue;
        for (int dx = -1; dx <= 1; ++dx) {
          int64_t xx = x + dx;
          if (xx < 0 || xx >= N) continue;
          int64_t c = (zz * N + yy) * N + xx;
          cols[n] = (int32_t)c;
          vals[n] = random_vals ? gen_value(gen_hash3(seed, (uint64_t)r, (uint64_t)c))
                                : (c == r ? 26.0 : -1.0);
          ++n;
        }
      }
    }
  }
  return n;
}

/* Uniform-k row: draws h(seed, i, t) & (n-1) for t = 0,1,... and keeps the
 * first k distinct columns, sorted ascending (n a power of two, k <= 64).
 * Values: gen_value(h(seed + 1, i, c)). */
GEN_HD void gen_uniform_row(int64_t n, int k, uint64_t seed, int64_t i, int32_t* cols,
                            double* vals) {
  int m = 0;
  for (uint64_t t = 0; m < k; ++t) {
    int32_t c = (int32_t)(gen_hash3(seed, (uint64_t)i, t) & (uint64_t)(n - 1));
    int dup = 0;
    for (int q = 0; q < m; ++q) dup |= (cols[q] == c);
    if (!dup) cols[m++] = c;
  }
  for (int a = 1; a < k; ++a) { /* insertion sort */
    int32_t c = cols[a];
    int b = a - 1;
    while (b >= 0 && cols[b] > c) { cols[b + 1] = cols[b]; --b; }
    cols[b + 1] = c;
  }
  for (int a = 0; a < k; ++a) vals[a] = gen_value(gen_hash3(seed + 1, (uint64_t)i, (uint64_t)cols[a]));
}

/* RMAT edge e (Graph500 recursion): at each of `scale`
 * levels draw u = h(seed, e, level) >> 11 (53 bits) and pick the quadrant by
 * the integer thresholds t1 < t2 < t3 (= floor(2^53·a), ·(a+b), ·(a+b+c)).
 * Returns (row << 32) | col. */
GEN_HD uint64_t gen_rmat_edge(int scale, uint64_t seed, uint64_t e, uint64_t t1, uint64_t t2,
                              uint64_t t3) {
  uint64_t r = 0, c = 0;
  for (int l = 0; l < scale; ++l) {
    uint64_t u = gen_hash3(seed, e, (uint64_t)l) >> 11;
    uint64_t rb = (u >= t2) ? 1u : 0u;                 /* quadrants c, d: lower half */
    uint64_t cb = (u >= t1 && u < t2) || (u >= t3) ? 1u : 0u; /* quadrants b, d: right half */
    r = (r << 1) | rb;
    c = (c << 1) | cb;
  }
  return (r << 32) | c;
}

#endif
