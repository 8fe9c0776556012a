/* oracle/oracle.c — the CPU ORACLE for the B200 SpMV path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / `--impl reference` leg may load this library.
 * The product (paper_2302_05662_b200/) never links, imports or calls it, and
 * this file shares no code, header, table or constant generator with it.
 *
 * Plain, slow, obviously-correct C in fp64, written from the paper's
 * definitions as read in SURVEY.md §8(c) (items O1–O12, plus O13 BELL) and DESIGN.md
 * "Readings". Citations: P:n = /root/reference/PAPER.md line n,
 * S:n = /root/reference/SPEC.md line n (interfaces/test ideas only).
 *
 * Pins (what checks this file against something other than itself) live in
 * tests/test_oracle_pins.py; every function below lists its pins. Parity of
 * format *choices* (tuner/selector) is "parity unpinned" — see DESIGN.md.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EXPORT __attribute__((visibility("default")))

/* Oracle status codes (own numbering; tests map them by name). */
enum {
  ORACLE_OK = 0,
  ORACLE_INVALID_ARG = 1,
  ORACLE_INDEX_OUT_OF_RANGE = 2,
  ORACLE_DUPLICATE = 3,
  ORACLE_UNSUPPORTED = 4
};

#define ORACLE_MAX_DIM 2147483647LL

/* ---------------------------------------------------------------------------
 * O1 canonicalize — input is COO, "the default sparse format ... in
 * SuiteSparse". Validate bounds, sort by (row, col), reject
 * duplicates, keep explicit zeros (SURVEY §8(c) reading 26).
 * Pins: permutation invariance, brute-force set comparison, Appendix D.
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t r, c;
  int64_t idx;
} trip_t;

static int cmp_trip(const void* a, const void* b) {
  const trip_t* x = (const trip_t*)a;
  const trip_t* y = (const trip_t*)b;
  if (x->r != y->r) return x->r < y->r ? -1 : 1;
  if (x->c != y->c) return x->c < y->c ? -1 : 1;
  return 0;
}

EXPORT int oracle_canonicalize(int64_t rows, int64_t cols, int64_t nnz, const int32_t* r,
                               const int32_t* c, const double* v, int32_t* r_out,
                               int32_t* c_out, double* v_out) {
  if (rows < 0 || cols < 0 || nnz < 0) return ORACLE_INVALID_ARG;
  if (rows > ORACLE_MAX_DIM || cols > ORACLE_MAX_DIM) return ORACLE_UNSUPPORTED;
  for (int64_t k = 0; k < nnz; ++k)
    if (r[k] < 0 || r[k] >= rows || c[k] < 0 || c[k] >= cols) return ORACLE_INDEX_OUT_OF_RANGE;
  trip_t* t = (trip_t*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(trip_t));
  for (int64_t k = 0; k < nnz; ++k) {
    t[k].r = r[k];
    t[k].c = c[k];
    t[k].idx = k;
  }
  qsort(t, (size_t)nnz, sizeof(trip_t), cmp_trip);
  for (int64_t k = 1; k < nnz; ++k)
    if (t[k].r == t[k - 1].r && t[k].c == t[k - 1].c) {
      free(t);
      return ORACLE_DUPLICATE;
    }
  for (int64_t k = 0; k < nnz; ++k) {
    r_out[k] = t[k].r;
    c_out[k] = t[k].c;
    v_out[k] = v[t[k].idx];
  }
  free(t);
  return ORACLE_OK;
}

/* ---------------------------------------------------------------------------
 * O2 CSR — "The boundaries of each row are saved in a third array called
 * Row Index". row_ptr[i] = lower_bound(R, i) = #{k : R[k] < i}
 * over the canonical (sorted) row array R, i = 0..rows.
 * Pins: S:125-126 identity/empty examples, row_ptr[rows] = nnz,
 * reconstruct-dense exactness, Appendix D.
 * ------------------------------------------------------------------------- */
EXPORT void oracle_csr(int64_t rows, int64_t nnz, const int32_t* R, int64_t* row_ptr) {
  for (int64_t i = 0; i <= rows; ++i) {
    int64_t lo = 0, hi = nnz; /* first k with R[k] >= i */
    while (lo < hi) {
      int64_t mid = lo + (hi - lo) / 2;
      if (R[mid] < i) lo = mid + 1;
      else hi = mid;
    }
    row_ptr[i] = lo;
  }
}

/* ---------------------------------------------------------------------------
 * O3 features — Table 2 (tab:Matrix_Features): n, nnz, Avg_nnz,
 * Var_nnz, ELL_ratio, Median, Mode, Std_nnz over the row lengths L_i, plus
 * max/min/#empty and the bandwidth the north star adds. Conventions
 * (SURVEY §8(c) reading 5): population variance, even-n median =
 * mean of the two middle order statistics, mode ties -> smallest
 * (S:325), empty rows included (wiki-talk median 0), ELL_ratio of an
 * all-empty matrix = 1. Arithmetic (reading 6): exact integer
 * moments S1 = ΣL, S2 = ΣL² (128-bit), then
 *   mean = S1/n; var = (n·S2 − S1²)/n/n; std = sqrt(var);
 *   ell_ratio = S1/(n·max)  (the ELL matrix is n × max_nnz).
 * Bandwidth: max over ALL entries of (i − j) and (j − i), clamped at 0.
 * Pins: Appendix B closed forms (5-pt, 27-pt, uniform), Appendix D,
 * brute force (sorted median / counted mode) in tests.
 * ------------------------------------------------------------------------- */
typedef struct {
  int64_t n_rows, n_cols, nnz, max_len, min_len, n_empty, mode, bw_lower, bw_upper, bandwidth;
  double mean, var, std, ell_ratio, median;
} oracle_features_t;

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

EXPORT int oracle_features(int64_t rows, int64_t cols, const int64_t* row_ptr,
                           const int32_t* col, oracle_features_t* f) {
  if (rows <= 0) return ORACLE_INVALID_ARG; /* n = 0 -> error */
  memset(f, 0, sizeof(*f));
  int64_t* L = (int64_t*)malloc((size_t)rows * sizeof(int64_t));
  unsigned __int128 S1 = 0, S2 = 0;
  int64_t mx = 0, mn = INT64_MAX, empty = 0;
  int64_t bl = 0, bu = 0;
  for (int64_t i = 0; i < rows; ++i) {
    L[i] = row_ptr[i + 1] - row_ptr[i];
    S1 += (unsigned __int128)L[i];
    S2 += (unsigned __int128)L[i] * (unsigned __int128)L[i];
    if (L[i] > mx) mx = L[i];
    if (L[i] < mn) mn = L[i];
    if (L[i] == 0) ++empty;
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      int64_t j = col[k];
      if (i - j > bl) bl = i - j;
      if (j - i > bu) bu = j - i;
    }
  }
  unsigned __int128 n = (unsigned __int128)rows;
  unsigned __int128 num = n * S2 - S1 * S1;
  f->n_rows = rows;
  f->n_cols = cols;
  f->nnz = (int64_t)S1;
  f->max_len = mx;
  f->min_len = mn;
  f->n_empty = empty;
  f->mean = (double)(int64_t)S1 / (double)rows;
  f->var = (double)num / (double)rows / (double)rows;
  f->std = sqrt(f->var);
  f->ell_ratio = (mx == 0) ? 1.0 : (double)(int64_t)S1 / (double)(rows * mx);
  qsort(L, (size_t)rows, sizeof(int64_t), cmp_i64);
  int64_t lo = L[(rows - 1) / 2], hi = L[rows / 2];
  f->median = ((double)lo + (double)hi) / 2.0;
  int64_t best = L[0], bestc = 0;
  for (int64_t a = 0; a < rows;) { /* runs of equal lengths in ascending order */
    int64_t b = a;
    while (b < rows && L[b] == L[a]) ++b;
    if (b - a > bestc) { bestc = b - a; best = L[a]; }
    a = b;
  }
  f->mode = best;
  f->bw_lower = bl;
  f->bw_upper = bu;
  f->bandwidth = bl > bu ? bl : bu;
  free(L);
  return ORACLE_OK;
}

/* ---------------------------------------------------------------------------
 * O4 ELL — "Dimensions of the Data matrix will be m × max_nnz".
 * Reading 9: column-major [K][n_pad], n_pad = ceil(rows/128)·128, slot
 * (i, k) at k·n_pad + i; slot k < L_i holds row i's k-th entry in column
 * order, otherwise padding (col −1, value +0.0). Phantom rows are padding.
 * Pins: S:134 example, padding = n_pad·K − nnz, reconstruct-dense,
 * Appendix D.
 * ------------------------------------------------------------------------- */
EXPORT int64_t oracle_ell_npad(int64_t rows) { return (rows + 127) / 128 * 128; }

EXPORT void oracle_ell(int64_t rows, const int64_t* row_ptr, const int32_t* col, const double* val,
                       int64_t K, int64_t n_pad, int32_t* colE, double* valE) {
  for (int64_t k = 0; k < K; ++k)
    for (int64_t i = 0; i < n_pad; ++i) {
      int64_t L = (i < rows) ? row_ptr[i + 1] - row_ptr[i] : 0;
      if (k < L) {
        colE[k * n_pad + i] = col[row_ptr[i] + k];
        valE[k * n_pad + i] = val[row_ptr[i] + k];
      } else {
        colE[k * n_pad + i] = -1;
        valE[k * n_pad + i] = 0.0;
      }
    }
}

/* ---------------------------------------------------------------------------
 * O5 SELL-C-σ — "Each slice of this format consists of a constant number of
 * rows ... The length of each slice is the maximum number of non-zero
 * elements per row in that slice" with a Slice Index array (Fig. 2
 * uses slice height 2). Reading 10 generalises to SELL-C-σ: perm
 * sorts each σ-window [wσ, min((w+1)σ, rows)) by (L desc, row asc)
 * (σ = 1: identity); slice s holds rows perm[sC + j], j < C (phantom lanes
 * have L = 0); w_s = max lane length; slice_ptr[s+1] = slice_ptr[s] + C·w_s;
 * element (s, j, k) at slice_ptr[s] + k·C + j; padding as in O4.
 * Requires C >= 1 and (σ = 1 or σ mod C = 0).
 * Pins: S:152 example, one-slice SELL = ELL padding,
 * reconstruct-dense, Appendix D (C = 2, σ = 1 and C = 4, σ = 4).
 * ------------------------------------------------------------------------- */
typedef struct {
  int64_t len, row;
} lenrow_t;

static int cmp_lenrow(const void* a, const void* b) {
  const lenrow_t* x = (const lenrow_t*)a;
  const lenrow_t* y = (const lenrow_t*)b;
  if (x->len != y->len) return x->len > y->len ? -1 : 1; /* length descending */
  return x->row < y->row ? -1 : (x->row > y->row ? 1 : 0); /* then row ascending */
}

EXPORT int oracle_sell_perm(int64_t rows, const int64_t* row_ptr, int64_t C, int64_t sigma,
                            int32_t* perm) {
  if (C < 1 || sigma < 1 || (sigma != 1 && sigma % C != 0)) return ORACLE_INVALID_ARG;
  lenrow_t* w = (lenrow_t*)malloc((size_t)(sigma > 0 ? sigma : 1) * sizeof(lenrow_t));
  for (int64_t s0 = 0; s0 < rows; s0 += sigma) {
    int64_t s1 = s0 + sigma < rows ? s0 + sigma : rows;
    for (int64_t i = s0; i < s1; ++i) {
      w[i - s0].len = row_ptr[i + 1] - row_ptr[i];
      w[i - s0].row = i;
    }
    qsort(w, (size_t)(s1 - s0), sizeof(lenrow_t), cmp_lenrow);
    for (int64_t i = s0; i < s1; ++i) perm[i] = (int32_t)w[i - s0].row;
  }
  free(w);
  return ORACLE_OK;
}

EXPORT int64_t oracle_sell_nslices(int64_t rows, int64_t C) { return (rows + C - 1) / C; }

/* slice_ptr has n_slices + 1 entries; returns the total slot count. */
EXPORT int64_t oracle_sell_slice_ptr(int64_t rows, const int64_t* row_ptr, const int32_t* perm,
                                     int64_t C, int64_t* slice_ptr) {
  int64_t ns = (rows + C - 1) / C;
  slice_ptr[0] = 0;
  for (int64_t s = 0; s < ns; ++s) {
    int64_t w = 0;
    for (int64_t j = 0; j < C; ++j) {
      int64_t q = s * C + j;
      if (q >= rows) continue;
      int64_t i = perm[q];
      int64_t L = row_ptr[i + 1] - row_ptr[i];
      if (L > w) w = L;
    }
    slice_ptr[s + 1] = slice_ptr[s] + C * w;
  }
  return slice_ptr[ns];
}

EXPORT void oracle_sell_fill(int64_t rows, const int64_t* row_ptr, const int32_t* col,
                             const double* val, const int32_t* perm, int64_t C,
                             const int64_t* slice_ptr, int32_t* colS, double* valS) {
  int64_t ns = (rows + C - 1) / C;
  for (int64_t s = 0; s < ns; ++s) {
    int64_t w = (slice_ptr[s + 1] - slice_ptr[s]) / C;
    for (int64_t k = 0; k < w; ++k)
      for (int64_t j = 0; j < C; ++j) {
        int64_t q = s * C + j;
        int64_t pos = slice_ptr[s] + k * C + j;
        int64_t i = (q < rows) ? perm[q] : -1;
        int64_t L = (i >= 0) ? row_ptr[i + 1] - row_ptr[i] : 0;
        if (k < L) {
          colS[pos] = col[row_ptr[i] + k];
          valS[pos] = val[row_ptr[i] + k];
        } else {
          colS[pos] = -1;
          valS[pos] = 0.0;
        }
      }
  }
}

/* ---------------------------------------------------------------------------
 * O6 HYB — not in the paper (reading 12): ELL part of width K_h plus a COO
 * tail. Automatic K_h is the Bell–Garland/CUSP rule written out:
 *   rows_gt = rows; for i in 0..max−1 { rows_gt −= hist[i];
 *     if (3·rows_gt < rows || rows_gt < 4096) { K_h = i; break; } }
 *   otherwise K_h = max.
 * The tail holds every entry with in-row rank >= K_h, in (row, col) order.
 * Pins: Appendix B (c1 -> 3 with a 7,936-entry tail; c2 27; c4 32),
 * Appendix D (auto 0; K_h = 2 tail), K_h = max => empty tail, K_h = 0 =>
 * pure COO, reconstruct-dense.
 * ------------------------------------------------------------------------- */
EXPORT int64_t oracle_hyb_auto_k(int64_t rows, const int64_t* row_ptr) {
  int64_t mx = 0;
  for (int64_t i = 0; i < rows; ++i)
    if (row_ptr[i + 1] - row_ptr[i] > mx) mx = row_ptr[i + 1] - row_ptr[i];
  int64_t* hist = (int64_t*)calloc((size_t)mx + 1, sizeof(int64_t));
  for (int64_t i = 0; i < rows; ++i) hist[row_ptr[i + 1] - row_ptr[i]]++;
  int64_t K = mx, rows_gt = rows;
  for (int64_t i = 0; i < mx; ++i) {
    rows_gt -= hist[i];
    if (3 * rows_gt < rows || rows_gt < 4096) {
      K = i;
      break;
    }
  }
  free(hist);
  return K;
}

EXPORT int64_t oracle_hyb_tail_nnz(int64_t rows, const int64_t* row_ptr, int64_t K) {
  int64_t t = 0;
  for (int64_t i = 0; i < rows; ++i) {
    int64_t L = row_ptr[i + 1] - row_ptr[i];
    if (L > K) t += L - K;
  }
  return t;
}

EXPORT void oracle_hyb_tail(int64_t rows, const int64_t* row_ptr, const int32_t* col,
                            const double* val, int64_t K, int32_t* tr, int32_t* tc, double* tv) {
  int64_t t = 0;
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t k = row_ptr[i] + K; k < row_ptr[i + 1]; ++k) {
      tr[t] = (int32_t)i;
      tc[t] = col[k];
      tv[t] = val[k];
      ++t;
    }
}

/* ---------------------------------------------------------------------------
 * O13 BELL — "a block of non-zero elements is considered as an element of the
 * ELL format ... 1) Data matrix, which is used to store blocks of non-zero
 * elements, and 2) Column Index matrix, which is used to store the block
 * indices" (Fig. 2(d) uses 2 × 2 blocks). Reading R11b:
 * block row I covers rows [I·bh, I·bh+bh), block column J covers columns
 * [J·bw, J·bw+bw); a block is stored iff it holds at least one entry; block
 * row I lists its blocks by increasing J; Kb = max blocks per block row;
 * column-major padding to nbr_pad = ceil(n_brows/128)·128 block rows:
 * bcol[k·nbr_pad + I] = J or −1, and value plane e = r·bw + c of slot k at
 * bval[(k·bh·bw + e)·nbr_pad + I] = A(I·bh + r, J·bw + c) or +0.0.
 * Pins: SPEC S:143-144 examples, reconstruct-dense, block-count brute force.
 * ------------------------------------------------------------------------- */
EXPORT int64_t oracle_bell_kb(int64_t rows, const int64_t* row_ptr, const int32_t* col, int64_t bh,
                              int64_t bw) {
  int64_t nbr = (rows + bh - 1) / bh, kb = 0;
  for (int64_t I = 0; I < nbr; ++I) {
    int64_t count = 0, last = -1;
    /* blocks of block row I in increasing J: repeatedly take the smallest J > last */
    for (;;) {
      int64_t best = -1;
      for (int64_t i = I * bh; i < (I + 1) * bh && i < rows; ++i)
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
          int64_t J = col[k] / bw;
          if (J > last && (best < 0 || J < best)) best = J;
        }
      if (best < 0) break;
      last = best;
      ++count;
    }
    if (count > kb) kb = count;
  }
  return kb;
}

EXPORT void oracle_bell(int64_t rows, const int64_t* row_ptr, const int32_t* col, const double* val,
                        int64_t bh, int64_t bw, int64_t kb, int64_t nbr_pad, int32_t* bcol, double* bval) {
  int64_t nbr = (rows + bh - 1) / bh, be = bh * bw;
  for (int64_t q = 0; q < kb * nbr_pad; ++q) bcol[q] = -1;
  for (int64_t q = 0; q < kb * be * nbr_pad; ++q) bval[q] = 0.0;
  for (int64_t I = 0; I < nbr; ++I) {
    int64_t last = -1;
    for (int64_t slot = 0; slot < kb; ++slot) {
      int64_t best = -1;
      for (int64_t i = I * bh; i < (I + 1) * bh && i < rows; ++i)
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
          int64_t J = col[k] / bw;
          if (J > last && (best < 0 || J < best)) best = J;
        }
      if (best < 0) break;
      last = best;
      bcol[slot * nbr_pad + I] = (int32_t)best;
      for (int64_t i = I * bh; i < (I + 1) * bh && i < rows; ++i)
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k)
          if (col[k] / bw == best) {
            int64_t e = (i - I * bh) * bw + (col[k] - best * bw);
            bval[(slot * be + e) * nbr_pad + I] = val[k];
          }
    }
  }
}

/* ---------------------------------------------------------------------------
 * O8 SpMV — "finds the dense vector product Y of a sparse matrix A and a
 * dense vector X such that Y = A × X", with the BLAS α/β extension
 * (reading 1): y_i = α·Σ_k a_ik·x_k + β·y_i, β = 0 => y not read, α = 0 =>
 * A not read. Per row, in column order, fp64 Neumaier-compensated sum of
 * the products (fp32 inputs are widened exactly; their products are exact
 * in fp64). Also returns a_i = Σ|a_ik·x_k| for the O9 tolerance.
 * Pins: dense brute force (O10), A·e_j = column j, A·1 = row sums, 5-point
 * Laplacian on x = (grid row)² gives −2 on interior rows, Dirichlet
 * eigenvectors, Appendix D.
 * ------------------------------------------------------------------------- */
static void spmv_row(int64_t i, const int64_t* row_ptr, const int32_t* col, const double* val,
                     const double* x, double alpha, double beta, const double* y_in, double* y_out,
                     double* abs_out) {
  double sum = 0.0, comp = 0.0, a = 0.0;
  if (alpha != 0.0) {
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      double t = val[k] * x[col[k]];
      double s = sum + t;
      if (fabs(sum) >= fabs(t)) comp += (sum - s) + t;
      else comp += (t - s) + sum;
      sum = s;
      a += fabs(t);
    }
  }
  double acc = sum + comp;
  y_out[i] = (beta == 0.0) ? alpha * acc : alpha * acc + beta * y_in[i];
  if (abs_out) abs_out[i] = a;
}

EXPORT void oracle_spmv_csr(int64_t rows, const int64_t* row_ptr, const int32_t* col,
                            const double* val, const double* x, double alpha, double beta,
                            const double* y_in, double* y_out, double* abs_out) {
  for (int64_t i = 0; i < rows; ++i) spmv_row(i, row_ptr, col, val, x, alpha, beta, y_in, y_out, abs_out);
}

/* The same O8 loop over all host cores (SURVEY §8(d) "CPU baseline": the CSR
 * naive loop once single-threaded and once with an OpenMP parallel-for over
 * rows, schedule(static)). Each row is still summed by one thread in column
 * order, so y is bitwise identical to oracle_spmv_csr (pinned by
 * test_omp_leg_bitwise). Timing only: the parity tests use the 1-thread loop. */
EXPORT void oracle_spmv_csr_omp(int64_t rows, const int64_t* row_ptr, const int32_t* col,
                                const double* val, const double* x, double alpha, double beta,
                                const double* y_in, double* y_out, double* abs_out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < rows; ++i) spmv_row(i, row_ptr, col, val, x, alpha, beta, y_in, y_out, abs_out);
}

EXPORT int oracle_omp_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ---------------------------------------------------------------------------
 * O10 dense brute force (n <= 64): scatter into a dense rows × cols matrix
 * and sum D_ij·x_j over increasing j in plain fp64. Used to pin O1/O2/O8.
 * ------------------------------------------------------------------------- */
EXPORT void oracle_dense_spmv(int64_t rows, int64_t cols, int64_t nnz, const int32_t* r,
                              const int32_t* c, const double* v, const double* x, double* y) {
  double* D = (double*)calloc((size_t)(rows * cols > 0 ? rows * cols : 1), sizeof(double));
  for (int64_t k = 0; k < nnz; ++k) D[(int64_t)r[k] * cols + c[k]] = v[k];
  for (int64_t i = 0; i < rows; ++i) {
    double s = 0.0;
    for (int64_t j = 0; j < cols; ++j) s += D[i * cols + j] * x[j];
    y[i] = s;
  }
  free(D);
}

/* ---------------------------------------------------------------------------
 * O11 power step (not in the paper; the eigensolver appears only as
 * motivation; SURVEY §8(c) reading 30):
 *   y = A·x_k;  s = Σ y²;  λ_k = x_k·y  (‖x_k‖ = 1);  x_{k+1} = y/√s.
 * Sums are Neumaier-compensated fp64. Pins: x0 = 1 -> y = row sums;
 * analytic dominant eigenvector -> λ = λ_max (Appendix B).
 * ------------------------------------------------------------------------- */
static double neumaier_dot(int64_t n, const double* a, const double* b) {
  double sum = 0.0, comp = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double t = a[i] * b[i];
    double s = sum + t;
    if (fabs(sum) >= fabs(t)) comp += (sum - s) + t;
    else comp += (t - s) + sum;
    sum = s;
  }
  return sum + comp;
}

static void power_step(int omp, int64_t rows, const int64_t* row_ptr, const int32_t* col,
                       const double* val, const double* x, double* y, double* x_next,
                       double* lambda, double* s_out) {
  if (omp) oracle_spmv_csr_omp(rows, row_ptr, col, val, x, 1.0, 0.0, NULL, y, NULL);
  else oracle_spmv_csr(rows, row_ptr, col, val, x, 1.0, 0.0, NULL, y, NULL);
  double s = neumaier_dot(rows, y, y);
  *lambda = neumaier_dot(rows, x, y);
  *s_out = s;
  double r = sqrt(s);
  for (int64_t i = 0; i < rows; ++i) x_next[i] = y[i] / r;
}

EXPORT void oracle_power_step(int64_t rows, const int64_t* row_ptr, const int32_t* col,
                              const double* val, const double* x, double* y, double* x_next,
                              double* lambda, double* s_out) {
  power_step(0, rows, row_ptr, col, val, x, y, x_next, lambda, s_out);
}

/* O11 with the all-core O8 loop (timing leg; the sums stay serial). */
EXPORT void oracle_power_step_omp(int64_t rows, const int64_t* row_ptr, const int32_t* col,
                                  const double* val, const double* x, double* y, double* x_next,
                                  double* lambda, double* s_out) {
  power_step(1, rows, row_ptr, col, val, x, y, x_next, lambda, s_out);
}

/* ---------------------------------------------------------------------------
 * O12 nnz-balanced row partition (not in the paper):
 * b_0 = 0, b_P = rows, b_k = lower_bound(row_ptr, ceil(k·nnz/P)) — the
 * first row index whose prefix count reaches the target.
 * Pins: Σ local nnz = nnz, per-rank imbalance < max row length, monotone.
 * ------------------------------------------------------------------------- */
EXPORT void oracle_partition(int64_t rows, const int64_t* row_ptr, int64_t P, int64_t* bounds) {
  int64_t nnz = row_ptr[rows];
  bounds[0] = 0;
  bounds[P] = rows;
  for (int64_t k = 1; k < P; ++k) {
    unsigned __int128 num = (unsigned __int128)k * (unsigned __int128)nnz;
    int64_t target = (int64_t)((num + (unsigned __int128)P - 1) / (unsigned __int128)P);
    int64_t b = 0;
    while (b <= rows && row_ptr[b] < target) ++b; /* naive linear lower_bound */
    bounds[k] = b;
  }
}
