// selector.cu — the learned format selector and overhead estimators
// (SURVEY.md §8(f) f3): the paper's run-time-mode pipeline (P:442-452:
// features -> predicted best format -> estimated overhead -> convert iff the
// predicted gain exceeds it) with a decision-tree classifier
// and overhead regressors (fig:overhead_prediction P:461-516).
// The model is trained offline by tools/train_selector.py on a corpus
// measured on B200 (tools/selector_corpus.py) and compiled in as
// selector_model.h. Host code only: inference is a handful of comparisons.
#include <cmath>

#include "handle.cuh"
#include "selector.cuh"
#include "selector_model.h"

namespace spmv {

// Feature vector (tools/train_selector.py feature_vector: same order, same
// IEEE double arithmetic) from the Table-2 features.
void selector_features(const spmv_features_t& f, int vbytes, double x[kSelectorFeatures]) {
  static_assert(kSelectorFeatures == model::kNumFeatures, "feature count mismatch with the trained model");
  const double n = (double)f.n_rows, nnz = (double)f.nnz, mean = f.mean;
  x[0] = std::log2(n + 1.0);
  x[1] = std::log2(nnz + 1.0);
  x[2] = mean;
  x[3] = f.var;
  x[4] = f.std;
  x[5] = f.ell_ratio;
  x[6] = f.median;
  x[7] = (double)f.mode;
  x[8] = (double)f.max_len;
  x[9] = (double)f.min_len;
  x[10] = (double)f.n_empty / (n > 1.0 ? n : 1.0);
  x[11] = (double)f.bandwidth / (n > 1.0 ? n : 1.0);
  x[12] = mean > 0 ? f.std / mean : 0.0;
  x[13] = mean > 0 ? (double)f.max_len / mean : 0.0;
  x[14] = (double)vbytes;
}

static double eval_tree(const model::Node* t, const double* x) {
  int i = 0;
  while (t[i].feature >= 0) i = (x[t[i].feature] <= t[i].threshold) ? t[i].left : t[i].right;
  return t[i].value;
}

int selector_class(const double* x) { return (int)eval_tree(model::kClassifier, x); }

double selector_speed_ratio(int cls, const double* x) {
  if (cls <= 0 || cls >= model::kNumClasses) return 1.0;
  return std::exp(eval_tree(model::kRatio[cls], x));
}

// Predictors of the overhead estimators (tools/train_selector.py
// overhead_predictors: same order, same arithmetic): the conversions and the
// feature pass are bandwidth-bound kernels plus a few launches, so their
// device time is a constant plus per-entry, per-row and per-ELL-slot costs
// (and, for ELL/SELL, the 8-bit dictionary's flag array of 2·bandwidth + 1 bins).
static void overhead_predictors(const spmv_features_t& f, double phi[model::kNumOverheadPredictors]) {
  const double n = (double)f.n_rows;
  phi[0] = 1.0;
  phi[1] = (double)f.nnz * 1e-6;
  phi[2] = n * 1e-6;
  phi[3] = std::ceil(n / 128.0) * 128.0 * (double)f.max_len * 1e-6;
  phi[4] = 2.0 * (double)(f.bandwidth < (1LL << 22) ? f.bandwidth : (1LL << 22)) * 1e-6;  // dictionary flags
  phi[5] = n * f.std * 1e-6;  // >= Σ|L_i − mean|: the row-length dispersion SELL pads
}

static double linear(const double* w, const double* phi, int k) {
  double s = 0.0;
  for (int i = 0; i < k; ++i) s += w[i] * phi[i];
  return s > 1e-6 ? s : 1e-6;
}

double selector_c_latency(int cls, const spmv_features_t& f) {
  if (cls < 0 || cls >= model::kNumClasses) return 0.0;
  double phi[model::kNumOverheadPredictors];
  overhead_predictors(f, phi);
  return linear(model::kCLatencyLin[cls], phi, model::kNumOverheadPredictors);
}

double selector_f_latency(const spmv_features_t& f) {
  double phi[model::kNumOverheadPredictors];
  overhead_predictors(f, phi);
  return linear(model::kFLatencyLin, phi, 3);
}

const char* selector_class_name(int cls) {
  return (cls >= 0 && cls < model::kNumClasses) ? model::kClassNames[cls] : "?";
}

void selector_class_format(int cls, int* fmt, spmv_format_params_t* p) {
  *p = spmv_format_params_t{};
  p->hyb_K = -1;
  switch (cls) {
    case 1: *fmt = SPMV_FMT_CSR; p->csr_alg = SPMV_CSR_MERGE; break;
    case 2: *fmt = SPMV_FMT_ELL; p->index16 = -1; break;   // the narrowest column encoding that fits
    case 3: *fmt = SPMV_FMT_SELL; p->index16 = -1; break;
    case 4: *fmt = SPMV_FMT_HYB; break;
    case 5: *fmt = SPMV_FMT_COO; break;
    case 6: *fmt = SPMV_FMT_BELL; p->bell_b = 2; break;
    case 7: *fmt = SPMV_FMT_BELL; p->bell_b = 3; break;
    case 8: *fmt = SPMV_FMT_CSR; p->csr_alg = SPMV_CSR_STREAM; break;
    default: *fmt = SPMV_FMT_CSR; p->csr_alg = SPMV_CSR_VECTOR; break;
  }
}

}  // namespace spmv
