// selector.cuh — learned format selector (selector.cu, model in selector_model.h).
#pragma once
#include "../../include/spmv.h"

namespace spmv {
constexpr int kSelectorFeatures = 15;
void selector_features(const spmv_features_t& f, int vbytes, double x[kSelectorFeatures]);
int selector_class(const double* x);
// Predicted t_class / t_CSR-vector (1 for class 0).
double selector_speed_ratio(int cls, const double* x);
// Predicted conversion latency of the class's format / feature-extraction
// latency (seconds): linear in the bytes the kernels move (nnz, rows, ELL
// slots), fitted without negative weights on warm device latencies.
double selector_c_latency(int cls, const spmv_features_t& f);
double selector_f_latency(const spmv_features_t& f);
const char* selector_class_name(int cls);
void selector_class_format(int cls, int* fmt, spmv_format_params_t* p);
}  // namespace spmv
