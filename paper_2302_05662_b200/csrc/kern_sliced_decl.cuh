// kern_sliced_decl.cuh — ELL/SELL kernel parameter block and variant-table
// getters (definitions in kern_sliced.cuh, instantiated in inst_sliced_*.cu).
#pragma once
#include "spmv_common.cuh"

namespace spmv {
namespace kern {

struct SlicedParams {
  const int32_t* col;
  const void* val;
  const int64_t* sp;    // SELL slice pointers (nullptr for ELL)
  const int32_t* perm;  // SELL row permutation (nullptr = identity)
  int64_t rows;
  int64_t nslices;
  int64_t ell_K, ell_stride;
  const void* x;
  void* y;
  Epilogue e;
};

using SlicedFn = void (*)(const SlicedParams);
template <class T, int C>
SlicedFn sliced_fn(int bi, int ri);

}  // namespace kern
}  // namespace spmv
