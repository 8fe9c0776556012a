// kern_coo_decl.cuh — COO segmented-reduction kernel parameter block and
// variant-table getter (definitions in kern_coo.cuh, inst_coo_*.cu).
#pragma once
#include <climits>

#include "spmv_common.cuh"

namespace spmv {
namespace kern {

struct CooParams {
  const int32_t* row;
  const int32_t* col;
  const void* val;
  int64_t nnz;
  const void* x;
  void* y;
  Epilogue e;
  ChunkRec* recs;
};

using CooFn = void (*)(const CooParams);
template <class T, int W>
CooFn coo_fn(int bi, int ri);

}  // namespace kern
}  // namespace spmv
