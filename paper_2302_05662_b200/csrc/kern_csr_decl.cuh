// kern_csr_decl.cuh — CSR kernel parameter block and variant-table getters
// (definitions in kern_csr.cuh, instantiated per (dtype, row_ptr type) in
// inst_csr_*.cu so the variants compile in parallel).
#pragma once
#include "spmv_common.cuh"

namespace spmv {
namespace kern {

struct CsrParams {
  const void* rp;
  const int32_t* col;
  const void* val;
  int64_t rows, nnz;
  const void* x;
  void* y;
  Epilogue e;
  ChunkRec* recs;
};

using CsrFn = void (*)(const CsrParams);
template <class T, class RP, int LANES>
CsrFn csr_vector_fn(int bi, int ri);
template <class T, class RP, int IPT>
CsrFn csr_merge_fn(int bi, int ri);

}  // namespace kern
}  // namespace spmv
