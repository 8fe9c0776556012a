// kern_bell_decl.cuh — BELL kernel parameter block and variant-table getter
// (definitions in kern_bell.cuh, instantiated in inst_bell_*.cu).
#pragma once
#include "spmv_common.cuh"

namespace spmv {
namespace kern {

struct BellParams {
  const int32_t* bcol;  // [kb][nbr_pad]
  const void* bval;     // [kb][b·b][nbr_pad]
  int64_t rows, cols, nbr, nbr_pad, kb;
  const void* x;
  void* y;
  Epilogue e;
};

using BellFn = void (*)(const BellParams);
template <class T, int BS>
BellFn bell_fn(int bi, int ri);

}  // namespace kern
}  // namespace spmv
