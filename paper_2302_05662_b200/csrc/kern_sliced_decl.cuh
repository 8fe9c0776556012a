// kern_sliced_decl.cuh — ELL/SELL kernel parameter block and variant-table
// getters (definitions in kern_sliced.cuh, instantiated in inst_sliced_*.cu).
#pragma once
#include "spmv_common.cuh"

namespace spmv {
namespace kern {

struct SlicedParams {
  const int32_t* col;       // int32 column indices (pad -1), or nullptr when col16 is used
  const int16_t* col16;     // 16-bit offsets: column = col_origin + row + d (pad -32768)
  const uint8_t* col8;      // 8-bit codes: column = col_origin + row + tab8[code] (pad 255)
  const int32_t* tab8;      // [256] offset of each code
  int64_t col_origin;
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
// ENC: column encoding, 0 = int32 columns, 1 = 16-bit offsets, 2 = 8-bit dictionary codes
template <class T, int C, int ENC, bool CARRY>
SlicedFn sliced_fn(int bi, int ri);
// launch knob flag of ELL/SELL: the carried-batch loop (see k_sliced)
constexpr int kSlicedCarry = 1 << 16;

}  // namespace kern
}  // namespace spmv
