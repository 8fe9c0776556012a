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

// Row-interleaved tile kernel (k_coo_tile): launch knob kCooTile | EPT, a
// block stages B·EPT consecutive entries in shared memory and walks them
// thread-per-row. nullptr for (block, EPT) pairs over the shared-memory cap.
constexpr int kCooTile = 0x100;
template <class T, int EPT>
CooFn coo_tile_fn(int bi, int ri);
template <class T>
constexpr size_t coo_tile_smem(int B, int EPT) {
  // row, col, val of the tile + segment starts (TILE + 1) + per-(pass, warp) head counts
  return (size_t)B * EPT * (4 + 4 + sizeof(T) + 4) + 4 + (size_t)EPT * (B / 32) * 4 + 16;
}

}  // namespace kern
}  // namespace spmv
