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
  const int64_t* coords;  // merge-path chunk start coordinates (x, y) pairs, nchunks+1
  int64_t nchunks;
  const uint32_t* rm_bits;  // row map (k_csr_nnz_map): row-start bit per entry
  const int32_t* rm_rows;   //   ids of the non-empty rows, in order
  const int64_t* rm_ord0;   //   row starts before each 256-entry chunk
  int rm_identity;          //   no empty rows: the j-th non-empty row is row j (no list lookups)
};

using CsrFn = void (*)(const CsrParams);
template <class T, class RP, int LANES>
CsrFn csr_vector_fn(int bi, int ri);
template <class T, class RP, int IPT>
CsrFn csr_merge_fn(int bi, int ri);
// CSR-vector with quad (128-bit) loads: knob kCsrQuad | LANES, LANES in {4, 8, 16, 32}
constexpr int kCsrQuad = 0x100;
template <class T, class RP, int LANES>
CsrFn csr_vector4_fn(int bi, int ri);
template <class T, class RP, int EPT>
CsrFn csr_stream_fn(int bi, int ri);
// Shared-memory stage of the CSR-stream pipeline holding `cap` entries: the
// column region (cap + 4 ints) then the value region (cap + 16/sizeof(T)
// values), both 16-byte aligned (the slack absorbs the alignment of the
// tile's first entry).
template <class T>
struct StreamStage {
  static constexpr int kValPad = 16 / (int)sizeof(T);
  __host__ __device__ static constexpr size_t col_bytes(int cap) { return ((size_t)(cap + 4) * 4 + 15) / 16 * 16; }
  __host__ __device__ static constexpr size_t bytes(int cap) {
    return col_bytes(cap) + ((size_t)(cap + kValPad) * sizeof(T) + 15) / 16 * 16;
  }
};
constexpr int kStreamStages = 2;
// Dynamic shared memory of a CSR-stream block: kStreamStages stages of
// B rows × EPT entries of (col, value).
template <class T>
constexpr size_t stream_smem_bytes(int block, int ept) {
  return (size_t)kStreamStages * StreamStage<T>::bytes(block * ept);
}
// Dynamic shared memory of a merge-path block of `block` threads.
// Per-warp slice: ITEMS fp64 products then ITEMS+1 int32 row ends, padded to 16 B.
__host__ __device__ constexpr size_t merge_warp_smem(int ipt) {
  return (((size_t)(32 * ipt) * 8 + (size_t)(32 * ipt + 1) * 4) + 15) / 16 * 16;
}
template <class T>
constexpr size_t merge_smem_bytes(int block, int ipt) {
  return (size_t)(block / 32) * merge_warp_smem(ipt);
}
// Merge-path tiles (k_csr_merge_tile): launch knob kMergeTile | IPT; a block
// owns block·IPT merge items (row ends + entries).
constexpr int kMergeTile = 0x100;
template <class T, class RP, int IPT>
CsrFn csr_merge_tile_fn(int bi, int ri);
template <class T>
constexpr size_t merge_tile_smem(int block, int ipt) {
  // col + value of up to block·IPT entries, then up to block·IPT + 2 row starts
  return (size_t)block * ipt * (4 + sizeof(T)) + ((size_t)block * ipt + 2) * 4 + 16;
}
// Pipelined merge-path (k_csr_merge_stream): knob kMergeStream | IPT; B
// consumer threads + one TMA producer warp, two stages of B·IPT merge items.
constexpr int kMergeStream = 0x200;
template <class T, class RP, int IPT>
CsrFn csr_merge_stream_fn(int bi, int ri);
template <class T, class RP>
struct MergeStage {
  // col + val (StreamStage layout), then row starts (RP, 16-byte slack on both ends)
  static constexpr int kRpPad = 16 / (int)sizeof(RP);
  __host__ __device__ static constexpr size_t rp_off(int items) { return StreamStage<T>::bytes(items); }
  __host__ __device__ static constexpr size_t bytes(int items) {
    return rp_off(items) + ((size_t)(items + 2 + 2 * kRpPad) * sizeof(RP) + 15) / 16 * 16;
  }
};
template <class T, class RP>
constexpr size_t merge_stream_smem(int block, int ipt) {
  return (size_t)kStreamStages * MergeStage<T, RP>::bytes(block * ipt);
}
// nnz-split CSR of the merge-path family (k_csr_nnz): knob kMergeNnz | W,
// a warp owns 32·W consecutive entries (W = 4 or 8).
constexpr int kMergeNnz = 0x400;
template <class T, class RP, int W>
CsrFn csr_nnz_fn(int bi, int ri);
// nnz-split CSR with a cached row map (k_csr_nnz_map): knob kMergeRowmap | 8,
// a warp owns 256 consecutive entries; rows from the row-start bits.
constexpr int kMergeRowmap = 0x800;
template <class T, class RP>
CsrFn csr_nnz_map_fn(int bi, int ri);
// nnz-split partition: coords[c] = row holding entry c·per (rows past the end), c = 0..nchunks.
void nnz_partition(const void* rp, bool rp64, int64_t rows, int64_t nnz, int64_t per, int64_t nchunks,
                   int64_t* coords, cudaStream_t s);
// Merge-path partition pre-pass: coords[2c], coords[2c+1] = start of chunk c.
void merge_partition(const void* rp, bool rp64, int64_t rows, int64_t nnz, int64_t items_per_chunk,
                     int64_t nchunks, int64_t* coords, cudaStream_t s);

}  // namespace kern
}  // namespace spmv
