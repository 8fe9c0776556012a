// merge-path partition pre-pass launcher (kernel in kern_csr.cuh)
#include "kern_csr.cuh"
namespace spmv {
namespace kern {
void merge_partition(const void* rp, bool rp64, int64_t rows, int64_t nnz, int64_t items_per_chunk,
                     int64_t nchunks, int64_t* coords, cudaStream_t s) {
  const unsigned g = grid_for(nchunks + 1, 256);
  if (rp64)
    LAUNCH(k_merge_partition<int64_t>, g, 256, 0, s, static_cast<const int64_t*>(rp), rows, nnz, items_per_chunk,
           nchunks, coords);
  else
    LAUNCH(k_merge_partition<int32_t>, g, 256, 0, s, static_cast<const int32_t*>(rp), rows, nnz, items_per_chunk,
           nchunks, coords);
}
void nnz_partition(const void* rp, bool rp64, int64_t rows, int64_t nnz, int64_t per, int64_t nchunks,
                   int64_t* coords, cudaStream_t s) {
  const unsigned g = grid_for(nchunks + 1, 256);
  if (rp64)
    LAUNCH(k_nnz_partition<int64_t>, g, 256, 0, s, static_cast<const int64_t*>(rp), rows, nnz, per, nchunks, coords);
  else
    LAUNCH(k_nnz_partition<int32_t>, g, 256, 0, s, static_cast<const int32_t*>(rp), rows, nnz, per, nchunks, coords);
}
}  // namespace kern
}  // namespace spmv
