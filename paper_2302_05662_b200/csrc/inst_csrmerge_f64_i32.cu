// instantiation unit: merge-path CSR variants, double values, int32_t row pointers
#include "kern_csr.cuh"
namespace spmv {
namespace kern {
template CsrFn csr_merge_fn<double, int32_t, 4>(int, int);
template CsrFn csr_nnz_fn<double, int32_t, 4>(int, int);
template CsrFn csr_nnz_map_fn<double, int32_t>(int, int);
template CsrFn csr_nnz_fn<double, int32_t, 8>(int, int);
template CsrFn csr_merge_fn<double, int32_t, 8>(int, int);
template CsrFn csr_merge_fn<double, int32_t, 16>(int, int);
template CsrFn csr_merge_tile_fn<double, int32_t, 4>(int, int);
template CsrFn csr_merge_tile_fn<double, int32_t, 8>(int, int);
template CsrFn csr_merge_tile_fn<double, int32_t, 16>(int, int);
template CsrFn csr_merge_tile_fn<double, int32_t, 32>(int, int);
template CsrFn csr_merge_stream_fn<double, int32_t, 4>(int, int);
template CsrFn csr_merge_stream_fn<double, int32_t, 8>(int, int);
template CsrFn csr_merge_stream_fn<double, int32_t, 16>(int, int);
template CsrFn csr_merge_stream_fn<double, int32_t, 32>(int, int);
}  // namespace kern
}  // namespace spmv
