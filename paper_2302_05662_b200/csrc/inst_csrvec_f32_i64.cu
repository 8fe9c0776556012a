// instantiation unit: CSR-vector variants, float values, int64_t row pointers
#include "kern_csr.cuh"
namespace spmv {
namespace kern {
template CsrFn csr_vector_fn<float, int64_t, 1>(int, int);
template CsrFn csr_vector_fn<float, int64_t, 2>(int, int);
template CsrFn csr_vector_fn<float, int64_t, 4>(int, int);
template CsrFn csr_vector_fn<float, int64_t, 8>(int, int);
template CsrFn csr_vector_fn<float, int64_t, 16>(int, int);
template CsrFn csr_vector_fn<float, int64_t, 32>(int, int);
template CsrFn csr_vector4_fn<float, int64_t, 4>(int, int);
template CsrFn csr_vector4_fn<float, int64_t, 8>(int, int);
template CsrFn csr_vector4_fn<float, int64_t, 16>(int, int);
template CsrFn csr_vector4_fn<float, int64_t, 32>(int, int);
}  // namespace kern
}  // namespace spmv
