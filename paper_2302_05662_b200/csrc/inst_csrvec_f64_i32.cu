// instantiation unit: CSR-vector variants, double values, int32_t row pointers
#include "kern_csr.cuh"
namespace spmv {
namespace kern {
template CsrFn csr_vector_fn<double, int32_t, 1>(int, int);
template CsrFn csr_vector_fn<double, int32_t, 2>(int, int);
template CsrFn csr_vector_fn<double, int32_t, 4>(int, int);
template CsrFn csr_vector_fn<double, int32_t, 8>(int, int);
template CsrFn csr_vector_fn<double, int32_t, 16>(int, int);
template CsrFn csr_vector_fn<double, int32_t, 32>(int, int);
template CsrFn csr_vector4_fn<double, int32_t, 4>(int, int);
template CsrFn csr_vector4_fn<double, int32_t, 8>(int, int);
template CsrFn csr_vector4_fn<double, int32_t, 16>(int, int);
template CsrFn csr_vector4_fn<double, int32_t, 32>(int, int);
}  // namespace kern
}  // namespace spmv
