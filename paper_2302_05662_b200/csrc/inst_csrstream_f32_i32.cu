// instantiation unit: CSR-stream variants, float values, int32_t row pointers
#include "kern_csr.cuh"
namespace spmv {
namespace kern {
template CsrFn csr_stream_fn<float, int32_t, 16>(int, int);
template CsrFn csr_stream_fn<float, int32_t, 32>(int, int);
template CsrFn csr_stream_fn<float, int32_t, 64>(int, int);
}  // namespace kern
}  // namespace spmv
