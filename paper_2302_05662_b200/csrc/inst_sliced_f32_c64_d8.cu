// instantiation unit: ELL/SELL variants, float values, C = 64 (8-bit dictionary column codes)
#include "kern_sliced.cuh"
namespace spmv {
namespace kern {
template SlicedFn sliced_fn<float, 64, 2, false>(int, int);
template SlicedFn sliced_fn<float, 64, 2, true>(int, int);
}  // namespace kern
}  // namespace spmv
