// instantiation unit: ELL/SELL variants, double values, C = 64 (8-bit dictionary column codes)
#include "kern_sliced.cuh"
namespace spmv {
namespace kern {
template SlicedFn sliced_fn<double, 64, 2, false>(int, int);
template SlicedFn sliced_fn<double, 64, 2, true>(int, int);
}  // namespace kern
}  // namespace spmv
