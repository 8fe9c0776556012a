// instantiation unit: ELL/SELL variants, double values, C = 128
#include "kern_sliced.cuh"
namespace spmv {
namespace kern {
template SlicedFn sliced_fn<double, 128, 0, false>(int, int);
template SlicedFn sliced_fn<double, 128, 0, true>(int, int);
template SlicedFn sliced_fn<double, 128, 1, false>(int, int);
template SlicedFn sliced_fn<double, 128, 1, true>(int, int);
}  // namespace kern
}  // namespace spmv
