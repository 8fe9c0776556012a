// instantiation unit: ELL/SELL variants, double values, C = 128
#include "kern_sliced.cuh"
namespace spmv {
namespace kern {
template SlicedFn sliced_fn<double, 128, false, false>(int, int);
template SlicedFn sliced_fn<double, 128, false, true>(int, int);
template SlicedFn sliced_fn<double, 128, true, false>(int, int);
template SlicedFn sliced_fn<double, 128, true, true>(int, int);
}  // namespace kern
}  // namespace spmv
