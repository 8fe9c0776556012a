// instantiation unit: ELL/SELL variants, float values, C = 64
#include "kern_sliced.cuh"
namespace spmv {
namespace kern {
template SlicedFn sliced_fn<float, 64, false, false>(int, int);
template SlicedFn sliced_fn<float, 64, false, true>(int, int);
template SlicedFn sliced_fn<float, 64, true, false>(int, int);
template SlicedFn sliced_fn<float, 64, true, true>(int, int);
}  // namespace kern
}  // namespace spmv
