// instantiation unit: ELL/SELL variants, float values, C = 64
#include "kern_sliced.cuh"
namespace spmv {
namespace kern {
template SlicedFn sliced_fn<float, 64, 0, false>(int, int);
template SlicedFn sliced_fn<float, 64, 0, true>(int, int);
template SlicedFn sliced_fn<float, 64, 1, false>(int, int);
template SlicedFn sliced_fn<float, 64, 1, true>(int, int);
}  // namespace kern
}  // namespace spmv
