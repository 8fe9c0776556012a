// instantiation unit: ELL/SELL variants, float values, C = 32
#include "kern_sliced.cuh"
namespace spmv {
namespace kern {
template SlicedFn sliced_fn<float, 32, false, false>(int, int);
template SlicedFn sliced_fn<float, 32, false, true>(int, int);
template SlicedFn sliced_fn<float, 32, true, false>(int, int);
template SlicedFn sliced_fn<float, 32, true, true>(int, int);
}  // namespace kern
}  // namespace spmv
