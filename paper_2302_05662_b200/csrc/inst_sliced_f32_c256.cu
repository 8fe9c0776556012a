// instantiation unit: ELL/SELL variants, float values, C = 256
#include "kern_sliced.cuh"
namespace spmv {
namespace kern {
template SlicedFn sliced_fn<float, 256, false, false>(int, int);
template SlicedFn sliced_fn<float, 256, false, true>(int, int);
template SlicedFn sliced_fn<float, 256, true, false>(int, int);
template SlicedFn sliced_fn<float, 256, true, true>(int, int);
}  // namespace kern
}  // namespace spmv
