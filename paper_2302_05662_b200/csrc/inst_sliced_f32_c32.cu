// instantiation unit: ELL/SELL variants, float values, C = 32
#include "kern_sliced.cuh"
namespace spmv {
namespace kern {
template SlicedFn sliced_fn<float, 32>(int, int);
}  // namespace kern
}  // namespace spmv
