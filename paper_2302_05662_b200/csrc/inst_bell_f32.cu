// instantiation unit: BELL variants, float values, block sizes 2, 3, 4
#include "kern_bell.cuh"
namespace spmv {
namespace kern {
template BellFn bell_fn<float, 2>(int, int);
template BellFn bell_fn<float, 3>(int, int);
template BellFn bell_fn<float, 4>(int, int);
}  // namespace kern
}  // namespace spmv
