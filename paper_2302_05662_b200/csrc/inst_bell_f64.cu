// instantiation unit: BELL variants, double values, block sizes 2, 3, 4
#include "kern_bell.cuh"
namespace spmv {
namespace kern {
template BellFn bell_fn<double, 2>(int, int);
template BellFn bell_fn<double, 3>(int, int);
template BellFn bell_fn<double, 4>(int, int);
}  // namespace kern
}  // namespace spmv
