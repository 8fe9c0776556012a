// instantiation unit: COO segmented-reduction variants, double values
#include "kern_coo.cuh"
namespace spmv {
namespace kern {
template CooFn coo_fn<double, 2>(int, int);
template CooFn coo_fn<double, 4>(int, int);
template CooFn coo_fn<double, 8>(int, int);
template CooFn coo_tile_fn<double, 4>(int, int);
template CooFn coo_tile_fn<double, 8>(int, int);
template CooFn coo_tile_fn<double, 16>(int, int);
template CooFn coo_tile_fn<double, 32>(int, int);
}  // namespace kern
}  // namespace spmv
