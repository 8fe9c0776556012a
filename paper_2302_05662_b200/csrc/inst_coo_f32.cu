// instantiation unit: COO segmented-reduction variants, float values
#include "kern_coo.cuh"
namespace spmv {
namespace kern {
template CooFn coo_fn<float, 2>(int, int);
template CooFn coo_fn<float, 4>(int, int);
template CooFn coo_fn<float, 8>(int, int);
template CooFn coo_tile_fn<float, 4>(int, int);
template CooFn coo_tile_fn<float, 8>(int, int);
template CooFn coo_tile_fn<float, 16>(int, int);
template CooFn coo_tile_fn<float, 32>(int, int);
}  // namespace kern
}  // namespace spmv
