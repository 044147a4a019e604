// Lookup kernel instantiations for 8 batch value(s) per tile (separate
// translation unit: the four widths compile in parallel).
#include "grid_lookup.cuh"

namespace pm2l {
namespace gk {
template cudaError_t launch_rows_t<8>(const TablesDev&, const GridDev&, const RowLaunch&,
                                        const double*, const LaunchOut&, cudaStream_t);
}  // namespace gk
}  // namespace pm2l
