// Kernel instantiations for W = 8 (256 threads per environment).
#include "tabx_lane.cuh"

namespace tabx {
cudaError_t launch_lanes_w8(const Params& P, int sm_count, cudaStream_t stream, int* grid) {
  return launch_lanes_t<8, 1>(P, sm_count, stream, grid);
}
cudaError_t launch_emit_w8(const Params& P, int sm_count, cudaStream_t stream) {
  return launch_emit_t<8, 1>(P, sm_count, stream);
}
}  // namespace tabx
