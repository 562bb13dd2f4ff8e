// Kernel instantiations for W = 1 (32 threads per environment).
#include "tabx_lane.cuh"

namespace tabx {
cudaError_t launch_lanes_w1(const Params& P, int sm_count, cudaStream_t stream, int* grid) {
  return launch_lanes_t<1, 4>(P, sm_count, stream, grid);
}
cudaError_t launch_emit_w1(const Params& P, int sm_count, cudaStream_t stream) {
  #ifndef TABX_EMIT_EPW
#define TABX_EMIT_EPW 8
#endif
  return launch_emit_t<1, TABX_EMIT_EPW>(P, sm_count, stream);
}
}  // namespace tabx
