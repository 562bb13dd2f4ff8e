// Kernel instantiations for W = 1 (32 threads per environment).
#include "tabx_lane.cuh"

namespace tabx {
cudaError_t launch_ctrl_w1(const Params& P, int nh, int sm_count, cudaStream_t stream) {
  return launch_ctrl_t<1>(P, nh, sm_count, stream);
}
cudaError_t launch_lanes_w1(const Params& P, int sm_count, cudaStream_t stream, int* grid) {
  return launch_lanes_t<1, 4, TABX_K1_EPB>(P, sm_count, stream, grid);
}
// observation-kernel envs (warps) per CTA at W = 1
#ifndef TABX_EMIT_EPW
#define TABX_EMIT_EPW 4
#endif
cudaError_t launch_emit_w1(const Params& P, int sm_count, cudaStream_t stream) {
  return launch_emit_t<1, TABX_EMIT_EPW>(P, sm_count, stream);
}
// Phase cycle counters of the instrumented build (zeros otherwise).
cudaError_t phase_cycles_w1(unsigned long long* host16, int reset) {
#if defined(TABX_PHASE_PROF) || defined(TABX_COUNT_PROF)
  cudaError_t e = cudaMemcpyFromSymbol(host16, tabx_phase_cycles, 16 * sizeof(unsigned long long));
  if (e == cudaSuccess && reset) {
    static const unsigned long long zero[16] = {};
    e = cudaMemcpyToSymbol(tabx_phase_cycles, zero, sizeof(zero));
  }
  return e;
#else
  (void)reset;
  for (int k = 0; k < 16; ++k) host16[k] = 0;
  return cudaSuccess;
#endif
}
}  // namespace tabx
