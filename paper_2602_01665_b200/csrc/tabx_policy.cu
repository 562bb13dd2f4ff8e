// Masked action sampling for the on-device rollout loop (SURVEY.md 8(f)
// rank 2, C5): Gumbel-max over the legal actions of each agent's logits and
// the log-probability of the sampled action under the masked softmax, in one
// pass (one thread per agent).  The noise is a counter-based hash of
// (seed, step, agent, action), so a captured graph replays a fresh draw per
// step by advancing `step` on the device.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "tabx_device.cuh"
#include "tabx_sample.cuh"

namespace tabx {

template <typename T>
__device__ __forceinline__ float load_logit(const T* p);
template <>
__device__ __forceinline__ float load_logit<float>(const float* p) {
  return *p;
}
template <>
__device__ __forceinline__ float load_logit<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}

template <typename T>
__global__ void masked_sample_kernel(const T* __restrict__ logits, int64_t ld,
                                     const uint8_t* __restrict__ mask, int64_t M, uint64_t seed,
                                     const uint64_t* __restrict__ step_ptr, uint64_t step_add,
                                     int64_t* __restrict__ actions, float* __restrict__ logp) {
  const uint64_t key = sample_key(seed, step_ptr, step_add);
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < M;
       r += (int64_t)gridDim.x * blockDim.x) {
    const T* l = logits + r * ld;
    float lg[TABX_NUM_ACTIONS];
#pragma unroll
    for (int a = 0; a < TABX_NUM_ACTIONS; ++a) lg[a] = load_logit<T>(l + a);
    sample_row(lg, mask + r * TABX_NUM_ACTIONS, key, r, actions, logp);
  }
}

cudaError_t launch_masked_sample(const void* logits, int bf16, int64_t ld, const uint8_t* mask,
                                 int64_t M, uint64_t seed, const uint64_t* step_ptr,
                                 uint64_t step_add, int64_t* actions, float* logp, int sm_count,
                                 cudaStream_t stream) {
  if (M <= 0) return cudaSuccess;
  const int threads = 256;
  int64_t blocks = (M + threads - 1) / threads;
  if (blocks > (int64_t)sm_count * 16) blocks = (int64_t)sm_count * 16;
  if (bf16)
    masked_sample_kernel<__nv_bfloat16><<<(int)blocks, threads, 0, stream>>>(
        (const __nv_bfloat16*)logits, ld, mask, M, seed, step_ptr, step_add, actions, logp);
  else
    masked_sample_kernel<float><<<(int)blocks, threads, 0, stream>>>(
        (const float*)logits, ld, mask, M, seed, step_ptr, step_add, actions, logp);
  return cudaGetLastError();
}

// float32 [rows, D] -> bfloat16 [rows, Dp] (Dp % 8 == 0, zero padded): the
// policy's aligned input, one 16-byte store of 8 bf16 per thread.
__global__ void pack_bf16_kernel(const float* __restrict__ src, int64_t rows, int D, int Dp,
                                 __nv_bfloat16* __restrict__ dst) {
  const int per_row = Dp >> 3;
  const int64_t n = rows * per_row;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = q / per_row;
    const int c0 = (int)(q - r * per_row) << 3;
    const float* s = src + r * D;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __float2bfloat16_rn(c0 + k < D ? s[c0 + k] : 0.0f);
    *reinterpret_cast<uint4*>(dst + r * Dp + c0) = *reinterpret_cast<const uint4*>(v);
  }
}

cudaError_t launch_pack_bf16(const float* src, int64_t rows, int D, int Dp, void* dst,
                             int sm_count, cudaStream_t stream) {
  const int64_t n = rows * (Dp >> 3);
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)sm_count * 32) blocks = (int64_t)sm_count * 32;
  pack_bf16_kernel<<<(int)blocks, 256, 0, stream>>>(src, rows, D, Dp, (__nv_bfloat16*)dst);
  return cudaGetLastError();
}

}  // namespace tabx
