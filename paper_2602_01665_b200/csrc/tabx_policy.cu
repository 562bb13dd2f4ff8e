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

namespace tabx {

__device__ __forceinline__ uint64_t sm_mix(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

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
  const uint64_t step = (step_ptr ? *step_ptr : 0ull) + step_add;
  const uint64_t key = sm_mix(seed + 0x9E3779B97F4A7C15ull * (step + 1));
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < M;
       r += (int64_t)gridDim.x * blockDim.x) {
    const T* l = logits + r * ld;
    const uint8_t* m = mask + r * TABX_NUM_ACTIONS;
    float v[TABX_NUM_ACTIONS];
    float mx = -INFINITY;
#pragma unroll
    for (int a = 0; a < TABX_NUM_ACTIONS; ++a) {
      v[a] = m[a] ? load_logit<T>(l + a) : -INFINITY;
      mx = fmaxf(mx, v[a]);
    }
    float se = 0.0f, best = -INFINITY;
    int arg = TABX_NUM_ACTIONS - 1;
    const uint64_t h = sm_mix(key ^ (uint64_t)r * 0xD1B54A32D192ED03ull);
#pragma unroll
    for (int a = 0; a < TABX_NUM_ACTIONS; ++a) {
      if (v[a] == -INFINITY) continue;
      se += __expf(v[a] - mx);
      const uint64_t z = sm_mix(h + (uint64_t)(a + 1) * 0x9E3779B97F4A7C15ull);
      const float u = ((float)(z >> 40) + 0.5f) * (1.0f / 16777216.0f);  // (0, 1)
      const float g = v[a] - __logf(-__logf(u));
      if (g > best) {
        best = g;
        arg = a;
      }
    }
    actions[r] = arg;
    logp[r] = v[arg] - mx - __logf(se);
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
