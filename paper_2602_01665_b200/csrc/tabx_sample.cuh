// Masked Gumbel-max sampling of one agent row (the rollout loop's sampler,
// C5): shared by the stand-alone sampler kernel (tabx_policy.cu) and the
// policy-MLP kernel's fused epilogue (tabx_mlp.cu), so both draw the same
// action and log-probability from the same logits.  The noise is a
// counter-based hash of (seed, step, agent, action).
#pragma once
#include <stdint.h>

#include "tabx.h"

namespace tabx {

// optional fused masked sampling of the policy-MLP logits (mask == nullptr: off)
struct MlpSample {
  const uint8_t* mask;  // [rows, TABX_NUM_ACTIONS]
  uint64_t seed;
  const uint64_t* step_ptr;
  uint64_t step_add;
  int64_t* actions;
  float* logp;
};

__device__ __forceinline__ uint64_t sm_mix(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// per-launch noise key: step = *step_ptr (device counter, may be null) + step_add
__device__ __forceinline__ uint64_t sample_key(uint64_t seed, const uint64_t* step_ptr,
                                               uint64_t step_add) {
  const uint64_t step = (step_ptr ? *step_ptr : 0ull) + step_add;
  return sm_mix(seed + 0x9E3779B97F4A7C15ull * (step + 1));
}

// lg: the row's first TABX_NUM_ACTIONS logits; m: its mask row (bytes)
__device__ __forceinline__ void sample_row(const float* lg, const uint8_t* __restrict__ m,
                                           uint64_t key, int64_t r, int64_t* __restrict__ actions,
                                           float* __restrict__ logp) {
  float v[TABX_NUM_ACTIONS];
  float mx = -INFINITY;
#pragma unroll
  for (int a = 0; a < TABX_NUM_ACTIONS; ++a) {
    v[a] = m[a] ? lg[a] : -INFINITY;
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

}  // namespace tabx
