/*
 * A C caller of the drop-in boundary (include/tabx.h) with no Python in the
 * loop: reads one tabx_config (raw struct bytes, written by the test from a
 * scenario document), creates a batch, steps it with host-chosen external
 * actions, and prints per-step checksums of the outputs a trainer reads back.
 *
 *   abi_driver <config.bin> <batch> <steps> <seed0>
 *
 * Lane seeds are seed0 + b; external actions are the deterministic pattern
 * (b + i + t) % 5 (moves / rotate, always legal for live units).
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "tabx.h"

#define CK(x)                                                         \
  do {                                                                \
    int rc_ = (x);                                                    \
    if (rc_) {                                                        \
      fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, tabx_last_error()); \
      return 1;                                                       \
    }                                                                 \
  } while (0)

int main(int argc, char** argv) {
  if (argc < 5) return 2;
  FILE* f = fopen(argv[1], "rb");
  if (!f) return 2;
  tabx_config cfg;
  if (fread(&cfg, sizeof(cfg), 1, f) != 1) return 2;
  fclose(f);
  const int64_t B = atoll(argv[2]);
  const int T = atoi(argv[3]);
  const uint64_t seed0 = strtoull(argv[4], NULL, 10);
  uint64_t* seeds = (uint64_t*)malloc(8 * B);
  for (int64_t b = 0; b < B; ++b) seeds[b] = seed0 + (uint64_t)b;
  tabx_handle* h = NULL;
  CK(tabx_create(&cfg, 1, NULL, seeds, B, 1, 0, NULL, &h));
  int64_t bb;
  int32_t N, Z, D, G;
  CK(tabx_dims(h, &bb, &N, &Z, &D, &G));
  float *obs, *glob, *rew;
  uint8_t *mask, *term, *trunc;
  int64_t* act_d;
  cudaMalloc((void**)&obs, 4 * B * N * D);
  cudaMalloc((void**)&glob, 4 * B * G);
  cudaMalloc((void**)&rew, 4 * B * N);
  cudaMalloc((void**)&mask, B * N * TABX_NUM_ACTIONS);
  cudaMalloc((void**)&term, B);
  cudaMalloc((void**)&trunc, B);
  cudaMalloc((void**)&act_d, 8 * B * N);
  tabx_outputs out;
  memset(&out, 0, sizeof(out));
  out.observations = obs;
  out.global_state = glob;
  out.rewards = rew;
  out.action_mask = mask;
  out.terminated = term;
  out.truncated = trunc;
  CK(tabx_init_output(h, &out));
  int64_t* act_h = (int64_t*)malloc(8 * B * N);
  float* rew_h = (float*)malloc(4 * B * N);
  float* obs_h = (float*)malloc(4 * B * N * D);
  for (int t = 0; t < T; ++t) {
    for (int64_t b = 0; b < B; ++b)
      for (int i = 0; i < N; ++i) act_h[b * N + i] = (b + i + t) % 5;
    cudaMemcpy(act_d, act_h, 8 * B * N, cudaMemcpyHostToDevice);
    CK(tabx_step(h, act_d, &out));
    tabx_error err;
    CK(tabx_get_error(h, &err, 1));
    if (err.code) {
      printf("error %d env %lld unit %d action %lld\n", err.code, (long long)err.env, err.unit,
             (long long)err.action);
      return 3;
    }
    cudaMemcpy(rew_h, rew, 4 * B * N, cudaMemcpyDeviceToHost);
    cudaMemcpy(obs_h, obs, 4 * B * N * D, cudaMemcpyDeviceToHost);
    double rs = 0.0, os = 0.0;
    for (int64_t k = 0; k < B * N; ++k) rs += rew_h[k] * (double)((k % 7) + 1);
    for (int64_t k = 0; k < B * N * D; ++k) os += obs_h[k] * (double)((k % 13) + 1);
    printf("%d %.17g %.17g\n", t, rs, os);
  }
  CK(tabx_destroy(h));
  return 0;
}
