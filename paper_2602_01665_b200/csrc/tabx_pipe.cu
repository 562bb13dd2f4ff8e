// Native pipelined host stepping (include/tabx.h, tabx_pipe_*): host int64
// actions in, host rewards / terminated / truncated out, every step, with the
// copies on their own streams overlapping the neighbouring steps' kernels.
// The Python HostStepper (bindings.py) did the same orchestration with ~13
// Python-level CUDA calls per step, which made small batches (C1, 256 envs:
// 0.025 ms of device work per step) host-bound; here a step is one C call.
//
// Per step k in slot s = k % depth:
//   (slot reuse) wait until step k - depth's results reached the host
//   up:   copy the host actions into the slot's device buffer, record h2d[s]
//   main: wait h2d[s]; tabx_step writing rewards / terminated / truncated into
//         the slot's device buffers; copy the latched error word; record
//         staged[s]
//   down: wait staged[s]; copy the slot's results to its pinned host
//         buffers; record d2h[s]
// tabx_pipe_result(k) waits d2h[s] and returns the pinned host pointers.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <new>
#include <string>

#include "../../include/tabx.h"

struct tabx_pipe {
  tabx_handle* h = nullptr;
  int device = 0;
  int depth = 0;
  int64_t B = 0;
  int N = 0;
  cudaStream_t main = nullptr, up = nullptr, down = nullptr;
  tabx_outputs outs[TABX_PIPE_MAX_DEPTH];
  int64_t* act_dev[TABX_PIPE_MAX_DEPTH] = {};
  float* rew_dev[TABX_PIPE_MAX_DEPTH] = {};
  uint8_t* flag_dev[TABX_PIPE_MAX_DEPTH] = {};  // [2, B]: terminated, truncated
  uint64_t* err_dev[TABX_PIPE_MAX_DEPTH] = {};
  float* rew_host[TABX_PIPE_MAX_DEPTH] = {};
  uint8_t* flag_host[TABX_PIPE_MAX_DEPTH] = {};
  uint64_t* err_host[TABX_PIPE_MAX_DEPTH] = {};
  cudaEvent_t h2d[TABX_PIPE_MAX_DEPTH] = {}, staged[TABX_PIPE_MAX_DEPTH] = {},
              d2h[TABX_PIPE_MAX_DEPTH] = {};
  int64_t used[TABX_PIPE_MAX_DEPTH];
  int64_t next = 0;
};

namespace {

struct Guard {
  int prev = -1;
  explicit Guard(int d) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != d) cudaSetDevice(d);
    else prev = -1;
  }
  ~Guard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

void free_pipe(tabx_pipe* p) {
  if (!p) return;
  if (p->up) cudaStreamSynchronize(p->up);
  if (p->down) cudaStreamSynchronize(p->down);
  for (int s = 0; s < TABX_PIPE_MAX_DEPTH; ++s) {
    cudaFree(p->act_dev[s]);
    cudaFree(p->rew_dev[s]);
    cudaFree(p->flag_dev[s]);
    cudaFree(p->err_dev[s]);
    cudaFreeHost(p->rew_host[s]);
    cudaFreeHost(p->flag_host[s]);
    cudaFreeHost(p->err_host[s]);
    if (p->h2d[s]) cudaEventDestroy(p->h2d[s]);
    if (p->staged[s]) cudaEventDestroy(p->staged[s]);
    if (p->d2h[s]) cudaEventDestroy(p->d2h[s]);
  }
  if (p->up) cudaStreamDestroy(p->up);
  if (p->down) cudaStreamDestroy(p->down);
  delete p;
}

}  // namespace

extern "C" {

int tabx_pipe_create(tabx_handle* h, int32_t depth, const tabx_outputs* base, void* stream,
                     tabx_pipe** out) {
  if (!h || !base || !out || depth < 1 || depth > TABX_PIPE_MAX_DEPTH) return TABX_E_ARGUMENT;
  int64_t B = 0;
  int32_t N = 0;
  int rc = tabx_dims(h, &B, &N, nullptr, nullptr, nullptr);
  if (rc) return rc;
  tabx_pipe* p = new (std::nothrow) tabx_pipe();
  if (!p) return TABX_E_CUDA;
  p->h = h;
  p->depth = depth;
  p->B = B;
  p->N = N;
  p->main = (cudaStream_t)stream;
  cudaGetDevice(&p->device);
  cudaError_t e = cudaStreamCreateWithFlags(&p->up, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->down, cudaStreamNonBlocking);
  for (int s = 0; s < depth && e == cudaSuccess; ++s) {
    p->used[s] = -1;
    p->outs[s] = *base;
    if (e == cudaSuccess) e = cudaMalloc(&p->act_dev[s], sizeof(int64_t) * B * N);
    if (e == cudaSuccess) e = cudaMalloc(&p->rew_dev[s], sizeof(float) * B * N);
    if (e == cudaSuccess) e = cudaMalloc(&p->flag_dev[s], 2 * B);
    if (e == cudaSuccess) e = cudaMalloc(&p->err_dev[s], 8);
    if (e == cudaSuccess) e = cudaHostAlloc(&p->rew_host[s], sizeof(float) * B * N, 0);
    if (e == cudaSuccess) e = cudaHostAlloc(&p->flag_host[s], 2 * B, 0);
    if (e == cudaSuccess) e = cudaHostAlloc(&p->err_host[s], 8, 0);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->h2d[s], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->staged[s], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->d2h[s], cudaEventDisableTiming);
    if (e == cudaSuccess) {
      p->outs[s].rewards = p->rew_dev[s];
      p->outs[s].terminated = p->flag_dev[s];
      p->outs[s].truncated = p->flag_dev[s] + B;
    }
  }
  if (e != cudaSuccess) {
    free_pipe(p);
    return TABX_E_CUDA;
  }
  *out = p;
  return TABX_OK;
}

int tabx_pipe_submit(tabx_pipe* p, const int64_t* host_actions, int64_t* ticket) {
  if (!p || !host_actions) return TABX_E_ARGUMENT;
  Guard g(p->device);
  const int64_t k = p->next;
  const int s = (int)(k % p->depth);
  // the slot's previous results must have reached the host
  if (p->used[s] >= 0 && cudaEventSynchronize(p->d2h[s]) != cudaSuccess) return TABX_E_CUDA;
  const size_t ab = sizeof(int64_t) * p->B * p->N;
  if (cudaMemcpyAsync(p->act_dev[s], host_actions, ab, cudaMemcpyHostToDevice, p->up) !=
          cudaSuccess ||
      cudaEventRecord(p->h2d[s], p->up) != cudaSuccess ||
      cudaStreamWaitEvent(p->main, p->h2d[s], 0) != cudaSuccess)
    return TABX_E_CUDA;
  int rc = tabx_step(p->h, p->act_dev[s], &p->outs[s]);
  if (rc) return rc;
  rc = tabx_copy_error_word(p->h, p->err_dev[s]);
  if (rc) return rc;
  if (cudaEventRecord(p->staged[s], p->main) != cudaSuccess ||
      cudaStreamWaitEvent(p->down, p->staged[s], 0) != cudaSuccess ||
      cudaMemcpyAsync(p->rew_host[s], p->rew_dev[s], sizeof(float) * p->B * p->N,
                      cudaMemcpyDeviceToHost, p->down) != cudaSuccess ||
      cudaMemcpyAsync(p->flag_host[s], p->flag_dev[s], 2 * p->B, cudaMemcpyDeviceToHost,
                      p->down) != cudaSuccess ||
      cudaMemcpyAsync(p->err_host[s], p->err_dev[s], 8, cudaMemcpyDeviceToHost, p->down) !=
          cudaSuccess ||
      cudaEventRecord(p->d2h[s], p->down) != cudaSuccess)
    return TABX_E_CUDA;
  p->used[s] = k;
  p->next = k + 1;
  if (ticket) *ticket = k;
  return TABX_OK;
}

int tabx_pipe_result(tabx_pipe* p, int64_t ticket, const float** rewards,
                     const uint8_t** terminated, const uint8_t** truncated,
                     int64_t* error_index) {
  if (!p || ticket < 0) return TABX_E_ARGUMENT;
  const int s = (int)(ticket % p->depth);
  if (p->used[s] != ticket) return TABX_E_ARGUMENT;  // no longer buffered
  Guard g(p->device);
  if (cudaEventSynchronize(p->d2h[s]) != cudaSuccess) return TABX_E_CUDA;
  if (rewards) *rewards = p->rew_host[s];
  if (terminated) *terminated = p->flag_host[s];
  if (truncated) *truncated = p->flag_host[s] + p->B;
  if (error_index) {
    const uint64_t w = *p->err_host[s];
    *error_index = w == ~0ull ? -1 : (int64_t)w;
  }
  return TABX_OK;
}

int tabx_pipe_destroy(tabx_pipe* p) {
  if (!p) return TABX_OK;
  Guard g(p->device);
  free_pipe(p);
  return TABX_OK;
}

}  // extern "C"
