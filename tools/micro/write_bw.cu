// Write-bandwidth ceilings on this GPU for the observation stream's pattern:
// (1) cudaMemsetAsync, (2) plain coalesced float4 stores, (3) per-warp TMA
// bulk stores of 3,088-byte chunks from shared memory, double-buffered, 24
// warps/SM (the observation kernel's geometry without its compute).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_bw write_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void st4(float4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_float4(0.f, 1.f, 2.f, 3.f);
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void tma_store(char* dst, size_t chunks, int chunk_bytes) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
  unsigned char* buf = sm + (size_t)w * 2 * chunk_bytes;
  for (int i = lane * 16; i < 2 * chunk_bytes; i += 512) *(uint4*)(buf + i) = make_uint4(1, 2, 3, 4);
  __syncwarp();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  int b = 0;
  for (size_t c = (size_t)blockIdx.x * wpb + w; c < chunks; c += (size_t)gridDim.x * wpb) {
    if (lane == 0) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * chunk_bytes),
                   "r"(sa(buf + b * chunk_bytes)), "r"(chunk_bytes) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    b ^= 1;
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t bytes = (size_t)8 << 30;
  char* d;
  cudaMalloc(&d, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    cudaMemsetAsync(d, rep, bytes);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("memset        %.0f GB/s\n", bytes / ms / 1e6);
    cudaEventRecord(a);
    st4<<<148 * 16, 512>>>((float4*)d, bytes / 16);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("float4 stores %.0f GB/s\n", bytes / ms / 1e6);
    for (int cb : {3088, 6176, 12352}) {
      const int wpb = 8;
      const size_t smem = (size_t)wpb * 2 * cb;
      cudaFuncSetAttribute(tma_store, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tma_store, wpb * 32, smem);
      const size_t chunks = bytes / cb;
      cudaEventRecord(a);
      tma_store<<<148 * per_sm, wpb * 32, smem>>>(d, chunks, cb);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("TMA %5d B chunks, %d warps/SM: %.0f GB/s (%s)\n", cb, per_sm * wpb,
             chunks * (double)cb / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
