// Policy MLP of the on-device rollout loop (C5) on the
// 5th-generation tensor cores: logits = W2 · bf16(relu(W1 · x + b1)) + b2 for
// every agent row x (bf16, K features), hidden = 128, 8 logits, in ONE pass
// over x.  The cuBLASLt pair it replaces reads x, writes the hidden
// activations, reads them back and writes the logits; here the hidden tile
// never leaves the SM (TMEM -> registers), so HBM sees x once and 16 B of
// logits per row.
//
// Two kernels (tabx_policy_mlp picks by K):
//   * mlp_policy_tma_kernel (K <= 704, the rollout's shapes): TMA-fed,
//     warp-specialised, W1 resident in shared memory; see its comment below.
//   * mlp_policy_kernel (larger K, where W1 does not fit beside the x
//     stages): 128 threads per CTA stage each K chunk of 80 features of x and
//     W1 with cp.async (zero-filled past K and past the last row) into the
//     no-swizzle K-major UMMA layout (8-row x 16-byte core matrices, LBO
//     128 B along K, SBO 1,280 B between 8-row groups), thread 0 issues the
//     MMAs, the same threads run the epilogue.
// Both share the epilogue (mlp_epilogue_cols): tcgen05.ld 32x32b.x32 of the
// accumulator rows, + b1, ReLU, bf16 rounding (the module's hidden dtype),
// times W2 (fp32 copy in shared memory, broadcast reads) into 8 logits; one
// 16-byte store per row.
#include <cuda_bf16.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "tabx_device.cuh"
#include "tabx_sample.cuh"

namespace tabx {

constexpr int MLP_THREADS = 128;
constexpr int MLP_M = 128;       // rows per tile (UMMA M, TMEM lanes)
constexpr int MLP_H = 128;       // hidden units (UMMA N, TMEM columns)
constexpr int MLP_OUT = 8;       // logits per row
constexpr int MLP_KC = 80;       // K features per chunk (5 x UMMA K = 16)
constexpr int MLP_STAGES = 5;
constexpr int MLP_SBO = (MLP_KC / 8) * 128;           // bytes between 8-row groups
constexpr int MLP_OPND = MLP_M * MLP_KC * 2;          // 20,480 B per operand per stage
constexpr int MLP_STAGE_BYTES = 2 * MLP_OPND;         // x chunk + W1 chunk
constexpr int MLP_SMEM = MLP_STAGES * MLP_STAGE_BYTES + MLP_H * MLP_OUT * 4 + MLP_H * 4 +
                         MLP_OUT * 4 + (MLP_STAGES + 1) * 8 + 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  long long t0 = 0;
  for (int spin = 0;; ++spin) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    // a lost arrival must not hang the device: trap after ~1 s
    if (spin == 1024) t0 = clock64();
    if (spin > 1024 && (spin & 1023) == 0 && clock64() - t0 > 2000000000ll) __trap();
  }
}

// UMMA shared-memory descriptor, no swizzle, K-major (version 1 = sm_100)
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// instruction descriptor: f32 accumulate, bf16 A and B, both K-major, N, M
constexpr uint32_t MLP_IDESC = (1u << 4) | (1u << 7) | (1u << 10) |
                               ((uint32_t)(MLP_H >> 3) << 17) | ((uint32_t)(MLP_M >> 4) << 24);

// smem byte offset of element (r, k) of a [128 x 80] chunk operand
__device__ __forceinline__ uint32_t chunk_off(int r, int kp) {
  return (uint32_t)((r >> 3) * MLP_SBO + kp * 128 + (r & 7) * 16);
}

#ifndef MLP_PROMO
#define MLP_PROMO 2
#endif
#ifndef MLP_EXP
#define MLP_EXP 0  // probe builds only: 1 = epilogue without its math, 2 = no MMAs
#endif
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Accumulates into lg the layer-2 contribution of hidden units
// [h0, h0 + 32 * NCB) of this thread's row (TMEM address ta = its lane and
// column h0): + b1, ReLU, bf16 rounding, times W2.  With empty_bar != 0 the
// thread arrives there once its last TMEM load has completed.
template <int NCB>
__device__ __forceinline__ void mlp_epilogue_cols(uint32_t ta, int h0, const float* w2s,
                                                  const float* b1s, float* lg,
                                                  uint32_t empty_bar) {
#pragma unroll
  for (int cb = 0; cb < NCB; ++cb) {
    uint32_t v[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, "
        "%10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, "
        "%26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(ta + (uint32_t)(cb * 32)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (empty_bar && cb == NCB - 1) {  // the accumulator may be overwritten
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(empty_bar);
    }
    if (MLP_EXP == 1) {
      lg[cb] += __uint_as_float(v[0]) + __uint_as_float(v[31]);
      continue;
    }
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int h = h0 + cb * 32 + q;
      float a = __fadd_rn(__uint_as_float(v[q]), b1s[h]);
      a = __bfloat162float(__float2bfloat16_rn(fmaxf(a, 0.0f)));
      const float4 wa = *reinterpret_cast<const float4*>(&w2s[h * MLP_OUT]);
      const float4 wb = *reinterpret_cast<const float4*>(&w2s[h * MLP_OUT + 4]);
      lg[0] = __fmaf_rn(a, wa.x, lg[0]);
      lg[1] = __fmaf_rn(a, wa.y, lg[1]);
      lg[2] = __fmaf_rn(a, wa.z, lg[2]);
      lg[3] = __fmaf_rn(a, wa.w, lg[3]);
      lg[4] = __fmaf_rn(a, wb.x, lg[4]);
      lg[5] = __fmaf_rn(a, wb.y, lg[5]);
      lg[6] = __fmaf_rn(a, wb.z, lg[6]);
      lg[7] = __fmaf_rn(a, wb.w, lg[7]);
    }
  }
}

__device__ __forceinline__ void store_logits(__nv_bfloat16* out, int64_t row, const float* lg) {
  __align__(16) __nv_bfloat16 ob[MLP_OUT];
#pragma unroll
  for (int o = 0; o < MLP_OUT; ++o) ob[o] = __float2bfloat16_rn(lg[o]);
  *reinterpret_cast<uint4*>(out + row * MLP_OUT) = *reinterpret_cast<const uint4*>(ob);
}

__global__ void __launch_bounds__(MLP_THREADS, 1)
    mlp_policy_kernel(const __nv_bfloat16* __restrict__ x, int64_t rows, int K, int64_t ldx,
                      const __nv_bfloat16* __restrict__ w1, const __nv_bfloat16* __restrict__ b1,
                      const __nv_bfloat16* __restrict__ w2, const __nv_bfloat16* __restrict__ b2,
                      __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* stages = sm;
  float* w2s = reinterpret_cast<float*>(sm + MLP_STAGES * MLP_STAGE_BYTES);  // [H][OUT]
  float* b1s = w2s + MLP_H * MLP_OUT;
  float* b2s = b1s + MLP_H;
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(b2s + MLP_OUT) + 7) & ~(uintptr_t)7);  // [STAGES] + acc
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + MLP_STAGES + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int q = tid; q < MLP_H * MLP_OUT; q += MLP_THREADS) {
    const int j = q / MLP_OUT, o = q % MLP_OUT;
    w2s[q] = __bfloat162float(w2[o * MLP_H + j]);
  }
  for (int q = tid; q < MLP_H; q += MLP_THREADS) b1s[q] = __bfloat162float(b1[q]);
  if (tid < MLP_OUT) b2s[tid] = __bfloat162float(b2[tid]);
  if (tid == 0) {
    for (int s = 0; s <= MLP_STAGES; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(MLP_H));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  const int nch = (K + MLP_KC - 1) / MLP_KC;
  const int64_t ntiles = (rows + MLP_M - 1) / MLP_M;
  const int64_t my_tiles =
      blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nchunks = my_tiles * nch;
  const uint32_t stage0 = smem_u32(stages);

  // stage chunk c (tile c / nch of this CTA, K chunk c % nch): x and W1 rows
  auto issue = [&](int64_t c) {
    const int64_t tile = blockIdx.x + (c / nch) * gridDim.x;
    const int j = (int)(c % nch);
    const uint32_t sa = stage0 + (uint32_t)(c % MLP_STAGES) * MLP_STAGE_BYTES;
    const uint32_t sb = sa + MLP_OPND;
    // piece p: 8 consecutive threads fill one 128-B core matrix (rows r&7)
    for (int p = tid; p < MLP_M * (MLP_KC / 8); p += MLP_THREADS) {
      const int r = (p & 7) | ((p / (8 * (MLP_KC / 8))) << 3);
      const int kp = (p >> 3) % (MLP_KC / 8);
      const int k = j * MLP_KC + kp * 8;
      const int64_t row = tile * MLP_M + r;
      const bool kin = k < K;
      const bool xin = kin && row < rows;
      cp16(sa + chunk_off(r, kp), xin ? (const void*)(x + row * ldx + k) : (const void*)x,
           xin ? 16u : 0u);
      cp16(sb + chunk_off(r, kp), kin ? (const void*)(w1 + (int64_t)r * K + k) : (const void*)w1,
           kin ? 16u : 0u);
    }
  };

  for (int64_t c = 0; c < MLP_STAGES - 1; ++c) {
    if (c < nchunks) issue(c);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t cn = c + MLP_STAGES - 1;
    if (cn < nchunks) {
      if (cn >= MLP_STAGES)  // the MMAs of chunk cn - STAGES read this stage
        mbar_wait(smem_u32(&bars[cn % MLP_STAGES]), (uint32_t)((cn / MLP_STAGES - 1) & 1));
      issue(cn);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(MLP_STAGES - 1) : "memory");
    // the generic-proxy writes of cp.async become visible to the tensor cores
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const int j = (int)(c % nch);
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t sa = stage0 + (uint32_t)(c % MLP_STAGES) * MLP_STAGE_BYTES;
      const uint32_t sb = sa + MLP_OPND;
#pragma unroll
      for (int kk = 0; kk < MLP_KC / 16; ++kk) {
        const uint64_t da = umma_desc(sa + kk * 256, 128, MLP_SBO);
        const uint64_t db = umma_desc(sb + kk * 256, 128, MLP_SBO);
        const uint32_t acc = (j > 0 || kk > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(MLP_IDESC), "r"(acc)
            : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::
                       "r"(smem_u32(&bars[c % MLP_STAGES]))
                   : "memory");
      if (j == nch - 1)
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&bars[MLP_STAGES]))
            : "memory");
    }
    if (j == nch - 1) {  // epilogue of this tile
      const int64_t it = c / nch;
      const int64_t tile = blockIdx.x + it * gridDim.x;
      mbar_wait(smem_u32(&bars[MLP_STAGES]), (uint32_t)(it & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float lg[MLP_OUT];
#pragma unroll
      for (int o = 0; o < MLP_OUT; ++o) lg[o] = b2s[o];
      mlp_epilogue_cols<MLP_H / 32>(tmem + ((uint32_t)(warp * 32) << 16), 0, w2s, b1s, lg, 0u);
      const int64_t row = tile * MLP_M + warp * 32 + lane;
      if (row < rows) store_logits(out, row, lg);
      // every warp has read the accumulator before the next tile's MMAs
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(MLP_H));
}

// ---------------------------------------------------------------------------
// Main kernel (K <= 704): TMA-fed, warp-specialised, W1 resident.  x and W1
// are read through 2-D tensor maps as [128 rows x 64 features] boxes with the
// 128-byte swizzle (the layout the UMMA descriptor's SWIZZLE_128B mode
// reads: rows 128 B apart, 8-row groups 1,024 B apart, K advanced by 32 B
// per 16-feature MMA inside the swizzle atom); the TMA unit zero-fills past
// K and past the last row.  W1 is loaded once per CTA (every SM re-reading
// W1 chunks from L2 each tile is a hot spot).  Roles: MLP_EW epilogue warps
// (warp w reads TMEM lanes 32 (w % 4).. and hidden slice w / 4; slices are
// summed through shared memory), then one warp whose lane 0 issues the TMA
// loads and one whose lane 0 issues the MMAs.  Two TMEM accumulators (256
// columns): the epilogue of tile t overlaps the MMAs of tile t + 1.
#ifndef MLP_EW
#define MLP_EW 16
#endif
constexpr int MLPT_EW = MLP_EW;                 // epilogue warps (4 per TMEM sub-partition)
constexpr int MLPT_PARTS = MLPT_EW / 4;         // hidden-unit slices per row
constexpr int MLPT_THREADS = 32 * (MLPT_EW + 2);  // + TMA warp + MMA warp
constexpr int MLPT_KB = 64;                     // features per box / chunk
constexpr int MLPT_BOX = MLP_M * MLPT_KB * 2;   // 16,384 B
constexpr int MLPT_SMEM_MAX = 232448;           // 227 KB opt-in per CTA
constexpr int MLPT_MISC =
    MLP_H * MLP_OUT * 4 + MLP_H * 4 + MLP_OUT * 4 + 2 * (MLPT_PARTS - 1) * MLP_M * MLP_OUT * 4 +
    32 * 8 + 16 + 1024;

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__global__ void __launch_bounds__(MLPT_THREADS, 1)
    mlp_policy_tma_kernel(const __grid_constant__ CUtensorMap tx,
                          const __grid_constant__ CUtensorMap tw, int64_t rows, int K,
                          const __nv_bfloat16* __restrict__ b1,
                          const __nv_bfloat16* __restrict__ w2,
                          const __nv_bfloat16* __restrict__ b2, __nv_bfloat16* __restrict__ out,
                          int nstages, const MlpSample sa) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  const uint32_t raw = smem_u32(sm_raw);
  unsigned char* sm = sm_raw + (((raw + 1023u) & ~1023u) - raw);  // 1,024-B aligned
  const int nch = (K + MLPT_KB - 1) / MLPT_KB;
  const uint32_t w1a = smem_u32(sm);
  const uint32_t stage0 = w1a + (uint32_t)nch * MLPT_BOX;
  float* w2s = reinterpret_cast<float*>(sm + (size_t)(nch + nstages) * MLPT_BOX);
  float* b1s = w2s + MLP_H * MLP_OUT;
  float* b2s = b1s + MLP_H;
  float* red = b2s + MLP_OUT;  // [2][PARTS-1][128][8] partial logits of slices 1..
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(red + 2 * (MLPT_PARTS - 1) * MLP_M * MLP_OUT) + 7) &
      ~(uintptr_t)7);
  uint64_t* full = bars;          // [nstages]  x box landed (TMA bytes)
  uint64_t* empty = bars + 8;     // [nstages]  MMAs done reading it
  uint64_t* acc_full = bars + 16; // [2]
  uint64_t* acc_empty = bars + 18;// [2]        256 epilogue arrivals
  uint64_t* wfull = bars + 20;    // W1 landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 21);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int q = tid; q < MLP_H * MLP_OUT; q += MLPT_THREADS) {
    const int j = q / MLP_OUT, o = q % MLP_OUT;
    w2s[q] = __bfloat162float(w2[o * MLP_H + j]);
  }
  for (int q = tid; q < MLP_H; q += MLPT_THREADS) b1s[q] = __bfloat162float(b1[q]);
  if (tid < MLP_OUT) b2s[tid] = __bfloat162float(b2[tid]);
  if (tid == 0) {
    for (int s = 0; s < nstages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])));
    }
    for (int a = 0; a < 2; ++a) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&acc_full[a])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&acc_empty[a])),
                   "n"(32 * MLPT_EW));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(wfull)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(2 * MLP_H));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  const int64_t ntiles = (rows + MLP_M - 1) / MLP_M;
  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nchunks = my_tiles * nch;

  // stage / phase counters advance incrementally: these two loops are single
  // threads whose instruction latency bounds the whole pipeline
  if (warp == MLPT_EW) {  // ---- TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tx)) : "memory");
      mbar_expect(smem_u32(wfull), (uint32_t)nch * MLPT_BOX);
      for (int j = 0; j < nch; ++j)
        tma_load_2d(w1a + (uint32_t)j * MLPT_BOX, &tw, j * MLPT_KB, 0, smem_u32(wfull));
      int st = 0, j = 0;
      uint32_t ph = 0;
      int row0 = (int)blockIdx.x * MLP_M;
      const int row_step = (int)gridDim.x * MLP_M;
      const uint32_t full0 = smem_u32(full), empty0 = smem_u32(empty);
      for (int64_t c = 0; c < nchunks; ++c) {
        if (c >= nstages) mbar_wait(empty0 + 8u * st, ph ^ 1u);
        mbar_expect(full0 + 8u * st, MLPT_BOX);
        tma_load_2d(stage0 + (uint32_t)st * MLPT_BOX, &tx, j * MLPT_KB, row0, full0 + 8u * st);
        if (++j == nch) {
          j = 0;
          row0 += row_step;
        }
        if (++st == nstages) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
    __syncwarp();
  } else if (warp == MLPT_EW + 1) {  // ---- MMA issuer
    if (lane == 0) {
      mbar_wait(smem_u32(wfull), 0u);
      const uint64_t da0 = umma_desc_sw128(stage0), db0 = umma_desc_sw128(w1a);
      const uint32_t full0 = smem_u32(full), empty0 = smem_u32(empty);
      int st = 0;
      uint32_t ph = 0;
      for (int64_t it = 0; it < my_tiles; ++it) {
        const int a = (int)(it & 1);
        if (it >= 2) mbar_wait(smem_u32(&acc_empty[a]), (uint32_t)(((it >> 1) - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc_t = tmem + (uint32_t)(a * MLP_H);
        for (int j = 0; j < nch; ++j) {
          mbar_wait(full0 + 8u * st, ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          // descriptor start-address field counts 16-byte units
          const uint64_t da = da0 + (uint64_t)(st * (MLPT_BOX >> 4));
          const uint64_t db = db0 + (uint64_t)(j * (MLPT_BOX >> 4));
#pragma unroll
          for (int kk = 0; kk < (MLP_EXP == 2 ? 0 : MLPT_KB / 16); ++kk) {
            const uint32_t accum = (j > 0 || kk > 0) ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "setp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc_t),
                "l"(da + 2u * kk), "l"(db + 2u * kk), "r"(MLP_IDESC), "r"(accum)
                : "memory");
          }
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                  empty0 + 8u * st)
              : "memory");
          if (++st == nstages) {
            st = 0;
            ph ^= 1u;
          }
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&acc_full[a]))
            : "memory");
      }
    }
    __syncwarp();
  } else {  // ---- epilogue: warp w -> TMEM lanes 32 (w % 4).., hidden slice w / 4
    constexpr int HS = MLP_H / MLPT_PARTS;  // hidden units per slice
    const int sub = warp & 3, part = warp >> 2;
    const uint64_t skey = sa.mask ? sample_key(sa.seed, sa.step_ptr, sa.step_add) : 0ull;
    for (int64_t it = 0; it < my_tiles; ++it) {
      const int a = (int)(it & 1);
      mbar_wait(smem_u32(&acc_full[a]), (uint32_t)((it / 2) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float lg[MLP_OUT];
#pragma unroll
      for (int o = 0; o < MLP_OUT; ++o) lg[o] = part ? 0.0f : b2s[o];
      mlp_epilogue_cols<HS / 32>(
          tmem + ((uint32_t)(sub * 32) << 16) + (uint32_t)(a * MLP_H + part * HS), part * HS,
          w2s, b1s, lg, smem_u32(&acc_empty[a]));
      const int r = sub * 32 + lane;
      if (part) {
        float* rr = red + (((size_t)a * (MLPT_PARTS - 1) + part - 1) * MLP_M + r) * MLP_OUT;
        *reinterpret_cast<float4*>(rr) = make_float4(lg[0], lg[1], lg[2], lg[3]);
        *reinterpret_cast<float4*>(rr + 4) = make_float4(lg[4], lg[5], lg[6], lg[7]);
      }
      // the warps of this sub-partition (one per slice)
      asm volatile("bar.sync %0, %1;" ::"r"(1 + sub), "n"(32 * MLPT_PARTS) : "memory");
      if (!part) {
#pragma unroll
        for (int q = 1; q < MLPT_PARTS; ++q) {
          const float* rr = red + (((size_t)a * (MLPT_PARTS - 1) + q - 1) * MLP_M + r) * MLP_OUT;
          const float4 u = *reinterpret_cast<const float4*>(rr);
          const float4 w = *reinterpret_cast<const float4*>(rr + 4);
          lg[0] += u.x; lg[1] += u.y; lg[2] += u.z; lg[3] += u.w;
          lg[4] += w.x; lg[5] += w.y; lg[6] += w.z; lg[7] += w.w;
        }
        const int64_t tile = blockIdx.x + it * gridDim.x;
        const int64_t row = tile * MLP_M + r;
        if (row < rows) {
          __align__(16) __nv_bfloat16 ob[MLP_OUT];
#pragma unroll
          for (int o = 0; o < MLP_OUT; ++o) ob[o] = __float2bfloat16_rn(lg[o]);
          if (out)
            *reinterpret_cast<uint4*>(out + row * MLP_OUT) = *reinterpret_cast<const uint4*>(ob);
          if (sa.mask) {  // the sampler on the bf16 logits, as the stand-alone kernel reads them
            float lv[TABX_NUM_ACTIONS];
#pragma unroll
            for (int o = 0; o < TABX_NUM_ACTIONS; ++o) lv[o] = __bfloat162float(ob[o]);
            sample_row(lv, sa.mask + row * TABX_NUM_ACTIONS, skey, row, sa.actions, sa.logp);
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(2 * MLP_H));
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static std::once_flag once;
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// [rows x K] bf16, row stride ld elements, as [128 x 64] 128B-swizzled boxes
static bool encode_rows(CUtensorMap* m, const void* base, int64_t rows, int K, int64_t ld) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  const cuuint32_t box[2] = {MLPT_KB, MLP_M};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             MLP_PROMO == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
             : MLP_PROMO == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                              : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_masked_sample(const void* logits, int bf16, int64_t ld, const uint8_t* mask,
                                 int64_t M, uint64_t seed, const uint64_t* step_ptr,
                                 uint64_t step_add, int64_t* actions, float* logp, int sm_count,
                                 cudaStream_t stream);

static int mlp_tma_stages(int K) {
  const int nch = (K + MLPT_KB - 1) / MLPT_KB;
  return (MLPT_SMEM_MAX - MLPT_MISC) / MLPT_BOX - nch;
}

// The fused sampler runs in the TMA kernel; the W1-streaming kernel (large K)
// needs a logits buffer and a separate sampler pass.
bool mlp_fused_sampling(int K) { return mlp_tma_stages(K) >= 3; }

cudaError_t launch_mlp_policy(const void* x, int64_t rows, int K, int64_t ldx, const void* w1,
                              const void* b1, const void* w2, const void* b2, void* out,
                              const MlpSample& sa, int sm_count, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  const int64_t ntiles = (rows + MLP_M - 1) / MLP_M;
  const int grid = (int)(ntiles < sm_count ? ntiles : sm_count);
  const int nch = (K + MLPT_KB - 1) / MLPT_KB;
  const int tma_stages = mlp_tma_stages(K);
  int per_sm = 0;  // (launch_geometry sets the shared-memory attribute once per device)
  CUtensorMap tx, tw;
  if (tma_stages >= 3 && encode_rows(&tx, x, rows, K, ldx) && encode_rows(&tw, w1, MLP_H, K, K)) {
    const int ns = tma_stages < 8 ? tma_stages : 8;
    const size_t smem = (size_t)(nch + ns) * MLPT_BOX + MLPT_MISC;
    cudaError_t e =
        launch_geometry((const void*)mlp_policy_tma_kernel, MLPT_THREADS, smem, &per_sm);
    if (e != cudaSuccess) return e;
    mlp_policy_tma_kernel<<<grid, MLPT_THREADS, smem, stream>>>(
        tx, tw, rows, K, (const __nv_bfloat16*)b1, (const __nv_bfloat16*)w2,
        (const __nv_bfloat16*)b2, (__nv_bfloat16*)out, ns, sa);
    return cudaGetLastError();
  }
  if (!out) return cudaErrorInvalidValue;  // (the C ABI rejects this case first)
  cudaError_t e = launch_geometry((const void*)mlp_policy_kernel, MLP_THREADS, MLP_SMEM, &per_sm);
  if (e != cudaSuccess) return e;
  mlp_policy_kernel<<<grid, MLP_THREADS, MLP_SMEM, stream>>>(
      (const __nv_bfloat16*)x, rows, K, ldx, (const __nv_bfloat16*)w1,
      (const __nv_bfloat16*)b1, (const __nv_bfloat16*)w2, (const __nv_bfloat16*)b2,
      (__nv_bfloat16*)out);
  e = cudaGetLastError();
  if (e != cudaSuccess || !sa.mask) return e;
  return launch_masked_sample(out, 1, MLP_OUT, sa.mask, rows, sa.seed, sa.step_ptr, sa.step_add,
                              sa.actions, sa.logp, sm_count, stream);
}

}  // namespace tabx
