// Fused step + observation kernel (W = 1, K0 path): one persistent CTA per
// SM, warp-specialised.
//
// The unfused step runs K1 (environment logic, float64 dependency chains:
// issue/latency-bound, 0.10 of HBM) and then K2 (observation stream:
// HBM-bound) back to back, so the SM's issue slots idle during K2 and HBM
// idles during K1.  Here the CTA's step warps run K1's per-environment body
// (run_lane, environment.py:207-348) over the CTA's environments while its
// emitter warps stream the observation rows of the environments already
// stepped (emit_lane, perception.py:52-201): the two limits overlap inside
// one SM.  setmaxnreg moves registers from the emitter warpgroups (which
// need ~80) to the step warpgroups (float64 state + caches).
//
// Hand-off: the CTA's environments are work items k = 0, 1, ... (env
// b = blockIdx.x + k * gridDim.x).  Step warps and emitter warps each take
// items in order from their own shared counter; a step warp publishes item k
// in a shared done-bitmap after its state write-back (release: fence.cta
// then the bit), and the emitter that took item k waits for the bit
// (acquire: the bit, then fence.cta) and reads the post-step state back from
// global memory (L2-resident: it was just written by this SM).  Step warps
// never wait on emitters, so the kernel is deadlock-free by construction.
// Same per-environment code as K1 + K2, so the same bits.
//
// Measured (B200, C3, 262,144 envs; tools/fab.sh): it LOSES, and is off by
// default (TABX_FUSED=1 turns it on).  K1 + K2 = 1.33 + 1.62 ms; fused:
// 8 step + 8 emitter warps (152 / 104 registers) 3.27 ms, 8 + 12 (128 / 72)
// 3.48, 12 + 4 (136 / 104) 5.65, 4 + 16 (128 / 88) 5.12, every warp
// stepping then emitting its own env (16 warps x 128) 3.27.  Both halves are
// per-warp latency-bound, not issue- or bandwidth-bound: a step warp takes
// ~11.5 us per environment whether 4 or 16 step warps share the SM, an
// emitter warp ~12.7 us; the 64 K-register file holds 16 step warps (128
// registers) OR ~24 emitter warps (80), and the fused kernel would need
// ~14 + ~13 of them resident at once to beat the sum of the two kernels.
#include "tabx_lane.cuh"

namespace tabx {

template <int R>
__device__ __forceinline__ void reg_alloc() {
  if constexpr (R > 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(R));
}
template <int R>
__device__ __forceinline__ void reg_dealloc() {
  if constexpr (R > 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(R));
}

struct FusedCtl {
  uint32_t next_step, next_emit, pad0, pad1;
};

__host__ __device__ __forceinline__ size_t fused_ctl_bytes(int items) {
  return (sizeof(FusedCtl) + (size_t)4 * ((items + 31) / 32) + 15) & ~(size_t)15;
}

// SW step warps, EW emitter warps (multiples of 4: setmaxnreg acts on whole
// warpgroups); RS / RE: registers per thread after the redistribution (0 =
// keep the launch allocation).
template <int NF, int ZF, bool F16, int SW, int EW, int RS, int RE>
__global__ void __launch_bounds__(32 * (SW + EW), 1) fused_kernel(const Params P, int items_max) {
  constexpr int N = NF, Z = ZF;
  constexpr int D = TABX_OWN_DIM + TABX_OTHER_DIM * (NF - 1) + TABX_ZONE_DIM * ZF;
  constexpr int G = TABX_OWN_DIM * NF + TABX_ZONE_DIM * ZF;
  constexpr int R = emit_rows(N, D, TABX_EMIT_BUDGET);
  constexpr int SF = emit_stage_floats(N, D, G, R);
  constexpr size_t env_bytes = (sizeof(EnvSmem<1>) + 15) & ~(size_t)15;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (P.sync->err_index != NO_ERROR) return;  // an action violated the mask: no mutation
  FusedCtl* ctl = reinterpret_cast<FusedCtl*>(smem_raw);
  uint32_t* done = reinterpret_cast<uint32_t*>(smem_raw + sizeof(FusedCtl));
  const size_t ctl_bytes = fused_ctl_bytes(items_max);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = blockIdx.x, grid = gridDim.x;
  const int items = (int)((P.B - c + grid - 1) / grid);  // envs of this CTA
  TABX_ASSERT(items <= items_max);
  for (int q = threadIdx.x; q < (items + 31) / 32; q += blockDim.x) done[q] = 0u;
  if (threadIdx.x == 0) {
    ctl->next_step = 0;
    ctl->next_emit = 0;
  }
  const uint32_t step_no = P.sync->step;
  const bool refresh = P.sync->refresh[step_no % 3] != 0;
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) P.sync->refresh[(step_no + 2) % 3] = 0;

  if (warp < SW) {
    // ---------------------------------------------------------- step warps
    reg_alloc<RS>();
    EnvSmem<1>& S = *reinterpret_cast<EnvSmem<1>*>(smem_raw + ctl_bytes + warp * env_bytes);
    {  // pair table (N <= 32), kernel lifetime
      int p = 0;
      for (int a = 0; a < N; ++a) {
        const int cnt = N - 1 - a;
        for (int q = lane; q < cnt; q += 32) S.ptab[p + q] = (uint16_t)((a << 8) | (a + 1 + q));
        p += cnt;
      }
      __syncwarp();
    }
    for (;;) {
      int k = 0;
      if (lane == 0) k = (int)atomicAdd(&ctl->next_step, 1u);
      k = __shfl_sync(0xffffffffu, k, 0);
      if (k >= items) break;
      const int64_t b = c + (int64_t)k * grid;
      TABX_POISON(&S, offsetof(EnvSmem<1>, ptab), lane, 32);
      __syncwarp();
      run_lane<1, MODE_STEP_K0, NF, ZF>(P, b, lane, S, nullptr, refresh, step_no);
      // release: every lane's state stores before the item's done bit
      __threadfence_block();
      __syncwarp();
      if (lane == 0) atomicOr(&done[k >> 5], 1u << (k & 31));
    }
  } else {
    // ------------------------------------------------------- emitter warps
    reg_dealloc<RE>();
    const int w = warp - SW;
    const EmitScratch<1> X = emit_scratch<1>(
        smem_raw + ctl_bytes + SW * env_bytes + (size_t)w * emit_warp_bytes<1>(N, Z, R, SF), N, Z,
        R);
    const DevState& st = P.st;
    int buf = 0;
    for (;;) {
      int k = 0;
      if (lane == 0) k = (int)atomicAdd(&ctl->next_emit, 1u);
      k = __shfl_sync(0xffffffffu, k, 0);
      if (k >= items) break;
      const int64_t b = c + (int64_t)k * grid;
      if (lane == 0) {
        const volatile uint32_t* dw = done + (k >> 5);
        const uint32_t bit = 1u << (k & 31);
        while (!(*dw & bit)) __nanosleep(64);
        __threadfence_block();  // acquire: the step warp's state stores
      }
      __syncwarp();
      const int32_t kc = st.cfg[b];
      const tabx_config* C = P.cfgs + kc;
      const DerivedCfg* DC = P.dcfgs + kc;
      const bool pending = (st.flags[b] & F_PEND) != 0;
      float* ob = pending ? P.out.final_observations : P.out.observations;
      float* gb = pending ? P.out.final_global_state : P.out.global_state;
      __nv_bfloat16* o16 = (F16 && !pending) ? (__nv_bfloat16*)P.out.observations_bf16 : nullptr;
      if (!ob && !gb && !o16) continue;
      load_view<1>(X, st, b, N, Z, C, DC, lane);
      emit_lane<1, F16>(X, ob, gb, b, N, Z, D, G, R, SF, C, DC, lane, buf, false, o16,
                        (int)P.out.observations_bf16_ld);
    }
    if (lane == 0) bulk_wait_all();
  }
}

// Sequential variant: every warp steps an environment and then streams its
// observation rows itself (no hand-off), EPB warps per CTA at the step
// kernel's 128 registers.  The emitter's view aliases the head of the
// warp's EnvSmem (dead once the step is written back; the pair table at its
// tail is kept); the stage buffers are the warp's own, so the TMA stores of
// one environment drain while the warp steps the next.
template <int NF, int ZF, bool F16, int EPB>
__global__ void __launch_bounds__(32 * EPB, 4) fused_seq_kernel(const Params P) {
  constexpr int N = NF, Z = ZF;
  constexpr int D = TABX_OWN_DIM + TABX_OTHER_DIM * (NF - 1) + TABX_ZONE_DIM * ZF;
  constexpr int G = TABX_OWN_DIM * NF + TABX_ZONE_DIM * ZF;
  constexpr int R = emit_rows(N, D, TABX_EMIT_BUDGET);
  constexpr int SF = emit_stage_floats(N, D, G, R);
  constexpr size_t env_bytes = (sizeof(EnvSmem<1>) + 15) & ~(size_t)15;
  static_assert(emit_view_bytes<1>(N) + emit_aux_bytes<1>(N, Z, R) <= offsetof(EnvSmem<1>, ptab),
                "emitter view must fit below the pair table");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (P.sync->err_index != NO_ERROR) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t step_no = P.sync->step;
  const bool refresh = P.sync->refresh[step_no % 3] != 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) P.sync->refresh[(step_no + 2) % 3] = 0;
  unsigned char* eb = smem_raw + warp * env_bytes;
  EnvSmem<1>& S = *reinterpret_cast<EnvSmem<1>*>(eb);
  EmitScratch<1> X = emit_scratch<1>(eb, N, Z, R);
  X.stage = reinterpret_cast<float*>(smem_raw + EPB * env_bytes +
                                     (size_t)warp * TABX_EMIT_NBUF * SF * sizeof(float));
  {
    int p = 0;
    for (int a = 0; a < N; ++a) {
      const int cnt = N - 1 - a;
      for (int q = lane; q < cnt; q += 32) S.ptab[p + q] = (uint16_t)((a << 8) | (a + 1 + q));
      p += cnt;
    }
    __syncwarp();
  }
  const DevState& st = P.st;
  int buf = 0;
  for (int64_t b = (int64_t)blockIdx.x * EPB + warp; b < P.B; b += (int64_t)gridDim.x * EPB) {
    TABX_POISON(&S, offsetof(EnvSmem<1>, ptab), lane, 32);
    __syncwarp();
    run_lane<1, MODE_STEP_K0, NF, ZF>(P, b, lane, S, nullptr, refresh, step_no);
    __syncwarp();  // the warp's own state stores, read back below (L1/L2)
    const int32_t kc = st.cfg[b];
    const tabx_config* C = P.cfgs + kc;
    const DerivedCfg* DC = P.dcfgs + kc;
    const bool pending = (st.flags[b] & F_PEND) != 0;
    float* ob = pending ? P.out.final_observations : P.out.observations;
    float* gb = pending ? P.out.final_global_state : P.out.global_state;
    __nv_bfloat16* o16 = (F16 && !pending) ? (__nv_bfloat16*)P.out.observations_bf16 : nullptr;
    if (!ob && !gb && !o16) continue;
    load_view<1>(X, st, b, N, Z, C, DC, lane);
    emit_lane<1, F16>(X, ob, gb, b, N, Z, D, G, R, SF, C, DC, lane, buf, false, o16,
                      (int)P.out.observations_bf16_ld);
  }
  if (lane == 0) bulk_wait_all();
}

template <int NF, int ZF, bool F16, int EPB>
cudaError_t launch_fused_seq(const Params& P, int sm_count, cudaStream_t stream) {
  constexpr int D = TABX_OWN_DIM + TABX_OTHER_DIM * (NF - 1) + TABX_ZONE_DIM * ZF;
  constexpr int G = TABX_OWN_DIM * NF + TABX_ZONE_DIM * ZF;
  constexpr int R = emit_rows(NF, D, TABX_EMIT_BUDGET);
  constexpr int SF = emit_stage_floats(NF, D, G, R);
  constexpr size_t env_bytes = (sizeof(EnvSmem<1>) + 15) & ~(size_t)15;
  const size_t smem = EPB * (env_bytes + (size_t)TABX_EMIT_NBUF * SF * sizeof(float));
  int per_sm = 0;
  auto kern = fused_seq_kernel<NF, ZF, F16, EPB>;
  cudaError_t e = launch_geometry((const void*)kern, 32 * EPB, smem, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorNotSupported;
  const int64_t need = (P.B + EPB - 1) / EPB, cap = (int64_t)sm_count * per_sm;
  int grid = (int)(need < cap ? need : cap);
  if (grid < 1) grid = 1;
  kern<<<grid, 32 * EPB, smem, stream>>>(P);
  return cudaGetLastError();
}

template <int NF, int ZF, bool F16, int SW, int EW, int RS, int RE>
cudaError_t launch_fused_v(const Params& P, int sm_count, cudaStream_t stream) {
  constexpr int D = TABX_OWN_DIM + TABX_OTHER_DIM * (NF - 1) + TABX_ZONE_DIM * ZF;
  constexpr int G = TABX_OWN_DIM * NF + TABX_ZONE_DIM * ZF;
  constexpr int R = emit_rows(NF, D, TABX_EMIT_BUDGET);
  constexpr int SF = emit_stage_floats(NF, D, G, R);
  constexpr size_t env_bytes = (sizeof(EnvSmem<1>) + 15) & ~(size_t)15;
  const int grid = (int)(P.B < sm_count ? P.B : sm_count);
  if (grid < 1) return cudaSuccess;
  const int64_t items = (P.B + grid - 1) / grid;
  if (items > (1 << 16)) return cudaErrorNotSupported;  // done-bitmap bound (8 KB)
  const size_t smem = fused_ctl_bytes((int)items) + SW * env_bytes +
                      (size_t)EW * emit_warp_bytes<1>(NF, ZF, R, SF);
  int per_sm = 0;
  auto kern = fused_kernel<NF, ZF, F16, SW, EW, RS, RE>;
  cudaError_t e = launch_geometry((const void*)kern, 32 * (SW + EW), smem, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorNotSupported;
  kern<<<grid, 32 * (SW + EW), smem, stream>>>(P, (int)items);
  return cudaGetLastError();
}

// Variant (TABX_FUSED_VARIANT, read at batch creation): step / emitter warp
// split and register redistribution.
template <int NF, int ZF, bool F16>
cudaError_t launch_fused_shape(const Params& P, int variant, int sm_count, cudaStream_t stream) {
  switch (variant) {
    case 1: return launch_fused_v<NF, ZF, F16, 8, 12, 128, 72>(P, sm_count, stream);
    case 2: return launch_fused_v<NF, ZF, F16, 4, 16, 128, 88>(P, sm_count, stream);
    case 3: return launch_fused_seq<NF, ZF, F16, 4>(P, sm_count, stream);
    default: return launch_fused_v<NF, ZF, F16, 8, 8, 152, 104>(P, sm_count, stream);
  }
}

// The fused path covers the W = 1 shapes with specialised kernels (C3, C2);
// cudaErrorNotSupported tells the caller to run K1 + K2 instead.
cudaError_t launch_fused_w1(const Params& P, int variant, int sm_count, cudaStream_t stream) {
  if (P.generic_shapes || P.mode != MODE_STEP_K0) return cudaErrorNotSupported;
  const bool f16 = P.out.observations_bf16 != nullptr;
  if (P.N == 20 && P.Z == 6)
    return f16 ? launch_fused_shape<20, 6, true>(P, variant, sm_count, stream)
               : launch_fused_shape<20, 6, false>(P, variant, sm_count, stream);
  if (P.N == 20 && P.Z == 0)
    return f16 ? launch_fused_shape<20, 0, true>(P, variant, sm_count, stream)
               : launch_fused_shape<20, 0, false>(P, variant, sm_count, stream);
  return cudaErrorNotSupported;
}

}  // namespace tabx

// ------------------------------------------------- single-launch small step --
// Small batches (below the controller-pass threshold, W = 1): the step is
// launch-latency bound (C1, 256 envs: K1 + K2 + K3 back to back, ~30 us for
// three dependent launches), so the whole step runs as ONE launch: each warp
// steps its environment with the in-kernel controller (run_lane MODE_STEP),
// streams its observation rows (terminal rows to final_* when the lane's
// auto-reset is pending), and then performs that reset itself (run_lane
// MODE_RESET: respawn, fresh caches, fresh observation).  The last CTA to
// finish advances the device step counter, as K3 does.  The batch-coupled
// cache refresh stays deferred to the next step's start (same ring), so the
// per-environment code and the bits are those of K1 + K2 + K3.
namespace tabx {

template <int NF, int ZF, int EPB>
__global__ void __launch_bounds__(32 * EPB, TABX_MIN_BLOCKS_W1(EPB)) step_small_kernel(const Params P) {
  constexpr size_t env_bytes = (sizeof(EnvSmem<1>) * EPB + 15) & ~(size_t)15;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (P.sync->err_index != NO_ERROR) return;  // an action violated the mask: no mutation
  const int N = NF ? NF : P.N, Z = ZF ? ZF : P.Z;
  EnvSmem<1>* envs = reinterpret_cast<EnvSmem<1>*>(smem_raw);
  const size_t view_bytes = reset_view_bytes<1>(P);
  const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* scratch = smem_raw + env_bytes + g * view_bytes;
  const uint32_t step_no = P.sync->step;
  const bool refresh = P.sync->refresh[step_no % 3] != 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) P.sync->refresh[(step_no + 2) % 3] = 0;
  {  // pair table (N <= 32)
    int p = 0;
    for (int a = 0; a < N; ++a) {
      const int cnt = N - 1 - a;
      for (int q = lane; q < cnt; q += 32) envs[g].ptab[p + q] = (uint16_t)((a << 8) | (a + 1 + q));
      p += cnt;
    }
    __syncwarp();
  }
  const int R = emit_rows(N, P.D, TABX_EMIT_BUDGET);
  const int SF = emit_stage_floats(N, P.D, P.G, R);
  const DevState& st = P.st;
  for (int64_t b = (int64_t)blockIdx.x * EPB + g; b < P.B; b += (int64_t)gridDim.x * EPB) {
    TABX_POISON(&envs[g], offsetof(EnvSmem<1>, ptab), lane, 32);
    __syncwarp();
    run_lane<1, MODE_STEP, NF, ZF>(P, b, lane, envs[g], nullptr, refresh, step_no);
    __syncwarp();  // the warp's own state stores, read back below
    const int32_t kc = st.cfg[b];
    const tabx_config* C = P.cfgs + kc;
    const DerivedCfg* DC = P.dcfgs + kc;
    const bool pending = (st.flags[b] & F_PEND) != 0;
    float* ob = pending ? P.out.final_observations : P.out.observations;
    float* gb = pending ? P.out.final_global_state : P.out.global_state;
    __nv_bfloat16* o16 = pending ? nullptr : (__nv_bfloat16*)P.out.observations_bf16;
    if (ob || gb || o16) {
      const EmitScratch<1> X = emit_scratch<1>(scratch, N, Z, R);
      int buf = 0;
      load_view<1>(X, st, b, N, Z, C, DC, lane);
      if (o16)
        emit_lane<1, true>(X, ob, gb, b, N, Z, P.D, P.G, R, SF, C, DC, lane, buf, true, o16,
                           (int)P.out.observations_bf16_ld);
      else
        emit_lane<1>(X, ob, gb, b, N, Z, P.D, P.G, R, SF, C, DC, lane, buf, true);
    }
    if (pending) {
      // K3 for this lane (its stage buffers were drained above)
      TABX_POISON(&envs[g], offsetof(EnvSmem<1>, ptab), lane, 32);
      __syncwarp();
      run_lane<1, MODE_RESET, NF, ZF>(P, b, lane, envs[g], scratch, refresh, step_no);
    }
  }
  if (lane == 0) bulk_wait_all();
  // the step ends here: the last CTA advances the device step counter
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t ticket = atomicAdd(&P.sync->blocks_done, 1u);
    if (ticket == gridDim.x - 1) {
      P.sync->blocks_done = 0;
      P.sync->any_pend = 0;
      P.sync->step = step_no + 1;
      __threadfence();
    }
  }
}

template <int NF, int ZF>
cudaError_t launch_small_shape(const Params& P, int sm_count, cudaStream_t stream) {
  constexpr int EPB = 4;
  const size_t env_bytes = (sizeof(EnvSmem<1>) * EPB + 15) & ~(size_t)15;
  const size_t smem = env_bytes + reset_view_bytes<1>(P) * EPB;
  int per_sm = 0;
  auto kern = step_small_kernel<NF, ZF, EPB>;
  cudaError_t e = launch_geometry((const void*)kern, 32 * EPB, smem, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorNotSupported;
  const int64_t need = (P.B + EPB - 1) / EPB, cap = (int64_t)sm_count * per_sm;
  int grid = (int)(need < cap ? need : cap);
  if (grid < 1) grid = 1;
  kern<<<grid, 32 * EPB, smem, stream>>>(P);
  return cudaGetLastError();
}

// The single-launch step for W = 1 batches stepped with the in-kernel
// controller (MODE_STEP); cudaErrorNotSupported otherwise.
cudaError_t launch_small_w1(const Params& P, int sm_count, cudaStream_t stream) {
  if (P.mode != MODE_STEP) return cudaErrorNotSupported;
  if (!P.generic_shapes && P.N == 6 && P.Z == 0) return launch_small_shape<6, 0>(P, sm_count, stream);
  return launch_small_shape<0, 0>(P, sm_count, stream);
}

}  // namespace tabx
