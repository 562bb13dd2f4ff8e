// Observation / global-state writer: a streaming kernel of its own.
//
// The step kernel leaves the post-step state and the stage-8 visibility /
// attackable rows in HBM; this kernel turns them into the float32
// observation tensor [B, N, obs_dim] and global state [B, global_dim]
// (perception.py:99-201).  One warp per environment, ~96 registers, many
// warps per SM: each warp stages the env's per-unit view (positions, 15 own
// features, N-bit rows) in shared memory, assembles the observation rows a
// few at a time in shared memory and streams them out with double-buffered
// TMA bulk stores.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "tabx_device.cuh"
#include "tabx_math.cuh"

namespace tabx {

// Per-warp view of one environment (units 0..32W-1).
template <int W>
struct EmitEnv {
  static constexpr int NT = 32 * W;
  double px[NT], py[NT];
  float own[NT][16] __attribute__((aligned(16)));
  uint32_t vis[NT * W], atk[NT * W];
  uint32_t flags[NT];  // bit0 active, bit1 enemy
};

__device__ __forceinline__ bool row_bit(const uint32_t* row, int j) {
  return (row[j >> 5] >> (j & 31)) & 1u;
}

// Own-feature block of unit u from its HBM state (perception.py:108-132).
__device__ __forceinline__ void own_from_state(float* o, const DevState& st, int64_t gu,
                                               const tabx_config* __restrict__ C,
                                               const DerivedCfg* __restrict__ DC, int u) {
  o[15] = 0.0f;
  if (!C->active[u]) {
#pragma unroll
    for (int f = 0; f < TABX_OWN_DIM; ++f) o[f] = 0.0f;
    return;
  }
  const double2 p = st.pos[gu];
  const double2 cs = st.hcs[gu];
  const double hp = st.health[gu], cd = st.cooldown[gu];
  const double mh = C->max_health[u], ucd = C->cooldown[u];
  o[0] = f32_quot(hp, mh, DC->rmh[u]);
  o[1] = f32_quot(mh, 1000.0, 0.001);
  o[2] = f32_quot(p.x, C->field_w, DC->rw);
  o[3] = f32_quot(p.y, C->field_h, DC->rh);
  o[4] = __double2float_rn(cs.x);
  o[5] = __double2float_rn(cs.y);
  o[6] = __double2float_rn(C->attack_range[u]);
  o[7] = __double2float_rn(C->damage[u]);
  o[8] = __double2float_rn(cd);
  o[9] = ucd > 0.0 ? f32_quot(cd, ucd, DC->rucd[u]) : 0.0f;
  o[10] = __double2float_rn(C->radius[u]);
  o[11] = __double2float_rn(C->mass[u]);
  o[12] = __double2float_rn(C->sight_angle[u]);
  o[13] = (st.ubits[gu] & U_ALIVE) ? 1.0f : 0.0f;
  o[14] = __double2float_rn(C->speed[u]);
}

// Load lane b's view into E (all 32 lanes of the warp).
template <int W>
__device__ __forceinline__ void load_view(EmitEnv<W>& E, const DevState& st, int64_t b, int N,
                                          const tabx_config* __restrict__ C,
                                          const DerivedCfg* __restrict__ DC, int lane) {
  for (int u = lane; u < N; u += 32) {
    const int64_t gu = b * N + u;
    const double2 p = st.pos[gu];
    E.px[u] = p.x;
    E.py[u] = p.y;
    own_from_state(E.own[u], st, gu, C, DC, u);
    E.flags[u] = (C->active[u] ? 1u : 0u) | (C->team[u] ? 2u : 0u);
#pragma unroll
    for (int k = 0; k < W; ++k) {
      E.vis[u * W + k] = st.vis[gu * W + k];
      E.atk[u * W + k] = st.atk[gu * W + k];
    }
  }
  __syncwarp();
}

// ---- TMA bulk stores (cp.async.bulk.global.shared::cta)
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bulk_s2g(void* g, const void* s, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(g),
               "r"(smem_addr(s)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
template <int K>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(K) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// dst[gs, gs+count) <- stage[pad, pad+count), pad = gs & 3: the 16-byte
// aligned interior by one TMA bulk store (lane 0), the <= 3-float head and
// tail by plain stores.
__device__ __forceinline__ void flush_stage(float* __restrict__ dst, int64_t gs, int count,
                                            const float* stage, int lane) {
  const int pad = (int)(gs & 3);
  const int64_t a0 = (gs + 3) & ~(int64_t)3;
  const int64_t a1 = (gs + count) & ~(int64_t)3;
  if (a1 > a0) {
    if (lane == 0) {
      bulk_s2g(dst + a0, stage + pad + (a0 - gs), (uint32_t)((a1 - a0) * 4));
      bulk_commit();
    }
    for (int e = lane; e < (int)(a0 - gs); e += 32) dst[gs + e] = stage[pad + e];
    for (int e = (int)(a1 - gs) + lane; e < count; e += 32) dst[gs + e] = stage[pad + e];
  } else {
    for (int e = lane; e < count; e += 32) dst[gs + e] = stage[pad + e];
  }
}

// Position of the n-th (0-based) set bit of w, by popc halving.
__device__ __forceinline__ int nth_bit(uint32_t w, int n) {
  int pos = 0;
  int c = __popc(w & 0xFFFFu);
  if (n >= c) { n -= c; w >>= 16; pos += 16; }
  c = __popc(w & 0xFFu);
  if (n >= c) { n -= c; w >>= 8; pos += 8; }
  c = __popc(w & 0xFu);
  if (n >= c) { n -= c; w >>= 4; pos += 4; }
  c = __popc(w & 0x3u);
  if (n >= c) { n -= c; w >>= 2; pos += 2; }
  if (n >= (int)(w & 1u)) pos += 1;
  return pos;
}

// Env b's observation rows and global-state row, one warp.  Rows are built
// in shared memory R at a time (zero fill with 16-byte stores, then the own
// block, the visible (observer, other) pair blocks enumerated from the N-bit
// visibility rows, and the zone blocks) and leave through double-buffered
// TMA bulk stores; hidden pairs -- most of the tensor -- cost only the fill.
template <int W>
__device__ void emit_lane(const EmitEnv<W>& E, float* __restrict__ obs, float* __restrict__ glob,
                          int64_t b, int N, int Z, int D, int G, int R, int SF, float* stage,
                          const tabx_config* __restrict__ C, const DerivedCfg* __restrict__ DC,
                          int lane) {
  const double fw = C->field_w, fh = C->field_h, rw = DC->rw, rh = DC->rh;
  const int M = N - 1;
  const int zoff = TABX_OWN_DIM + TABX_OTHER_DIM * M;
  int buf = 0;
  if (obs) {
    for (int r0 = 0; r0 < N; r0 += R) {
      const int nr = min(R, N - r0);
      const int64_t gs = (b * N + r0) * (int64_t)D;
      float* st = stage + buf * SF;
      const int pad = (int)(gs & 3);
      float* row0 = st + pad;
      if (lane == 0) bulk_wait_read<1>();
      __syncwarp();
      {
        const int n4 = (pad + nr * D + 3) >> 2;
        float4* z4 = reinterpret_cast<float4*>(st);
        const float4 zero = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        int q = lane;
        for (; q + 96 < n4; q += 128) {
          z4[q] = zero;
          z4[q + 32] = zero;
          z4[q + 64] = zero;
          z4[q + 96] = zero;
        }
        for (; q < n4; q += 32) z4[q] = zero;
      }
      __syncwarp();
      for (int e = lane; e < nr * TABX_OWN_DIM; e += 32) {
        const int rr = e / TABX_OWN_DIM, f = e - rr * TABX_OWN_DIM;
        row0[rr * D + f] = E.own[r0 + rr][f];
      }
      // visible pairs of the chunk's rows (vis excludes inactive rows/columns)
      int total = 0;
      for (int rr = 0; rr < nr; ++rr) {
        const int r = r0 + rr;
#pragma unroll
        for (int k = 0; k < W; ++k)
          total += __popc(E.vis[r * W + k] & ~(k == (r >> 5) ? 1u << (r & 31) : 0u));
      }
      for (int s = lane; s < total; s += 32) {
        int rr = 0, n = s, j = -1;
        for (; rr < nr; ++rr) {
          const int r = r0 + rr;
          for (int k = 0; k < W && j < 0; ++k) {
            const uint32_t w = E.vis[r * W + k] & ~(k == (r >> 5) ? 1u << (r & 31) : 0u);
            const int c = __popc(w);
            if (n < c) {
              j = (k << 5) + nth_bit(w, n);
            } else {
              n -= c;
            }
          }
          if (j >= 0) break;
        }
        const int r = r0 + rr;
        const int kk = j - (j > r ? 1 : 0);
        float* blk = row0 + rr * D + TABX_OWN_DIM + TABX_OTHER_DIM * kk;
        const float4* oj = reinterpret_cast<const float4*>(E.own[j]);
        const float4 o0 = oj[0], o1 = oj[1], o2 = oj[2], o3 = oj[3];
        blk[0] = o0.x;
        blk[1] = o0.y;
        blk[2] = f32_quot(E.px[j] - E.px[r], fw, rw);
        blk[3] = f32_quot(E.py[j] - E.py[r], fh, rh);
        blk[4] = o1.x;
        blk[5] = o1.y;
        blk[6] = o1.z;
        blk[7] = o1.w;
        blk[8] = o2.x;
        blk[9] = o2.y;
        blk[10] = o2.z;
        blk[11] = o2.w;
        blk[12] = o3.x;
        blk[13] = o3.y;
        blk[14] = o3.z;
        blk[15] = (E.flags[j] & 2u) ? 1.0f : 0.0f;
        blk[16] = row_bit(&E.atk[r * W], j) ? 1.0f : 0.0f;
      }
      // zone blocks: lane z of each active row (unused slots stay zero)
      if (lane < Z) {
        const int z = lane;
        const int ty = C->zone_type[z];
        for (int rr = 0; rr < nr && ty != TABX_ZONE_NONE; ++rr) {
          const int r = r0 + rr;
          if (!(E.flags[r] & 1u)) continue;
          float* zb = row0 + rr * D + zoff + TABX_ZONE_DIM * z;
          zb[ty - 1] = 1.0f;
          zb[3] = f32_quot(C->zone_cx[z] - E.px[r], fw, rw);
          zb[4] = f32_quot(C->zone_cy[z] - E.py[r], fh, rh);
          zb[5] = __double2float_rn(C->zone_ax[z]);
          zb[6] = __double2float_rn(C->zone_ay[z]);
          zb[7] = __double2float_rn(C->zone_effect[z]);
        }
      }
      fence_proxy_async();
      __syncwarp();
      flush_stage(obs, gs, nr * D, st, lane);
      buf ^= 1;
    }
  }
  if (glob) {
    const int64_t gs = b * (int64_t)G;
    float* st = stage + buf * SF;
    float* row = st + (int)(gs & 3);
    if (lane == 0) bulk_wait_read<1>();
    __syncwarp();
    for (int e = lane; e < N * TABX_OWN_DIM; e += 32) {
      const int u = e / TABX_OWN_DIM;
      row[e] = E.own[u][e - u * TABX_OWN_DIM];
    }
    for (int q = lane; q < Z * TABX_ZONE_DIM; q += 32) {
      const int z = q >> 3, f = q & 7;
      const int ty = C->zone_type[z];
      float v;
      if (ty == TABX_ZONE_NONE) {
        v = 0.0f;
      } else {
        switch (f) {
          case 0: case 1: case 2: v = ty == f + 1 ? 1.0f : 0.0f; break;
          case 3: v = f32_quot(C->zone_cx[z], fw, rw); break;
          case 4: v = f32_quot(C->zone_cy[z], fh, rh); break;
          case 5: v = __double2float_rn(C->zone_ax[z]); break;
          case 6: v = __double2float_rn(C->zone_ay[z]); break;
          default: v = __double2float_rn(C->zone_effect[z]); break;
        }
      }
      row[N * TABX_OWN_DIM + q] = v;
    }
    fence_proxy_async();
    __syncwarp();
    flush_stage(glob, gs, G, st, lane);
  }
  if (lane == 0) bulk_wait_read<0>();
  __syncwarp();
}

// Stage geometry: R rows per chunk within `budget` bytes per buffer.
__host__ __device__ __forceinline__ int emit_rows(int N, int D, int budget) {
  int R = budget / (4 * D);
  if (R < 1) R = 1;
  if (R > N) R = N;
  return R;
}
__host__ __device__ __forceinline__ int emit_stage_floats(int N, int D, int G, int R) {
  const int need = (R * D > G ? R * D : G) + 8;
  return (need + 3) & ~3;
}

// K2: observations of every lane after a step (final_* buffers for lanes
// whose auto-reset is pending: their terminal observation) or after
// init_output.  EPW environments per CTA, one warp each; dynamic shared
// memory = EPW x (view + 2 stage buffers of SF floats).
#ifndef TABX_EMIT_BUDGET
#define TABX_EMIT_BUDGET 3200  // stage bytes per buffer per warp (W = 1)
#endif
#ifndef TABX_EMIT_MIN_BLOCKS
#define TABX_EMIT_MIN_BLOCKS 3
#endif
template <int W, int EPW>
__global__ void __launch_bounds__(32 * EPW, TABX_EMIT_MIN_BLOCKS)
    emit_kernel(const Params P, int R, int SF) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  EmitEnv<W>* views = reinterpret_cast<EmitEnv<W>*>(smem_raw);
  float* stages = reinterpret_cast<float*>(smem_raw + ((sizeof(EmitEnv<W>) * EPW + 15) & ~15));
  if (P.mode == MODE_STEP && P.sync->err_index != NO_ERROR) return;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const DevState& st = P.st;
  for (int64_t b = (int64_t)blockIdx.x * EPW + w; b < P.B; b += (int64_t)gridDim.x * EPW) {
    const int32_t k = st.cfg[b];
    const tabx_config* C = P.cfgs + k;
    const DerivedCfg* DC = P.dcfgs + k;
    const bool pending = (st.flags[b] & F_PEND) != 0;
    float* ob = pending ? P.out.final_observations : P.out.observations;
    float* gb = pending ? P.out.final_global_state : P.out.global_state;
    if (!ob && !gb) continue;
    load_view<W>(views[w], st, b, P.N, C, DC, lane);
    emit_lane<W>(views[w], ob, gb, b, P.N, P.Z, P.D, P.G, R, SF, stages + (size_t)w * 2 * SF, C,
                 DC, lane);
  }
  if (lane == 0) bulk_wait_all();
}

template <int W, int EPW>
cudaError_t launch_emit_t(const Params& P, int sm_count, cudaStream_t stream) {
  const int R = emit_rows(P.N, P.D, W == 1 ? TABX_EMIT_BUDGET : 8192);
  const int SF = emit_stage_floats(P.N, P.D, P.G, R);
  const size_t smem = ((sizeof(EmitEnv<W>) * EPW + 15) & ~(size_t)15) +
                      (size_t)EPW * 2 * SF * sizeof(float);
  static size_t cached_smem = 0;
  static int per_sm = 0;
  if (smem != cached_smem) {
    cudaError_t e = cudaFuncSetAttribute(emit_kernel<W, EPW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, emit_kernel<W, EPW>, 32 * EPW,
                                                      smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    cached_smem = smem;
  }
  int64_t need = (P.B + EPW - 1) / EPW;
  int64_t cap = (int64_t)sm_count * per_sm;
  int grid = (int)(need < cap ? need : cap);
  if (grid < 1) grid = 1;
  emit_kernel<W, EPW><<<grid, 32 * EPW, smem, stream>>>(P, R, SF);
  return cudaGetLastError();
}

}  // namespace tabx
