// Observation / global-state writer: a streaming kernel of its own.
//
// The step kernel leaves the post-step state and the stage-8 visibility /
// attackable rows in HBM; this kernel turns them into the float32
// observation tensor [B, N, obs_dim] and global state [B, global_dim]
// (perception.py:99-201).  One warp per environment, low register count,
// many warps per SM: each warp stages the env's per-unit view (positions,
// 15 own features, N-bit rows) in shared memory and then streams the env's
// observation block with coalesced 16-byte evict-first stores.  Blocks of
// hidden (observer, other) pairs -- most of the tensor -- cost one visibility
// test per float4.
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

// Observation element (r, c) of the env (perception.py:159-192).
template <int W>
__device__ __forceinline__ float obs_elem(const EmitEnv<W>& E, const tabx_config* __restrict__ C,
                                          const DerivedCfg* __restrict__ DC, int zoff, int r,
                                          int c) {
  if (c < TABX_OWN_DIM) return E.own[r][c];
  if (c < zoff) {
    const int c2 = c - TABX_OWN_DIM;
    const int k = c2 / TABX_OTHER_DIM, f = c2 - k * TABX_OTHER_DIM;
    const int j = k + (k >= r ? 1 : 0);
    if (!row_bit(&E.vis[r * W], j)) return 0.0f;
    switch (f) {
      case 2: return f32_quot(E.px[j] - E.px[r], C->field_w, DC->rw);
      case 3: return f32_quot(E.py[j] - E.py[r], C->field_h, DC->rh);
      case 15: return (E.flags[j] & 2u) ? 1.0f : 0.0f;
      case 16: return row_bit(&E.atk[r * W], j) ? 1.0f : 0.0f;
      default: return E.own[j][f];
    }
  }
  const int c3 = c - zoff;
  const int z = c3 >> 3, f = c3 & 7;
  const int ty = C->zone_type[z];
  if (ty == TABX_ZONE_NONE) return 0.0f;
  switch (f) {
    case 0: case 1: case 2: return ty == f + 1 ? 1.0f : 0.0f;
    case 3: return f32_quot(C->zone_cx[z] - E.px[r], C->field_w, DC->rw);
    case 4: return f32_quot(C->zone_cy[z] - E.py[r], C->field_h, DC->rh);
    case 5: return __double2float_rn(C->zone_ax[z]);
    case 6: return __double2float_rn(C->zone_ay[z]);
    default: return __double2float_rn(C->zone_effect[z]);
  }
}

// Stream env b's observation rows and global-state row (one warp).
template <int W>
__device__ void emit_lane(const EmitEnv<W>& E, float* __restrict__ obs, float* __restrict__ glob,
                          int64_t b, int N, int Z, int D, int G,
                          const tabx_config* __restrict__ C, const DerivedCfg* __restrict__ DC,
                          int lane) {
  const int M = N - 1;
  const int zoff = TABX_OWN_DIM + TABX_OTHER_DIM * M;
  if (obs) {
    const int64_t E_ = (int64_t)N * D;
    const int64_t start = b * E_;
    if ((start & 3) == 0 && (E_ & 3) == 0) {
      // row groups of g rows span a multiple of 4 floats
      const int g = (D & 3) == 0 ? 1 : ((D & 1) == 0 ? 2 : 4);
      const int span4 = (g * D) >> 2;
      for (int rg = 0; rg < N; rg += g) {
        float4* __restrict__ dst = reinterpret_cast<float4*>(obs + start + (int64_t)rg * D);
        for (int q = lane; q < span4; q += 32) {
          const int e0 = q << 2;
          const int rr = (e0 >= D) + (e0 >= 2 * D) + (e0 >= 3 * D);
          int r = rg + rr;
          int c = e0 - rr * D;
          float v[4];
          // fast path: the 4 floats lie in hidden pair blocks of one row
          bool done = false;
          if (c >= TABX_OWN_DIM && c + 3 < zoff) {
            const int k0 = (c - TABX_OWN_DIM) / TABX_OTHER_DIM;
            const int k1 = (c + 3 - TABX_OWN_DIM) / TABX_OTHER_DIM;
            const int j0 = k0 + (k0 >= r ? 1 : 0), j1 = k1 + (k1 >= r ? 1 : 0);
            if (!row_bit(&E.vis[r * W], j0) && !row_bit(&E.vis[r * W], j1)) {
              v[0] = v[1] = v[2] = v[3] = 0.0f;
              done = true;
            }
          }
          if (!done) {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              v[t] = (E.flags[r] & 1u) ? obs_elem<W>(E, C, DC, zoff, r, c) : 0.0f;
              if (++c == D) {
                c = 0;
                ++r;
              }
            }
          }
          __stcs(dst + q, make_float4(v[0], v[1], v[2], v[3]));
        }
      }
    } else {
      for (int64_t e = lane; e < E_; e += 32) {
        const int r = (int)(e / D), c = (int)(e - (int64_t)r * D);
        obs[start + e] = (E.flags[r] & 1u) ? obs_elem<W>(E, C, DC, zoff, r, c) : 0.0f;
      }
    }
  }
  if (glob) {
    float* row = glob + b * (int64_t)G;
    const int own_cols = N * TABX_OWN_DIM;
    for (int c = lane; c < G; c += 32) {
      float v;
      if (c < own_cols) {
        const int u = c / TABX_OWN_DIM;
        v = E.own[u][c - u * TABX_OWN_DIM];
      } else {
        const int o = c - own_cols;
        const int z = o >> 3, f = o & 7;
        const int ty = C->zone_type[z];
        if (ty == TABX_ZONE_NONE) {
          v = 0.0f;
        } else {
          switch (f) {
            case 0: case 1: case 2: v = ty == f + 1 ? 1.0f : 0.0f; break;
            case 3: v = f32_quot(C->zone_cx[z], C->field_w, DC->rw); break;
            case 4: v = f32_quot(C->zone_cy[z], C->field_h, DC->rh); break;
            case 5: v = __double2float_rn(C->zone_ax[z]); break;
            case 6: v = __double2float_rn(C->zone_ay[z]); break;
            default: v = __double2float_rn(C->zone_effect[z]); break;
          }
        }
      }
      __stcs(row + c, v);
    }
  }
}

// K2: observations of every lane after a step (final_* buffers for lanes
// whose auto-reset is pending: their terminal observation) or after
// init_output.  EPW environments per CTA, one warp each.
template <int W, int EPW>
__global__ void __launch_bounds__(32 * EPW) emit_kernel(const Params P) {
  __shared__ EmitEnv<W> envs[EPW];
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
    load_view<W>(envs[w], st, b, P.N, C, DC, lane);
    emit_lane<W>(envs[w], ob, gb, b, P.N, P.Z, P.D, P.G, C, DC, lane);
    __syncwarp();
  }
}

template <int W, int EPW>
cudaError_t launch_emit_t(const Params& P, int sm_count, cudaStream_t stream) {
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaError_t e =
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, emit_kernel<W, EPW>, 32 * EPW, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
  }
  int64_t need = (P.B + EPW - 1) / EPW;
  int64_t cap = (int64_t)sm_count * per_sm;
  int grid = (int)(need < cap ? need : cap);
  if (grid < 1) grid = 1;
  emit_kernel<W, EPW><<<grid, 32 * EPW, 0, stream>>>(P);
  return cudaGetLastError();
}

}  // namespace tabx
