// Kernel instantiations for W = 1 (32 threads per environment).
#include "tabx_lane.cuh"

namespace tabx {
// ------------------------------------------------------------------ K0 ---
// Heuristic controller pass (heuristics.py:103-243) ahead of K1, for W == 1.
// Inside K1 the decision runs on the heuristic team's lanes only (10 of 32
// in C3) with the rest of the warp idle; here one lane is one heuristic unit
// and a warp packs the heuristic units of G environments, over a compact
// per-env view staged in shared memory.  Same inputs as K1's in-kernel call
// (the pre-step state, the cached vis/atk rows), so the same decision; the
// action goes to P.ctrl_act and the scripted-controller memory straight to
// the state, where K1 reads it.  On a step that refreshes the caches (a batch
// refill) the refresh kernel has rewritten the rows first; a step with a
// latched action error is skipped (no mutation).
struct CtrlView {
  double px[32], py[32], ch[32], sh[32], rad[32], mh[32];
  uint32_t uf[32], zin[32], vis[32], atk[32];
  uint32_t m_active[1], m_alive[1];
};

#ifndef TABX_K0_MINB
#define TABX_K0_MINB 6
#endif
__global__ void __launch_bounds__(128, TABX_K0_MINB) ctrl_kernel(const Params P, int G, int NH) {
  if (P.sync->err_index != NO_ERROR) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  CtrlView* V = reinterpret_cast<CtrlView*>(smem_raw) + wib * G;
  const int N = P.N, Z = P.Z;
  const DevState& st = P.st;
  const int wpb = blockDim.x >> 5;
  const int64_t stride = (int64_t)gridDim.x * wpb * G;
  const int g = lane / NH, k = lane - g * NH;
  for (int64_t b0 = ((int64_t)blockIdx.x * wpb + wib) * G; b0 < P.B; b0 += stride) {
    if (lane < G) {
      V[lane].m_active[0] = 0u;
      V[lane].m_alive[0] = 0u;
    }
    __syncwarp();
    // the view K1 publishes at the top of its step (publish / build_masks)
    for (int q = lane; q < G * N; q += 32) {
      const int gq = q / N, j = q - gq * N;
      const int64_t b = b0 + gq;
      if (b >= P.B) continue;
      const tabx_config* __restrict__ C = P.cfgs + st.cfg[b];
      const int64_t u = b * N + j;
      const double2 p = st.pos[u];
      const double2 cs = st.hcs[u];
      const double mh = C->max_health[j];
      const bool act = C->active[j] != 0;
      const bool alive = (st.ubits[u] & U_ALIVE) != 0;
      CtrlView& W1 = V[gq];
      W1.px[j] = p.x;
      W1.py[j] = p.y;
      W1.ch[j] = cs.x;
      W1.sh[j] = cs.y;
      W1.rad[j] = C->radius[j];
      W1.mh[j] = mh;
      W1.uf[j] = (act ? UF_ACTIVE : 0u) | (alive ? UF_ALIVE : 0u) |
                 (C->team[j] ? UF_ENEMY : 0u) | (C->kinematic[j] ? UF_KIN : 0u) |
                 (st.health[u] < mh ? UF_INJURED : 0u);
      W1.zin[j] = st.zbits[u];
      if (act) atomicOr(&W1.m_active[0], 1u << j);
      if (alive) atomicOr(&W1.m_alive[0], 1u << j);
    }
    __syncwarp();
    const int64_t b = b0 + g;
    if (g < G && b < P.B) {
      const int32_t cf = st.cfg[b];
      const tabx_config* __restrict__ C = P.cfgs + cf;
      const DerivedCfg* __restrict__ DC = P.dcfgs + cf;
      // an env with more heuristic units than the launch packs (a config
      // added after a graph capture) takes extra rounds on the same lanes
      const int nheur = (st.flags[b] & F_DONE) ? 0 : DC->n_heur;
      for (int kk = k; kk < nheur; kk += NH) {
        const int i = DC->hlist[kk];
        const int64_t u = b * N + i;
        const uint8_t ub = st.ubits[u];
        if (ub & U_ALIVE) {  // free: alive, active (hlist), lane running
          CtrlView& W1 = V[g];
          const int team = C->team[i] ? 1 : 0;
          const double hd = st.heading[u], cd = st.cooldown[u];
          const uint32_t mask7 =
              0x1Fu | ((cd <= 0.0) ? 0x20u : 0u) | (C->enable_noop ? 0x40u : 0u);
          const double speff = C->speed[i] * swamp_mult(C, Z, W1.zin[i], DC->swamp_m);
          const uint64_t seed = st.seed[b];
          const uint64_t t = (uint64_t)(int64_t)st.t[b];
          const double ue = uniform53(seed, t, TAG_EXPLORE, (uint64_t)i);
          const double up = uniform53(seed, t, TAG_PICK, (uint64_t)i);
          W1.vis[i] = st.vis[u];
          W1.atk[i] = st.atk[u];
          const double2 m = st.mem_pos[u];
          const int r = scripted_body<1>(W1, C, i, N, Z, hd, cd, speff * C->dt, mask7, ue, up,
                                         C->epsilon[team], C->aggressive[team], DC->bush_m, m.x,
                                         m.y, (ub & U_MEMV) != 0);
          P.ctrl_act[u] = (int8_t)(r & SA_ACT_MASK);
          if (r & SA_HAS) {
            const int tg = r >> SA_TGT_SHIFT;
            st.mem_pos[u] = make_double2(W1.px[tg], W1.py[tg]);
          }
          const bool mv = (r & (SA_HAS | SA_MEMOK)) != 0;
          st.ubits[u] = (uint8_t)((ub & ~U_MEMV) | (mv ? U_MEMV : 0));
        }
      }
    }
    __syncwarp();
  }
}

// nh: heuristic units per env (upper bound over the config table), >= 1
cudaError_t launch_ctrl_w1(const Params& P, int nh, int sm_count, cudaStream_t stream) {
  int G = 32 / nh;
  if (G > 8) G = 8;
  if (G < 1) G = 1;
  const int threads = 128;
  const size_t smem = sizeof(CtrlView) * G * (threads / 32);
  static size_t cached_smem = 0;
  static int cached_per_sm = 0;
  int per_sm = cached_per_sm;
  if (smem != cached_smem) {
    cudaError_t e = cudaFuncSetAttribute(ctrl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ctrl_kernel, threads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    cached_smem = smem;
    cached_per_sm = per_sm;
  }
  const int64_t groups = (P.B + G - 1) / G;
  const int64_t need = (groups + threads / 32 - 1) / (threads / 32);
  const int64_t cap = (int64_t)sm_count * per_sm;
  const int grid = (int)(need < cap ? (need < 1 ? 1 : need) : cap);
  ctrl_kernel<<<grid, threads, smem, stream>>>(P, G, nh);
  return cudaGetLastError();
}

cudaError_t launch_lanes_w1(const Params& P, int sm_count, cudaStream_t stream, int* grid) {
  return launch_lanes_t<1, 4>(P, sm_count, stream, grid);
}
cudaError_t launch_emit_w1(const Params& P, int sm_count, cudaStream_t stream) {
  #ifndef TABX_EMIT_EPW
#define TABX_EMIT_EPW 8
#endif
  return launch_emit_t<1, TABX_EMIT_EPW>(P, sm_count, stream);
}
// Phase cycle counters of the instrumented build (zeros otherwise).
cudaError_t phase_cycles_w1(unsigned long long* host16, int reset) {
#ifdef TABX_PHASE_PROF
  cudaError_t e = cudaMemcpyFromSymbol(host16, tabx_phase_cycles, 16 * sizeof(unsigned long long));
  if (e == cudaSuccess && reset) {
    static const unsigned long long zero[16] = {};
    e = cudaMemcpyToSymbol(tabx_phase_cycles, zero, sizeof(zero));
  }
  return e;
#else
  (void)reset;
  for (int k = 0; k < 16; ++k) host16[k] = 0;
  return cudaSuccess;
#endif
}
}  // namespace tabx
