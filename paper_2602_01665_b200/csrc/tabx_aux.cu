// Auxiliary kernels: action validation, spawn, state export/import,
// statistics reduction, libm test hook, and the lane-kernel dispatcher.
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <tuple>

#include "tabx_device.cuh"
#include "tabx_math.cuh"

namespace tabx {

cudaError_t launch_lanes_w1(const Params& P, int sm_count, cudaStream_t stream, int* grid);
cudaError_t launch_lanes_w2(const Params& P, int sm_count, cudaStream_t stream, int* grid);
cudaError_t launch_lanes_w4(const Params& P, int sm_count, cudaStream_t stream, int* grid);
cudaError_t launch_lanes_w8(const Params& P, int sm_count, cudaStream_t stream, int* grid);
cudaError_t launch_emit_w1(const Params& P, int sm_count, cudaStream_t stream);
cudaError_t launch_emit_w2(const Params& P, int sm_count, cudaStream_t stream);
cudaError_t launch_emit_w4(const Params& P, int sm_count, cudaStream_t stream);
cudaError_t launch_emit_w8(const Params& P, int sm_count, cudaStream_t stream);

cudaError_t launch_geometry(const void* kernel, int threads, size_t smem, int* per_sm) {
  static std::mutex mu;
  // resident blocks per (kernel, device, threads, smem); the dynamic
  // shared-memory limit per (kernel, device) only ever rises (lowering it
  // would break a cached larger launch of the same kernel)
  static std::map<std::tuple<const void*, int, int, size_t>, int> occ;
  static std::map<std::pair<const void*, int>, size_t> limit;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const auto key = std::make_tuple(kernel, dev, threads, smem);
  std::lock_guard<std::mutex> lock(mu);
  auto it = occ.find(key);
  if (it != occ.end()) {
    *per_sm = it->second;
    return cudaSuccess;
  }
  size_t& lim = limit[std::make_pair(kernel, dev)];
  if (smem > lim) {
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    lim = smem;
  }
  int n = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem);
  if (e != cudaSuccess) return e;
  n = n < 1 ? 1 : n;
  occ.emplace(key, n);
  *per_sm = n;
  return cudaSuccess;
}

cudaError_t launch_emit(const Params& P, int W, int sm_count, cudaStream_t stream) {
  switch (W) {
    case 1: return launch_emit_w1(P, sm_count, stream);
    case 2: return launch_emit_w2(P, sm_count, stream);
    case 4: return launch_emit_w4(P, sm_count, stream);
    default: return launch_emit_w8(P, sm_count, stream);
  }
}

// External action validation (environment.py:166-178): first offender in
// row-major order is latched with atomicMin before any lane mutates.
__global__ void validate_kernel(const int64_t* __restrict__ actions, DevState st,
                                const tabx_config* __restrict__ cfgs, int64_t B, int N,
                                Sync* sync) {
  const int64_t n = B * N;
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = u / N;
    const int i = (int)(u - b * N);
    // every input issued before the first test: one DRAM round trip per
    // unit instead of a chain of dependent ones behind early exits
    const uint8_t fl = st.flags[b];
    const int32_t k = st.cfg[b];
    const uint8_t ub = st.ubits[u];
    const int64_t a = actions[u];
    const double cd = st.cooldown[u];
    const tabx_config* C = cfgs + k;
    const bool ext = !(fl & F_DONE) && C->active[i] && (ub & U_ALIVE) &&
                     C->controller[C->team[i] ? 1 : 0] == TABX_CTRL_EXTERNAL;
    if (!ext) continue;
    bool ok;
    if (a < 0 || a >= TABX_NUM_ACTIONS) {
      ok = false;
    } else if (a == A_ATTACK) {
      ok = cd <= 0.0;
    } else if (a == A_NOOP) {
      ok = C->enable_noop != 0;
    } else {
      ok = true;
    }
    if (!ok) atomicMin(&sync->err_index, (unsigned long long)u);
  }
}

// fill_env for lanes [b0, b1) (arrays.py:244-321); also used at creation.
// With a lane list, entry k spawns lane lanes[k], first switching it to
// config slots[k] and seed seeds[k] when those are given.
// A single lane (reset_env) takes its slot / seed as immediates instead
// (imm_slot >= 0, has_imm_seed), so the host never stages them in memory.
__global__ void spawn_kernel(DevState st, const tabx_config* __restrict__ cfgs,
                             const DerivedCfg* __restrict__ dcfgs, int64_t b0, int64_t b1, int N,
                             int W, int reset_stats, const int64_t* __restrict__ lanes,
                             const int32_t* __restrict__ slots, const uint64_t* __restrict__ seeds,
                             int32_t imm_slot, uint64_t imm_seed, int has_imm_seed) {
  for (int64_t k = b0 + blockIdx.x; k < b1; k += gridDim.x) {
    const int64_t b = lanes ? lanes[k] : k;
    if (slots || seeds || imm_slot >= 0 || has_imm_seed) {
      if (threadIdx.x == 0) {
        if (slots) st.cfg[b] = slots[k];
        if (seeds) st.seed[b] = seeds[k];
        if (imm_slot >= 0) st.cfg[b] = imm_slot;
        if (has_imm_seed) st.seed[b] = imm_seed;
      }
      __syncthreads();
    }
    const tabx_config* C = cfgs + st.cfg[b];
    const DerivedCfg* DC = dcfgs + st.cfg[b];
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const int64_t u = b * N + i;
      if (C->active[i]) {
        st.pos[u] = make_double2(C->spawn_x[i], C->spawn_y[i]);
        st.heading[u] = C->spawn_heading[i];
        st.health[u] = C->max_health[i];
        st.ubits[u] = U_ALIVE;
      } else {
        st.ubits[u] = 0;
      }
      st.vel[u] = make_double2(0.0, 0.0);
      st.imp_dv[u] = make_double2(0.0, 0.0);
      st.cooldown[u] = 0.0;
      st.reveal[u] = 0.0;
      st.mem_pos[u] = make_double2(0.0, 0.0);
      const double h = st.heading[u];
      st.hcs[u] = make_double2(libm_cos(h), libm_sin(h));
      st.zbits[u] = zone_bits(C, DC, C->n_zones, st.pos[u].x, st.pos[u].y);
      for (int k = 0; k < W; ++k) {
        st.vis[u * W + k] = 0u;
        st.atk[u * W + k] = 0u;
      }
    }
    if (threadIdx.x == 0) {
      // env_steps statistic: the steps of an episode cut short by this
      // respawn were never added to st_len (only finished episodes are)
      if (reset_stats)
        st.st_base[b] = 0;
      else if (!(st.flags[b] & F_DONE))
        st.st_base[b] += st.t[b];
      st.t[b] = 0;
      st.prev_gap[b] = 0.0;
      st.ep_return[b] = 0.0;
      st.flags[b] = 0;
      st.winner[b] = -1;
      st.reason[b] = R_NONE;
      st.first_kill[b] = -1;
      if (reset_stats) {
        st.st_episodes[b] = st.st_wins[b] = st.st_fk_ally[b] = st.st_ties[b] = st.st_elims[b] = 0;
        st.st_len[b] = 0;
        st.st_ret[b] = 0.0;
      }
    }
  }
}

// Row k of the destination <- lane lanes[k] (lanes == nullptr: lane k).
__global__ void export_kernel(DevState st, tabx_state d, const int64_t* __restrict__ lanes,
                              int64_t rows, int N, int W) {
  const int64_t n = rows * N;
  for (int64_t du = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; du < n;
       du += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = du / N;
    const int i = (int)(du - k * N);
    const int64_t b = lanes ? lanes[k] : k;
    const int64_t u = b * N + i;
    if (i == 0) {
      if (d.seed) d.seed[k] = st.seed[b];
      if (d.episode) d.episode[k] = st.episode[b];
      if (d.t) d.t[k] = st.t[b];
      if (d.prev_gap) d.prev_gap[k] = st.prev_gap[b];
      if (d.ep_return) d.ep_return[k] = st.ep_return[b];
      if (d.done) d.done[k] = (st.flags[b] & F_DONE) ? 1 : 0;
      if (d.terminated) d.terminated[k] = (st.flags[b] & F_TERM) ? 1 : 0;
      if (d.truncated) d.truncated[k] = (st.flags[b] & F_TRUNC) ? 1 : 0;
      if (d.winner) d.winner[k] = st.winner[b];
      if (d.reason) d.reason[k] = st.reason[b];
      if (d.first_kill) d.first_kill[k] = st.first_kill[b];
      if (d.config) d.config[k] = st.cfg[b];
    }
    if (d.pos) { d.pos[2 * du] = st.pos[u].x; d.pos[2 * du + 1] = st.pos[u].y; }
    if (d.heading) d.heading[du] = st.heading[u];
    if (d.vel) { d.vel[2 * du] = st.vel[u].x; d.vel[2 * du + 1] = st.vel[u].y; }
    if (d.imp_dv) { d.imp_dv[2 * du] = st.imp_dv[u].x; d.imp_dv[2 * du + 1] = st.imp_dv[u].y; }
    if (d.health) d.health[du] = st.health[u];
    if (d.cooldown) d.cooldown[du] = st.cooldown[u];
    if (d.reveal) d.reveal[du] = st.reveal[u];
    if (d.alive) d.alive[du] = (st.ubits[u] & U_ALIVE) ? 1 : 0;
    if (d.mem_pos) { d.mem_pos[2 * du] = st.mem_pos[u].x; d.mem_pos[2 * du + 1] = st.mem_pos[u].y; }
    if (d.mem_valid) d.mem_valid[du] = (st.ubits[u] & U_MEMV) ? 1 : 0;
    for (int j = 0; j < N; ++j) {
      const uint32_t vb = (st.vis[u * W + (j >> 5)] >> (j & 31)) & 1u;
      const uint32_t ab = (st.atk[u * W + (j >> 5)] >> (j & 31)) & 1u;
      if (d.vis) d.vis[du * N + j] = (uint8_t)vb;
      if (d.atk) d.atk[du * N + j] = (uint8_t)ab;
    }
  }
}

__global__ void import_kernel(DevState st, tabx_state s, const tabx_config* __restrict__ cfgs,
                              const DerivedCfg* __restrict__ dcfgs, int64_t B, int N, int W) {
  const int64_t n = B * N;
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = u / N;
    const int i = (int)(u - b * N);
    if (i == 0) {
      if (s.seed) st.seed[b] = s.seed[b];
      if (s.episode) st.episode[b] = s.episode[b];
      if (s.t) st.t[b] = (int32_t)s.t[b];
      if (s.prev_gap) st.prev_gap[b] = s.prev_gap[b];
      if (s.ep_return) st.ep_return[b] = s.ep_return[b];
      if (s.done && s.terminated && s.truncated)
        st.flags[b] = (s.done[b] ? F_DONE : 0) | (s.terminated[b] ? F_TERM : 0) |
                      (s.truncated[b] ? F_TRUNC : 0);
      if (s.winner) st.winner[b] = (int8_t)s.winner[b];
      if (s.reason) st.reason[b] = (int8_t)s.reason[b];
      if (s.first_kill) st.first_kill[b] = (int8_t)s.first_kill[b];
      if (s.config) st.cfg[b] = s.config[b];
    }
    if (s.pos) st.pos[u] = make_double2(s.pos[2 * u], s.pos[2 * u + 1]);
    if (s.heading) st.heading[u] = s.heading[u];
    if (s.vel) st.vel[u] = make_double2(s.vel[2 * u], s.vel[2 * u + 1]);
    if (s.imp_dv) st.imp_dv[u] = make_double2(s.imp_dv[2 * u], s.imp_dv[2 * u + 1]);
    if (s.health) st.health[u] = s.health[u];
    if (s.cooldown) st.cooldown[u] = s.cooldown[u];
    if (s.reveal) st.reveal[u] = s.reveal[u];
    if (s.mem_pos) st.mem_pos[u] = make_double2(s.mem_pos[2 * u], s.mem_pos[2 * u + 1]);
    if (s.alive && s.mem_valid)
      st.ubits[u] = (s.alive[u] ? U_ALIVE : 0) | (s.mem_valid[u] ? U_MEMV : 0);
    {
      // derived caches follow the imported heading / position
      const int32_t k = s.config ? s.config[b] : st.cfg[b];
      const double h = s.heading ? s.heading[u] : st.heading[u];
      const double x = s.pos ? s.pos[2 * u] : st.pos[u].x;
      const double y = s.pos ? s.pos[2 * u + 1] : st.pos[u].y;
      st.hcs[u] = make_double2(libm_cos(h), libm_sin(h));
      st.zbits[u] = zone_bits(cfgs + k, dcfgs + k, cfgs[k].n_zones, x, y);
    }
    if (s.vis && s.atk) {
      for (int k = 0; k < W; ++k) {
        uint32_t vw = 0, aw = 0;
        for (int jj = 0; jj < 32; ++jj) {
          const int j = (k << 5) + jj;
          if (j >= N) break;
          if (s.vis[u * N + j]) vw |= 1u << jj;
          if (s.atk[u * N + j]) aw |= 1u << jj;
        }
        st.vis[u * W + k] = vw;
        st.atk[u * W + k] = aw;
      }
    }
  }
}

// Per-config derived values (reciprocals, masks, roster sizes).
__global__ void derive_kernel(const tabx_config* __restrict__ cfgs, DerivedCfg* dcfgs, int k0,
                              int k1) {
  for (int k = k0 + blockIdx.x; k < k1; k += gridDim.x) {
    const tabx_config* C = cfgs + k;
    DerivedCfg* D = dcfgs + k;
    for (int i = threadIdx.x; i < C->n_units; i += blockDim.x) {
      D->rmh[i] = 1.0 / C->max_health[i];
      D->rucd[i] = C->cooldown[i] > 0.0 ? 1.0 / C->cooldown[i] : 0.0;
    }
    for (int z = threadIdx.x; z < C->n_zones; z += blockDim.x) {
      D->rax[z] = C->zone_type[z] ? 1.0 / C->zone_ax[z] : 0.0;
      D->ray[z] = C->zone_type[z] ? 1.0 / C->zone_ay[z] : 0.0;
    }
    // zone blocks of the observation / global state (perception.py:170-201)
    for (int q = threadIdx.x; q < TABX_MAX_ZONES * TABX_ZONE_DIM; q += blockDim.x) {
      const int z = q / TABX_ZONE_DIM, f = q % TABX_ZONE_DIM;
      const int ty = z < C->n_zones ? C->zone_type[z] : TABX_ZONE_NONE;
      float vo = 0.0f, vg = 0.0f;
      if (ty != TABX_ZONE_NONE) {
        switch (f) {
          case 0: case 1: case 2: vo = vg = (ty == f + 1) ? 1.0f : 0.0f; break;
          case 3: vg = __double2float_rn(C->zone_cx[z] / C->field_w); break;
          case 4: vg = __double2float_rn(C->zone_cy[z] / C->field_h); break;
          case 5: vo = vg = __double2float_rn(C->zone_ax[z]); break;
          case 6: vo = vg = __double2float_rn(C->zone_ay[z]); break;
          default: vo = vg = __double2float_rn(C->zone_effect[z]); break;
        }
      }
      D->zobs[q] = vo;
      D->zglob[q] = vg;
    }
    if (threadIdx.x == 0) {
      D->rw = 1.0 / C->field_w;
      double rmx = 0.0;
      for (int i = 0; i < C->n_units; ++i)
        if (C->active[i] && C->radius[i] > rmx) rmx = C->radius[i];
      D->rad_max = rmx;
      D->rh = 1.0 / C->field_h;
      uint32_t lm = 0, bm = 0, sm = 0;
      for (int z = 0; z < C->n_zones; ++z) {
        if (C->zone_type[z] == TABX_ZONE_LAVA) lm |= 1u << z;
        if (C->zone_type[z] == TABX_ZONE_BUSH) bm |= 1u << z;
        if (C->zone_type[z] == TABX_ZONE_SWAMP) sm |= 1u << z;
      }
      D->lava_m = lm;
      D->bush_m = bm;
      D->swamp_m = sm;
      int na = 0, ne = 0;
      for (int i = 0; i < C->n_units; ++i) {
        if (!C->active[i]) continue;
        if (C->team[i]) ++ne; else ++na;
      }
      D->n_ally = na;
      D->n_enemy = ne;
      int nh = 0;
      for (int i = 0; i < C->n_units; ++i)
        if (C->active[i] && C->controller[C->team[i] ? 1 : 0] == TABX_CTRL_HEURISTIC)
          D->hlist[nh++] = (uint8_t)i;
      D->n_heur = nh;
    }
  }
}

// Deterministic single-block reduction of the per-lane statistics.
// env_steps of lane b = st_len (finished episodes) + st_base + t of the
// running episode; st_base = -t at the last statistics reset (the part of
// that episode counted before) + t of episodes cut short by a respawn.
__global__ void stats_kernel(DevState st, int64_t B, double* out, int reset) {
  __shared__ double part[8][256];
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t b = threadIdx.x; b < B; b += blockDim.x) {
    const bool done = (st.flags[b] & F_DONE) != 0;
    const int64_t running = done ? 0 : (int64_t)st.t[b];
    acc[0] += st.st_episodes[b];
    acc[1] += st.st_wins[b];
    acc[2] += st.st_fk_ally[b];
    acc[3] += st.st_ties[b];
    acc[4] += (double)st.st_len[b];
    acc[5] += st.st_ret[b];
    acc[6] += st.st_elims[b];
    acc[7] += (double)(st.st_len[b] + st.st_base[b] + running);
    if (reset) {
      st.st_episodes[b] = st.st_wins[b] = st.st_fk_ally[b] = st.st_ties[b] = st.st_elims[b] = 0;
      st.st_len[b] = 0;
      st.st_ret[b] = 0.0;
      st.st_base[b] = -running;
    }
  }
  for (int k = 0; k < 8; ++k) part[k][threadIdx.x] = acc[k];
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s)
      for (int k = 0; k < 8; ++k) part[k][threadIdx.x] += part[k][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int k = 0; k < 8; ++k) out[k] = part[k][0];
}

__global__ void sincos_debug_kernel(const double* x, double* s, double* c, int64_t n) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const sincos_t r = libm_sincos(x[k]);
    s[k] = r.s;
    c[k] = r.c;
  }
}

cudaError_t launch_ctrl_w1(const Params& P, int nh, int sm_count, cudaStream_t stream);
cudaError_t launch_ctrl_w2(const Params& P, int nh, int sm_count, cudaStream_t stream);
cudaError_t launch_ctrl_w4(const Params& P, int nh, int sm_count, cudaStream_t stream);
cudaError_t launch_ctrl_w8(const Params& P, int nh, int sm_count, cudaStream_t stream);
cudaError_t launch_ctrl(const Params& P, int W, int nh, int sm_count, cudaStream_t stream) {
  switch (W) {
    case 1: return launch_ctrl_w1(P, nh, sm_count, stream);
    case 2: return launch_ctrl_w2(P, nh, sm_count, stream);
    case 4: return launch_ctrl_w4(P, nh, sm_count, stream);
    default: return launch_ctrl_w8(P, nh, sm_count, stream);
  }
}

cudaError_t launch_lanes(const Params& P, int W, int sm_count, cudaStream_t stream,
                         int* grid_out) {
  switch (W) {
    case 1: return launch_lanes_w1(P, sm_count, stream, grid_out);
    case 2: return launch_lanes_w2(P, sm_count, stream, grid_out);
    case 4: return launch_lanes_w4(P, sm_count, stream, grid_out);
    default: return launch_lanes_w8(P, sm_count, stream, grid_out);
  }
}

static int grid_for(int64_t n, int threads, int sm_count) {
  int64_t g = (n + threads - 1) / threads;
  int64_t cap = (int64_t)sm_count * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

cudaError_t launch_validate(const int64_t* actions, const DevState& st, const tabx_config* cfgs,
                            int64_t B, int N, Sync* sync, int sm_count, cudaStream_t stream) {
  validate_kernel<<<grid_for(B * N, 256, sm_count), 256, 0, stream>>>(actions, st, cfgs, B, N,
                                                                      sync);
  return cudaGetLastError();
}

cudaError_t launch_spawn(const DevState& st, const tabx_config* cfgs, const DerivedCfg* dcfgs,
                         int64_t b0, int64_t b1, int N, int W, int reset_stats, int sm_count,
                         cudaStream_t stream) {
  int64_t n = b1 - b0;
  int grid = (int)(n < (int64_t)sm_count * 32 ? n : (int64_t)sm_count * 32);
  if (grid < 1) return cudaSuccess;
  spawn_kernel<<<grid, 32 * W, 0, stream>>>(st, cfgs, dcfgs, b0, b1, N, W, reset_stats, nullptr,
                                             nullptr, nullptr, -1, 0, 0);
  return cudaGetLastError();
}

cudaError_t launch_spawn_one(const DevState& st, const tabx_config* cfgs, const DerivedCfg* dcfgs,
                             int64_t b, int32_t slot, uint64_t seed, int has_seed, int N, int W,
                             cudaStream_t stream) {
  spawn_kernel<<<1, 32 * W, 0, stream>>>(st, cfgs, dcfgs, b, b + 1, N, W, 0, nullptr, nullptr,
                                          nullptr, slot, seed, has_seed);
  return cudaGetLastError();
}

cudaError_t launch_spawn_lanes(const DevState& st, const tabx_config* cfgs,
                               const DerivedCfg* dcfgs, const int64_t* lanes, const int32_t* slots,
                               const uint64_t* seeds, int64_t n, int N, int W, int sm_count,
                               cudaStream_t stream) {
  int grid = (int)(n < (int64_t)sm_count * 32 ? n : (int64_t)sm_count * 32);
  if (grid < 1) return cudaSuccess;
  spawn_kernel<<<grid, 32 * W, 0, stream>>>(st, cfgs, dcfgs, 0, n, N, W, 0, lanes, slots, seeds,
                                             -1, 0, 0);
  return cudaGetLastError();
}

cudaError_t launch_export(const DevState& st, const tabx_state& d, const int64_t* lanes,
                          int64_t rows, int N, int W, int sm_count, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  export_kernel<<<grid_for(rows * N, 256, sm_count), 256, 0, stream>>>(st, d, lanes, rows, N, W);
  return cudaGetLastError();
}

cudaError_t launch_import(const DevState& st, const tabx_state& s, const tabx_config* cfgs,
                          const DerivedCfg* dcfgs, int64_t B, int N, int W, int sm_count,
                          cudaStream_t stream) {
  import_kernel<<<grid_for(B * N, 256, sm_count), 256, 0, stream>>>(st, s, cfgs, dcfgs, B, N, W);
  return cudaGetLastError();
}

cudaError_t launch_derive(const tabx_config* cfgs, DerivedCfg* dcfgs, int k0, int k1,
                          cudaStream_t stream) {
  if (k1 <= k0) return cudaSuccess;
  derive_kernel<<<k1 - k0, 128, 0, stream>>>(cfgs, dcfgs, k0, k1);
  return cudaGetLastError();
}

cudaError_t launch_stats(const DevState& st, int64_t B, double* out, int reset,
                         cudaStream_t stream) {
  stats_kernel<<<1, 256, 0, stream>>>(st, B, out, reset);
  return cudaGetLastError();
}

cudaError_t launch_sincos_debug(const double* x, double* s, double* c, int64_t n,
                                cudaStream_t stream) {
  sincos_debug_kernel<<<grid_for(n, 256, 148), 256, 0, stream>>>(x, s, c, n);
  return cudaGetLastError();
}

}  // namespace tabx
