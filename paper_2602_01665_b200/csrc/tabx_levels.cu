// Level sampling / mutation on the device: the
// reference's sample_level / mutate_level (pkg/src/skirmish/scenario.py:696-826)
// for a batch of levels, one warp per level.  The warp copies the source
// config row into the destination row; lane 0 then replays the reference's
// draw sequence on the level's own PCG64 stream -- numpy's bit generator
// bit for bit (128-bit LCG step, XSL-RR output, next_double = (x >> 11) *
// 2^-53, uniform = lo + (hi - lo) * next_double, bounded integers by
// Lemire's method on the bit generator's buffered 32-bit halves) -- and
// rewrites the drawn fields and the unit roles that depend on them
// (template.py / arrays.py:265-267).  Compiled with -fmad=false like the
// step: every expression is the reference's float64 one.
#include <cuda_runtime.h>
#include <stdint.h>

#include "tabx_device.cuh"

namespace tabx {

struct Pcg64 {
  uint64_t s_hi, s_lo, i_hi, i_lo;
  uint32_t has32, u32;

  // numpy pcg64: state = state * MULT + inc; output XSL-RR of the new state
  __device__ uint64_t next64() {
    const uint64_t m_hi = 0x2360ed051fc65da4ull, m_lo = 0x4385df649fccf645ull;
    const uint64_t lo = s_lo * m_lo;
    const uint64_t hi = __umul64hi(s_lo, m_lo) + s_hi * m_lo + s_lo * m_hi;
    s_lo = lo + i_lo;
    s_hi = hi + i_hi + (s_lo < lo ? 1ull : 0ull);
    const uint64_t x = s_hi ^ s_lo;
    const unsigned r = (unsigned)(s_hi >> 58);
    return (x >> r) | (x << ((64u - r) & 63u));
  }
  __device__ uint32_t next32() {
    if (has32) {
      has32 = 0;
      return u32;
    }
    const uint64_t v = next64();
    has32 = 1;
    u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  __device__ double next_double() {
    return (double)(next64() >> 11) * (1.0 / 9007199254740992.0);
  }
  // Generator.uniform(lo, hi)
  __device__ double uniform(double lo, double hi) {
    const double range = hi - lo;
    return lo + range * next_double();
  }
  // Generator.integers(0, n) for 1 <= n <= 2^32 - 1 (buffered Lemire)
  __device__ int bounded(int n) {
    const uint32_t rng = (uint32_t)(n - 1);
    if (rng == 0) return 0;
    const uint32_t excl = rng + 1u;
    uint64_t m = (uint64_t)next32() * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      const uint32_t thr = (0xFFFFFFFFu - rng) % excl;
      while (left < thr) {
        m = (uint64_t)next32() * excl;
        left = (uint32_t)m;
      }
    }
    return (int)(m >> 32);
  }
};

// Python min(max(x, lo), hi) (first argument wins ties)
__device__ __forceinline__ double py_clip(double x, double lo, double hi) {
  const double a = lo > x ? lo : x;
  return hi < a ? hi : a;
}

__device__ __forceinline__ void set_roles(tabx_config* C, int i) {
  C->role_assassin[i] = C->speed[i] >= 1.4 ? 1 : 0;  // arrays.py:31
  C->role_ranger[i] = (C->attack_range[i] >= 10.0 && C->damage[i] > 0.0) ? 1 : 0;
  C->role_healer[i] = C->damage[i] < 0.0 ? 1 : 0;
}

__device__ __forceinline__ void default_effect_range(int ty, double& lo, double& hi) {
  if (ty == TABX_ZONE_LAVA) {  // LAVA_DAMAGE_RANGE, scenario.py:41
    lo = 2.0;
    hi = 10.0;
  } else {  // SWAMP_MULT_RANGE, scenario.py:42
    lo = 0.2;
    hi = 0.8;
  }
}

__device__ void level_body(tabx_config* C, const tabx_level_spec& S, int op, double delta,
                           Pcg64& g) {
  const int N = C->n_units;
  int nz = 0;  // the scenario's zones fill the leading slots
  while (nz < C->n_zones && C->zone_type[nz] != TABX_ZONE_NONE) ++nz;
  // open unit fields in sorted-name order: attack_damage, max_health, speed
  double* ufield[3] = {C->damage, C->max_health, C->speed};

  if (op == TABX_LEVEL_SAMPLE) {
    if (S.open_units) {
      for (int i = 0; i < N; ++i) {
        if (!C->active[i]) continue;
        for (int f = 0; f < 3; ++f)
          if (S.unit_open[f]) ufield[f][i] = g.uniform(S.unit_lo[f], S.unit_hi[f]);
        set_roles(C, i);
      }
    }
    if (S.open_zones) {
      for (int z = 0; z < nz; ++z) {
        const int old = C->zone_type[z];
        const int ty = S.zone_types[g.bounded(S.n_zone_types)];
        C->zone_cx[z] = g.uniform(S.box_x0, S.box_x1);
        C->zone_cy[z] = g.uniform(S.box_y0, S.box_y1);
        if (S.axis_open) {
          C->zone_ax[z] = g.uniform(S.axis_lo, S.axis_hi);
          C->zone_ay[z] = g.uniform(S.axis_lo, S.axis_hi);
        }
        if (ty == TABX_ZONE_BUSH) {
          C->zone_effect[z] = 0.0;
        } else if (S.effect_open[ty]) {
          C->zone_effect[z] = g.uniform(S.effect_lo[ty], S.effect_hi[ty]);
        } else if (ty != old) {
          double lo, hi;
          default_effect_range(ty, lo, hi);
          C->zone_effect[z] = g.uniform(lo, hi);
        }
        C->zone_type[z] = ty;
      }
    }
    if (S.open_heuristic) {
      for (int t = 0; t < 2; ++t) {
        if (C->controller[t] != TABX_CTRL_HEURISTIC) continue;
        if (S.eps_open) C->epsilon[t] = g.uniform(S.eps_lo, S.eps_hi);
        if (S.agg_open) C->aggressive[t] = g.uniform(S.agg_lo, S.agg_hi);
      }
    }
    return;
  }

  if (op == TABX_LEVEL_PERTURB) {
    auto bump = [&](double v, double lo, double hi) {
      const double width = hi - lo;
      const double nudged = v + g.uniform(-delta * width, delta * width);
      return py_clip(nudged, lo, hi);
    };
    if (S.open_units) {
      for (int i = 0; i < N; ++i) {
        if (!C->active[i]) continue;
        for (int f = 0; f < 3; ++f)
          if (S.unit_open[f]) ufield[f][i] = bump(ufield[f][i], S.unit_lo[f], S.unit_hi[f]);
        set_roles(C, i);
      }
    }
    if (S.open_zones) {
      for (int z = 0; z < nz; ++z) {
        C->zone_cx[z] = bump(C->zone_cx[z], S.box_x0, S.box_x1);
        C->zone_cy[z] = bump(C->zone_cy[z], S.box_y0, S.box_y1);
        if (S.axis_open) {
          C->zone_ax[z] = bump(C->zone_ax[z], S.axis_lo, S.axis_hi);
          C->zone_ay[z] = bump(C->zone_ay[z], S.axis_lo, S.axis_hi);
        }
        const int ty = C->zone_type[z];
        if (S.effect_open[ty])
          C->zone_effect[z] = bump(C->zone_effect[z], S.effect_lo[ty], S.effect_hi[ty]);
      }
    }
    if (S.open_heuristic) {
      for (int t = 0; t < 2; ++t) {
        if (C->controller[t] != TABX_CTRL_HEURISTIC) continue;
        if (S.eps_open) C->epsilon[t] = bump(C->epsilon[t], S.eps_lo, S.eps_hi);
        if (S.agg_open) C->aggressive[t] = bump(C->aggressive[t], S.agg_lo, S.agg_hi);
      }
    }
    return;
  }

  if (nz == 0) return;  // single-zone edits of a zoneless level are no-ops
  const int z = g.bounded(nz);
  if (op == TABX_LEVEL_SWAP_AXES) {
    const double a = C->zone_ax[z];
    C->zone_ax[z] = C->zone_ay[z];
    C->zone_ay[z] = a;
    return;
  }
  // retype
  const int ty = S.zone_types[g.bounded(S.n_zone_types)];
  if (ty == TABX_ZONE_BUSH) {
    C->zone_effect[z] = 0.0;
  } else {
    double lo, hi;
    if (S.effect_open[ty]) {
      lo = S.effect_lo[ty];
      hi = S.effect_hi[ty];
    } else {
      default_effect_range(ty, lo, hi);
    }
    C->zone_effect[z] = g.uniform(lo, hi);
  }
  C->zone_type[z] = ty;
}

__global__ void levels_kernel(tabx_config* cfgs, const int32_t* __restrict__ src_slots,
                              int32_t dst_first, int32_t count, tabx_level_spec spec, int op,
                              double delta, tabx_pcg64* rngs) {
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  for (int k = blockIdx.x * warps + (threadIdx.x >> 5); k < count; k += gridDim.x * warps) {
    tabx_config* dst = cfgs + dst_first + k;
    const int32_t src = src_slots ? src_slots[k] : dst_first + k;
    if (src != dst_first + k) {
      const int4* s4 = reinterpret_cast<const int4*>(cfgs + src);
      int4* d4 = reinterpret_cast<int4*>(dst);
      constexpr int n4 = (int)(sizeof(tabx_config) / 16);
      for (int q = lane; q < n4; q += 32) d4[q] = s4[q];
      constexpr int tail = (int)(sizeof(tabx_config) % 16);
      if (tail && lane < tail)
        reinterpret_cast<char*>(dst)[n4 * 16 + lane] =
            reinterpret_cast<const char*>(cfgs + src)[n4 * 16 + lane];
    }
    __syncwarp();
    if (lane == 0) {
      tabx_pcg64 r = rngs[k];
      Pcg64 g{r.state_hi, r.state_lo, r.inc_hi, r.inc_lo, r.has_uint32, r.uinteger};
      level_body(dst, spec, op, delta, g);
      r.state_hi = g.s_hi;
      r.state_lo = g.s_lo;
      r.has_uint32 = g.has32;
      r.uinteger = g.u32;
      rngs[k] = r;
    }
    __syncwarp();
  }
}

cudaError_t launch_levels(tabx_config* cfgs, const int32_t* src_slots, int32_t dst_first,
                          int32_t count, const tabx_level_spec& spec, int op, double delta,
                          tabx_pcg64* rngs, int sm_count, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  const int warps = 4;
  int grid = (count + warps - 1) / warps;
  if (grid > sm_count * 8) grid = sm_count * 8;
  levels_kernel<<<grid, 32 * warps, 0, stream>>>(cfgs, src_slots, dst_first, count, spec, op,
                                                 delta, rngs);
  return cudaGetLastError();
}

}  // namespace tabx
