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
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "tabx_device.cuh"
#include "tabx_math.cuh"

namespace tabx {

// Per-warp view of one environment, laid out in dynamic shared memory for
// the batch's N units: positions, the 15 own features (16-float rows), the
// N-bit visibility / attackable rows, unit flags.
// floats per unit row of the view's own-feature table (15 used): a multiple
// of 4 keeps the rows 16-byte aligned for the float4 reads of the pair
// blocks, and 20 (not 16) spreads eight consecutive rows over distinct bank
// groups (fewer shared-memory bank conflicts in those reads)
#ifndef TABX_OWN_STRIDE
#define TABX_OWN_STRIDE 20
#endif
template <int W>
struct EmitEnv {
  double* px;
  double* py;
  float (*own)[TABX_OWN_STRIDE];
  uint32_t* vis;
  uint32_t* atk;
  uint32_t* flags;  // bit0 active, bit1 enemy
};

// Per-warp emitter scratch: the view and, for W == 1, the env's visible
// (observer, other) pairs in row-major order with each observer's start in
// that list; then two stage buffers.
template <int W>
struct EmitScratch {
  EmitEnv<W> E;
  uint16_t* rstart;  // [N + 1]
  uint16_t* plist;   // [N * (N - 1)], (observer << 5) | other
  float* stage;
};
__host__ __device__ __forceinline__ constexpr size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }
template <int W>
__host__ __device__ __forceinline__ constexpr size_t emit_view_bytes(int N) {
  return align16((size_t)16 * N) + (size_t)4 * TABX_OWN_STRIDE * N +
         align16((size_t)4 * N * (2 * W + 1));
}
template <int W>
__host__ __device__ __forceinline__ constexpr size_t emit_aux_bytes(int N, int Z, int R) {
  return W == 1 ? align16(((size_t)N + 1 + (size_t)N * (N - 1)) * sizeof(uint16_t)) : 0;
}

__device__ __forceinline__ bool row_bit(const uint32_t* row, int j) {
  return (row[j >> 5] >> (j & 31)) & 1u;
}

// Own-feature block of unit u from its state values (perception.py:108-132).
__device__ __forceinline__ void own_from_vals(float* o, double2 p, double2 cs, double hp,
                                              double cd, uint8_t ub,
                                              const tabx_config* __restrict__ C,
                                              const DerivedCfg* __restrict__ DC, int u) {
  o[15] = 0.0f;
  if (!C->active[u]) {
#pragma unroll
    for (int f = 0; f < TABX_OWN_DIM; ++f) o[f] = 0.0f;
    return;
  }
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
  o[13] = (ub & U_ALIVE) ? 1.0f : 0.0f;
  o[14] = __double2float_rn(C->speed[u]);
}

// Own-feature block of unit u from its HBM state.
__device__ __forceinline__ void own_from_state(float* o, const DevState& st, int64_t gu,
                                               const tabx_config* __restrict__ C,
                                               const DerivedCfg* __restrict__ DC, int u) {
  if (!C->active[u]) {
    own_from_vals(o, make_double2(0.0, 0.0), make_double2(0.0, 0.0), 0.0, 0.0, 0, C, DC, u);
    return;
  }
  own_from_vals(o, st.pos[gu], st.hcs[gu], st.health[gu], st.cooldown[gu], st.ubits[gu], C, DC,
                u);
}

// One unit's view inputs held in registers (W = 1: lane u = unit u), so the
// emitter can issue the NEXT environment's loads before streaming the
// current one's rows (TABX_EMIT_VIEW_PREFETCH).
struct ViewRegs {
  double2 p, cs;
  double hp, cd;
  uint32_t vis, atk;
  uint8_t ub;
};
__device__ __forceinline__ void fetch_view_regs(ViewRegs& V, const DevState& st, int64_t b, int N,
                                                int lane) {
  if (lane < N) {
    const int64_t gu = b * N + lane;
    V.p = st.pos[gu];
    V.cs = st.hcs[gu];
    V.hp = st.health[gu];
    V.cd = st.cooldown[gu];
    V.ub = st.ubits[gu];
    V.vis = st.vis[gu];
    V.atk = st.atk[gu];
  }
}

// Load lane b's view into E (all 32 lanes of the warp).
template <int W>
__device__ __forceinline__ void load_view(const EmitScratch<W>& X, const DevState& st, int64_t b,
                                          int N, int Z, const tabx_config* __restrict__ C,
                                          const DerivedCfg* __restrict__ DC, int lane) {
  const EmitEnv<W>& E = X.E;
  // (checked build) the view and pair list, not the stage buffers a bulk
  // store may still be reading
  TABX_POISON(X.E.px, (size_t)((const unsigned char*)X.stage - (const unsigned char*)X.E.px),
              lane, 32);
  __syncwarp();
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
  if constexpr (W == 1) {
    // visible-pair list: exclusive scan of the per-observer counts (vis
    // already excludes inactive observers / others; drop the self bit)
    const bool valid = lane < N;
    uint32_t w = valid ? (E.vis[lane] & ~(1u << lane)) : 0u;
    const int c = __popc(w);
    int incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += v;
    }
    TABX_JITTER(300);
    if (valid) X.rstart[lane + 1] = (uint16_t)incl;
    if (lane == 0) X.rstart[0] = 0;
    for (int n = incl - c; w; w &= w - 1, ++n)
      X.plist[n] = (uint16_t)((lane << 5) | (__ffs(w) - 1));
  }
  __syncwarp();
}


// load_view for W = 1 from the registers fetch_view_regs filled.
__device__ __forceinline__ void load_view_regs(const EmitScratch<1>& X, const ViewRegs& V, int N,
                                               const tabx_config* __restrict__ C,
                                               const DerivedCfg* __restrict__ DC, int lane) {
  const EmitEnv<1>& E = X.E;
  TABX_POISON(X.E.px, (size_t)((const unsigned char*)X.stage - (const unsigned char*)X.E.px),
              lane, 32);
  __syncwarp();
  const bool valid = lane < N;
  if (valid) {
    const int u = lane;
    E.px[u] = V.p.x;
    E.py[u] = V.p.y;
    own_from_vals(E.own[u], V.p, V.cs, V.hp, V.cd, V.ub, C, DC, u);
    E.flags[u] = (C->active[u] ? 1u : 0u) | (C->team[u] ? 2u : 0u);
    E.vis[u] = V.vis;
    E.atk[u] = V.atk;
  }
  uint32_t w = valid ? (V.vis & ~(1u << lane)) : 0u;
  const int c = __popc(w);
  int incl = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  TABX_JITTER(300);
  if (valid) X.rstart[lane + 1] = (uint16_t)incl;
  if (lane == 0) X.rstart[0] = 0;
  for (int n = incl - c; w; w &= w - 1, ++n) X.plist[n] = (uint16_t)((lane << 5) | (__ffs(w) - 1));
  __syncwarp();
}

// W = 1 fixed-shape emitter: 1 = fetch the next env's view into registers
// before streaming this env's rows
#ifndef TABX_EMIT_VIEW_PREFETCH
#define TABX_EMIT_VIEW_PREFETCH -1  // -1: per shape (EmitTune), 0 / 1: off / on
#endif

// bf16 policy-feed stores with the streaming cache hint (st.global.cs)
#ifndef TABX_EMIT_F16_STCS
#define TABX_EMIT_F16_STCS 1  // C5 +1% (4 paired runs)
#endif

// stage buffers per warp (2: fill one while the bulk store drains the other)
#ifndef TABX_EMIT_NBUF
#define TABX_EMIT_NBUF 2
#endif

// ---- TMA bulk stores (cp.async.bulk.global.shared::cta)
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// L2 policy of the row stream's bulk stores.  Evict-first (the rows are
// never read back on the device path) measured faster for the one-warp-per-
// env emitter (W = 1: C3 262,144 envs K2 1.665 -> 1.611 ms, C3 65,536
// -2%, C2 262,144 -1%, C2 65,536 +0.7%) and slower for W = 4 (C4 15.5 ->
// 15.9 ms), so it is used for W = 1 only; TABX_EMIT_EVICT_FIRST=0 turns it off.
#ifndef TABX_EMIT_EVICT_FIRST
#define TABX_EMIT_EVICT_FIRST 1
#endif
template <bool EF>
__device__ __forceinline__ void bulk_s2g(void* g, const void* s, uint32_t bytes) {
  if constexpr (EF && TABX_EMIT_EVICT_FIRST) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;\n" ::"l"(g),
        "r"(smem_addr(s)), "r"(bytes), "l"(pol)
        : "memory");
  } else {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(g),
                 "r"(smem_addr(s)), "r"(bytes)
                 : "memory");
  }
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
template <bool EF>
__device__ __forceinline__ void flush_stage(float* __restrict__ dst, int64_t gs, int count,
                                            const float* stage, int lane) {
  const int pad = (int)(gs & 3);
  const int64_t a0 = (gs + 3) & ~(int64_t)3;
  const int64_t a1 = (gs + count) & ~(int64_t)3;
  TABX_ASSERT(gs >= 0 && count > 0 && ((uintptr_t)(dst + a0) & 15u) == 0);
  if (a1 > a0) {
    if (lane == 0) bulk_s2g<EF>(dst + a0, stage + pad + (a0 - gs), (uint32_t)((a1 - a0) * 4));
    // <= 3 head floats on lanes 0..2, <= 3 tail floats on lanes 4..6
    const int head = (int)(a0 - gs), t0 = (int)(a1 - gs);
    const int e = lane < 4 ? lane : t0 + lane - 4;
    if (lane < 4 ? lane < head : (lane < 8 && e < count)) dst[gs + e] = stage[pad + e];
  } else {
    for (int e = lane; e < count; e += 32) dst[gs + e] = stage[pad + e];
  }
  // one (possibly empty) bulk group per flush keeps the double-buffer
  // accounting exact: wait_group.read 1 frees the buffer before the last
  if (lane == 0) bulk_commit();
}

// a chunk of `count` floats starting at global float gs fits its stage
// buffer of SF floats at the alignment pad gs & 3
__device__ __forceinline__ bool pad_fits(int64_t gs, int count, int SF) {
  return (int)(gs & 3) + count <= SF;
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
// block, the visible (observer, other) pair blocks, and the zone blocks) and
// leave through double-buffered TMA bulk stores; hidden pairs -- most of the
// tensor -- cost only the fill.  `buf` (the stage buffer to fill next)
// persists across the envs a warp emits so the buffer rotation never waits
// on the store just issued; drain = wait for every store before returning.
// o16 (optional): the bfloat16 policy-feed copy of the observation rows,
// row stride ld16 (tabx.h observations_bf16), written from the same stage.
template <int W, bool F16 = false>
__device__ void emit_lane(const EmitScratch<W>& X, float* __restrict__ obs,
                          float* __restrict__ glob, int64_t b, int N, int Z, int D, int G, int R,
                          int SF, const tabx_config* __restrict__ C,
                          const DerivedCfg* __restrict__ DC, int lane, int& buf, bool drain,
                          __nv_bfloat16* __restrict__ o16 = nullptr, int ld16 = 0,
                          int rbeg = 0, int rstep = 1) {
  const EmitEnv<W>& E = X.E;
  const double fw = C->field_w, fh = C->field_h, rw = DC->rw, rh = DC->rh;
  const int M = N - 1;
  const int zoff = TABX_OWN_DIM + TABX_OTHER_DIM * M;
  const int ZD = Z * TABX_ZONE_DIM;
  // Zone blocks of a chunk (W == 1, R * ZD <= 96 and R * 2Z <= 32): each lane
  // owns up to three template slots e = lane + 32k of the chunk's zone region
  // (row e / ZD, feature e % ZD) and one relative-position item (row, zone,
  // axis); the decode, the template values and the zone centres are per-env
  // registers, so a chunk costs a few stores and one quotient per lane.
  const bool zfast = W == 1 && R * ZD <= 96 && R * 2 * Z <= 32;
  float zt[3];
  int zinfo[3];  // (row + 1) << 16 | offset in the chunk; 0 = no slot
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int e = lane + 32 * k;
    const int rr = ZD > 0 ? e / ZD : 0, q = ZD > 0 ? e - rr * ZD : 0;
    const bool on = ZD > 0 && rr < R;
    zinfo[k] = on ? ((rr + 1) << 16) | (rr * D + zoff + q) : 0;
    zt[k] = on ? DC->zobs[q] : 0.0f;
  }
  const int rel_rr = Z > 0 ? lane / (2 * Z) : 0;
  const int rel_z = Z > 0 ? (lane - rel_rr * 2 * Z) >> 1 : 0, rel_ax = lane & 1;
  const bool rel_on = Z > 0 && rel_rr < R && C->zone_type[rel_z] != TABX_ZONE_NONE;
  const double rel_c = rel_on ? (rel_ax ? C->zone_cy[rel_z] : C->zone_cx[rel_z]) : 0.0;
  const double rel_f = rel_ax ? fh : fw, rel_rf = rel_ax ? rh : rw;
  const int rel_off = rel_rr * D + zoff + rel_z * TABX_ZONE_DIM + 3 + rel_ax;
  if (obs || (F16 && o16)) {
    // (rbeg, rstep: this warp's share of the chunks when several warps
    // emit one environment, emit_kernel_cta)
    for (int r0 = rbeg * R; r0 < N; r0 += rstep * R) {
      const int nr = min(R, N - r0);
      const int64_t gs = (b * N + r0) * (int64_t)D;
      TABX_ASSERT(nr > 0 && (pad_fits(gs, nr * D, SF)));
      TABX_JITTER(301);
      float* st = X.stage + buf * SF;
      const int pad = (int)(gs & 3);
      float* row0 = st + pad;
      if (lane == 0) bulk_wait_read<TABX_EMIT_NBUF - 1>();
      __syncwarp();
      {
        const int n4 = (pad + nr * D + 3) >> 2;
        float4* z4 = reinterpret_cast<float4*>(st);
        const float4 zero = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if (lane + 32 * t < n4) z4[lane + 32 * t] = zero;
        for (int q = lane + 256; q < n4; q += 32) z4[q] = zero;
      }
      __syncwarp();
      TABX_JITTER(304);  // lanes start the chunk's writes out of step
      for (int e = lane; e < nr * TABX_OWN_DIM; e += 32) {
        const int rr = e / TABX_OWN_DIM, f = e - rr * TABX_OWN_DIM;
        row0[rr * D + f] = E.own[r0 + rr][f];
      }
      // visible pairs of the chunk's rows (vis excludes inactive rows/columns)
      auto pair_block = [&](int r, int j) {
        TABX_ASSERT(r >= r0 && r < r0 + nr && j >= 0 && j < N && j != r);
        const int kk = j - (j > r ? 1 : 0);
        float* blk = row0 + (r - r0) * D + TABX_OWN_DIM + TABX_OTHER_DIM * kk;
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
      };
      if constexpr (W == 1) {
        const int p1 = X.rstart[r0 + nr];
        for (int p = X.rstart[r0] + lane; p < p1; p += 32) {
          const int rj = X.plist[p];
          pair_block(rj >> 5, rj & 31);
        }
      } else {
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
          pair_block(r0 + rr, j);
        }
      }
      // zone blocks of the active rows: the config's template with the
      // observer-relative position (unused zone slots stay zero)
      if (zfast) {
#pragma unroll
        for (int k = 0; k < 3; ++k)
        {
          const int rr = (zinfo[k] >> 16) - 1;
          if (rr >= 0 && rr < nr && (E.flags[r0 + rr] & 1u)) row0[zinfo[k] & 0xFFFF] = zt[k];
        }
        __syncwarp();  // the relative positions overwrite template slots
        if (rel_on && rel_rr < nr) {
          const int r = r0 + rel_rr;
          if (E.flags[r] & 1u)
            row0[rel_off] = f32_quot(rel_c - (rel_ax ? E.py[r] : E.px[r]), rel_f, rel_rf);
        }
      } else {
        for (int rr = 0; rr < nr; ++rr) {
          const int r = r0 + rr;
          if (!(E.flags[r] & 1u)) continue;
          float* zb = row0 + rr * D + zoff;
          for (int q = lane; q < ZD; q += 32) {
            const int z = q >> 3, f = q & 7;
            float v = DC->zobs[q];
            if ((f == 3 || f == 4) && C->zone_type[z] != TABX_ZONE_NONE)
              v = f == 3 ? f32_quot(C->zone_cx[z] - E.px[r], fw, rw)
                         : f32_quot(C->zone_cy[z] - E.py[r], fh, rh);
            zb[q] = v;
          }
        }
      }
      TABX_JITTER(302);
      fence_proxy_async();
      __syncwarp();
      if (obs) flush_stage<W == 1>(obs, gs, nr * D, st, lane);
      if (F16 && o16) {
        // 8 bfloat16 (16 bytes) per store, zero past obs_dim; the stage is
        // only read, beside the bulk store reading it.  Rows start 8-byte
        // aligned in the stage (D even), so float2 loads.
        const int per_row = ld16 >> 3;
        for (int rr = 0; rr < nr; ++rr) {
          const float* src = row0 + rr * D;
          __nv_bfloat16* dst = o16 + (b * N + r0 + rr) * (int64_t)ld16;
          for (int c = lane; c < per_row; c += 32) {
            const int c0 = c << 3;
            __align__(16) __nv_bfloat162 v[4];
            if ((D & 1) == 0 && ((pad + rr * D) & 1) == 0 && c0 + 8 <= D) {
              const float2* s2 = reinterpret_cast<const float2*>(src + c0);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float2 f = s2[k];
                v[k] = __floats2bfloat162_rn(f.x, f.y);
              }
            } else {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                v[k] = __floats2bfloat162_rn(c0 + 2 * k < D ? src[c0 + 2 * k] : 0.0f,
                                             c0 + 2 * k + 1 < D ? src[c0 + 2 * k + 1] : 0.0f);
            }
#if TABX_EMIT_F16_STCS
            __stcs(reinterpret_cast<uint4*>(dst + c0), *reinterpret_cast<const uint4*>(v));
#else
            *reinterpret_cast<uint4*>(dst + c0) = *reinterpret_cast<const uint4*>(v);
#endif
          }
        }
      }
      buf = buf + 1 == TABX_EMIT_NBUF ? 0 : buf + 1;
    }
  }
  if (glob) {
    const int64_t gs = b * (int64_t)G;
    float* st = X.stage + buf * SF;
    float* row = st + (int)(gs & 3);
    if (lane == 0) bulk_wait_read<TABX_EMIT_NBUF - 1>();
    __syncwarp();
    for (int e = lane; e < N * TABX_OWN_DIM; e += 32) {
      const int u = e / TABX_OWN_DIM;
      row[e] = E.own[u][e - u * TABX_OWN_DIM];
    }
    for (int q = lane; q < ZD; q += 32) row[N * TABX_OWN_DIM + q] = DC->zglob[q];
    TABX_JITTER(303);
    fence_proxy_async();
    __syncwarp();
    flush_stage<W == 1>(glob, gs, G, st, lane);
    buf = buf + 1 == TABX_EMIT_NBUF ? 0 : buf + 1;
  }
  if (drain) {
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
  }
}

// Stage geometry: R rows per chunk within `budget` bytes per buffer.
__host__ __device__ __forceinline__ constexpr int emit_rows(int N, int D, int budget) {
  int R = budget / (4 * D);
  if (R < 1) R = 1;
  if (R > N) R = N;
  return R;
}
__host__ __device__ __forceinline__ constexpr int emit_stage_floats(int N, int D, int G, int R) {
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
// resident CTAs per SM the register budget is cut for (W = 1: 6 CTAs of 4
// warps = 24 warps/SM at 80 registers; W > 1: 3)
#ifndef TABX_EMIT_MIN_BLOCKS_W1
#define TABX_EMIT_MIN_BLOCKS_W1 0  // 0: per shape (EmitTune); the generic kernel: 6
#endif
#ifndef TABX_EMIT_MIN_BLOCKS
#define TABX_EMIT_MIN_BLOCKS 3
#endif
// Bytes of one warp's emitter scratch (view, zone-relative table, stages).
template <int W>
__host__ __device__ __forceinline__ size_t emit_warp_bytes(int N, int Z, int R, int SF) {
  return emit_view_bytes<W>(N) + emit_aux_bytes<W>(N, Z, R) + (size_t)TABX_EMIT_NBUF * SF * sizeof(float);
}
template <int W>
__device__ __forceinline__ EmitScratch<W> emit_scratch(unsigned char* base, int N, int Z, int R) {
  EmitScratch<W> X;
  unsigned char* p = base;
  X.E.px = reinterpret_cast<double*>(p);
  X.E.py = X.E.px + N;
  p += align16((size_t)16 * N);
  X.E.own = reinterpret_cast<float(*)[TABX_OWN_STRIDE]>(p);
  p += (size_t)4 * TABX_OWN_STRIDE * N;
  X.E.vis = reinterpret_cast<uint32_t*>(p);
  X.E.atk = X.E.vis + N * W;
  X.E.flags = X.E.atk + N * W;
  p += align16((size_t)4 * N * (2 * W + 1));
  X.rstart = reinterpret_cast<uint16_t*>(p);
  X.plist = X.rstart + N + 1;
  X.stage = reinterpret_cast<float*>(p + emit_aux_bytes<W>(N, Z, R));
  return X;
}

template <int W, int EPW, bool F16>
__global__ void __launch_bounds__(32 * EPW,
                                  (W == 1 ? (TABX_EMIT_MIN_BLOCKS_W1 > 0 ? TABX_EMIT_MIN_BLOCKS_W1 : 6)
                                          : TABX_EMIT_MIN_BLOCKS))
    emit_kernel(const Params P, int R, int SF) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (is_step_mode(P.mode) && P.sync->err_index != NO_ERROR) return;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const EmitScratch<W> X =
      emit_scratch<W>(smem_raw + (size_t)w * emit_warp_bytes<W>(P.N, P.Z, R, SF), P.N, P.Z, R);
  const DevState& st = P.st;
  int buf = 0;
  const int64_t stride = (int64_t)gridDim.x * EPW;
  int64_t b = (int64_t)blockIdx.x * EPW + w;
  // config index and flags one env ahead (see emit_kernel_fixed)
  int32_t k_next = b < P.B ? st.cfg[b] : 0;
  uint8_t f_next = b < P.B ? st.flags[b] : 0;
  for (; b < P.B; b += stride) {
    const int32_t k = k_next;
    const uint8_t fl = f_next;
    if (b + stride < P.B) {
      k_next = st.cfg[b + stride];
      f_next = st.flags[b + stride];
    }
    const tabx_config* C = P.cfgs + k;
    const DerivedCfg* DC = P.dcfgs + k;
    const bool pending = (fl & F_PEND) != 0;
    float* ob = pending ? P.out.final_observations : P.out.observations;
    float* gb = pending ? P.out.final_global_state : P.out.global_state;
    // the policy feed always holds the current observation: K3 writes it for
    // the lanes it resets
    __nv_bfloat16* o16 = (F16 && !pending) ? (__nv_bfloat16*)P.out.observations_bf16 : nullptr;
    if (!ob && !gb && !o16) continue;
    load_view<W>(X, st, b, P.N, P.Z, C, DC, lane);
    emit_lane<W, F16>(X, ob, gb, b, P.N, P.Z, P.D, P.G, R, SF, C, DC, lane, buf, false, o16,
                      (int)P.out.observations_bf16_ld);
  }
  if (lane == 0) bulk_wait_all();
}

template <int W, int EPW, bool F16>
cudaError_t launch_emit_f(const Params& P, int sm_count, cudaStream_t stream) {
  const int R = emit_rows(P.N, P.D, W == 1 ? TABX_EMIT_BUDGET : 8192);
  const int SF = emit_stage_floats(P.N, P.D, P.G, R);
  const size_t smem = (size_t)EPW * emit_warp_bytes<W>(P.N, P.Z, R, SF);
  int per_sm = 1;
  cudaError_t e = launch_geometry((const void*)emit_kernel<W, EPW, F16>, 32 * EPW, smem, &per_sm);
  if (e != cudaSuccess) return e;
  int64_t need = (P.B + EPW - 1) / EPW;
  int64_t cap = (int64_t)sm_count * per_sm;
  int grid = (int)(need < cap ? need : cap);
  if (grid < 1) grid = 1;
  emit_kernel<W, EPW, F16><<<grid, 32 * EPW, smem, stream>>>(P, R, SF);
  return cudaGetLastError();
}

// The bfloat16 policy feed is its own instantiation: the plain observation
// stream carries none of its code.
// Instantiations with the unit / zone counts (and so the row geometry) fixed
// at compile time, for the common shapes: constant trip counts and offsets,
// fewer live registers (no spills).  Same body as emit_kernel.
// Per-shape tuning of the fixed-shape emitter (W = 1): resident CTAs per SM
// the register budget is cut for, and whether the next env's view inputs are
// fetched into registers before this env's rows stream out (VPF).  Measured
// (B200, tools/kab.sh): C3 (20, 6) at 262,144 envs 1.655 ms (6 CTAs, no VPF)
// -> 1.466 ms (4 CTAs = 16 warps at 113 registers, VPF; 5 CTAs without VPF
// 1.541); C2 (20, 0) at 65,536 envs 0.363 -> 0.345 ms with 5 CTAs and no VPF
// (VPF at 4 CTAs: 0.362).  At 6 CTAs (80 registers, 24 warps) the view loads
// at each env's start were a quarter of the emitter's stall samples and
// 219 KB of shared memory left little L1 for the config rows they read.
// With the bf16 policy feed (the C5 rollout at 16,384 envs) the original
// 6 CTAs without VPF stay faster (C5 43.2 vs 42.4 M env-steps/s).
template <int NF, int ZF, bool F16>
struct EmitTune {
  // resident warps per SM (the register budget follows from it)
  static constexpr int warps = F16 ? 24 : (NF == 20 && ZF == 6) ? 16 : (NF == 20 && ZF == 0) ? 20 : 24;
  static constexpr bool vpf = !F16 && NF == 20 && ZF == 6;
};

template <int W, int EPW, bool F16, int NF, int ZF>
__global__ void __launch_bounds__(32 * EPW,
                                  (W == 1 ? (TABX_EMIT_MIN_BLOCKS_W1 > 0
                                                 ? TABX_EMIT_MIN_BLOCKS_W1
                                                 : (EmitTune<NF, ZF, F16>::warps / EPW > 0
                                                        ? EmitTune<NF, ZF, F16>::warps / EPW
                                                        : 1))
                                          : TABX_EMIT_MIN_BLOCKS))
    emit_kernel_fixed(const Params P) {
  constexpr int N = NF, Z = ZF;
  constexpr int D = TABX_OWN_DIM + TABX_OTHER_DIM * (NF - 1) + TABX_ZONE_DIM * ZF;
  constexpr int G = TABX_OWN_DIM * NF + TABX_ZONE_DIM * ZF;
  constexpr int R = emit_rows(N, D, W == 1 ? TABX_EMIT_BUDGET : 8192);
  constexpr int SF = emit_stage_floats(N, D, G, R);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (is_step_mode(P.mode) && P.sync->err_index != NO_ERROR) return;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const EmitScratch<W> X =
      emit_scratch<W>(smem_raw + (size_t)w * emit_warp_bytes<W>(N, Z, R, SF), N, Z, R);
  const DevState& st = P.st;
  int buf = 0;
  const int64_t stride = (int64_t)gridDim.x * EPW;
  int64_t b = (int64_t)blockIdx.x * EPW + w;
  // the env's config index and flags are loaded one env ahead, and its
  // per-unit state is pulled into L2 one env ahead, so a warp's view load
  // does not start with a dependent chain of DRAM round trips
  int32_t k_next = b < P.B ? st.cfg[b] : 0;
  uint8_t f_next = b < P.B ? st.flags[b] : 0;
  // (W = 1, TABX_EMIT_VIEW_PREFETCH) the next env's view inputs are loaded
  // into registers before this env's rows stream out
  constexpr bool VPF =
      W == 1 && (TABX_EMIT_VIEW_PREFETCH < 0 ? EmitTune<NF, ZF, F16>::vpf : TABX_EMIT_VIEW_PREFETCH != 0);
  ViewRegs V_next;
  if (VPF && b < P.B) fetch_view_regs(V_next, st, b, N, lane);
  for (; b < P.B; b += stride) {
    const int32_t k = k_next;
    const uint8_t fl = f_next;
    ViewRegs V = V_next;
    if (b + stride < P.B) {
      k_next = st.cfg[b + stride];
      f_next = st.flags[b + stride];
      if (VPF) fetch_view_regs(V_next, st, b + stride, N, lane);
    }
    const tabx_config* C = P.cfgs + k;
    const DerivedCfg* DC = P.dcfgs + k;
    const bool pending = (fl & F_PEND) != 0;
    float* ob = pending ? P.out.final_observations : P.out.observations;
    float* gb = pending ? P.out.final_global_state : P.out.global_state;
    __nv_bfloat16* o16 = (F16 && !pending) ? (__nv_bfloat16*)P.out.observations_bf16 : nullptr;
    if (!ob && !gb && !o16) continue;
    if constexpr (VPF)
      load_view_regs(X, V, N, C, DC, lane);
    else
      load_view<W>(X, st, b, N, Z, C, DC, lane);
    emit_lane<W, F16>(X, ob, gb, b, N, Z, D, G, R, SF, C, DC, lane, buf, false, o16,
                      (int)P.out.observations_bf16_ld);
  }
  if (lane == 0) bulk_wait_all();
}

template <int W, int EPW, bool F16, int NF, int ZF>
cudaError_t launch_emit_fixed(const Params& P, int sm_count, cudaStream_t stream) {
  constexpr int D = TABX_OWN_DIM + TABX_OTHER_DIM * (NF - 1) + TABX_ZONE_DIM * ZF;
  constexpr int G = TABX_OWN_DIM * NF + TABX_ZONE_DIM * ZF;
  constexpr int R = emit_rows(NF, D, W == 1 ? TABX_EMIT_BUDGET : 8192);
  constexpr int SF = emit_stage_floats(NF, D, G, R);
  const size_t smem = (size_t)EPW * emit_warp_bytes<W>(NF, ZF, R, SF);
  int per_sm = 1;
  cudaError_t e = launch_geometry((const void*)emit_kernel_fixed<W, EPW, F16, NF, ZF>, 32 * EPW,
                                  smem, &per_sm);
  if (e != cudaSuccess) return e;
  int64_t need = (P.B + EPW - 1) / EPW;
  int64_t cap = (int64_t)sm_count * per_sm;
  int grid = (int)(need < cap ? need : cap);
  if (grid < 1) grid = 1;
  emit_kernel_fixed<W, EPW, F16, NF, ZF><<<grid, 32 * EPW, smem, stream>>>(P);
  return cudaGetLastError();
}

template <int W, int EPW, bool F16>
cudaError_t launch_emit_shape(const Params& P, int sm_count, cudaStream_t stream) {
  // the C3 / C2 / C1 / C4 shapes (as the step kernel); any other: generic
  if (P.generic_shapes) return launch_emit_f<W, EPW, F16>(P, sm_count, stream);
  if constexpr (W == 1) {
    if (P.N == 20 && P.Z == 6) return launch_emit_fixed<1, EPW, F16, 20, 6>(P, sm_count, stream);
    if (P.N == 20 && P.Z == 0) return launch_emit_fixed<1, EPW, F16, 20, 0>(P, sm_count, stream);
    if (P.N == 6 && P.Z == 0) return launch_emit_fixed<1, EPW, F16, 6, 0>(P, sm_count, stream);
  }
  if constexpr (W == 4) {
    if (P.N == 100 && P.Z == 0)
      return launch_emit_fixed<4, EPW, F16, 100, 0>(P, sm_count, stream);
  }
  return launch_emit_f<W, EPW, F16>(P, sm_count, stream);
}

// W > 1: one environment per CTA of WPE warps.  The CTA loads the env's
// view once into shared memory (N units over 32 WPE threads) and the warps
// split its row chunks (warp w: chunks w, w + WPE, ...; warp 0 also the
// global-state row), each through its own double-buffered TMA stage.  The
// one-warp-per-env emitter holds a whole view (13 KB at N = 100) plus two
// 6.8 KB stages per warp, which capped it at 8 warps/SM; sharing the view
// fits 12.
template <int W, int WPE, bool F16, int NF, int ZF>
__global__ void __launch_bounds__(32 * WPE) emit_kernel_cta(const Params P, int R, int SF) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (is_step_mode(P.mode) && P.sync->err_index != NO_ERROR) return;
  const int N = NF ? NF : P.N, Z = NF ? ZF : P.Z;
  const int D = NF ? TABX_OWN_DIM + TABX_OTHER_DIM * (NF - 1) + TABX_ZONE_DIM * ZF : P.D;
  const int G = NF ? TABX_OWN_DIM * NF + TABX_ZONE_DIM * ZF : P.G;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const size_t vb = emit_view_bytes<W>(N);
  EmitScratch<W> X = emit_scratch<W>(smem_raw, N, Z, R);
  X.stage = reinterpret_cast<float*>(smem_raw + vb) + (size_t)w * TABX_EMIT_NBUF * SF;
  const EmitEnv<W>& E = X.E;
  const DevState& st = P.st;
  int buf = 0;
  for (int64_t b = blockIdx.x; b < P.B; b += gridDim.x) {
    const int32_t k = st.cfg[b];
    const tabx_config* C = P.cfgs + k;
    const DerivedCfg* DC = P.dcfgs + k;
    const bool pending = (st.flags[b] & F_PEND) != 0;
    float* ob = pending ? P.out.final_observations : P.out.observations;
    float* gb = pending ? P.out.final_global_state : P.out.global_state;
    __nv_bfloat16* o16 = (F16 && !pending) ? (__nv_bfloat16*)P.out.observations_bf16 : nullptr;
    if (!ob && !gb && !o16) continue;  // CTA-uniform
    __syncthreads();  // every warp is done with the previous env's view
    TABX_POISON(X.E.px, vb, tid, 32 * WPE);
    __syncthreads();
    for (int u = tid; u < N; u += 32 * WPE) {
      const int64_t gu = b * N + u;
      const double2 p = st.pos[gu];
      E.px[u] = p.x;
      E.py[u] = p.y;
      own_from_state(E.own[u], st, gu, C, DC, u);
      E.flags[u] = (C->active[u] ? 1u : 0u) | (C->team[u] ? 2u : 0u);
#pragma unroll
      for (int kk = 0; kk < W; ++kk) {
        E.vis[u * W + kk] = st.vis[gu * W + kk];
        E.atk[u * W + kk] = st.atk[gu * W + kk];
      }
    }
    __syncthreads();
    emit_lane<W, F16>(X, ob, w == 0 ? gb : nullptr, b, N, Z, D, G, R, SF, C, DC, lane, buf, false,
                      o16, (int)P.out.observations_bf16_ld, w, WPE);
  }
  if (lane == 0) bulk_wait_all();
}

// W > 1: warps per environment of the observation kernel (0: the one-warp
// emitter).  Measured (tools/wprobe.py, kab): W = 2 (40 units) 1.96 -> 1.62 ms
// with 2 (4: 2.03); W = 4 (C4, 100 units) neutral with 4, +0.7% with 2: kept
// at one; W = 8 (150 units) 6.91 -> 5.97 ms with 2, 4.88 ms with 4.
#ifndef TABX_EMIT_WPE_W2
#define TABX_EMIT_WPE_W2 2
#endif
#ifndef TABX_EMIT_WPE_W4
#define TABX_EMIT_WPE_W4 0
#endif
#ifndef TABX_EMIT_WPE_W8
#define TABX_EMIT_WPE_W8 4
#endif
template <int W>
constexpr int emit_wpe() {
  return W == 2 ? TABX_EMIT_WPE_W2 : W == 4 ? TABX_EMIT_WPE_W4 : W == 8 ? TABX_EMIT_WPE_W8 : 0;
}

template <int W, bool F16, int NF, int ZF>
cudaError_t launch_emit_cta(const Params& P, int sm_count, cudaStream_t stream) {
  constexpr int WPE = emit_wpe<W>() > 0 ? emit_wpe<W>() : 1;
  const int R = emit_rows(P.N, P.D, 8192);
  const int SF = emit_stage_floats(P.N, P.D, P.G, R);
  const size_t smem = emit_view_bytes<W>(P.N) + (size_t)WPE * TABX_EMIT_NBUF * SF * sizeof(float);
  int per_sm = 0;
  auto kern = emit_kernel_cta<W, WPE, F16, NF, ZF>;
  cudaError_t e = launch_geometry((const void*)kern, 32 * WPE, smem, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorNotSupported;
  const int64_t cap = (int64_t)sm_count * per_sm;
  int grid = (int)(P.B < cap ? P.B : cap);
  if (grid < 1) grid = 1;
  kern<<<grid, 32 * WPE, smem, stream>>>(P, R, SF);
  return cudaGetLastError();
}

template <int W, int EPW>
cudaError_t launch_emit_t(const Params& P, int sm_count, cudaStream_t stream) {
  if constexpr (W > 1 && emit_wpe<W>() > 0) {
    if constexpr (W == 4) {
      if (!P.generic_shapes && P.N == 100 && P.Z == 0)
        return P.out.observations_bf16 ? launch_emit_cta<4, true, 100, 0>(P, sm_count, stream)
                                       : launch_emit_cta<4, false, 100, 0>(P, sm_count, stream);
    }
    return P.out.observations_bf16 ? launch_emit_cta<W, true, 0, 0>(P, sm_count, stream)
                                   : launch_emit_cta<W, false, 0, 0>(P, sm_count, stream);
  }
  return P.out.observations_bf16 ? launch_emit_shape<W, EPW, true>(P, sm_count, stream)
                                 : launch_emit_shape<W, EPW, false>(P, sm_count, stream);
}

}  // namespace tabx
