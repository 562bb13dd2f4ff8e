// The batched environment step on sm_100a.
//
// One environment per "env group" of NT = 32*W threads, thread i = unit i
// (N <= NT).  W = 1 (N <= 32) packs EPB environments per CTA, one per warp,
// synchronised with __syncwarp only; W > 1 runs one environment per CTA.
// A persistent grid-stride loop walks the lanes.  Unit state lives in
// registers, the cross-unit views (positions, headings, flags, cache rows)
// in shared memory; the O(N^2) pair passes are row-owned (thread i scans
// j = 0..N-1) with the visibility / attackable rows built as N-bit masks.
// Order-dependent reductions (Gauss-Seidel contacts, numpy's pairwise team
// sums) run on one thread over shared memory, exactly in reference order.
// The observation block of each environment is generated column-by-column
// from shared memory and streamed out with 16-byte stores.
//
// Every stage cites the reference line it restates; arithmetic is float64,
// compiled with -fmad=false so no product is fused that numpy rounds.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "tabx_device.cuh"
#include "tabx_emit.cuh"
#include "tabx_math.cuh"

namespace tabx {

// ------------------------------------------------------------------ rng --
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// rng.py:31-37
__device__ __forceinline__ uint64_t key_hash(uint64_t seed, uint64_t step, uint64_t tag,
                                             uint64_t lane) {
  uint64_t h = mix64(seed + 0x9E3779B97F4A7C15ull * tag);
  h = mix64(h + step * 0xC2B2AE3D27D4EB4Full);
  return mix64(h + lane * 0x165667B19E3779F9ull);
}

// rng.py:40-43
__device__ __forceinline__ double uniform53(uint64_t seed, uint64_t step, uint64_t tag,
                                            uint64_t lane) {
  return (double)(key_hash(seed, step, tag, lane) >> 11) * (1.0 / 9007199254740992.0);
}

// ------------------------------------------------- phase instrumentation --
// Built only with -DTABX_PHASE_PROF (tools): lane 0 of each env accumulates
// SM clock cycles per step phase into tabx_phase_cycles (read back with
// tabx_debug_phase_cycles).  The default build compiles the marks to nothing.
#if defined(TABX_PHASE_PROF) && !defined(TABX_COUNT_PROF)
#define TABX_PHASE_BEGIN() long long ph_t0_ = clock64()
#define TABX_PHASE(k)                                                  \
  do {                                                                 \
    const long long ph_t1_ = clock64();                                \
    if ((threadIdx.x & 31) == 0)                                       \
      atomicAdd(&tabx_phase_cycles[k], (unsigned long long)(ph_t1_ - ph_t0_)); \
    ph_t0_ = ph_t1_;                                                   \
  } while (0)
// divergent regions: the lowest active lane reports
#define TABX_PHASE_DIV(k)                                              \
  do {                                                                 \
    const long long ph_t1_ = clock64();                                \
    if ((threadIdx.x & 31) == __ffs(__activemask()) - 1)               \
      atomicAdd(&tabx_phase_cycles[k], (unsigned long long)(ph_t1_ - ph_t0_)); \
    ph_t0_ = ph_t1_;                                                   \
  } while (0)
#else
#define TABX_PHASE_DIV(k) TABX_JITTER(100 + (k))
#define TABX_PHASE_BEGIN() \
  do {                     \
  } while (0)
#define TABX_PHASE(k) TABX_JITTER(k)
#endif


// W > 1: cull the O(N^2) contact and visibility pair passes with a sort of
// the units along y and a sweep over the |dy| window:
// a pair with |dy| beyond the window cannot touch / be in sight, since the
// reference's float64 distance is never below |dy|
#ifndef TABX_SWEEP
#define TABX_SWEEP 1
#endif

#ifndef TABX_VIS_UNROLL
#define TABX_VIS_UNROLL 4
#endif
constexpr int kVisUnroll = TABX_VIS_UNROLL;  // unroll of the visibility filter loop

// ------------------------------------------------------------- helpers --
constexpr uint32_t UF_ACTIVE = 1, UF_ALIVE = 2, UF_ENEMY = 4, UF_KIN = 8, UF_INJURED = 16;

template <int W>
struct EnvSmem {
  static constexpr int NT = 32 * W;
  double px[NT], py[NT], ch[NT], sh[NT], rad[NT], mh[NT], rv[NT], dmg[NT];
  double vx[NT], vy[NT], sx[NT], sy[NT];
  uint32_t vis[NT * W], atk[NT * W], touch[NT * W];
  // W > 1 sort-and-sweep culling: float32 y keys (+inf for inactive units),
  // the units in ascending key order and each unit's rank in it
  float ykey[NT], skey[NT];  // skey[r] = key of the unit of rank r
  int16_t ord[NT], rnk[NT];
  unsigned long long rk_key[NT];  // per-warp sorted runs of (key bits, index) (rank_by_y)
  uint32_t dymax;  // float bits: largest |y| move since the keys were taken
  uint32_t uf[NT];
  uint32_t zin[NT];
  int32_t tgt[NT];
  uint32_t ball[8][W];  // env_ballot slots, one per call site (one barrier each)
  // env-wide unit sets as N-bit masks (word k = units 32k..32k+31)
  uint32_t m_active[W], m_alive[W], m_enemy[W], m_rev[W], m_inbush[W];
  uint32_t m_zone[TABX_MAX_ZONES][W];
  double red[2];
  double part[16];
  // W == 1: unordered pairs (i<j) in row-major order, (i << 8) | j, and the
  // touching-pair bit masks of one step (32 pairs per word, same order)
  uint16_t ptab[W == 1 ? 496 : 1];
  uint32_t tmask[W == 1 ? 16 : 1];
};

template <int W>
__device__ __forceinline__ void env_sync() {
  if (W == 1) {
    __syncwarp();
  } else {
    __syncthreads();
  }
}

// Env-wide ballot: word k holds predicates of units 32k..32k+31.  W > 1:
// every call site has its own slot SL of S.ball, written once per step, so a
// ballot costs one barrier (a slot is rewritten only in the next step, after
// that step's opening barrier).
template <int W, int SL>
__device__ __forceinline__ void env_ballot(bool p, EnvSmem<W>& S, int i, uint32_t (&m)[W]) {
  static_assert(SL >= 0 && SL < 8, "ballot slot");
  uint32_t b = __ballot_sync(0xffffffffu, p);
  if (W == 1) {
    m[0] = b;
  } else {
    if ((i & 31) == 0) S.ball[SL][i >> 5] = b;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < W; ++k) m[k] = S.ball[SL][k];
  }
}

// Two predicates through slots SL and SL + 1 with one barrier.
template <int W, int SL>
__device__ __forceinline__ void env_ballot2(bool p0, bool p1, EnvSmem<W>& S, int i,
                                            uint32_t (&m0)[W], uint32_t (&m1)[W]) {
  static_assert(SL >= 0 && SL + 1 < 8, "ballot slot");
  const uint32_t b0 = __ballot_sync(0xffffffffu, p0), b1 = __ballot_sync(0xffffffffu, p1);
  if (W == 1) {
    m0[0] = b0;
    m1[0] = b1;
  } else {
    if ((i & 31) == 0) {
      S.ball[SL][i >> 5] = b0;
      S.ball[SL + 1][i >> 5] = b1;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < W; ++k) {
      m0[k] = S.ball[SL][k];
      m1[k] = S.ball[SL + 1][k];
    }
  }
}

template <int W, int SL>
__device__ __forceinline__ bool env_any(bool p, EnvSmem<W>& S, int i) {
  uint32_t m[W];
  env_ballot<W, SL>(p, S, i, m);
  uint32_t a = 0;
#pragma unroll
  for (int k = 0; k < W; ++k) a |= m[k];
  return a != 0;
}

// Rank of every unit by its published y key (ties by index), all threads:
// S.ord[rank] = unit, S.rnk[unit] = rank, S.skey[rank] = key.  Each warp
// sorts its 32 (key, index) pairs with a shuffle bitonic network, then every
// element's rank is its place in its run plus the number of smaller
// elements in each other warp's run (binary searches); one barrier.
template <int W>
__device__ __forceinline__ void rank_by_y(EnvSmem<W>& S, int i, int N) {
  const uint32_t full = 0xffffffffu;
  const int lane = i & 31, w = i >> 5;
  const float f = S.ykey[i];  // +inf for inactive units and threads past N
  // one 64-bit key, unique per unit: the float's order-preserving bits, then
  // the index (ties by index)
  const uint32_t fb = __float_as_uint(f);
  const uint32_t ob = (fb & 0x80000000u) ? ~fb : (fb | 0x80000000u);
  unsigned long long key = ((unsigned long long)ob << 32) | (unsigned)i;
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(full, key, stride);
      const bool up = (lane & size) == 0;
      const bool lower = (lane & stride) == 0;
      // the lower position keeps the smaller key in an ascending block
      if ((ok < key) == (lower == up)) key = ok;
    }
  }
  S.rk_key[i] = key;
  env_sync<W>();
  int r = lane;
#pragma unroll
  for (int w2 = 0; w2 < W; ++w2) {
    if (w2 == w) continue;
    const unsigned long long* rk = S.rk_key + w2 * 32;
    int lo = 0, hi = 32;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (rk[mid] < key) lo = mid + 1; else hi = mid;
    }
    r += lo;
  }
#ifdef TABX_SELFTEST_RACE
  // negative control: half the threads publish their ranks 20 us late
  if ((threadIdx.x * 0x9E3779B9u) >> 31) __nanosleep(20000);
#endif
  const int id = (int)(key & 0xffffffffu);
  if (id < N) {
    S.ord[r] = (int16_t)id;
    S.rnk[id] = (int16_t)r;
    S.skey[r] = S.ykey[id];
  }
}

// First rank in [0, N) whose sorted key is >= v (N if none).
template <int W>
__device__ __forceinline__ int lower_rank(const EnvSmem<W>& S, int N, float v) {
  int lo = 0, hi = N;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (S.skey[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
// First rank in [0, N) whose sorted key is > v (N if none).
template <int W>
__device__ __forceinline__ int upper_rank(const EnvSmem<W>& S, int N, float v) {
  int lo = 0, hi = N;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (S.skey[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Upper bound of |dy| - (key_j - key_i) for keys within `win` of key_i:
// the keys are float32 roundings of float64 ys (relative error 2^-24 each)
// and their difference rounds once more; 2^-21 leaves an 8x margin.
__device__ __forceinline__ float sweep_limit(float yi, double win) {
  const float w = (float)win;
  return w + (2.0f * fabsf(yi) + 2.0f * w) * 0x1p-21f + 1e-30f;
}

// Env-wide unit masks from the per-unit state just published (all threads).
template <int W>
__device__ __forceinline__ void build_masks(EnvSmem<W>& S, int i, bool valid, bool active,
                                            bool alive, bool enemy, double rv, uint32_t zin,
                                            int Z, uint32_t bush_m) {
  // word k of every mask is warp k's ballot: each warp writes its own words
  // (no cross-warp exchange here; the caller's barrier publishes them)
  const uint32_t full = 0xffffffffu;
  const uint32_t ma = __ballot_sync(full, valid && active);
  const uint32_t ml = __ballot_sync(full, valid && alive);
  const uint32_t me = __ballot_sync(full, valid && enemy);
  const uint32_t mr = __ballot_sync(full, valid && rv > 0.0);
  uint32_t inb = 0u;
  for (int z = 0; z < Z; ++z) {
    const uint32_t mz = __ballot_sync(full, valid && ((zin >> z) & 1u));
    if ((i & 31) == 0) S.m_zone[z][i >> 5] = mz;
    if ((bush_m >> z) & 1u) inb |= mz;
  }
  if ((i & 31) == 0) {
    S.m_active[i >> 5] = ma;
    S.m_alive[i >> 5] = ml;
    S.m_enemy[i >> 5] = me;
    S.m_rev[i >> 5] = mr;
    S.m_inbush[i >> 5] = inb;
  }
}

__device__ __forceinline__ bool bit_of(const uint32_t* row, int j) {
  return (row[j >> 5] >> (j & 31)) & 1u;
}

// float32(fl64(x / y)) without the float64 division: q = x * fl(1/y) is
// within 3 ulp of fl64(x / y), so both round to the same float32 unless q
// sits within a few ulp of a float32 rounding midpoint (low 29 mantissa bits
// near 0x10000000) -- then, and for float32-subnormal magnitudes, divide.
// Only the swamps the unit stands in contribute (the reference multiplies the
// others' 1.0, which is exact), in ascending zone order.
__device__ __forceinline__ double swamp_mult(const tabx_config* __restrict__ C, int Z,
                                             uint32_t zin, uint32_t swamp_m) {
  double m = 1.0;
  for (uint32_t hit = zin & swamp_m; hit; hit &= hit - 1) m = m * C->zone_effect[__ffs(hit) - 1];
  return m;
}

// lava burn rate: numpy last-axis sum over Z (environment.py:273)
__device__ __forceinline__ double lava_sum(const tabx_config* __restrict__ C, int Z, uint32_t zin,
                                           uint32_t lava_m) {
  uint32_t hit = zin & lava_m;
  if (Z < 8) {  // sequential from 0.0; the 0.0 terms of other zones are exact no-ops
    double r = 0.0;
    for (; hit; hit &= hit - 1) r += C->zone_effect[__ffs(hit) - 1];
    return r;
  }
  double v[TABX_MAX_ZONES];
  for (int z = 0; z < Z; ++z) v[z] = ((hit >> z) & 1u) ? C->zone_effect[z] : 0.0;
  return pairwise_sum(v, Z);
}

// Index of the floor(u*n)-th legal action (environment.py:198-201).
__device__ __forceinline__ int kth_legal(uint32_t mask7, double u) {
  const int n = __popc(mask7);
  long long kk = (long long)(u * (double)n);
  if (kk > n - 1) kk = n - 1;
  // position of the kk-th set bit of the 7-bit mask, by popc halving
  int k = (int)kk, pos = 0;
  uint32_t w = mask7;
  int c = __popc(w & 0xFu);
  if (k >= c) { k -= c; w >>= 4; pos += 4; }
  c = __popc(w & 0x3u);
  if (k >= c) { k -= c; w >>= 2; pos += 2; }
  if (k >= (int)(w & 1u)) pos += 1;
  return pos;
}

// Move choice: argmin / argmax of squared distance over the 4 axis moves
// (heuristics.py:75-84); ties go to the lowest action id.
__device__ __forceinline__ int best_move(double px, double py, double gx, double gy, double step,
                                         bool away) {
  const double dxs[4] = {0.0, 0.0, 1.0, -1.0};
  const double dys[4] = {1.0, -1.0, 0.0, 0.0};
  int best = 0;
  double bv = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    double cx = px + dxs[k] * step;
    double cy = py + dys[k] * step;
    double ex = cx - gx, ey = cy - gy;
    double v = ex * ex + ey * ey;
    if (k == 0 || (away ? (v > bv) : (v < bv))) {
      bv = v;
      best = k;
    }
  }
  return best;
}

struct UnitStatic {
  double rad, mh, mass, inv_mass, speed, dmg, range, ucd, sangle, cos_half, srange;
  bool active, enemy, kin, assassin, ranger, healer;
};

__device__ __forceinline__ UnitStatic load_static(const tabx_config* __restrict__ C, int i,
                                                  bool valid) {
  UnitStatic u;
  if (valid) {
    u.rad = C->radius[i];
    u.mh = C->max_health[i];
    u.mass = C->mass[i];
    u.inv_mass = C->inv_mass[i];
    u.speed = C->speed[i];
    u.dmg = C->damage[i];
    u.range = C->attack_range[i];
    u.ucd = C->cooldown[i];
    u.sangle = C->sight_angle[i];
    u.cos_half = C->sight_cos_half[i];
    u.srange = C->sight_range[i];
    u.active = C->active[i] != 0;
    u.enemy = C->team[i] != 0;
    u.kin = C->kinematic[i] != 0;
    u.assassin = C->role_assassin[i] != 0;
    u.ranger = C->role_ranger[i] != 0;
    u.healer = C->role_healer[i] != 0;
  } else {
    u.rad = 0.0;
    u.mh = 1.0;
    u.mass = 1.0;
    u.inv_mass = 1.0;
    u.speed = u.dmg = u.range = u.ucd = u.sangle = u.srange = 0.0;
    u.cos_half = 1.0;
    u.active = u.enemy = u.kin = u.assassin = u.ranger = u.healer = false;
  }
  return u;
}

// MUFU reciprocal square root (rel. error < 2^-22.9, subnormals flushed): the
// float32 wedge filter only needs it far inside its 2e-5 margin, and a
// flushed tiny distance is already routed to the exact test (d2 > 1e-30).
__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// sqrt(a2) < sqrt(b2) for the correctly rounded float64 sqrt, deciding on
// the squares unless they are within 1e-14 (where the roots may round equal).
__device__ __forceinline__ bool closer(double a2, double b2) {
  if (!(a2 < b2)) return false;
  if (a2 < b2 * (1.0 - 1e-14)) return true;
  TABX_COUNT(8);
  return slow_sqrt(a2) < slow_sqrt(b2);
}

struct Seen {
  double dist;
  bool seen;
};

// Reference float64 verdict of the view wedge + range test (perception.py:52-66).
static __device__ __noinline__ Seen exact_seen(double dx, double dy, double ch, double sh, double srange,
                                        double cos_half) {
  Seen r;
  r.dist = sqrt(dx * dx + dy * dy);
  const double lx = dx * ch + dy * sh;
  const double cdev = r.dist > 0.0 ? lx / r.dist : 1.0;
  r.seen = r.dist <= srange && cdev >= cos_half;
  return r;
}

// Reference float64 strike-box test (combat.py:30-40).
static __device__ __noinline__ bool exact_box(double dx, double dy, double ch, double sh, double reach,
                                       double rad, double rj) {
  const double lx = dx * ch + dy * sh;
  const double ly = (-dx) * sh + dy * ch;
  const double gx = lx - np_clip(lx, 0.0, reach);
  const double gy = ly - np_clip(ly, -rad, rad);
  return gx * gx + gy * gy <= rj * rj;
}

// Visibility / attackable rows of observer i and its nearest attackable
// target (perception.py:52-96, combat.py:16-83).  Writes the two N-bit rows
// to S.vis / S.atk and returns the target or -1.
//
// Pass 1 (branch-free over all j): classify each pair in float32 -- sight
// range against sight_range^2, view wedge via rsqrt -- with margins two orders
// of magnitude above the float32 error bound, into "surely seen" and "unsure"
// bit masks.  Pass 2 evaluates the rare unsure pairs with the reference's
// float64 expressions.  Bush concealment is then pure mask algebra over the
// env-wide masks, and the strike box + exact distance (which orders the
// target) run only over the few attackable candidates.  Verdicts are exactly
// the float64 ones.
template <int W, bool SWEEP = false>
__device__ __forceinline__ int cache_row_body(EnvSmem<W>& S, int i, int N, double cos_half,
                                              double srange, double dmg, double reach, double rad,
                                              uint32_t bush_m) {
  uint32_t vis[W], atk[W];
#pragma unroll
  for (int k = 0; k < W; ++k) vis[k] = atk[k] = 0u;
  int tgt = -1;
  const uint32_t uf_i = S.uf[i];
  if (uf_i & UF_ACTIVE) {  // vis requires both active; atk requires vis
    TABX_COUNT(9);
    const double px = S.px[i], py = S.py[i], ch = S.ch[i], sh = S.sh[i];
    const float chf = (float)ch, shf = (float)sh;
    const float sr2 = (float)(srange * srange);
    const float sr2_lo = sr2 * 0.99999f, sr2_hi = sr2 * 1.00001f;
    const float cf = (float)cos_half;
    const float cf_lo = cf - 2e-5f, cf_hi = cf + 2e-5f;
    uint32_t seen[W], unsure[W];
#pragma unroll
    for (int k = 0; k < W; ++k) seen[k] = unsure[k] = 0u;
    // SWEEP (W > 1, ranks of this stage's positions in S): only the units
    // whose y key lies within the sight range of this one's, a contiguous
    // run of the y order around its rank; every other unit has |dy| >
    // srange and so dist > srange (not seen)
    int q0 = 0, q1 = N;
    if constexpr (SWEEP) {
      // keys and order of the contact pass; every unit moved by at most dymax
      const float yi = S.ykey[i];
      const float lim = sweep_limit(yi, srange + 2.0 * (double)__uint_as_float(S.dymax));
      // keys k with |k - yi| <= lim: ranks [q0, q1) (binary searches; the
      // float bounds yi -+ lim round outward by at most an ulp, covered by
      // lim's margin)
      q0 = lower_rank<W>(S, N, yi - lim);
      q1 = upper_rank<W>(S, N, yi + lim);
    }
#pragma unroll (kVisUnroll)
    for (int q = q0; q < q1; ++q) {
      const int j = SWEEP ? (int)S.ord[q] : q;
      const float dxf = (float)(S.px[j] - px), dyf = (float)(S.py[j] - py);
      const float d2f = dxf * dxf + dyf * dyf;
      const float cdevf = (dxf * chf + dyf * shf) * rsqrt_approx(d2f);
      const bool inr = (d2f <= sr2_lo) & (d2f > 1e-30f);
      const bool outr = (d2f >= sr2_hi) & (d2f > 0.0f);
      const bool wt = cdevf >= cf_hi, wf = cdevf <= cf_lo;
      seen[j >> 5] |= (uint32_t)(inr & wt) << (j & 31);
      unsure[j >> 5] |= (uint32_t)(!outr & !(inr & (wt | wf))) << (j & 31);
    }
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const uint32_t keep = S.m_active[k] & ~(k == (i >> 5) ? 1u << (i & 31) : 0u);
      seen[k] &= keep;
      unsure[k] &= keep;
    }
#pragma unroll
    for (int k = 0; k < W; ++k) {
      uint32_t m = unsure[k];
      while (m) {
        const int j = (k << 5) + __ffs(m) - 1;
        m &= m - 1;
        TABX_COUNT(0);
        const Seen e = exact_seen(S.px[j] - px, S.py[j] - py, ch, sh, srange, cos_half);
        if (e.seen) seen[k] |= 1u << (j & 31);
      }
    }
    // concealment: j in a bush, on the other team, not sharing a bush with i,
    // reveal timer run out (perception.py:86-96)
    const bool enemy_i = (uf_i & UF_ENEMY) != 0;
    const uint32_t bush_i = S.zin[i] & bush_m;
    uint32_t shared[W];
#pragma unroll
    for (int k = 0; k < W; ++k) shared[k] = 0u;
    for (uint32_t zb = bush_i; zb; zb &= zb - 1) {
      const int z = __ffs(zb) - 1;
#pragma unroll
      for (int k = 0; k < W; ++k) shared[k] |= S.m_zone[z][k];
    }
    const bool can_hit = (uf_i & UF_ALIVE) && dmg != 0.0;
    uint32_t cand[W];
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const uint32_t foe = enemy_i ? ~S.m_enemy[k] : S.m_enemy[k];
      const uint32_t hidden = S.m_inbush[k] & foe & ~shared[k] & ~S.m_rev[k];
      vis[k] = seen[k] & ~hidden;
      const uint32_t role = dmg > 0.0 ? foe : ~foe;
      cand[k] = can_hit ? (vis[k] & role & S.m_alive[k]) : 0u;
    }
    vis[i >> 5] |= 1u << (i & 31);  // distance 0, cos_dev 1: sees itself
    const float reachf = (float)reach, radf = (float)rad;
    double best = 0.0;  // squared distance of the target so far
#pragma unroll
    for (int k = 0; k < W; ++k) {
      uint32_t m = cand[k];
      while (m) {
        const int j = (k << 5) + __ffs(m) - 1;
        m &= m - 1;
        const double dx = S.px[j] - px;
        const double dy = S.py[j] - py;
        const double rj = S.rad[j];
        const float dxf = (float)dx, dyf = (float)dy, rjf = (float)rj;
        const float lxf = dxf * chf + dyf * shf;
        const float lyf = (-dxf) * shf + dyf * chf;
        const float gxf = lxf - fminf(fmaxf(lxf, 0.0f), reachf);
        const float gyf = lyf - fminf(fmaxf(lyf, -radf), radf);
        const float gapf = gxf * gxf + gyf * gyf;
        const float rj2f = rjf * rjf;
        const float L = fabsf(lxf) + fabsf(lyf) + reachf + radf + rjf;
        const float mb = 3e-5f * L * L;
        bool box;
        if (gapf < rj2f - mb) {
          box = true;
        } else if (gapf > rj2f + mb) {
          box = false;
        } else {
          TABX_COUNT(1);
          box = exact_box(dx, dy, ch, sh, reach, rad, rj);
        }
        if (!box) continue;
        atk[k] |= 1u << (j & 31);
        TABX_COUNT(5);
        // nearest attackable, first index on ties of the rounded distances
        // (combat.py argmin over sqrt(dx^2 + dy^2)): squares compared, the
        // roots only for near-ties (closer)
        const double d2 = dx * dx + dy * dy;
        if (tgt < 0 || closer(d2, best)) {
          best = d2;
          tgt = j;
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < W; ++k) {
    S.vis[i * W + k] = vis[k];
    S.atk[i * W + k] = atk[k];
  }
  return tgt;
}

template <int W>
__device__ __noinline__ int cache_row_call(EnvSmem<W>& S, int i, int N, double cos_half,
                                           double srange, double dmg, double reach, double rad,
                                           uint32_t bush_m) {
  return cache_row_body<W>(S, i, N, cos_half, srange, dmg, reach, rad, bush_m);
}

// Out-of-line variant for the rare call sites (refresh, init, auto-reset).
template <int W>
__device__ __forceinline__ int cache_row_of(EnvSmem<W>& S, int i, int N, const UnitStatic& U,
                                            uint32_t bush_m) {
  return cache_row_call<W>(S, i, N, U.cos_half, U.srange, U.dmg, U.range, U.rad, bush_m);
}

// Inline variant for the every-step call (stage 8).
template <int W>
__device__ __forceinline__ int cache_row_inl(EnvSmem<W>& S, int i, int N, const UnitStatic& U,
                                             uint32_t bush_m) {
  return cache_row_body<W, (W > 1 && TABX_SWEEP)>(S, i, N, U.cos_half, U.srange, U.dmg, U.range,
                                                   U.rad, bush_m);
}

// Team health ratio sums in numpy pairwise order (arrays.py:390-400); one
// thread, values staged in S.vx (ally) / S.vy (enemy).
template <int W>
__device__ __forceinline__ void team_ratios(EnvSmem<W>& S, int i, int N, bool active, bool enemy,
                                            double hp, double mh, int n_ally, int n_enemy,
                                            double& ra, double& re) {
  S.vx[i] = (active && !enemy) ? hp / mh : 0.0;
  S.vy[i] = (active && enemy) ? hp / mh : 0.0;
  env_sync<W>();
  const double ca = (double)(n_ally > 1 ? n_ally : 1);
  const double ce = (double)(n_enemy > 1 ? n_enemy : 1);
  if (N >= 8 && N <= 128) {
    // numpy's 8-accumulator block (n <= 128): threads 0-7 / 8-15 run the ally /
    // enemy accumulators, threads 0 and 8 combine them in numpy's tree order
    // (W > 1 too: one thread summing 2 x 100 values serially held the other
    // warps at the next barrier)
    const int lim = N - (N % 8);
    if (i < 16) {
      const double* v = i < 8 ? S.vx : S.vy;
      double r = v[i & 7];
      for (int q = 8 + (i & 7); q < lim; q += 8) r += v[q];
      S.part[i] = r;
    }
    env_sync<W>();
    if (i == 0 || i == 8) {
      const double* v = i == 0 ? S.vx : S.vy;
      const double* pp = S.part + i;
      double r = ((pp[0] + pp[1]) + (pp[2] + pp[3])) + ((pp[4] + pp[5]) + (pp[6] + pp[7]));
      for (int q = lim; q < N; ++q) r += v[q];
      S.red[i >> 3] = r / (i == 0 ? ca : ce);
    }
  } else if (i == 0) {
    S.red[0] = pairwise_sum(S.vx, N) / ca;
    S.red[1] = pairwise_sum(S.vy, N) / ce;
  }
  env_sync<W>();
  ra = S.red[0];
  re = S.red[1];
  env_sync<W>();
}

// Heuristic opponent decision for unit i (heuristics.py:103-243).
// Returns the action packed with the scripted-controller memory update.
constexpr int SA_ACT_MASK = 0xff, SA_HAS = 0x100, SA_MEMOK = 0x200, SA_TGT_SHIFT = 16;
#ifdef TABX_INLINE_SCRIPTED
#define TABX_SCRIPTED_QUAL __device__ __forceinline__
#else
#define TABX_SCRIPTED_QUAL __device__ __noinline__
#endif
// SV: the env view the decision reads (EnvSmem<W> in K1; CtrlView in K0):
// px, py, ch, sh, rad, mh, uf, zin, the unit's vis / atk rows, m_active,
// m_alive.
template <int W, class SV>
__device__ __forceinline__ int scripted_body(const SV& S, const tabx_config* __restrict__ C, int i,
                                             int N, int Z, double hd, double cd, double step,
                                             uint32_t mask7, double u_explore, double u_pick,
                                             double eps, double xi, uint32_t bush_m, double mx,
                                             double my, bool memv) {
  TABX_PHASE_BEGIN();
  const UnitStatic U = load_static(C, i, true);
  const uint32_t* vis = &S.vis[i * W];
  const uint32_t* atk = &S.atk[i * W];
  const double px = S.px[i], py = S.py[i];
  // target candidates: visible, alive & active, not self
  // squared distances; closer() orders them exactly as their float64 roots
  double bf = 0.0, bi = 0.0, bn = 0.0, bm = 0.0, bmd = 0.0;
  int tf = -1, ti = -1, tn = -1, tm = -1;
  for (int k = 0; k < W; ++k) {
   uint32_t cm = vis[k] & S.m_active[k] & S.m_alive[k] & ~(k == (i >> 5) ? 1u << (i & 31) : 0u);
   while (cm) {
    const int j = (k << 5) + __ffs(cm) - 1;
    cm &= cm - 1;
    const uint32_t uj = S.uf[j];
    const double dx = S.px[j] - px, dy = S.py[j] - py;
    const double d = dx * dx + dy * dy;
    const bool foe = ((uj & UF_ENEMY) != 0) != U.enemy;
    if (!foe) {
      if (tf < 0 || closer(d, bf)) { bf = d; tf = j; }
      if ((uj & UF_INJURED) && (ti < 0 || closer(d, bi))) { bi = d; ti = j; }
    } else {
      if (tn < 0 || closer(d, bn)) { bn = d; tn = j; }
      const double m = S.mh[j];
      if (tm < 0 || m < bm || (m == bm && closer(d, bmd))) { bm = m; bmd = d; tm = j; }
    }
   }
  }
  int tgt;
  bool has;
  if (U.healer) {
    has = tf >= 0;
    tgt = ti >= 0 ? ti : (tf >= 0 ? tf : 0);
  } else if (U.assassin) {
    has = tm >= 0;
    tgt = tm >= 0 ? tm : 0;
  } else {
    has = tn >= 0;
    tgt = tn >= 0 ? tn : 0;
  }
  const bool has_near = tn >= 0;
  const double tpx = S.px[tgt], tpy = S.py[tgt], tr = S.rad[tgt];
  TABX_PHASE_DIV(14);

  // memory validity (heuristics.py:208-209), needed for the update either way
  const double gx = px - mx, gy = py - my;
  const bool mem_ok = memv && (sqrt(gx * gx + gy * gy) > U.rad);

  int act = -1;
  if (has && bit_of(atk, tgt) && cd <= 0.0) act = A_ATTACK;
  if (act < 0 && has) {
    // _aligned_after_rotate (heuristics.py:87-100): heading + rot_step unwrapped
    const double h2 = hd + C->rot_step;
    const sincos_t sc2 = libm_sincos(h2);
    const double c2 = sc2.c, s2 = sc2.s;
    const double dx = tpx - px, dy = tpy - py;
    const double lx = dx * c2 + dy * s2;
    const double ly = (-dx) * s2 + dy * c2;
    const double cx = np_clip(lx, 0.0, U.range);
    const double cy = np_clip(ly, -U.rad, U.rad);
    const double ex = lx - cx, ey = ly - cy;
    const bool box = ex * ex + ey * ey <= tr * tr;
    const double dist = sqrt(dx * dx + dy * dy);
    const double cdev = dist > 0.0 ? lx / dist : 1.0;
    if (box && cdev >= U.cos_half) act = A_ROTATE;
  }
  TABX_PHASE_DIV(15);
  if (act < 0 && U.ranger && has_near && sqrt(bn) < xi * U.range)
    act = best_move(px, py, S.px[tn], S.py[tn], step, true);
  if (act < 0 && has) {
    const double touch = U.rad + tr + 0.5;
    double gxd, gyd;
    if (U.healer) {
      gxd = tpx;
      gyd = tpy;
    } else if (U.assassin) {
      gxd = tpx - S.ch[tgt] * touch;
      gyd = tpy - S.sh[tgt] * touch;
    } else {
      const double standoff = np_max(0.8 * U.range, touch);
      gxd = tpx + S.ch[tgt] * standoff;
      gyd = tpy + S.sh[tgt] * standoff;
    }
    act = best_move(px, py, gxd, gyd, step, false);
  }
  if (act < 0 && mem_ok) act = best_move(px, py, mx, my, step, false);
  if (act < 0 && Z > 0 && U.ranger && bush_m != 0u && (S.zin[i] & bush_m) == 0u) {
    int nb = -1;
    double bd = 0.0;
    for (int z = 0; z < Z; ++z) {
      if (!((bush_m >> z) & 1u)) continue;
      const double ex = C->zone_cx[z] - px, ey = C->zone_cy[z] - py;
      const double d = sqrt(ex * ex + ey * ey);
      if (nb < 0 || d < bd) { bd = d; nb = z; }
    }
    act = best_move(px, py, C->zone_cx[nb], C->zone_cy[nb], step, false);
  }
  if (act < 0) act = A_ROTATE;
  // epsilon exploration (the pick draw is made by the caller, beside the
  // explore draw: two independent hash chains interleave)
  if (u_explore < eps) act = kth_legal(mask7, u_pick);
  // packed result: action, memory update (has -> remember tgt; memv = has || mem_ok)
  return act | (has ? SA_HAS : 0) | (mem_ok ? SA_MEMOK : 0) | (tgt << SA_TGT_SHIFT);
}

// K1's out-of-line call: everything arrives by value (scalars in registers,
// the unit's vis/atk rows in S.vis / S.atk): reference parameters of a
// non-inlined call would force the caller's copies into local memory
template <int W>
TABX_SCRIPTED_QUAL int scripted_action(const EnvSmem<W>& S, const tabx_config* __restrict__ C, int i,
                                       int N, int Z, double hd, double cd, double step,
                                       uint32_t mask7, double u_explore, double u_pick,
                                       double eps, double xi, uint32_t bush_m, double mx,
                                       double my, bool memv) {
  return scripted_body<W>(S, C, i, N, Z, hd, cd, step, mask7, u_explore, u_pick, eps, xi, bush_m,
                          mx, my, memv);
}

// ---------------------------------------------------------------- lane ---
// NF / ZF: unit / zone counts fixed at compile time (0 = P.N / P.Z): the
// step kernel's instantiations for the common shapes, where every per-unit
// and per-zone loop gets a constant trip count
template <int W, int M, int NF = 0, int ZF = 0>
__device__ void run_lane(const Params& P, int64_t b, int i, EnvSmem<W>& S,
                         unsigned char* emit, bool refresh, uint32_t step_no) {
  const int N = NF ? NF : P.N, Z = ZF ? ZF : P.Z;
  const bool valid = i < N;
  const int64_t u = b * N + i;
  const DevState& st = P.st;
  TABX_ASSERT(b >= 0 && b < P.B && N <= 32 * W && Z <= TABX_MAX_ZONES && P.st.cfg[b] >= 0);
  const tabx_config* __restrict__ C = P.cfgs + st.cfg[b];
  const DerivedCfg* __restrict__ DC = P.dcfgs + st.cfg[b];
  const UnitStatic U = load_static(C, i, valid);
  const uint32_t bush_m = DC->bush_m, lava_m = DC->lava_m, swamp_m = DC->swamp_m;
  const double dt = C->dt, fw = C->field_w, fh = C->field_h, rw = DC->rw, rh = DC->rh;
  const double rmh = valid ? DC->rmh[i] : 1.0, rucd = valid ? DC->rucd[i] : 0.0;

  TABX_PHASE_BEGIN();
  // ---- lane + unit state
  uint8_t lf = st.flags[b];
  const bool running = !(lf & F_DONE);
  int32_t t = st.t[b];
  uint64_t seed = st.seed[b];
  double prev_gap = st.prev_gap[b];
  double ep_ret = st.ep_return[b];
  int winner = st.winner[b], reason = st.reason[b], fk = st.first_kill[b];

  double px = 0.0, py = 0.0, hd = 0.0, hp = 0.0, cd = 0.0, rv = 0.0;
  double ivx = 0.0, ivy = 0.0, vlx = 0.0, vly = 0.0, mx = 0.0, my = 0.0;
  double ch = 1.0, sh = 0.0;  // libm cos/sin of hd, cached in the state
  uint32_t zin = 0u;          // zone bits at (px, py), cached in the state
  bool alive = false, memv = false;
  if (valid) {
    const double2 p = st.pos[u];
    px = p.x;
    py = p.y;
    hd = st.heading[u];
    hp = st.health[u];
    cd = st.cooldown[u];
    rv = st.reveal[u];
    const double2 iv = st.imp_dv[u];
    ivx = iv.x;
    ivy = iv.y;
    // realized velocity is output-only (written back only by running lanes);
    // the scripted-controller memory only exists for heuristic-team units
    // (under K0 the memory is K0's to update: K1 neither reads nor writes it)
    if (M == MODE_STEP && C->controller[U.enemy ? 1 : 0] == TABX_CTRL_HEURISTIC) {
      const double2 m = st.mem_pos[u];
      mx = m.x;
      my = m.y;
    }
    const uint8_t ub = st.ubits[u];
    alive = ub & U_ALIVE;
    memv = ub & U_MEMV;
    const double2 cs = st.hcs[u];
    ch = cs.x;
    sh = cs.y;
    zin = st.zbits[u];
  }

  auto publish = [&](void) {
    S.px[i] = px;
    S.py[i] = py;
    S.ch[i] = ch;
    S.sh[i] = sh;
    S.rad[i] = U.rad;
    S.mh[i] = U.mh;
    S.rv[i] = rv;
    S.dmg[i] = U.dmg;
    S.uf[i] = (U.active ? UF_ACTIVE : 0u) | (alive ? UF_ALIVE : 0u) | (U.enemy ? UF_ENEMY : 0u) |
              (U.kin ? UF_KIN : 0u) | (hp < U.mh ? UF_INJURED : 0u);
    S.zin[i] = zin;
  };

  const int n_ally = DC->n_ally, n_enemy = DC->n_enemy;

  uint32_t vis[W], atk[W];
  int tgt = -1;

  if (M == MODE_RESET) {
    // deferred auto-reset of a finished lane (environment.py:502-517): reseed,
    // respawn from the config template, fresh caches and prev_gap, then the
    // fresh observation / mask replace the step's (final ones were written by
    // the emit kernel)
    if (!(lf & F_PEND)) return;
    const int64_t episode = st.episode[b] + 1;
    seed = key_hash(seed, (uint64_t)episode, TAG_RESEED, 0);
    if (valid && U.active) {
      px = C->spawn_x[i];
      py = C->spawn_y[i];
      hd = C->spawn_heading[i];
      hp = U.mh;
      alive = true;
    } else {
      alive = false;
    }
    ivx = ivy = vlx = vly = 0.0;
    cd = rv = 0.0;
    mx = my = 0.0;
    memv = false;
    t = 0;
    ep_ret = 0.0;
    lf = 0;
    winner = -1;
    reason = R_NONE;
    fk = -1;
    {
      const sincos_t sc = libm_sincos(hd);
      ch = sc.c;
      sh = sc.s;
    }
    zin = valid ? zone_bits(C, DC, Z, px, py) : 0u;
    publish();
    build_masks<W>(S, i, valid, U.active, alive, U.enemy, rv, zin, Z, bush_m);
    env_sync<W>();
    cache_row_of<W>(S, i, N, U, bush_m);
    double ra, re;
    team_ratios<W>(S, i, N, U.active, U.enemy, hp, U.mh, n_ally, n_enemy, ra, re);
    prev_gap = ra - re;
    const tabx_outputs& O = P.out;
    if (valid) {
      st.pos[u] = make_double2(px, py);
      st.heading[u] = hd;
      st.vel[u] = make_double2(0.0, 0.0);
      st.imp_dv[u] = make_double2(0.0, 0.0);
      st.health[u] = hp;
      st.cooldown[u] = 0.0;
      st.reveal[u] = 0.0;
      st.mem_pos[u] = make_double2(0.0, 0.0);
      st.hcs[u] = make_double2(ch, sh);
      st.zbits[u] = zin;
      st.ubits[u] = alive ? U_ALIVE : 0;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        st.vis[u * W + k] = S.vis[i * W + k];
        st.atk[u * W + k] = S.atk[i * W + k];
      }
      if (O.action_mask) {
        const bool c2 = alive && U.active;
        uint8_t* m = O.action_mask + u * TABX_NUM_ACTIONS;
        for (int a = 0; a < 5; ++a) m[a] = c2;
        m[5] = c2;
        m[6] = (c2 && C->enable_noop) || !c2;
      }
    }
    if (i == 0) {
      st.episode[b] = episode;
      st.seed[b] = seed;
      st.t[b] = 0;
      st.prev_gap[b] = prev_gap;
      st.ep_return[b] = 0.0;
      st.flags[b] = 0;
      st.winner[b] = -1;
      st.reason[b] = R_NONE;
      st.first_kill[b] = -1;
      P.sync->refresh[(step_no + 1) % 3] = 1;
    }
    env_sync<W>();
    if (emit && i < 32) {
      const int R = emit_rows(N, P.D, W == 1 ? TABX_EMIT_BUDGET : 8192);
      const int SF = emit_stage_floats(N, P.D, P.G, R);
      const EmitScratch<W> X = emit_scratch<W>(emit, N, Z, R);
      int buf = 0;
      load_view<W>(X, st, b, N, Z, C, DC, i);
      if (O.observations_bf16)
        emit_lane<W, true>(X, O.observations, O.global_state, b, N, Z, P.D, P.G, R, SF, C, DC, i,
                           buf, true, (__nv_bfloat16*)O.observations_bf16,
                           (int)O.observations_bf16_ld);
      else
        emit_lane<W>(X, O.observations, O.global_state, b, N, Z, P.D, P.G, R, SF, C, DC, i, buf,
                     true);
    }
    env_sync<W>();
    return;
  }

  if (!is_step_mode(M)) {
    // init_output / refresh_caches (environment.py:147-151, :351-374)
    publish();
    build_masks<W>(S, i, valid, U.active, alive, U.enemy, rv, zin, Z, bush_m);
    env_sync<W>();
    if (M == MODE_REFRESH) {
      if (refresh) {
        cache_row_of<W>(S, i, N, U, bush_m);
        if (valid)
#pragma unroll
          for (int k = 0; k < W; ++k) {
            st.vis[u * W + k] = S.vis[i * W + k];
            st.atk[u * W + k] = S.atk[i * W + k];
          }
      }
      env_sync<W>();
      return;
    }
    cache_row_of<W>(S, i, N, U, bush_m);
#pragma unroll
    for (int k = 0; k < W; ++k) {
      vis[k] = S.vis[i * W + k];
      atk[k] = S.atk[i * W + k];
    }
    double ra, re;
    team_ratios<W>(S, i, N, U.active, U.enemy, hp, U.mh, n_ally, n_enemy, ra, re);
    prev_gap = ra - re;
    const tabx_outputs& O = P.out;
    if (valid) {
      const bool ctl = alive && U.active;
      if (O.action_mask) {
        uint8_t* m = O.action_mask + u * TABX_NUM_ACTIONS;
        for (int a = 0; a < 5; ++a) m[a] = ctl;
        m[5] = ctl && cd <= 0.0;
        m[6] = (ctl && C->enable_noop) || !ctl;
      }
      if (O.rewards) O.rewards[u] = 0.0f;
      if (O.actions) O.actions[u] = A_NOOP;
      if (O.interactions)
        for (int j = 0; j < N; ++j) O.interactions[u * N + j] = 0;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        st.vis[u * W + k] = vis[k];
        st.atk[u * W + k] = atk[k];
      }
    }
    if (i == 0) {
      st.prev_gap[b] = prev_gap;
      if (O.terminated) O.terminated[b] = (lf & F_TERM) ? 1 : 0;
      if (O.truncated) O.truncated[b] = (lf & F_TRUNC) ? 1 : 0;
      if (O.done) O.done[b] = (lf & F_DONE) ? 1 : 0;
      if (O.dense_reward) O.dense_reward[b] = 0.0;
      if (O.winner) O.winner[b] = winner;
      if (O.reason) O.reason[b] = reason;
      if (O.first_kill) O.first_kill[b] = fk;
      if (O.episode_return) O.episode_return[b] = ep_ret;
      if (O.episode_length) O.episode_length[b] = t;
      if (O.reset_mask) O.reset_mask[b] = 0;
    }
    env_sync<W>();
    return;
  }

  // ======================= step (environment.py:207-348) ==================
  if (M == MODE_STEP_K0) {
    // no in-kernel controller: the contact pass reads flags and radii (the
    // positions are published after integration) and, W > 1, the active set;
    // stage 8 republishes everything
    S.rad[i] = U.rad;
    S.uf[i] = (U.active ? UF_ACTIVE : 0u) | (alive ? UF_ALIVE : 0u);
    if (W > 1) {
      uint32_t m[W];
      env_ballot<W, 0>(valid && U.active, S, i, m);
      if ((i & 31) == 0) S.m_active[i >> 5] = m[i >> 5];
    }
  } else {
    publish();
    build_masks<W>(S, i, valid, U.active, alive, U.enemy, rv, zin, Z, bush_m);
  }
  env_sync<W>();

  TABX_PHASE(0);
  // 1. pre-step action mask (arrays.py:373-387)
  const bool ctl = alive && U.active;
  const uint32_t mask7 = ctl ? (0x1Fu | ((cd <= 0.0) ? 0x20u : 0u) | (C->enable_noop ? 0x40u : 0u))
                             : 0x40u;
  // effective speed after swamps at the pre-move position (arrays.py:338-343)
  const double speff = U.speed * swamp_mult(C, Z, zin, swamp_m);
  TABX_PHASE(9);
  // 2. action resolution (environment.py:154-204)
  const int team = U.enemy ? 1 : 0;
  const int ctrl = C->controller[team];
  const bool free_u = valid && ctl && running;
  const bool heur = free_u && ctrl == TABX_CTRL_HEURISTIC;
  int act = A_NOOP;
  if (free_u && P.actions) act = (int)P.actions[u];
  if (M == MODE_STEP_K0) {
    // K0 made the decision (its memory update is in the state read above)
    if (heur) act = (int)P.ctrl_act[u];
  } else if (env_any<W, 1>(heur, S, i)) {
    // cached vis/atk of the previous stage 8, or fresh after a batch refill
    if (refresh) {
      cache_row_of<W>(S, i, N, U, bush_m);
#pragma unroll
      for (int k = 0; k < W; ++k) {
        vis[k] = S.vis[i * W + k];
        atk[k] = S.atk[i * W + k];
      }
    } else if (valid) {
#pragma unroll
      for (int k = 0; k < W; ++k) {
        vis[k] = st.vis[u * W + k];
        atk[k] = st.atk[u * W + k];
      }
    } else {
#pragma unroll
      for (int k = 0; k < W; ++k) vis[k] = atk[k] = 0u;
    }
    TABX_PHASE(10);
    if (heur) {
      if (!refresh) {  // the refreshed rows are already in S.vis / S.atk
#pragma unroll
        for (int k = 0; k < W; ++k) {
          S.vis[i * W + k] = vis[k];
          S.atk[i * W + k] = atk[k];
        }
      }
      const double ue = uniform53(seed, (uint64_t)(int64_t)t, TAG_EXPLORE, (uint64_t)i);
      const double up = uniform53(seed, (uint64_t)(int64_t)t, TAG_PICK, (uint64_t)i);
      const double stepl = speff * dt;
      const int r = scripted_action<W>(S, C, i, N, Z, hd, cd, stepl, mask7, ue, up,
                                       C->epsilon[team], C->aggressive[team], bush_m, mx, my,
                                       memv);
      act = r & SA_ACT_MASK;
      if (r & SA_HAS) {
        const int tg = r >> SA_TGT_SHIFT;
        mx = S.px[tg];
        my = S.py[tg];
      }
      memv = (r & (SA_HAS | SA_MEMOK)) != 0;
    }
    TABX_PHASE(11);
  }
  if (free_u && ctrl == TABX_CTRL_RANDOM)
    act = kth_legal(mask7, uniform53(seed, (uint64_t)(int64_t)t, TAG_RANDOM, (uint64_t)i));
  if (!free_u) act = A_NOOP;

  TABX_PHASE(1);
  // 3-4. commanded velocity, integration, timers (environment.py:215-228)
  const bool moving = act < 4 && alive && U.active && !U.kin;
  const double vmag = moving ? speff : 0.0;
  const int ad = act < 0 ? 0 : (act > 3 ? 3 : act);
  const double dirx = ad == 2 ? 1.0 : (ad == 3 ? -1.0 : 0.0);
  const double diry = ad == 0 ? 1.0 : (ad == 1 ? -1.0 : 0.0);
  const double vux = dirx * vmag + ivx;
  const double vuy = diry * vmag + ivy;
  if (U.active && !U.kin && running) {
    px = px + vux * dt;
    py = py + vuy * dt;
  }
  const double tick = (U.active && running) ? dt : 0.0;
  cd = np_max(cd - tick, 0.0);
  rv = np_max(rv - tick, 0.0);
  if (W > 1 && TABX_SWEEP) {  // this step's touching rows (read after the barriers below)
#pragma unroll
    for (int k = 0; k < W; ++k) S.touch[i * W + k] = 0u;
  }
  env_sync<W>();
  TABX_JITTER(200);  // (checked build) publish the new positions out of step
  S.px[i] = px;
  S.py[i] = py;
  const double py_key = py;  // y the sweep keys are taken at
  if (W > 1 && TABX_SWEEP) {
    S.ykey[i] = (valid && U.active) ? (float)py : __int_as_float(0x7f800000);
    if (i == 0) S.dymax = 0u;
  }
  if (W > 1 && TABX_SWEEP) {
    // (the ranking's own barrier publishes the positions too)
    rank_by_y<W>(S, i, N);
#ifndef TABX_SELFTEST_RACE  // negative control of the checked build: the contact
                            // sweep reads the order without this barrier
    env_sync<W>();
#endif
  } else {
    env_sync<W>();
  }

  // 5. contacts: detection (physics.py:27-49), Gauss-Seidel (physics.py:52-94)
  // float32 filter on squared distance vs rs^2 (margin 1e-5 relative);
  // near-contact pairs get the reference's float64 depth test
  bool any_touch = false;
  uint32_t rowm[W];  // W > 1: rows (observers a) with a touching pair (a, c > a)
#pragma unroll
  for (int k = 0; k < W; ++k) rowm[k] = 0u;
  if (W == 1) {
    // all 32 lanes over the N(N-1)/2 pairs; one ballot word per 32 pairs keeps
    // the ascending (i, j) order the Gauss-Seidel solve needs
    const int NP = N * (N - 1) / 2;
    uint32_t anyw = 0u;
    for (int k = 0; (k << 5) < NP; ++k) {
      const int p = (k << 5) + i;
      bool hit = false;
      if (p < NP && running) {
        const uint32_t ij = S.ptab[p];
        const int a = (int)(ij >> 8), c = (int)(ij & 255u);
        TABX_ASSERT(a < c && c < N);
        if (S.uf[a] & S.uf[c] & UF_ACTIVE) {
          const double dx = S.px[c] - S.px[a], dy = S.py[c] - S.py[a];
          const double rs = S.rad[a] + S.rad[c];
          const float dxf = (float)dx, dyf = (float)dy;
          const float d2f = dxf * dxf + dyf * dyf;
          const float rs2f = (float)(rs * rs);
          if (d2f < rs2f * 0.99999f && d2f > 1e-30f) {
            hit = true;
          } else if (!(d2f > rs2f * 1.00001f)) {
            TABX_COUNT(2);
            const double dist = slow_sqrt(dx * dx + dy * dy);
            hit = (dist == 0.0 ? rs : rs - dist) > 0.0;
          }
        }
      }
      const uint32_t bm = __ballot_sync(0xffffffffu, hit);
      if (i == 0) S.tmask[k] = bm;
      anyw |= bm;
    }
    any_touch = anyw != 0u;
  } else if (TABX_SWEEP) {
    // each active unit scans forward in y order while the key gap is within
    // the largest contact distance 2 rad_max; every unordered pair with
    // |dy| <= 2 rad_max is seen once (from its lower-ranked unit); a hit sets
    // bit c of row a in S.touch (rows were cleared before the hand-off)
    if (running && valid && U.active) {
      const float yi = S.ykey[i];
      const float lim = sweep_limit(yi, 2.0 * DC->rad_max);
      for (int q = S.rnk[i] + 1; q < N; ++q) {
        if (!(S.skey[q] - yi <= lim)) break;  // ascending keys (+inf last)
        const int j = S.ord[q];
        const int a = i < j ? i : j, c = i < j ? j : i;
        const double dx = S.px[c] - S.px[a], dy = S.py[c] - S.py[a];
        const double rs = S.rad[a] + S.rad[c];
        const float dxf = (float)dx, dyf = (float)dy;
        const float d2f = dxf * dxf + dyf * dyf;
        const float rs2f = (float)(rs * rs);
        bool hit = false;
        if (d2f < rs2f * 0.99999f && d2f > 1e-30f) {
          hit = true;
        } else if (!(d2f > rs2f * 1.00001f)) {
          TABX_COUNT(3);
          const double dist = slow_sqrt(dx * dx + dy * dy);
          hit = (dist == 0.0 ? rs : rs - dist) > 0.0;
        }
        if (hit) atomicOr(&S.touch[a * W + (c >> 5)], 1u << (c & 31));
      }
    }
    env_sync<W>();
    bool mine = false;
#pragma unroll
    for (int k = 0; k < W; ++k) mine |= S.touch[i * W + k] != 0u;
    env_ballot<W, 2>(mine, S, i, rowm);
#pragma unroll
    for (int k = 0; k < W; ++k) any_touch |= rowm[k] != 0u;
  } else {
    uint32_t trow[W];
#pragma unroll
    for (int k = 0; k < W; ++k) trow[k] = 0u;
    bool mine = false;
    if (valid && U.active && running) {
      uint32_t unsure[W];
#pragma unroll
      for (int k = 0; k < W; ++k) unsure[k] = 0u;
      for (int j = i + 1; j < N; ++j) {
        const float dxf = (float)(S.px[j] - px), dyf = (float)(S.py[j] - py);
        const float d2f = dxf * dxf + dyf * dyf;
        const float rs2f = (float)((U.rad + S.rad[j]) * (U.rad + S.rad[j]));
        const bool sure = (d2f < rs2f * 0.99999f) & (d2f > 1e-30f);
        const bool maybe = !sure & !(d2f > rs2f * 1.00001f);
        trow[j >> 5] |= (uint32_t)sure << (j & 31);
        unsure[j >> 5] |= (uint32_t)maybe << (j & 31);
      }
#pragma unroll
      for (int k = 0; k < W; ++k) {
        trow[k] &= S.m_active[k];
        uint32_t m = unsure[k] & S.m_active[k];
        while (m) {
          const int j = (k << 5) + __ffs(m) - 1;
          m &= m - 1;
          const double dx = S.px[j] - px, dy = S.py[j] - py;
          const double rs = U.rad + S.rad[j];
          TABX_COUNT(4);
          const double dist = slow_sqrt(dx * dx + dy * dy);
          const double depth = dist == 0.0 ? rs : rs - dist;
          if (depth > 0.0) trow[k] |= 1u << (j & 31);
        }
        mine |= trow[k] != 0u;
      }
    }
#pragma unroll
    for (int k = 0; k < W; ++k) S.touch[i * W + k] = trow[k];
    env_ballot<W, 2>(mine, S, i, rowm);
#pragma unroll
    for (int k = 0; k < W; ++k) any_touch |= rowm[k] != 0u;
  }
  TABX_PHASE(10);  // (K0 mode: slot 10 = integrate + contact detection)
  double vfx = vux, vfy = vuy;
  if (any_touch) {
    S.vx[i] = vux;
    S.vy[i] = vuy;
    S.sx[i] = 0.0;
    S.sy[i] = 0.0;
    env_sync<W>();
    if (i == 0) {
      const double e = C->restitution, slop = C->slop, beta = C->correction;
      const int NP = N * (N - 1) / 2;
      // rows in ascending order (W > 1: only those with a touching pair)
      for (int kk = 0; kk < (W == 1 ? 1 : W); ++kk)
      for (uint32_t rows = W == 1 ? 1u : rowm[kk]; rows; rows &= rows - 1) {
        const int a0 = W == 1 ? 0 : (kk << 5) + __ffs(rows) - 1;
        for (int k = 0; k < (W == 1 ? (NP + 31) >> 5 : W); ++k) {
          uint32_t m = W == 1 ? S.tmask[k] : S.touch[a0 * W + k];
          while (m) {
            int a = a0;
            int bb = (k << 5) + __ffs(m) - 1;
            m &= m - 1;
            if (W == 1) {  // pair index -> (a, bb)
              const uint32_t ij = S.ptab[bb];
              a = (int)(ij >> 8);
              bb = (int)(ij & 255u);
            }
            const double wa = C->inv_mass[a], wb = C->inv_mass[bb];
            const double w = wa + wb;
            if (!(w > 0.0)) continue;
            const double dx = S.px[bb] - S.px[a], dy = S.py[bb] - S.py[a];
            const double dist = sqrt(dx * dx + dy * dy);
            const double rs = S.rad[a] + S.rad[bb];
            const bool coinc = dist == 0.0;
            const double depth = coinc ? rs : rs - dist;
            const double nx = coinc ? 1.0 : dx / dist;
            const double ny = coinc ? 0.0 : dy / dist;
            const double rel = (S.vx[bb] - S.vx[a]) * nx + (S.vy[bb] - S.vy[a]) * ny;
            const double jm = rel <= 0.0 ? (-(1.0 + e) * rel) / w : 0.0;
            S.vx[a] = S.vx[a] - (jm * wa) * nx;
            S.vy[a] = S.vy[a] - (jm * wa) * ny;
            S.vx[bb] = S.vx[bb] + (jm * wb) * nx;
            S.vy[bb] = S.vy[bb] + (jm * wb) * ny;
            const double corr = (beta * np_max(depth - slop, 0.0)) / w;
            S.sx[a] = S.sx[a] - (corr * wa) * nx;
            S.sy[a] = S.sy[a] - (corr * wa) * ny;
            S.sx[bb] = S.sx[bb] + (corr * wb) * nx;
            S.sy[bb] = S.sy[bb] + (corr * wb) * ny;
          }
        }
      }
    }
    env_sync<W>();
    vfx = S.vx[i];
    vfy = S.vy[i];
    px = px + S.sx[i];
    py = py + S.sy[i];
  }
  if (running) {
    ivx = vfx - vux;
    ivy = vfy - vuy;
    vlx = vfx;
    vly = vfy;
  }

  TABX_PHASE(2);
  // 6. boundary penalty + clip (physics.py:97-120)
  if (running && valid) {
    const bool out = px < 0.0 || px > fw || py < 0.0 || py > fh;
    if (out && alive && U.active) hp = np_max(hp - (C->boundary_coeff * U.mh) * dt, 0.0);
    if (U.active && !U.kin) {
      px = np_clip(px, 0.0, fw);
      py = np_clip(py, 0.0, fh);
    }
  }
  // 7. rotation (environment.py:249-252)
  if (act == A_ROTATE && alive && U.active && running) {
    hd = np_remainder(hd + C->rot_step, 6.283185307179586);
    {
      const sincos_t sc = libm_sincos(hd);
      ch = sc.c;
      sh = sc.s;
    }
  }

  TABX_PHASE(3);
  // 8. caches at the post-move state (environment.py:254-257)
  zin = valid ? zone_bits(C, DC, Z, px, py) : 0u;
  TABX_PHASE(12);
  env_sync<W>();
  publish();
  if (W > 1 && TABX_SWEEP && valid && U.active) {
    // the y order of the contact pass stands; windows widen by twice the
    // largest move since (contact correction, boundary clip), rounded up
    const float d = (float)fabs(py - py_key) * (1.0f + 0x1p-20f);
    if (d > 0.0f) atomicMax(&S.dymax, __float_as_uint(d));
  }
  build_masks<W>(S, i, valid, U.active, alive, U.enemy, rv, zin, Z, bush_m);
  env_sync<W>();
  TABX_PHASE(13);
  tgt = cache_row_inl<W>(S, i, N, U, bush_m);
#pragma unroll
  for (int k = 0; k < W; ++k) {
    vis[k] = S.vis[i * W + k];
    atk[k] = S.atk[i * W + k];
  }

  TABX_PHASE(4);
  // 9. combat (combat.py:86-113; environment.py:259-265)
  const bool swing = act == A_ATTACK && alive && U.active && cd <= 0.0;
  const bool landed = running && swing && tgt >= 0;
  TABX_ASSERT(tgt >= -1 && tgt < N && act >= 0 && act < TABX_NUM_ACTIONS);
  S.tgt[i] = landed ? tgt : -1;
  env_sync<W>();
  // per-victim damage: landed attackers in ascending order (combat.py:108)
  uint32_t lm[W];
  env_ballot<W, 3>(landed, S, i, lm);
  double delta = 0.0;
  bool was_hit = false;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    for (uint32_t m = lm[k]; m; m &= m - 1) {
      const int a = (k << 5) + __ffs(m) - 1;
      if (S.tgt[a] == i) {
        delta += S.dmg[a];
        was_hit = true;
      }
    }
  }
  if (running) {
    if (U.active && alive) hp = np_clip(hp - delta, 0.0, U.mh);
    if (swing) cd = U.ucd;
  }
  // 10. reveal on contact (environment.py:267-268)
  if (landed || was_hit) rv = C->reveal_duration;
  // 11. lava (environment.py:270-277)
  if (alive && U.active && running && valid) {
    const double burn = lava_sum(C, Z, S.zin[i], lava_m) * dt;
    hp = np_clip(hp - burn, 0.0, U.mh);
  }
  // 12. deaths, first kill (environment.py:279-286)
  const bool still = alive && hp > 0.0;
  const bool died = alive && !still;
  alive = still;
  bool any_died = false, ally_died = false;
  {
    uint32_t md[W], ma[W];
    env_ballot2<W, 4>(died, died && !U.enemy, S, i, md, ma);
#pragma unroll
    for (int k = 0; k < W; ++k) {
      any_died |= md[k] != 0u;
      ally_died |= ma[k] != 0u;
    }
  }
  if (any_died && fk < 0) fk = ally_died ? ENEMY : ALLY;

  TABX_PHASE(5);
  // rewards and termination (environment.py:288-328)
  double ra, re;
  team_ratios<W>(S, i, N, U.active, U.enemy, hp, U.mh, n_ally, n_enemy, ra, re);
  const double gap = ra - re;
  const double dense = running ? gap - prev_gap : 0.0;
  if (running) {
    prev_gap = gap;
    t += 1;
  }
  int na = 0, ne = 0;
  {
    uint32_t mA[W], mE[W];
    env_ballot2<W, 6>(alive && U.active && !U.enemy, alive && U.active && U.enemy, S, i, mA, mE);
#pragma unroll
    for (int k = 0; k < W; ++k) {
      na += __popc(mA[k]);
      ne += __popc(mE[k]);
    }
  }
  const bool elim = running && (na == 0 || ne == 0);
  const bool trunc = running && !elim && t >= C->max_steps;
  int win = -1, why = R_NONE;
  if (elim) {
    win = (ne == 0 && na > 0) ? ALLY : ENEMY;
    why = R_ELIM;
  } else if (trunc) {
    win = ra > re ? ALLY : ENEMY;
    why = ra == re ? R_TIE : R_TRUNC;
  }
  const bool fin = elim || trunc;
  const double terminal = fin ? (win == ALLY ? 1.0 : -1.0) : 0.0;
  const double ally_reward = dense + terminal;
  ep_ret = ep_ret + (running ? ally_reward : 0.0);
  if (elim) lf |= F_TERM;
  if (trunc) lf |= F_TRUNC;
  if (fin) {
    lf |= F_DONE;
    winner = win;
    reason = why;
  }
  const double reward_i =
      ((U.enemy ? -1.0 : 1.0) * (U.active ? 1.0 : 0.0)) * (running ? ally_reward : 0.0);

  TABX_PHASE(6);
  // ---- outputs of this step (observation uses stage-8 caches, post-step state)
  const tabx_outputs& O = P.out;
  const bool resets = P.auto_reset && (lf & F_DONE);
  if (resets) {
    lf |= F_PEND;  // the reset kernel respawns after the emit kernel
    if (i == 0) P.sync->any_pend = 1;
  }
  if (valid) {
    if (O.rewards) O.rewards[u] = (float)reward_i;
    if (O.actions) O.actions[u] = act;
    if (O.interactions)
      for (int j = 0; j < N; ++j) O.interactions[u * N + j] = (landed && tgt == j) ? 1 : 0;
    if (O.action_mask && !resets) {
      const bool c2 = alive && U.active;
      uint8_t* m = O.action_mask + u * TABX_NUM_ACTIONS;
      for (int a = 0; a < 5; ++a) m[a] = c2;
      m[5] = c2 && cd <= 0.0;
      m[6] = (c2 && C->enable_noop) || !c2;
    }
  }
  if (i == 0) {
    if (O.terminated) O.terminated[b] = (lf & F_TERM) ? 1 : 0;
    if (O.truncated) O.truncated[b] = (lf & F_TRUNC) ? 1 : 0;
    if (O.done) O.done[b] = (lf & F_DONE) ? 1 : 0;
    if (O.dense_reward) O.dense_reward[b] = dense;
    if (O.winner) O.winner[b] = winner;
    if (O.reason) O.reason[b] = reason;
    if (O.first_kill) O.first_kill[b] = fk;
    if (O.episode_return) O.episode_return[b] = ep_ret;
    if (O.episode_length) O.episode_length[b] = t;
    if (O.reset_mask) O.reset_mask[b] = resets ? 1 : 0;
    if (fin) {
      st.st_episodes[b] += 1;
      st.st_wins[b] += (win == ALLY) ? 1 : 0;
      st.st_fk_ally[b] += (fk == ALLY) ? 1 : 0;
      st.st_ties[b] += (why == R_TIE) ? 1 : 0;
      st.st_elims[b] += elim ? 1 : 0;
      st.st_len[b] += t;
      st.st_ret[b] += ep_ret;
    }
  }

  TABX_PHASE(7);
  // ---- state write-back
  if (valid) {
    st.pos[u] = make_double2(px, py);
    st.heading[u] = hd;
    if (running) st.vel[u] = make_double2(vlx, vly);
    st.imp_dv[u] = make_double2(ivx, ivy);
    st.health[u] = hp;
    st.cooldown[u] = cd;
    st.reveal[u] = rv;
    if (M == MODE_STEP && C->controller[U.enemy ? 1 : 0] == TABX_CTRL_HEURISTIC)
      st.mem_pos[u] = make_double2(mx, my);
    st.hcs[u] = make_double2(ch, sh);
    st.zbits[u] = zin;
    st.ubits[u] = (alive ? U_ALIVE : 0) | (memv ? U_MEMV : 0);
#pragma unroll
    for (int k = 0; k < W; ++k) {
      st.vis[u * W + k] = vis[k];
      st.atk[u * W + k] = atk[k];
    }
  }
  if (i == 0) {
    st.t[b] = t;
    st.prev_gap[b] = prev_gap;
    st.ep_return[b] = ep_ret;
    st.flags[b] = lf;
    st.winner[b] = (int8_t)winner;
    st.reason[b] = (int8_t)reason;
    st.first_kill[b] = (int8_t)fk;
  }
  TABX_PHASE(8);
  env_sync<W>();
}

// Per-env shared memory of the reset kernel's emitter: view + 2 stage buffers.
template <int W>
__host__ __device__ __forceinline__ size_t reset_view_bytes(const Params& P) {
  const int R = emit_rows(P.N, P.D, W == 1 ? TABX_EMIT_BUDGET : 8192);
  const int SF = emit_stage_floats(P.N, P.D, P.G, R);
  return emit_warp_bytes<W>(P.N, P.Z, R, SF);
}

#ifndef TABX_K1_EPB
#define TABX_K1_EPB 16  // W = 1: environments (warps) per step-kernel CTA (4: C3 K1 +10%)
#endif
// W = 1: 16 warps/SM at 128 registers whatever the CTA size
#define TABX_MIN_BLOCKS_W1(EPB) ((16 / (EPB)) > 0 ? (16 / (EPB)) : 1)
// W > 1 (one env per CTA of 32 W threads): resident warps per SM the
// register budget is cut for (C4 step kernels: unconstrained 254 registers
// at 8 warps/SM 11.2 ms; 16 warps at 128 registers 7.8 ms; 24 warps at 80
// registers 7.3 ms)
#ifndef TABX_WN_WARPS
#define TABX_WN_WARPS 24
#endif
#define TABX_MIN_BLOCKS_WN(W) (TABX_WN_WARPS / (W) > 1 ? TABX_WN_WARPS / (W) : 1)
// K1 (MODE_STEP / MODE_INIT / MODE_REFRESH) and K3 (MODE_RESET).
// One kernel per mode (M): the step kernel carries no reset / emitter code,
// which keeps its instruction footprint and register allocation to its own.
template <int W, int EPB, int M, int NF = 0, int ZF = 0>
__global__ void __launch_bounds__(32 * W * EPB, (W == 1 ? TABX_MIN_BLOCKS_W1(EPB) : TABX_MIN_BLOCKS_WN(W)))
    lane_kernel(const Params P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  EnvSmem<W>* envs = reinterpret_cast<EnvSmem<W>*>(smem_raw);
  const size_t env_bytes = (sizeof(EnvSmem<W>) * EPB + 15) & ~(size_t)15;
  const size_t view_bytes = reset_view_bytes<W>(P);
  unsigned char* view_base = smem_raw + env_bytes;

  uint32_t step_no = 0;
  bool refresh = false;
  if (is_step_mode(M) || M == MODE_RESET) {
    if (P.sync->err_index != NO_ERROR) return;  // an action violated the mask: no mutation
    step_no = P.sync->step;
    refresh = P.sync->refresh[step_no % 3] != 0;
    if (is_step_mode(M) && blockIdx.x == 0 && threadIdx.x == 0)
      P.sync->refresh[(step_no + 2) % 3] = 0;
  } else if (M == MODE_REFRESH) {
    step_no = P.sync->step;
    refresh = P.sync->refresh[step_no % 3] != 0;
    if (!refresh) return;  // nothing pending: the cached rows stand
  }
  const int g = threadIdx.x / (32 * W);
  const int i = threadIdx.x % (32 * W);
  if (W == 1) {  // pair table of this env group (N <= 32)
    int p = 0;
    for (int a = 0; a < P.N; ++a) {
      const int cnt = P.N - 1 - a;
      for (int q = i; q < cnt; q += 32) envs[g].ptab[p + q] = (uint16_t)((a << 8) | (a + 1 + q));
      p += cnt;
    }
    __syncwarp();
  }
  // K3 on a step where no lane finished: nothing to scan
  const bool work = M != MODE_RESET || P.sync->any_pend != 0;
  for (int64_t b = (int64_t)blockIdx.x * EPB + g; work && b < P.B;
       b += (int64_t)gridDim.x * EPB) {
    if (M == MODE_RESET && !(P.st.flags[b] & F_PEND)) continue;  // env-uniform
    // (checked build) everything but the kernel-lifetime pair table
    TABX_POISON(&envs[g], offsetof(EnvSmem<W>, ptab), i, 32 * W);
    env_sync<W>();
    run_lane<W, M, NF, ZF>(P, b, i, envs[g],
                M == MODE_RESET ? view_base + g * view_bytes
                                     : nullptr,
                refresh, step_no);
  }

  if (M == MODE_RESET) {
    // the reset kernel ends the step: advance the device step counter
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
}

// ------------------------------------------------------------------ K0 ---
// Heuristic controller pass (heuristics.py:103-243) ahead of K1.  Inside K1
// the decision runs on the heuristic team's lanes only (10 of 32 in C3, 50
// of 128 in C4) with the rest of the warp idle; here one lane is one
// heuristic unit, over a compact per-env view staged in shared memory: for
// W == 1 a warp packs the heuristic units of G environments, for W > 1 a
// warp takes one environment and its lanes stride over its heuristic units.
// Same inputs as K1's in-kernel call (the pre-step state, the cached vis/atk
// rows), so the same decision; the action goes to P.ctrl_act and the
// scripted-controller memory straight to the state (K1 under K0 neither
// reads nor writes it).  On a step that refreshes the caches (a batch refill)
// the refresh kernel has rewritten the rows first; a step with a latched
// action error is skipped (no mutation).
template <int W>
struct CtrlView {
  static constexpr int NT = 32 * W;
  double px[NT], py[NT], ch[NT], sh[NT], rad[NT], mh[NT];
  uint32_t uf[NT], zin[NT], vis[NT * W], atk[NT * W];
  uint32_t m_active[W], m_alive[W];
};

// K0 resident CTAs per SM the register budget is cut for: W = 1 6 (80
// registers; 4 and 5 measured neutral at C3), W > 1 4 (128 registers; C4
// refresh + K0 + K1 7.18 -> 7.05 ms)
#ifndef TABX_K0_THREADS
#define TABX_K0_THREADS 128  // threads per K0 CTA
#endif
#ifndef TABX_K0_MINB
#define TABX_K0_MINB(W) (((W) == 1 ? 768 : 512) / TABX_K0_THREADS)
#endif
template <int W>
__global__ void __launch_bounds__(TABX_K0_THREADS, TABX_K0_MINB(W)) ctrl_kernel(const Params P, int G, int NH) {
  if (P.sync->err_index != NO_ERROR) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  CtrlView<W>* V = reinterpret_cast<CtrlView<W>*>(smem_raw) + wib * G;
  const int N = P.N, Z = P.Z;
  const DevState& st = P.st;
  const int wpb = blockDim.x >> 5;
  const int64_t stride = (int64_t)gridDim.x * wpb * G;
  const int g = lane / NH, k = lane - g * NH;
  for (int64_t b0 = ((int64_t)blockIdx.x * wpb + wib) * G; b0 < P.B; b0 += stride) {
    TABX_POISON(V, sizeof(CtrlView<W>) * G, lane, 32);
    __syncwarp();
    for (int q = lane; q < G * W; q += 32) {
      V[q / W].m_active[q % W] = 0u;
      V[q / W].m_alive[q % W] = 0u;
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
      CtrlView<W>& view = V[gq];
      view.px[j] = p.x;
      view.py[j] = p.y;
      view.ch[j] = cs.x;
      view.sh[j] = cs.y;
      view.rad[j] = C->radius[j];
      view.mh[j] = mh;
      view.uf[j] = (act ? UF_ACTIVE : 0u) | (alive ? UF_ALIVE : 0u) |
                 (C->team[j] ? UF_ENEMY : 0u) | (C->kinematic[j] ? UF_KIN : 0u) |
                 (st.health[u] < mh ? UF_INJURED : 0u);
      view.zin[j] = st.zbits[u];
      if (act) atomicOr(&view.m_active[j >> 5], 1u << (j & 31));
      if (alive) atomicOr(&view.m_alive[j >> 5], 1u << (j & 31));
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
        TABX_ASSERT(i >= 0 && i < N);
        const int64_t u = b * N + i;
        const uint8_t ub = st.ubits[u];
        if (ub & U_ALIVE) {  // free: alive, active (hlist), lane running
          CtrlView<W>& view = V[g];
          const int team = C->team[i] ? 1 : 0;
          const double hd = st.heading[u], cd = st.cooldown[u];
          const uint32_t mask7 =
              0x1Fu | ((cd <= 0.0) ? 0x20u : 0u) | (C->enable_noop ? 0x40u : 0u);
          const double speff = C->speed[i] * swamp_mult(C, Z, view.zin[i], DC->swamp_m);
          const uint64_t seed = st.seed[b];
          const uint64_t t = (uint64_t)(int64_t)st.t[b];
          const double ue = uniform53(seed, t, TAG_EXPLORE, (uint64_t)i);
          const double up = uniform53(seed, t, TAG_PICK, (uint64_t)i);
#pragma unroll
          for (int w = 0; w < W; ++w) {
            view.vis[i * W + w] = st.vis[u * W + w];
            view.atk[i * W + w] = st.atk[u * W + w];
          }
          const double2 m = st.mem_pos[u];
          const int r = scripted_body<W>(view, C, i, N, Z, hd, cd, speff * C->dt, mask7, ue, up,
                                         C->epsilon[team], C->aggressive[team], DC->bush_m, m.x,
                                         m.y, (ub & U_MEMV) != 0);
          TABX_ASSERT((r & SA_ACT_MASK) < TABX_NUM_ACTIONS);
          TABX_JITTER(200);
          P.ctrl_act[u] = (int8_t)(r & SA_ACT_MASK);
          if (r & SA_HAS) {
            const int tg = r >> SA_TGT_SHIFT;
            st.mem_pos[u] = make_double2(view.px[tg], view.py[tg]);
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
template <int W>
cudaError_t launch_ctrl_t(const Params& P, int nh, int sm_count, cudaStream_t stream) {
  int G = nh < 32 ? 32 / nh : 1;
  if (G > 8) G = 8;
  if (W > 1) G = 1;
  const int NH = nh < 32 ? nh : 32;
  const int threads = TABX_K0_THREADS;
  const size_t smem = sizeof(CtrlView<W>) * G * (threads / 32);
  int per_sm = 1;
  cudaError_t e = launch_geometry((const void*)ctrl_kernel<W>, threads, smem, &per_sm);
  if (e != cudaSuccess) return e;
  const int64_t groups = (P.B + G - 1) / G;
  const int64_t need = (groups + threads / 32 - 1) / (threads / 32);
  const int64_t cap = (int64_t)sm_count * per_sm;
  const int grid = (int)(need < cap ? (need < 1 ? 1 : need) : cap);
  ctrl_kernel<W><<<grid, threads, smem, stream>>>(P, G, NH);
  return cudaGetLastError();
}

// ------------------------------------------------------------ launchers --
template <int W, int EPB, int M, int NF = 0, int ZF = 0>
cudaError_t launch_lanes_m(const Params& P, int sm_count, cudaStream_t stream, int* grid_out) {
  const int threads = 32 * W * EPB;
  const size_t env_bytes = (sizeof(EnvSmem<W>) * EPB + 15) & ~(size_t)15;
  const size_t smem = env_bytes + (M == MODE_RESET ? reset_view_bytes<W>(P) * EPB : 0);
  int per_sm = 1;
  cudaError_t e =
      launch_geometry((const void*)lane_kernel<W, EPB, M, NF, ZF>, threads, smem, &per_sm);
  if (e != cudaSuccess) return e;
  int64_t need = (P.B + EPB - 1) / EPB;
  int64_t cap = (int64_t)sm_count * per_sm;
  int grid = (int)(need < cap ? need : cap);
  if (grid < 1) grid = 1;
  if (grid_out) *grid_out = grid;
  lane_kernel<W, EPB, M, NF, ZF><<<grid, threads, smem, stream>>>(P);
  return cudaGetLastError();
}

// EPB: environments per CTA of the reset / init / refresh kernels; ES: of
// the step kernels (W = 1)
template <int W, int EPB, int ES = EPB>
cudaError_t launch_lanes_t(const Params& P, int sm_count, cudaStream_t stream, int* grid_out) {
  switch (P.mode) {
    case MODE_STEP: return launch_lanes_m<W, ES, MODE_STEP>(P, sm_count, stream, grid_out);
    case MODE_STEP_K0:
      // shape-specialised step kernels (C3 / C2 / C1 / C4 shapes); any other
      // shape, or TABX_GENERIC_SHAPES=1, takes the generic one
      if constexpr (W == 1) {
        if (!P.generic_shapes && P.N == 20 && P.Z == 6)
          return launch_lanes_m<1, ES, MODE_STEP_K0, 20, 6>(P, sm_count, stream, grid_out);
        if (!P.generic_shapes && P.N == 20 && P.Z == 0)
          return launch_lanes_m<1, ES, MODE_STEP_K0, 20, 0>(P, sm_count, stream, grid_out);
        if (!P.generic_shapes && P.N == 6 && P.Z == 0)
          return launch_lanes_m<1, ES, MODE_STEP_K0, 6, 0>(P, sm_count, stream, grid_out);
      }
      if constexpr (W == 4) {
        if (!P.generic_shapes && P.N == 100 && P.Z == 0)
          return launch_lanes_m<4, ES, MODE_STEP_K0, 100, 0>(P, sm_count, stream, grid_out);
      }
      return launch_lanes_m<W, ES, MODE_STEP_K0>(P, sm_count, stream, grid_out);
    case MODE_INIT: return launch_lanes_m<W, EPB, MODE_INIT>(P, sm_count, stream, grid_out);
    case MODE_REFRESH:
      return launch_lanes_m<W, EPB, MODE_REFRESH>(P, sm_count, stream, grid_out);
    default: return launch_lanes_m<W, EPB, MODE_RESET>(P, sm_count, stream, grid_out);
  }
}

}  // namespace tabx
