// Device-side data structures shared by the step kernels and the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tabx.h"
#include <math.h>

namespace tabx {

// ---- checked build (-DTABX_CHECKS; test infrastructure):
// device asserts on indices and store ranges, per-lane random delays at
// the step's phase boundaries (a shared-memory hand-off missing its
// __syncwarp / __syncthreads then reads a stale value, which the bit-exact
// parity tests see), and shared memory poisoned before each environment
// (a read of a value this environment never wrote is a NaN / garbage).
#ifdef TABX_CHECKS
#include <stdio.h>
#define TABX_ASSERT(c)                                                             \
  do {                                                                             \
    if (!(c)) {                                                                    \
      printf("TABX_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
             (int)blockIdx.x, (int)threadIdx.x);                                   \
      __trap();                                                                    \
    }                                                                              \
  } while (0)
__device__ __forceinline__ void tabx_jitter(unsigned k) {
  unsigned x = (unsigned)clock() ^ (threadIdx.x * 0x9E3779B9u) ^ (blockIdx.x * 0x85EBCA6Bu) ^
               (k * 0xC2B2AE35u);
  x ^= x >> 15;
  x *= 0x2C1B3C6Du;
  x ^= x >> 12;
  __nanosleep(x & 1023u);
}
#define TABX_JITTER(k) ::tabx::tabx_jitter(k)
// fill [p, p + bytes) with 0xFF bytes (float NaN, int -1) from `n` threads
__device__ __forceinline__ void tabx_poison(void* p, size_t bytes, int t, int n) {
  uint32_t* w = reinterpret_cast<uint32_t*>(p);
  for (size_t q = t; q < bytes / 4; q += n) w[q] = 0xFFFFFFFFu;
}
#define TABX_POISON(p, bytes, t, n) ::tabx::tabx_poison(p, bytes, t, n)
#else
#define TABX_ASSERT(c) \
  do {                 \
  } while (0)
#define TABX_JITTER(k) \
  do {                 \
  } while (0)
#define TABX_POISON(p, bytes, t, n) \
  do {                              \
  } while (0)
#endif

// ---- path counters (-DTABX_COUNT_PROF, tools/count_prof.py): how often the
// exact float64 fallbacks run; slot k of tabx_phase_cycles (the phase-profile
// array, read back with tabx_debug_phase_cycles)
#if defined(TABX_PHASE_PROF) || defined(TABX_COUNT_PROF)
__device__ unsigned long long tabx_phase_cycles[16];
#endif
#ifdef TABX_COUNT_PROF
#define TABX_COUNT(k) atomicAdd(&::tabx::tabx_phase_cycles[k], 1ull)
#else
#define TABX_COUNT(k) \
  do {                \
  } while (0)
#endif

constexpr int A_ROTATE = 4;
constexpr int A_ATTACK = 5;
constexpr int A_NOOP = 6;
constexpr int ALLY = 0;
constexpr int ENEMY = 1;
constexpr int R_NONE = 0, R_ELIM = 1, R_TRUNC = 2, R_TIE = 3;
constexpr unsigned long long NO_ERROR = ~0ull;

constexpr int TAG_RESEED = 2, TAG_EXPLORE = 3, TAG_PICK = 4, TAG_RANDOM = 5;

// lane flag bits (DevState::flags)
constexpr uint8_t F_DONE = 1, F_TERM = 2, F_TRUNC = 4;
constexpr uint8_t F_PEND = 8;  // auto-reset pending (step kernel -> reset kernel)
// unit bits (DevState::ubits)
constexpr uint8_t U_ALIVE = 1, U_MEMV = 2;

// Internal structure-of-arrays state (handle-owned HBM).  Per-unit arrays are
// [B*N] (unit u = b*N + i); the visibility / attackable caches are N-bit row
// masks, [B*N*W] words.
struct DevState {
  uint64_t* seed;
  int64_t* episode;
  int32_t* t;
  double* prev_gap;
  double* ep_return;
  uint8_t* flags;
  int8_t* winner;
  int8_t* reason;
  int8_t* first_kill;
  int32_t* cfg;
  double2* pos;
  double* heading;
  double2* vel;
  double2* imp_dv;
  double* health;
  double* cooldown;
  double* reveal;
  double2* mem_pos;
  double2* hcs;      // cached (cos, sin) of heading, libm-exact
  uint32_t* zbits;   // zone-membership bits at the current position
  uint8_t* ubits;
  uint32_t* vis;
  uint32_t* atk;
  // per-lane episode statistics (deterministic on-demand reduction)
  uint32_t* st_episodes;
  uint32_t* st_wins;
  uint32_t* st_fk_ally;
  uint32_t* st_ties;
  uint32_t* st_elims;
  int64_t* st_len;
  double* st_ret;
  int64_t* st_base;  // env_steps bookkeeping (stats_kernel)
};

// Control block: action-error latch, device step counter and the
// three-slot "some lane was refilled" flag ring (cache refresh).
struct Sync {
  unsigned long long err_index;
  uint32_t step;
  uint32_t blocks_done;
  int32_t refresh[3];
  int32_t any_pend;  // some lane awaits its auto-reset (K1 sets, K3 clears)
};

// Per-config values derived once on the device (not part of the ABI):
// reciprocals for the fast exact-rounding paths, float copies for filters.
struct DerivedCfg {
  double rw, rh;                      // 1/field_w, 1/field_h
  double rad_max;                     // largest radius of an active unit (contact sweep window)
  double rax[TABX_MAX_ZONES], ray[TABX_MAX_ZONES];
  double rmh[TABX_MAX_UNITS];         // 1/max_health
  double rucd[TABX_MAX_UNITS];        // 1/cooldown (0 if cooldown == 0)
  uint32_t lava_m, bush_m, swamp_m;   // zone-type bit masks
  int32_t n_ally, n_enemy;            // team roster sizes (active units)
  // active units of heuristic-controlled teams (K0's work list, ascending)
  int32_t n_heur;
  uint8_t hlist[TABX_MAX_UNITS];
  // float32 zone blocks (perception.py:170-201), zeros for unused slots:
  // observation block with the two relative-position features left 0, and
  // the global-state block (absolute position / field size)
  float zobs[TABX_MAX_ZONES * TABX_ZONE_DIM];
  float zglob[TABX_MAX_ZONES * TABX_ZONE_DIM];
};

// MODE_STEP_K0: the step kernel when K0 (the heuristic-controller pass) made
// the heuristic decisions; it carries no controller code of its own
enum Mode : int { MODE_STEP = 0, MODE_INIT = 1, MODE_REFRESH = 2, MODE_RESET = 3, MODE_STEP_K0 = 4 };
__host__ __device__ constexpr bool is_step_mode(int m) { return m == MODE_STEP || m == MODE_STEP_K0; }

struct Params {
  DevState st;
  const tabx_config* cfgs;
  const DerivedCfg* dcfgs;
  Sync* sync;
  const int64_t* actions;  // [B*N] or nullptr
  tabx_outputs out;
  int64_t B;
  int N, Z, D, G;
  int auto_reset;
  int mode;
  // K0 (heuristic controller pass): its action per unit, or nullptr
  // when K1 runs the controller itself
  int8_t* ctrl_act;
  int generic_shapes;  // 1: no shape-specialised kernel instantiations
};

__device__ __noinline__ static bool zone_exact(double ex, double ey, double ax, double ay) {
  TABX_COUNT(6);
  const double qx = ex / ax;
  const double qy = ey / ay;
  return qx * qx + qy * qy <= 1.0;
}

// Zone membership bits at (x, y) (arrays.py:329-335).  The reference
// divides by the semi-axes; here the quotients are first estimated with the
// precomputed reciprocals (error < 3 ulp) and the exact division is redone
// only when the ellipse sum lands within 1e-9 of 1.
__device__ __forceinline__ uint32_t zone_bits(const tabx_config* __restrict__ C,
                                              const DerivedCfg* __restrict__ DC, int Z, double x,
                                              double y) {
  uint32_t bits = 0;
  (void)Z;
  // the typed zones (lava | bush | swamp) by their bits: no per-zone type load
  for (uint32_t m = DC->lava_m | DC->bush_m | DC->swamp_m; m; m &= m - 1) {
    const int z = __ffs(m) - 1;
    const double ex = x - C->zone_cx[z];
    const double ey = y - C->zone_cy[z];
    const double ax = ex * DC->rax[z], ay = ey * DC->ray[z];
    const double s = ax * ax + ay * ay;
    bool in;
    if (s < 1.0 - 1e-9) {
      in = true;
    } else if (s > 1.0 + 1e-9) {
      in = false;
    } else {
      in = zone_exact(ex, ey, C->zone_ax[z], C->zone_ay[z]);
    }
    if (in) bits |= 1u << z;
  }
  return bits;
}

// Rare exact fallbacks live out of line: a call cannot be speculated, so the
// float64 division / square-root sequences only run on the lanes that need
// them instead of being if-converted into every warp's path.
static __device__ __noinline__ double slow_div(double x, double y) { return x / y; }
static __device__ __noinline__ double slow_sqrt(double x) { return sqrt(x); }

__device__ __forceinline__ float f32_quot(double x, double y, double ry) {
  double q = x * ry;
  const uint32_t lo = (uint32_t)__double2loint(q), hi = (uint32_t)__double2hiint(q);
  // low 29 bits within 8 of the float32 rounding midpoint 0x10000000
  const bool mid = ((lo - 0x0FFFFFF8u) & 0x1FFFFFFFu) <= 16u;
  // |q| outside [2^-125, 2^123) (float32 subnormal / overflow range, inf, nan)
  // and not zero
  const uint32_t e = (hi >> 20) & 0x7FFu;
  const bool odd = (e - 898u) > 247u && ((hi & 0x7FFFFFFFu) | lo) != 0u;
  if (mid || odd) {
    TABX_COUNT(7);
    q = slow_div(x, y);
  }
  return __double2float_rn(q);
}

// Launch geometry of a kernel with `smem` bytes of dynamic shared memory on
// the CURRENT device: raises the kernel's dynamic shared-memory limit there
// (a per-device attribute) and returns its resident blocks per SM.  Results
// are cached per (kernel, device, smem) behind a mutex, so a step costs one
// launch per kernel, stays capturable in a CUDA graph, and handles on
// several devices (or threads) each get the attribute set on their own GPU.
cudaError_t launch_geometry(const void* kernel, int threads, size_t smem, int* per_sm);
}  // namespace tabx
