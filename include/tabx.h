/*
 * tabx.h -- C ABI of the B200-native batched environment step.
 *
 * Drop-in boundary for the reference engine's batch path.  Each entry point
 * replaces one piece of the reference's Python interface:
 *
 *   tabx_create        BatchSim.__init__            pkg/src/skirmish/environment.py:472-484
 *                      (+ make_batch lane seeding  pkg/bindings/src/skirmish_bindings/__init__.py:51-75)
 *   tabx_init_output   init_output / BatchSim.last  environment.py:351-374
 *   tabx_step          BatchSim.step -> step_kernel environment.py:500-519, :207-348
 *                      (+ bindings step            bindings/.../__init__.py:89-123)
 *   tabx_reset_env     BatchSim.reset_env           environment.py:490-498
 *   tabx_export_state  BatchSim.sim (SimArrays)     arrays.py:45-132
 *   tabx_import_state  (parity injection into SimArrays)
 *   tabx_get_error     ActionMaskError              environment.py:166-178, core.py:34
 *   tabx_episode_stats rollout.summarize inputs     rollout.py:122-147
 *
 * Conventions: plain pointers and sizes only.  Every pointer inside
 * tabx_outputs / tabx_state is a DEVICE pointer on the handle's device;
 * tabx_config / seeds are HOST pointers.  All work is enqueued on the
 * handle's stream; nothing synchronises except tabx_get_error /
 * tabx_episode_stats.  Every function returns TABX_OK (0) or an error code;
 * tabx_last_error() describes the last failure on the calling thread.
 * A handle must not be shared between threads (bindings/.../__init__.py:9-10).
 */
#ifndef TABX_H_
#define TABX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TABX_ABI_VERSION 6

#define TABX_MAX_UNITS 256
#define TABX_MAX_ZONES 32
#define TABX_MAX_CONFIGS 256
#define TABX_NUM_ACTIONS 7
#define TABX_OWN_DIM 15
#define TABX_OTHER_DIM 17
#define TABX_ZONE_DIM 8
#define TABX_NUM_STATS 8

/* status codes */
#define TABX_OK 0
#define TABX_E_ARGUMENT 1     /* bad pointer / size / index                 */
#define TABX_E_CUDA 2         /* CUDA runtime failure (see tabx_last_error) */
#define TABX_E_ACTION_MASK 3  /* an external action violated the mask       */
#define TABX_E_SHAPE 4        /* config capacities differ from the handle's */
#define TABX_E_ALIGNMENT 5    /* obs / global-state buffer not 16-B aligned */
#define TABX_E_CAPACITY 6     /* every config-table slot is in use          */

/* controller ids (core.py:138) */
#define TABX_CTRL_EXTERNAL 0
#define TABX_CTRL_HEURISTIC 1
#define TABX_CTRL_RANDOM 2

/* zone ids (arrays.py:24-27) */
#define TABX_ZONE_NONE 0
#define TABX_ZONE_LAVA 1
#define TABX_ZONE_BUSH 2
#define TABX_ZONE_SWAMP 3

/*
 * One scenario resolved to a device template: static unit columns, spawn
 * state, team controllers, physics and zones (arrays.py:244-321).  Angles are
 * radians and cos(sight_angle/2) is precomputed on the host with numpy so the
 * spawn state is bit-identical to the reference's fill_env.  Padding slots
 * (i >= number of configured units, i < n_units) carry the reference's
 * padding values (max_health 1, radius 0, mass 1, inv_mass 1, cos_half 1).
 */
typedef struct tabx_config {
  int32_t n_units;       /* capacity N = max_units, 1..TABX_MAX_UNITS */
  int32_t n_zones;       /* capacity Z = max_zones, 0..TABX_MAX_ZONES */
  int32_t max_steps;
  int32_t enable_noop;
  int32_t controller[2]; /* per team, TABX_CTRL_* */
  double epsilon[2];     /* heuristic exploration rate per team */
  double aggressive[2];  /* heuristic kiting threshold per team */
  double dt, restitution, slop, correction, rot_step, boundary_coeff, reveal_duration;
  double field_w, field_h;
  uint8_t active[TABX_MAX_UNITS];
  uint8_t team[TABX_MAX_UNITS];
  uint8_t kinematic[TABX_MAX_UNITS];
  uint8_t role_assassin[TABX_MAX_UNITS];
  uint8_t role_ranger[TABX_MAX_UNITS];
  uint8_t role_healer[TABX_MAX_UNITS];
  double max_health[TABX_MAX_UNITS];
  double radius[TABX_MAX_UNITS];
  double mass[TABX_MAX_UNITS];
  double inv_mass[TABX_MAX_UNITS];
  double speed[TABX_MAX_UNITS];
  double damage[TABX_MAX_UNITS];
  double attack_range[TABX_MAX_UNITS];
  double cooldown[TABX_MAX_UNITS];
  double sight_angle[TABX_MAX_UNITS];
  double sight_cos_half[TABX_MAX_UNITS];
  double sight_range[TABX_MAX_UNITS];
  double spawn_x[TABX_MAX_UNITS];
  double spawn_y[TABX_MAX_UNITS];
  double spawn_heading[TABX_MAX_UNITS];
  int32_t zone_type[TABX_MAX_ZONES];
  double zone_cx[TABX_MAX_ZONES];
  double zone_cy[TABX_MAX_ZONES];
  double zone_ax[TABX_MAX_ZONES];
  double zone_ay[TABX_MAX_ZONES];
  double zone_effect[TABX_MAX_ZONES];
} tabx_config;

/*
 * Per-step outputs (BatchOutput, environment.py:113-136), caller-owned
 * device buffers written in place; NULL skips a field.  observations and
 * global_state are float32 (the reference computes float64; values are the
 * float64 results rounded to nearest float32).  Bool arrays are one byte.
 * final_* rows are written only for lanes that auto-reset this step
 * (reset_mask[b] = 1); other rows are left untouched, so the reference's
 * final_observations equals where(reset_mask, final_observations, observations).
 * observations, final_observations, global_state and final_global_state
 * must be 16-byte aligned (they are written with TMA bulk stores); calls
 * given a misaligned one return TABX_E_ALIGNMENT before launching anything.
 */
typedef struct tabx_outputs {
  float* observations;        /* [B, N, obs_dim]          */
  float* global_state;        /* [B, global_dim]          */
  float* rewards;             /* [B, N]                   */
  uint8_t* action_mask;       /* [B, N, 7]                */
  uint8_t* terminated;        /* [B]                      */
  uint8_t* truncated;         /* [B]                      */
  uint8_t* done;              /* [B]                      */
  double* dense_reward;       /* [B]                      */
  int64_t* actions;           /* [B, N] executed actions  */
  uint8_t* interactions;      /* [B, N, N]                */
  int64_t* winner;            /* [B]                      */
  int64_t* reason;            /* [B]                      */
  int64_t* first_kill;        /* [B]                      */
  double* episode_return;     /* [B]                      */
  int64_t* episode_length;    /* [B]                      */
  float* final_observations;  /* [B, N, obs_dim]          */
  float* final_global_state;  /* [B, global_dim]          */
  uint8_t* reset_mask;        /* [B]                      */
  /* Optional policy feed (not in the reference): the current observation
   * rows again as bfloat16 (round to nearest even), row stride
   * observations_bf16_ld elements (>= obs_dim, a multiple of 8; the columns
   * from obs_dim on are zero), i.e. 16-byte aligned rows a policy network
   * reads directly.  Lanes that auto-reset get their fresh observation. */
  void* observations_bf16;      /* [B, N, observations_bf16_ld] bf16 */
  int64_t observations_bf16_ld;
} tabx_outputs;

/*
 * Dynamic state in the reference's SimArrays dtypes (arrays.py:45-117),
 * device pointers, for export (parity checks) and import (state injection).
 * vis/atk are [B, N, N] bools (row = observer / attacker).
 */
typedef struct tabx_state {
  uint64_t* seed;       /* [B]       */
  int64_t* episode;     /* [B]       */
  int64_t* t;           /* [B]       */
  double* pos;          /* [B, N, 2] */
  double* heading;      /* [B, N]    */
  double* vel;          /* [B, N, 2] */
  double* imp_dv;       /* [B, N, 2] */
  double* health;       /* [B, N]    */
  double* cooldown;     /* [B, N]    */
  double* reveal;       /* [B, N]    */
  uint8_t* alive;       /* [B, N]    */
  double* prev_gap;     /* [B]       */
  double* ep_return;    /* [B]       */
  uint8_t* done;        /* [B]       */
  uint8_t* terminated;  /* [B]       */
  uint8_t* truncated;   /* [B]       */
  int64_t* winner;      /* [B]       */
  int64_t* reason;      /* [B]       */
  int64_t* first_kill;  /* [B]       */
  double* mem_pos;      /* [B, N, 2] */
  uint8_t* mem_valid;   /* [B, N]    */
  uint8_t* vis;         /* [B, N, N] */
  uint8_t* atk;         /* [B, N, N] */
  int32_t* config;      /* [B] index into the handle's config table */
} tabx_state;

/* First offending external action in row-major (env, unit) order. */
typedef struct tabx_error {
  int32_t code;   /* TABX_OK or TABX_E_ACTION_MASK */
  int32_t unit;
  int64_t env;
  int64_t action;
} tabx_error;

/*
 * Level generation (scenario.py:563-826).
 * tabx_pcg64 is numpy's PCG64 bit-generator state (bit_generator.state:
 * 128-bit state and increment, has_uint32 / uinteger buffer).
 * tabx_level_spec is a LevelGenSpec resolved on the host: open categories,
 * the unit ranges in sorted-name order (attack_damage, max_health, speed),
 * the zone types in spec order, the centre box, axis range, effect ranges
 * indexed by TABX_ZONE_*, and the heuristic ranges.
 */
typedef struct tabx_pcg64 {
  uint64_t state_hi, state_lo;
  uint64_t inc_hi, inc_lo;
  uint32_t has_uint32, uinteger;
} tabx_pcg64;

typedef struct tabx_level_spec {
  int32_t open_units, open_zones, open_heuristic;
  int32_t unit_open[3];
  double unit_lo[3], unit_hi[3];
  int32_t n_zone_types;
  int32_t zone_types[3];
  double box_x0, box_x1, box_y0, box_y1;
  int32_t axis_open;
  double axis_lo, axis_hi;
  int32_t effect_open[4];
  double effect_lo[4], effect_hi[4];
  int32_t eps_open;
  double eps_lo, eps_hi;
  int32_t agg_open;
  double agg_lo, agg_hi;
} tabx_level_spec;

#define TABX_LEVEL_SAMPLE 0    /* sample_level(spec, rng), scenario.py:696-747 */
#define TABX_LEVEL_PERTURB 1   /* mutate_level(.., "perturb"), :773-812 */
#define TABX_LEVEL_SWAP_AXES 2 /* mutate_level(.., "swap_axes"), :814-818 */
#define TABX_LEVEL_RETYPE 3    /* mutate_level(.., "retype"), :819-826 */

typedef struct tabx_handle tabx_handle;

int tabx_abi_version(void);
const char* tabx_last_error(void);

/* Size of obs/global rows for capacities N, Z (perception.py:40-49). */
int32_t tabx_obs_dim(int32_t n_units, int32_t n_zones);
int32_t tabx_global_dim(int32_t n_units, int32_t n_zones);

/*
 * Create a batch of `batch` lanes on `device`.  configs[0..n_configs) share
 * n_units / n_zones; env_config[b] (host, may be NULL = all 0) picks lane b's
 * config; seeds[b] (host) is lane b's episode seed.  Lanes are spawned
 * immediately; call tabx_init_output to produce the first observations.
 * stream is a cudaStream_t (NULL = legacy default stream).
 */
int tabx_create(const tabx_config* configs, int32_t n_configs, const int32_t* env_config,
                const uint64_t* seeds, int64_t batch, int32_t auto_reset, int32_t device,
                void* stream, tabx_handle** out);
int tabx_destroy(tabx_handle* h);
int tabx_set_stream(tabx_handle* h, void* stream);
int tabx_dims(const tabx_handle* h, int64_t* batch, int32_t* n_units, int32_t* n_zones,
              int32_t* obs_dim, int32_t* global_dim);

/* init_output: refresh caches, prev_gap, observations, masks for all lanes. */
int tabx_init_output(tabx_handle* h, const tabx_outputs* out);

/*
 * One step of every lane.  actions: device int64 [B, N] or NULL (the
 * reference's step(None): non-scripted units NOOP).  When actions are given
 * and a team is external, they are validated first; on a violation no lane
 * is mutated and tabx_get_error reports TABX_E_ACTION_MASK.  Asynchronous.
 */
int tabx_step(tabx_handle* h, const int64_t* actions, const tabx_outputs* out);

/*
 * reset_env(b, config, seed): respawn lane b (optionally with a new config
 * and/or a new seed), then run init_output for the whole batch into `out`
 * (environment.py:490-498).  A config equal (byte for byte) to a row of the
 * handle's config table reuses that slot; otherwise it takes a slot no lane
 * uses any more (slots are reference-counted per lane) or a new one.  The
 * slot lane b runs on afterwards is stored in *slot_out (may be NULL).
 * Asynchronous: nothing waits on the stream (the config row is staged in
 * pinned memory, slot and seed are kernel arguments).
 */
int tabx_reset_env(tabx_handle* h, int64_t b, const tabx_config* config, uint64_t seed,
                   int32_t has_seed, const tabx_outputs* out, int32_t* slot_out);

/*
 * Respawn every lane with new seeds (host [B]) and episode counters 0, and
 * zero the statistics: the bindings' reset() (bindings/.../__init__.py:78-86).
 * Call tabx_init_output afterwards.
 */
int tabx_respawn_all(tabx_handle* h, const uint64_t* seeds, const int32_t* env_config);

int tabx_export_state(tabx_handle* h, const tabx_state* dst);
/*
 * Trace gather (rollout.py:150-188 records): row k of
 * dst (n_lanes rows, the tabx_state layout) <- lane lanes[k] (device int64
 * [n_lanes]).  Asynchronous on the handle's stream; unlike tabx_export_state
 * it never materialises a pending cache refresh, so it does not perturb the
 * batch (vis/atk rows are the stored caches).
 */
int tabx_export_lanes(tabx_handle* h, const int64_t* lanes, int64_t n_lanes,
                      const tabx_state* dst);
int tabx_import_state(tabx_handle* h, const tabx_state* src);

/*
 * Enqueue (on the handle's stream, no synchronisation) a copy of the latched
 * first offending (env * N + unit) index of an action-mask violation
 * (uint64, all ones = none) into dst (device or pinned host), for pipelined
 * callers that read it back together with their step results.
 */
int tabx_copy_error_word(tabx_handle* h, uint64_t* dst);

/* Synchronises the stream; reports (and with clear != 0 clears) the action error. */
int tabx_get_error(tabx_handle* h, tabx_error* err, int32_t clear);

/*
 * Episode statistics accumulated on device since creation or the last reset
 * (host double[TABX_NUM_STATS], synchronises): episodes, ally_wins,
 * first_kill_ally, truncation_ties, sum_length, sum_return, eliminations,
 * env_steps.  dst_device (may be NULL) receives the same vector on device for
 * an NCCL all-reduce.
 */
int tabx_episode_stats(tabx_handle* h, double* dst_host, double* dst_device, int32_t reset);

/*
 * Per-kernel timing of tabx_step (CUDA events on the handle's stream around
 * the step kernel, the observation kernel and the reset kernel).  With
 * enable != 0 accumulation restarts; tabx_get_profile synchronises and
 * returns the summed milliseconds ms[3] and the number of steps timed.
 */
int tabx_set_profiling(tabx_handle* h, int32_t enable);
int tabx_get_profile(tabx_handle* h, double* ms, int64_t* steps);

/*
 * Which kernels the last tabx_step ran: *fused = 0 for the separate step,
 * observation and reset kernels; 1 when the fused step + observation kernel
 * did (W = 1, heuristic-controller pass on, a shape with specialised kernels,
 * and TABX_FUSED=1 at creation: it is off by default); 2 for the
 * single-launch step (W = 1 batches below TABX_SINGLE_MAX_ENVS = 4,096 lanes
 * stepped with the in-kernel controller: step, observation rows and
 * auto-resets in one kernel).  With fused = 1 the profile's ms[0] covers the
 * refresh check + controller pass and ms[1] the fused kernel; with 2, ms[1]
 * is the single kernel.
 */
int tabx_step_path(const tabx_handle* h, int32_t* fused);

/*
 * Native pipelined host stepping (the trainer's host-array loop; the Python
 * bindings.HostStepper drives it).  tabx_pipe_create keeps `depth` (<=
 * TABX_PIPE_MAX_DEPTH) slots of device / pinned host buffers; `base` is the
 * handle's outputs (observations, masks, ... stay where they point; each
 * step's rewards / terminated / truncated go to the slot's own buffers);
 * `stream` is the handle's stream.  tabx_pipe_submit copies host int64
 * actions [B*N] (pinned memory for an asynchronous copy) to the device on an
 * upload stream, runs tabx_step, and downloads the slot's results on a
 * download stream, returning a ticket; it first waits until the results of
 * the step `depth` tickets earlier reached the host.  tabx_pipe_result
 * waits for ticket's results and returns pointers to them in pinned host
 * memory (valid until the slot is reused) and the latched action-error
 * index (-1: none; the caller clears the latch with tabx_get_error).
 */
#define TABX_PIPE_MAX_DEPTH 4
typedef struct tabx_pipe tabx_pipe;
int tabx_pipe_create(tabx_handle* h, int32_t depth, const tabx_outputs* base, void* stream,
                     tabx_pipe** out);
int tabx_pipe_submit(tabx_pipe* p, const int64_t* host_actions, int64_t* ticket);
int tabx_pipe_result(tabx_pipe* p, int64_t ticket, const float** rewards,
                     const uint8_t** terminated, const uint8_t** truncated,
                     int64_t* error_index);
int tabx_pipe_destroy(tabx_pipe* p);

/*
 * Config table management.  The table starts with the configs given to
 * tabx_create (plus those added by tabx_reset_env); tabx_reserve_configs
 * grows its capacity (synchronises; reallocates the table, so CUDA graphs
 * captured before must be re-captured), tabx_num_configs reports rows and
 * capacity, tabx_get_config copies one row to the host (synchronises).
 * tabx_config_slot reports how many lanes the host knows on `slot` and
 * whether the slot is pinned (never recycled: rows written by tabx_levels,
 * and every slot that existed when tabx_respawn_lanes / tabx_import_state
 * moved lanes by device data).
 */
int tabx_reserve_configs(tabx_handle* h, int32_t capacity);
int tabx_num_configs(tabx_handle* h, int32_t* count, int32_t* capacity);
int tabx_get_config(tabx_handle* h, int32_t slot, tabx_config* dst);
int tabx_config_slot(tabx_handle* h, int32_t slot, int64_t* lanes, int32_t* pinned);

/*
 * A batch of levels on the device, one per entry k < count: row
 * dst_first + k of the config table <- op applied to row src_slots[k]
 * (device int32 [count]; NULL = in place), drawing from rngs[k] (device
 * tabx_pcg64 [count], advanced in place exactly as numpy's generator would
 * be).  Source rows must not be destination rows of other entries.  The
 * table grows to dst_first + count rows (within the capacity).  Async.
 */
int tabx_levels(tabx_handle* h, int32_t op, const tabx_level_spec* spec, double delta,
                const int32_t* src_slots, int32_t dst_first, int32_t count, tabx_pcg64* rngs);

/*
 * Respawn lanes lanes[k] (device int64 [n]), first switching them to config
 * slots[k] (device int32, may be NULL) and seeds[k] (device uint64, may be
 * NULL): fill_env for a lane list (arrays.py:244-321).  Follow with
 * tabx_init_output, as reset_env does (environment.py:490-498).  Async.
 */
int tabx_respawn_lanes(tabx_handle* h, const int64_t* lanes, const int32_t* slots,
                       const uint64_t* seeds, int64_t n);

/* sizeof of the ABI structs, so bindings can check their mirrors. */
int tabx_struct_sizes(int64_t* config, int64_t* outputs, int64_t* state, int64_t* level_spec,
                      int64_t* pcg64);

/*
 * Policy helper of the on-device rollout loop (C5): for each of m agents,
 * Gumbel-max sample over the legal actions (mask row of 7 bytes) of its
 * logits (float32, or bfloat16 with logits_bf16 != 0; row stride ld >= 7
 * elements) and the sampled action's log-probability under the masked
 * softmax.  Noise = counter hash of (seed, *step_ptr + step_add, agent,
 * action); step_ptr (device, may be NULL) lets a replayed CUDA graph draw
 * fresh noise.  Asynchronous on `stream`.
 */
int tabx_masked_sample(const void* logits, int32_t logits_bf16, int64_t ld,
                       const uint8_t* mask, int64_t m, uint64_t seed, const uint64_t* step_ptr,
                       uint64_t step_add, int64_t* actions, float* logp, void* stream);

/*
 * Policy input of the rollout loop: float32 rows [rows, d] (observations) ->
 * bfloat16 rows [rows, dp], dp a multiple of 8, zero padded (16-byte aligned
 * GEMM operand).  Asynchronous on `stream`.
 */
int tabx_pack_bf16(const float* src, int64_t rows, int32_t d, int32_t dp, void* dst,
                   void* stream);

/*
 * Policy MLP of the rollout loop (C5) on the tcgen05 tensor cores, one pass
 * over the input: logits[r] = W2 · bf16(relu(W1 · x[r] + b1)) + b2 for rows
 * r < rows.  x: bfloat16 [rows, ldx] (first k features used; k and ldx
 * multiples of 8, 16-byte aligned), W1 bfloat16 [128, k], b1 [128], W2
 * bfloat16 [8, 128], b2 [8] (torch Linear layouts), logits bfloat16
 * [rows, 8], 16-byte aligned.  fp32 accumulation; the hidden activations are
 * rounded to bfloat16 like the torch module's.  Asynchronous on `stream`.
 */
int tabx_policy_mlp(const void* x, int64_t rows, int32_t k, int64_t ldx, const void* w1,
                    const void* b1, const void* w2, const void* b2, void* logits, void* stream);

/*
 * tabx_policy_mlp with the masked sampler (tabx_masked_sample semantics, on
 * the bfloat16 logits) fused into its epilogue: actions / logp per row from
 * mask [rows, 7] and the noise counter (seed, *step_ptr + step_add).  logits
 * may be NULL (not written) when k <= 704; larger k needs the buffer (the
 * sampler then runs as a second kernel).  Asynchronous on `stream`.
 */
int tabx_policy_mlp_sample(const void* x, int64_t rows, int32_t k, int64_t ldx, const void* w1,
                           const void* b1, const void* w2, const void* b2, void* logits,
                           const uint8_t* mask, uint64_t seed, const uint64_t* step_ptr,
                           uint64_t step_add, int64_t* actions, float* logp, void* stream);

/*
 * Tool hook: SM cycles per step phase summed over envs (all step kernels),
 * nonzero only in a build with -DTABX_PHASE_PROF (tools/phase_prof.py).
 */
int tabx_debug_phase_cycles(uint64_t* host16, int32_t reset);

/* Test hook: libm-equal sin/cos of n device doubles (tabx_math.cuh). */
int tabx_debug_sincos(const double* x, double* s, double* c, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TABX_H_ */
