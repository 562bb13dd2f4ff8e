// C ABI (include/tabx.h): handle lifetime, config table, launches.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "tabx_device.cuh"
#include "tabx_sample.cuh"

namespace tabx {
cudaError_t launch_lanes(const Params& P, int W, int sm_count, cudaStream_t stream, int* grid);
cudaError_t launch_ctrl(const Params& P, int W, int nh, int sm_count, cudaStream_t stream);
cudaError_t launch_emit(const Params& P, int W, int sm_count, cudaStream_t stream);
cudaError_t launch_fused_w1(const Params& P, int variant, int sm_count, cudaStream_t stream);
cudaError_t launch_small_w1(const Params& P, int sm_count, cudaStream_t stream);
bool mlp_fused_sampling(int K);
cudaError_t launch_mlp_policy(const void* x, int64_t rows, int K, int64_t ldx, const void* w1,
                              const void* b1, const void* w2, const void* b2, void* out,
                              const MlpSample& sa, int sm_count, cudaStream_t stream);
cudaError_t launch_validate(const int64_t* actions, const DevState& st, const tabx_config* cfgs,
                            int64_t B, int N, Sync* sync, int sm_count, cudaStream_t stream);
cudaError_t launch_spawn(const DevState& st, const tabx_config* cfgs, const DerivedCfg* dcfgs,
                         int64_t b0, int64_t b1, int N, int W, int reset_stats, int sm_count,
                         cudaStream_t stream);
cudaError_t launch_derive(const tabx_config* cfgs, DerivedCfg* dcfgs, int k0, int k1,
                          cudaStream_t stream);
cudaError_t launch_levels(tabx_config* cfgs, const int32_t* src_slots, int32_t dst_first,
                          int32_t count, const tabx_level_spec& spec, int op, double delta,
                          tabx_pcg64* rngs, int sm_count, cudaStream_t stream);
cudaError_t launch_spawn_one(const DevState& st, const tabx_config* cfgs, const DerivedCfg* dcfgs,
                             int64_t b, int32_t slot, uint64_t seed, int has_seed, int N, int W,
                             cudaStream_t stream);
cudaError_t launch_spawn_lanes(const DevState& st, const tabx_config* cfgs,
                               const DerivedCfg* dcfgs, const int64_t* lanes, const int32_t* slots,
                               const uint64_t* seeds, int64_t n, int N, int W, int sm_count,
                               cudaStream_t stream);
cudaError_t phase_cycles_w1(unsigned long long* host16, int reset);
cudaError_t phase_cycles_w2(unsigned long long* host16, int reset);
cudaError_t phase_cycles_w4(unsigned long long* host16, int reset);
cudaError_t phase_cycles_w8(unsigned long long* host16, int reset);
cudaError_t launch_masked_sample(const void* logits, int bf16, int64_t ld, const uint8_t* mask,
                                 int64_t M, uint64_t seed, const uint64_t* step_ptr,
                                 uint64_t step_add, int64_t* actions, float* logp, int sm_count,
                                 cudaStream_t stream);
cudaError_t launch_pack_bf16(const float* src, int64_t rows, int D, int Dp, void* dst,
                             int sm_count, cudaStream_t stream);
cudaError_t launch_export(const DevState& st, const tabx_state& d, const int64_t* lanes,
                          int64_t rows, int N, int W, int sm_count, cudaStream_t stream);
cudaError_t launch_import(const DevState& st, const tabx_state& s, const tabx_config* cfgs,
                          const DerivedCfg* dcfgs, int64_t B, int N, int W, int sm_count,
                          cudaStream_t stream);
cudaError_t launch_stats(const DevState& st, int64_t B, double* out, int reset,
                         cudaStream_t stream);
cudaError_t launch_sincos_debug(const double* x, double* s, double* c, int64_t n,
                                cudaStream_t stream);
}  // namespace tabx

using namespace tabx;

struct tabx_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t B = 0;
  int N = 0, Z = 0, W = 1, D = 0, G = 0;
  int auto_reset = 0;
  int sm_count = 148;
  bool any_external = false;
  // K0 (heuristic controller pass): per-unit actions, and the
  // heuristic units per env over the config table (recounted when it changes)
  int8_t* ctrl_act = nullptr;
  int cfg_version = 0, ctrl_version = -1, ctrl_nh = 0;
  int generic_shapes = 0;  // TABX_GENERIC_SHAPES=1: skip the shape-specialised kernels
  // fused step + observation kernel (W = 1, K0 path; tabx_fused.cu): its
  // variant, -1 = off (the default; TABX_FUSED=1 turns it on); whether the
  // last step ran it
  int fused = 0;
  int fused_ran = 0;  // 1: fused step + observation kernel, 2: single-launch small step
  // single-launch step (K1 + K2 + K3 in one kernel) for W = 1 batches below
  // this many lanes stepped with the in-kernel controller (TABX_SINGLE_MAX_ENVS,
  // 0 = off)
  int64_t single_max = 4096;
  std::vector<tabx_config> cfg_host;  // host mirror of the table rows
  std::vector<char> cfg_host_ok;       // 0: row written on the device (tabx_levels)
  int cfg_cap = TABX_MAX_CONFIGS;
  // Config-slot recycling.  lane_slot mirrors st.cfg for every change the
  // host makes (create, reset_env, respawn_all); refcnt[k] counts the lanes
  // on slot k.  A slot whose count drops to 0 is reused by the next new
  // config.  Slots the host cannot track — rows written on the device
  // (tabx_levels) and every slot that existed when lanes were moved by device
  // data (tabx_respawn_lanes with slots, tabx_import_state with config) — are
  // pinned: never recycled.  row_hash / by_hash find an identical row in O(1).
  std::vector<int32_t> lane_slot;
  std::vector<int64_t> refcnt;
  std::vector<char> pinned;
  std::vector<uint64_t> row_hash;
  std::unordered_multimap<uint64_t, int32_t> by_hash;
  std::vector<int32_t> free_slots;
  // pinned staging ring for config rows uploaded by tabx_reset_env (a
  // cudaMemcpyAsync from pageable memory would block on the stream)
  static constexpr int STAGE_SLOTS = 8;
  tabx_config* stage = nullptr;
  cudaEvent_t stage_ev[STAGE_SLOTS] = {};
  int stage_next = 0;
  tabx_config* cfg_dev = nullptr;
  DerivedCfg* dcfg_dev = nullptr;
  DevState st{};
  void* arena = nullptr;
  Sync* sync = nullptr;
  double* stats_dev = nullptr;
  const int64_t* last_actions = nullptr;
  // optional per-kernel timing of tabx_step (bench roofline): ring of event sets
  static constexpr int PROF_SLOTS = 256;
  bool profiling = false;
  cudaEvent_t prof_ev[PROF_SLOTS][4] = {};
  int prof_next = 0, prof_pending = 0;
  double prof_ms[3] = {0.0, 0.0, 0.0};
  int64_t prof_steps = 0;
};

static void prof_collect(tabx_handle* h, int slot) {
  float ms[3];
  cudaEventSynchronize(h->prof_ev[slot][3]);
  for (int k = 0; k < 3; ++k) {
    cudaEventElapsedTime(&ms[k], h->prof_ev[slot][k], h->prof_ev[slot][k + 1]);
    h->prof_ms[k] += ms[k];
  }
  h->prof_steps += 1;
}

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

static int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return TABX_E_CUDA;
}

#define TABX_CUDA(call, what)                 \
  do {                                        \
    cudaError_t e_ = (call);                  \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

static int words_for(int N) {
  int w = (N + 31) / 32;
  if (w <= 1) return 1;
  if (w <= 2) return 2;
  if (w <= 4) return 4;
  return 8;
}

static Params make_params(tabx_handle* h, int mode, const int64_t* actions,
                          const tabx_outputs* out) {
  Params P;
  P.st = h->st;
  P.cfgs = h->cfg_dev;
  P.dcfgs = h->dcfg_dev;
  P.sync = h->sync;
  P.actions = actions;
  if (out) {
    P.out = *out;
  } else {
    memset(&P.out, 0, sizeof(P.out));
  }
  P.B = h->B;
  P.N = h->N;
  P.Z = h->Z;
  P.D = h->D;
  P.G = h->G;
  P.auto_reset = h->auto_reset;
  P.mode = mode;
  P.ctrl_act = nullptr;
  P.generic_shapes = h->generic_shapes;
  return P;
}

// Heuristic-controlled active units per env, maximised over the config
// table (rows written on the device count as all N).
static int ctrl_units(tabx_handle* h) {
  if (h->ctrl_version == h->cfg_version) return h->ctrl_nh;
  const int lim = h->N;
  int nh = 0;
  for (size_t k = 0; k < h->cfg_host.size(); ++k) {
    if (!h->cfg_host_ok[k]) {
      nh = lim;
      break;
    }
    const tabx_config& c = h->cfg_host[k];
    int n = 0;
    for (int i = 0; i < lim; ++i)
      if (c.active[i] && c.controller[c.team[i] ? 1 : 0] == TABX_CTRL_HEURISTIC) ++n;
    if (n > nh) nh = n;
  }
  h->ctrl_nh = nh;
  h->ctrl_version = h->cfg_version;
  return nh;
}

static int check_outputs(const tabx_outputs* out, int D) {
  if (!out) return TABX_OK;
  // rows leave through TMA bulk stores (cp.async.bulk), which need a
  // 16-byte-aligned base
  const float* ptrs[4] = {out->observations, out->final_observations, out->global_state,
                          out->final_global_state};
  for (const float* p : ptrs)
    if (p && (((uintptr_t)p) & 15u))
      return fail(TABX_E_ALIGNMENT,
                  "observation / global-state buffers must be 16-byte aligned");
  if (out->observations_bf16 && ((((uintptr_t)out->observations_bf16) & 15u) ||
                                 (out->observations_bf16_ld & 7) ||
                                 out->observations_bf16_ld < D))
    return fail(TABX_E_ALIGNMENT,
                "bfloat16 observation rows must be 16-byte aligned (ld a multiple of 8)");
  return TABX_OK;
}

static uint64_t config_hash(const tabx_config* c) {
  // FNV-1a over 64-bit words (the struct is a multiple of 8 bytes)
  const uint64_t* w = reinterpret_cast<const uint64_t*>(c);
  uint64_t x = 0xcbf29ce484222325ull;
  for (size_t k = 0; k < sizeof(tabx_config) / 8; ++k) {
    x ^= w[k];
    x *= 0x100000001b3ull;
  }
  return x;
}

static void slot_unindex(tabx_handle* h, int32_t k) {
  auto range = h->by_hash.equal_range(h->row_hash[k]);
  for (auto it = range.first; it != range.second; ++it)
    if (it->second == k) {
      h->by_hash.erase(it);
      return;
    }
}

// Recount the per-slot lane counts from the host mirror; rebuild the free list.
static void recount_slots(tabx_handle* h) {
  const size_t n = h->cfg_host.size();
  h->refcnt.assign(n, 0);
  for (int32_t k : h->lane_slot) h->refcnt[k] += 1;
  h->free_slots.clear();
  for (size_t k = n; k-- > 0;)
    if (!h->refcnt[k] && !h->pinned[k]) {
      slot_unindex(h, (int32_t)k);
      h->free_slots.push_back((int32_t)k);
    }
}

// Lanes were moved by device-side data: the mirror is no longer exact, so
// every existing slot is kept forever (counts stay upper bounds).
static void pin_all_slots(tabx_handle* h) {
  for (size_t k = 0; k < h->pinned.size(); ++k) h->pinned[k] = 1;
  h->free_slots.clear();
}

static void move_lane(tabx_handle* h, int64_t b, int32_t k) {
  const int32_t old = h->lane_slot[b];
  if (old == k) return;
  h->lane_slot[b] = k;
  h->refcnt[k] += 1;
  if (--h->refcnt[old] == 0 && !h->pinned[old]) {
    slot_unindex(h, old);
    h->free_slots.push_back(old);
  }
}

// The pinned staging ring for config rows (tabx_reset_env).  Allocated at
// creation: a page-locked allocation can take ~100 ms, which on first use
// made the first new-config reset_env the protocol's worst case.
static cudaError_t alloc_stage(tabx_handle* h) {
  if (h->stage) return cudaSuccess;
  cudaError_t e = cudaHostAlloc((void**)&h->stage, sizeof(tabx_config) * tabx_handle::STAGE_SLOTS,
                                cudaHostAllocDefault);
  for (int q = 0; e == cudaSuccess && q < tabx_handle::STAGE_SLOTS; ++q)
    e = cudaEventCreateWithFlags(&h->stage_ev[q], cudaEventDisableTiming);
  return e;
}

static int stage_config(tabx_handle* h, const tabx_config* c, const tabx_config** staged) {
  TABX_CUDA(alloc_stage(h), "config staging allocation");
  const int q = h->stage_next;
  h->stage_next = (q + 1) % tabx_handle::STAGE_SLOTS;
  // the copy that last used this staging row must have read it (normally
  // long done: STAGE_SLOTS uploads ago)
  TABX_CUDA(cudaEventSynchronize(h->stage_ev[q]), "staging wait");
  memcpy(h->stage + q, c, sizeof(tabx_config));
  *staged = h->stage + q;
  return TABX_OK;
}

static int stage_done(tabx_handle* h, const tabx_config* staged) {
  const int q = (int)(staged - h->stage);
  TABX_CUDA(cudaEventRecord(h->stage_ev[q], h->stream), "staging record");
  return TABX_OK;
}

// The table slot holding a row equal to *c (same bytes), else a recycled
// free slot or a new one with *c uploaded and derived on the stream.
static int find_or_add_config(tabx_handle* h, const tabx_config* c, int32_t* idx) {
  if (c->n_units != h->N || c->n_zones != h->Z)
    return fail(TABX_E_SHAPE, "batched environments must share max_units and max_zones");
  const uint64_t hs = config_hash(c);
  auto range = h->by_hash.equal_range(hs);
  for (auto it = range.first; it != range.second; ++it) {
    const int32_t k = it->second;
    if (h->cfg_host_ok[k] && !memcmp(&h->cfg_host[k], c, sizeof(tabx_config))) {
      *idx = k;
      return TABX_OK;
    }
  }
  int32_t k;
  if (!h->free_slots.empty()) {
    k = h->free_slots.back();
    h->free_slots.pop_back();
    h->cfg_host[k] = *c;
    h->cfg_host_ok[k] = 1;
  } else {
    if ((int)h->cfg_host.size() >= h->cfg_cap)
      return fail(TABX_E_CAPACITY,
                  "config table full: every slot is in use by a lane (tabx_reserve_configs)");
    h->cfg_host.push_back(*c);
    h->cfg_host_ok.push_back(1);
    h->refcnt.push_back(0);
    h->pinned.push_back(0);
    h->row_hash.push_back(0);
    k = (int32_t)h->cfg_host.size() - 1;
  }
  h->row_hash[k] = hs;
  h->by_hash.emplace(hs, k);
  ++h->cfg_version;
  const tabx_config* staged = nullptr;
  int rc = stage_config(h, c, &staged);
  if (rc) return rc;
  TABX_CUDA(cudaMemcpyAsync(h->cfg_dev + k, staged, sizeof(tabx_config), cudaMemcpyHostToDevice,
                            h->stream),
            "config upload");
  rc = stage_done(h, staged);
  if (rc) return rc;
  TABX_CUDA(launch_derive(h->cfg_dev, h->dcfg_dev, (int)k, (int)k + 1, h->stream), "derive");
  if (c->controller[0] == TABX_CTRL_EXTERNAL || c->controller[1] == TABX_CTRL_EXTERNAL)
    h->any_external = true;
  *idx = k;
  return TABX_OK;
}

extern "C" {

int tabx_abi_version(void) { return TABX_ABI_VERSION; }

const char* tabx_last_error(void) { return g_err.c_str(); }

int32_t tabx_obs_dim(int32_t n, int32_t z) {
  return TABX_OWN_DIM + (n - 1) * TABX_OTHER_DIM + z * TABX_ZONE_DIM;
}

int32_t tabx_global_dim(int32_t n, int32_t z) { return n * TABX_OWN_DIM + z * TABX_ZONE_DIM; }

int tabx_create(const tabx_config* configs, int32_t n_configs, const int32_t* env_config,
                const uint64_t* seeds, int64_t batch, int32_t auto_reset, int32_t device,
                void* stream, tabx_handle** out) {
  if (!configs || n_configs < 1 || !seeds || batch < 1 || !out)
    return fail(TABX_E_ARGUMENT, "tabx_create: bad argument");
  const int N = configs[0].n_units, Z = configs[0].n_zones;
  if (N < 1 || N > TABX_MAX_UNITS || Z < 0 || Z > TABX_MAX_ZONES)
    return fail(TABX_E_ARGUMENT, "unit / zone capacity out of range");
  for (int k = 1; k < n_configs; ++k)
    if (configs[k].n_units != N || configs[k].n_zones != Z)
      return fail(TABX_E_SHAPE, "batched environments must share max_units and max_zones");
  if (env_config)
    for (int64_t b = 0; b < batch; ++b)
      if (env_config[b] < 0 || env_config[b] >= n_configs)
        return fail(TABX_E_ARGUMENT, "env_config index out of range");
  DeviceGuard guard(device);
  tabx_handle* h = new tabx_handle();
  h->device = device;
  h->stream = (cudaStream_t)stream;
  h->B = batch;
  h->N = N;
  h->Z = Z;
  h->W = words_for(N);
  h->D = tabx_obs_dim(N, Z);
  h->G = tabx_global_dim(N, Z);
  h->auto_reset = auto_reset ? 1 : 0;
  cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, device);

  const int64_t B = batch, U = batch * N, W = h->W;
  // arena layout (all sub-arrays 256-byte aligned)
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  size_t o_seed = take(8 * B), o_ep = take(8 * B), o_t = take(4 * B), o_pg = take(8 * B),
         o_ret = take(8 * B), o_flags = take(B), o_win = take(B), o_rea = take(B),
         o_fk = take(B), o_cfg = take(4 * B), o_pos = take(16 * U), o_hd = take(8 * U),
         o_vel = take(16 * U), o_imp = take(16 * U), o_hp = take(8 * U), o_cd = take(8 * U),
         o_rv = take(8 * U), o_mem = take(16 * U), o_hcs = take(16 * U), o_zb = take(4 * U),
         o_ub = take(U), o_vis = take(4 * U * W),
         o_atk = take(4 * U * W), o_se = take(4 * B), o_sw = take(4 * B), o_sf = take(4 * B),
         o_stie = take(4 * B), o_sel = take(4 * B), o_sl = take(8 * B), o_sr = take(8 * B),
         o_sync = take(sizeof(Sync)), o_stats = take(8 * TABX_NUM_STATS), o_ctl = take(U),
         o_sb = take(8 * B);
  cudaError_t e = cudaMalloc(&h->arena, off);
  if (e != cudaSuccess) {
    delete h;
    return cuda_fail(e, "state allocation");
  }
  e = cudaMalloc((void**)&h->cfg_dev, sizeof(tabx_config) * TABX_MAX_CONFIGS);
  if (e == cudaSuccess)
    e = cudaMalloc((void**)&h->dcfg_dev, sizeof(DerivedCfg) * TABX_MAX_CONFIGS);
  if (e != cudaSuccess) {
    cudaFree(h->cfg_dev);
    cudaFree(h->arena);
    delete h;
    return cuda_fail(e, "config table allocation");
  }
  char* a = (char*)h->arena;
  DevState& st = h->st;
  st.seed = (uint64_t*)(a + o_seed);
  st.episode = (int64_t*)(a + o_ep);
  st.t = (int32_t*)(a + o_t);
  st.prev_gap = (double*)(a + o_pg);
  st.ep_return = (double*)(a + o_ret);
  st.flags = (uint8_t*)(a + o_flags);
  st.winner = (int8_t*)(a + o_win);
  st.reason = (int8_t*)(a + o_rea);
  st.first_kill = (int8_t*)(a + o_fk);
  st.cfg = (int32_t*)(a + o_cfg);
  st.pos = (double2*)(a + o_pos);
  st.heading = (double*)(a + o_hd);
  st.vel = (double2*)(a + o_vel);
  st.imp_dv = (double2*)(a + o_imp);
  st.health = (double*)(a + o_hp);
  st.cooldown = (double*)(a + o_cd);
  st.reveal = (double*)(a + o_rv);
  st.mem_pos = (double2*)(a + o_mem);
  st.hcs = (double2*)(a + o_hcs);
  st.zbits = (uint32_t*)(a + o_zb);
  st.ubits = (uint8_t*)(a + o_ub);
  st.vis = (uint32_t*)(a + o_vis);
  st.atk = (uint32_t*)(a + o_atk);
  st.st_episodes = (uint32_t*)(a + o_se);
  st.st_wins = (uint32_t*)(a + o_sw);
  st.st_fk_ally = (uint32_t*)(a + o_sf);
  st.st_ties = (uint32_t*)(a + o_stie);
  st.st_elims = (uint32_t*)(a + o_sel);
  st.st_len = (int64_t*)(a + o_sl);
  st.st_ret = (double*)(a + o_sr);
  st.st_base = (int64_t*)(a + o_sb);
  h->sync = (Sync*)(a + o_sync);
  h->stats_dev = (double*)(a + o_stats);
  // K0 is the default from TABX_K0_MIN_ENVS lanes on (4096; below
  // that the step is launch-latency bound and two extra launches cost more
  // than K0 saves); TABX_NO_K0=1 keeps the decision inside K1 always
  const char* no_k0 = getenv("TABX_NO_K0");
  const char* k0_min = getenv("TABX_K0_MIN_ENVS");
  const int64_t k0_envs = k0_min ? atoll(k0_min) : 4096;
  if (B >= k0_envs && !(no_k0 && no_k0[0] == '1'))
    h->ctrl_act = (int8_t*)(a + o_ctl);
  const char* gen = getenv("TABX_GENERIC_SHAPES");
  h->generic_shapes = (gen && gen[0] == '1') ? 1 : 0;
  const char* fz = getenv("TABX_FUSED");
  const char* fzv = getenv("TABX_FUSED_VARIANT");
  // off by default: measured 10% slower than K1 + K2
  h->fused = (fz && fz[0] == '1') ? (fzv ? atoi(fzv) : 0) : -1;
  const char* smx = getenv("TABX_SINGLE_MAX_ENVS");
  if (smx) h->single_max = atoll(smx);

  int rc = TABX_OK;
  for (int k = 0; k < n_configs; ++k) {
    h->cfg_host.push_back(configs[k]);
    h->cfg_host_ok.push_back(1);
    h->pinned.push_back(0);
    h->row_hash.push_back(config_hash(configs + k));
    h->by_hash.emplace(h->row_hash.back(), k);
    if (configs[k].controller[0] == TABX_CTRL_EXTERNAL ||
        configs[k].controller[1] == TABX_CTRL_EXTERNAL)
      h->any_external = true;
  }
  h->lane_slot.assign((size_t)B, 0);
  if (env_config) h->lane_slot.assign(env_config, env_config + B);
  recount_slots(h);
  e = cudaMemcpyAsync(h->cfg_dev, configs, sizeof(tabx_config) * n_configs,
                      cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess) e = launch_derive(h->cfg_dev, h->dcfg_dev, 0, n_configs, h->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->arena, 0, off, h->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(st.seed, seeds, 8 * B, cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess && env_config)
    e = cudaMemcpyAsync(st.cfg, env_config, 4 * B, cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(&h->sync->err_index, 0xFF, 8, h->stream);
  if (e == cudaSuccess)
    e = launch_spawn(st, h->cfg_dev, h->dcfg_dev, 0, B, N, (int)W, 1, h->sm_count, h->stream);
  if (e == cudaSuccess) e = alloc_stage(h);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);  // host arrays may be freed
  if (e != cudaSuccess) {
    rc = cuda_fail(e, "tabx_create");
    if (h->stage) {
      for (int q = 0; q < tabx_handle::STAGE_SLOTS; ++q)
        if (h->stage_ev[q]) cudaEventDestroy(h->stage_ev[q]);
      cudaFreeHost(h->stage);
    }
    cudaFree(h->dcfg_dev);
    cudaFree(h->cfg_dev);
    cudaFree(h->arena);
    delete h;
    return rc;
  }
  *out = h;
  return TABX_OK;
}

int tabx_destroy(tabx_handle* h) {
  if (!h) return TABX_OK;
  DeviceGuard guard(h->device);
  cudaStreamSynchronize(h->stream);
  if (h->prof_ev[0][0])
    for (int s = 0; s < tabx_handle::PROF_SLOTS; ++s)
      for (int k = 0; k < 4; ++k) cudaEventDestroy(h->prof_ev[s][k]);
  if (h->stage) {
    for (int q = 0; q < tabx_handle::STAGE_SLOTS; ++q) cudaEventDestroy(h->stage_ev[q]);
    cudaFreeHost(h->stage);
  }
  cudaFree(h->dcfg_dev);
  cudaFree(h->cfg_dev);
  cudaFree(h->arena);
  delete h;
  return TABX_OK;
}

int tabx_set_stream(tabx_handle* h, void* stream) {
  if (!h) return fail(TABX_E_ARGUMENT, "null handle");
  h->stream = (cudaStream_t)stream;
  return TABX_OK;
}

int tabx_dims(const tabx_handle* h, int64_t* batch, int32_t* n_units, int32_t* n_zones,
              int32_t* obs_dim, int32_t* global_dim) {
  if (!h) return fail(TABX_E_ARGUMENT, "null handle");
  if (batch) *batch = h->B;
  if (n_units) *n_units = h->N;
  if (n_zones) *n_zones = h->Z;
  if (obs_dim) *obs_dim = h->D;
  if (global_dim) *global_dim = h->G;
  return TABX_OK;
}

int tabx_init_output(tabx_handle* h, const tabx_outputs* out) {
  if (!h) return fail(TABX_E_ARGUMENT, "null handle");
  int rc = check_outputs(out, h->D);
  if (rc) return rc;
  DeviceGuard guard(h->device);
  Params P = make_params(h, MODE_INIT, nullptr, out);
  TABX_CUDA(launch_lanes(P, h->W, h->sm_count, h->stream, nullptr), "init_output launch");
  TABX_CUDA(launch_emit(P, h->W, h->sm_count, h->stream), "emit launch");
  // fresh caches everywhere: nothing left to refresh
  TABX_CUDA(cudaMemsetAsync(h->sync->refresh, 0, sizeof(h->sync->refresh), h->stream),
            "refresh clear");
  return TABX_OK;
}

int tabx_step(tabx_handle* h, const int64_t* actions, const tabx_outputs* out) {
  if (!h) return fail(TABX_E_ARGUMENT, "null handle");
  int rc = check_outputs(out, h->D);
  if (rc) return rc;
  DeviceGuard guard(h->device);
  if (actions && h->any_external) {
    TABX_CUDA(launch_validate(actions, h->st, h->cfg_dev, h->B, h->N, h->sync, h->sm_count,
                              h->stream),
              "validate launch");
  }
  h->last_actions = actions;
  // K1 step logic -> K2 observation streaming -> K3 deferred auto-resets
  Params P = make_params(h, MODE_STEP, actions, out);
  cudaEvent_t* ev = nullptr;
  if (h->profiling) {
    const int slot = h->prof_next;
    if (h->prof_pending == tabx_handle::PROF_SLOTS) {
      prof_collect(h, slot);
      --h->prof_pending;
    }
    ev = h->prof_ev[slot];
    h->prof_next = (slot + 1) % tabx_handle::PROF_SLOTS;
    ++h->prof_pending;
    cudaEventRecord(ev[0], h->stream);
  }
  if (h->ctrl_act) {
    const int nh = ctrl_units(h);
    if (nh > 0) {
      // K0 path: a pending batch refresh is materialised first (the rows K0
      // reads), then K0 decides, then the controller-free step kernel
      Params R = make_params(h, MODE_REFRESH, nullptr, nullptr);
      TABX_CUDA(launch_lanes(R, h->W, h->sm_count, h->stream, nullptr), "refresh launch");
      P.ctrl_act = h->ctrl_act;
      TABX_CUDA(launch_ctrl(P, h->W, nh, h->sm_count, h->stream), "controller launch");
      P.mode = MODE_STEP_K0;
    }
  }
  // fused step + observation kernel where it covers the shape; otherwise
  // K1 then K2.  Profile slots: [refresh + K0 | fused] or [.. + K1 | K2].
  h->fused_ran = 0;
  if (h->W == 1 && P.mode == MODE_STEP && h->B < h->single_max) {
    // the whole step in one launch (small batches are launch-latency bound)
    if (ev) cudaEventRecord(ev[1], h->stream);
    const cudaError_t se = launch_small_w1(P, h->sm_count, h->stream);
    if (se == cudaSuccess) {
      if (ev) {
        cudaEventRecord(ev[2], h->stream);
        cudaEventRecord(ev[3], h->stream);
      }
      h->fused_ran = 2;
      return TABX_OK;
    }
    if (se != cudaErrorNotSupported) TABX_CUDA(se, "single-launch step");
  }
  if (h->W == 1 && h->fused >= 0 && P.mode == MODE_STEP_K0) {
    if (ev) cudaEventRecord(ev[1], h->stream);
    const cudaError_t fe = launch_fused_w1(P, h->fused, h->sm_count, h->stream);
    if (fe == cudaSuccess) {
      h->fused_ran = 1;
    } else if (fe != cudaErrorNotSupported) {
      TABX_CUDA(fe, "fused step launch");
    }
  }
  if (!h->fused_ran) {
    TABX_CUDA(launch_lanes(P, h->W, h->sm_count, h->stream, nullptr), "step launch");
    if (ev) cudaEventRecord(ev[1], h->stream);
    TABX_CUDA(launch_emit(P, h->W, h->sm_count, h->stream), "emit launch");
  }
  if (ev) cudaEventRecord(ev[2], h->stream);
  P.mode = MODE_RESET;
  TABX_CUDA(launch_lanes(P, h->W, h->sm_count, h->stream, nullptr), "reset launch");
  if (ev) cudaEventRecord(ev[3], h->stream);
  return TABX_OK;
}

int tabx_reset_env(tabx_handle* h, int64_t b, const tabx_config* config, uint64_t seed,
                   int32_t has_seed, const tabx_outputs* out, int32_t* slot_out) {
  if (!h || b < 0 || b >= h->B) return fail(TABX_E_ARGUMENT, "tabx_reset_env: bad lane");
  int rc = check_outputs(out, h->D);
  if (rc) return rc;
  DeviceGuard guard(h->device);
  int32_t idx = -1;  // -1: keep the lane's slot
  if (config) {
    rc = find_or_add_config(h, config, &idx);
    if (rc) return rc;
    move_lane(h, b, idx);
  }
  // slot and seed travel as kernel arguments: nothing here waits on the stream
  TABX_CUDA(launch_spawn_one(h->st, h->cfg_dev, h->dcfg_dev, b, idx, seed, has_seed, h->N, h->W,
                             h->stream),
            "spawn launch");
  if (slot_out) *slot_out = h->lane_slot[b];
  return tabx_init_output(h, out);
}

int tabx_respawn_all(tabx_handle* h, const uint64_t* seeds, const int32_t* env_config) {
  if (!h || !seeds) return fail(TABX_E_ARGUMENT, "tabx_respawn_all: bad argument");
  DeviceGuard guard(h->device);
  if (env_config)
    for (int64_t b = 0; b < h->B; ++b)
      if (env_config[b] < 0 || env_config[b] >= (int32_t)h->cfg_host.size())
        return fail(TABX_E_ARGUMENT, "env_config index out of range");
  TABX_CUDA(cudaMemcpyAsync(h->st.seed, seeds, 8 * h->B, cudaMemcpyHostToDevice, h->stream),
            "seeds");
  TABX_CUDA(cudaMemsetAsync(h->st.episode, 0, 8 * h->B, h->stream), "episodes");
  if (env_config) {
    TABX_CUDA(cudaMemcpyAsync(h->st.cfg, env_config, 4 * h->B, cudaMemcpyHostToDevice, h->stream),
              "env config");
  } else {
    TABX_CUDA(cudaMemsetAsync(h->st.cfg, 0, 4 * h->B, h->stream), "env config");
  }
  TABX_CUDA(cudaMemsetAsync(&h->sync->err_index, 0xFF, 8, h->stream), "error clear");
  TABX_CUDA(launch_spawn(h->st, h->cfg_dev, h->dcfg_dev, 0, h->B, h->N, h->W, 1, h->sm_count,
                         h->stream),
            "spawn launch");
  TABX_CUDA(cudaStreamSynchronize(h->stream), "respawn sync");  // host arrays may be freed
  if (env_config)
    h->lane_slot.assign(env_config, env_config + h->B);
  else
    h->lane_slot.assign((size_t)h->B, 0);
  recount_slots(h);
  return TABX_OK;
}

int tabx_export_state(tabx_handle* h, const tabx_state* dst) {
  if (!h || !dst) return fail(TABX_E_ARGUMENT, "tabx_export_state: bad argument");
  DeviceGuard guard(h->device);
  // caches pending a batch refresh are materialised first (refresh_caches)
  Params P = make_params(h, MODE_REFRESH, nullptr, nullptr);
  TABX_CUDA(launch_lanes(P, h->W, h->sm_count, h->stream, nullptr), "refresh launch");
  TABX_CUDA(launch_export(h->st, *dst, nullptr, h->B, h->N, h->W, h->sm_count, h->stream),
            "export");
  return TABX_OK;
}

int tabx_export_lanes(tabx_handle* h, const int64_t* lanes, int64_t n_lanes,
                      const tabx_state* dst) {
  if (!h || !dst || n_lanes < 0 || (n_lanes > 0 && !lanes))
    return fail(TABX_E_ARGUMENT, "tabx_export_lanes: bad argument");
  DeviceGuard guard(h->device);
  TABX_CUDA(launch_export(h->st, *dst, lanes, n_lanes, h->N, h->W, h->sm_count, h->stream),
            "export lanes");
  return TABX_OK;
}

int tabx_reserve_configs(tabx_handle* h, int32_t capacity) {
  if (!h || capacity < 1) return fail(TABX_E_ARGUMENT, "tabx_reserve_configs: bad argument");
  if (capacity <= h->cfg_cap) return TABX_OK;
  DeviceGuard guard(h->device);
  tabx_config* c2 = nullptr;
  DerivedCfg* d2 = nullptr;
  cudaError_t e = cudaMalloc((void**)&c2, sizeof(tabx_config) * (size_t)capacity);
  if (e == cudaSuccess) e = cudaMalloc((void**)&d2, sizeof(DerivedCfg) * (size_t)capacity);
  const size_t n = h->cfg_host.size();
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(c2, h->cfg_dev, sizeof(tabx_config) * n, cudaMemcpyDeviceToDevice,
                        h->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d2, h->dcfg_dev, sizeof(DerivedCfg) * n, cudaMemcpyDeviceToDevice,
                        h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) {
    cudaFree(c2);
    cudaFree(d2);
    return cuda_fail(e, "tabx_reserve_configs");
  }
  cudaFree(h->cfg_dev);
  cudaFree(h->dcfg_dev);
  h->cfg_dev = c2;
  h->dcfg_dev = d2;
  h->cfg_cap = capacity;
  return TABX_OK;
}

int tabx_num_configs(tabx_handle* h, int32_t* count, int32_t* capacity) {
  if (!h) return fail(TABX_E_ARGUMENT, "tabx_num_configs: bad argument");
  if (count) *count = (int32_t)h->cfg_host.size();
  if (capacity) *capacity = h->cfg_cap;
  return TABX_OK;
}

int tabx_config_slot(tabx_handle* h, int32_t slot, int64_t* lanes, int32_t* pinned) {
  if (!h || slot < 0 || slot >= (int32_t)h->cfg_host.size())
    return fail(TABX_E_ARGUMENT, "tabx_config_slot: bad argument");
  if (lanes) *lanes = h->refcnt[slot];
  if (pinned) *pinned = h->pinned[slot];
  return TABX_OK;
}

int tabx_get_config(tabx_handle* h, int32_t slot, tabx_config* dst) {
  if (!h || !dst || slot < 0 || slot >= (int32_t)h->cfg_host.size())
    return fail(TABX_E_ARGUMENT, "tabx_get_config: bad argument");
  DeviceGuard guard(h->device);
  TABX_CUDA(cudaMemcpyAsync(dst, h->cfg_dev + slot, sizeof(tabx_config), cudaMemcpyDeviceToHost,
                            h->stream),
            "config read");
  TABX_CUDA(cudaStreamSynchronize(h->stream), "config read sync");
  return TABX_OK;
}

int tabx_levels(tabx_handle* h, int32_t op, const tabx_level_spec* spec, double delta,
                const int32_t* src_slots, int32_t dst_first, int32_t count, tabx_pcg64* rngs) {
  if (!h || !spec || count < 0 || (count > 0 && !rngs) || op < TABX_LEVEL_SAMPLE ||
      op > TABX_LEVEL_RETYPE || spec->n_zone_types < 1 || spec->n_zone_types > 3)
    return fail(TABX_E_ARGUMENT, "tabx_levels: bad argument");
  if (dst_first < 0 || dst_first > (int32_t)h->cfg_host.size() ||
      (int64_t)dst_first + count > h->cfg_cap)
    return fail(TABX_E_CAPACITY, "tabx_levels: destination rows outside the config table");
  for (int k = 0; k < spec->n_zone_types; ++k)
    if (spec->zone_types[k] < TABX_ZONE_LAVA || spec->zone_types[k] > TABX_ZONE_SWAMP)
      return fail(TABX_E_ARGUMENT, "tabx_levels: bad zone type");
  if (count == 0) return TABX_OK;
  DeviceGuard guard(h->device);
  TABX_CUDA(launch_levels(h->cfg_dev, src_slots, dst_first, count, *spec, op, delta, rngs,
                          h->sm_count, h->stream),
            "levels");
  TABX_CUDA(launch_derive(h->cfg_dev, h->dcfg_dev, dst_first, dst_first + count, h->stream),
            "levels derive");
  // rows written on the device: the host mirror no longer describes them
  const size_t end = (size_t)dst_first + (size_t)count;
  if (h->cfg_host.size() < end) {
    h->cfg_host.resize(end);
    h->cfg_host_ok.resize(end, 0);
    h->refcnt.resize(end, 0);
    h->pinned.resize(end, 0);
    h->row_hash.resize(end, 0);
  }
  for (size_t k = (size_t)dst_first; k < end; ++k) {
    if (h->cfg_host_ok[k]) slot_unindex(h, (int32_t)k);
    h->cfg_host_ok[k] = 0;
    h->pinned[k] = 1;  // caller-managed rows
  }
  h->free_slots.erase(std::remove_if(h->free_slots.begin(), h->free_slots.end(),
                                     [&](int32_t k) { return h->pinned[k] != 0; }),
                      h->free_slots.end());
  ++h->cfg_version;
  return TABX_OK;
}

int tabx_respawn_lanes(tabx_handle* h, const int64_t* lanes, const int32_t* slots,
                       const uint64_t* seeds, int64_t n) {
  if (!h || n < 0 || (n > 0 && !lanes))
    return fail(TABX_E_ARGUMENT, "tabx_respawn_lanes: bad argument");
  if (n == 0) return TABX_OK;
  DeviceGuard guard(h->device);
  if (slots) pin_all_slots(h);
  TABX_CUDA(launch_spawn_lanes(h->st, h->cfg_dev, h->dcfg_dev, lanes, slots, seeds, n, h->N, h->W,
                               h->sm_count, h->stream),
            "respawn lanes");
  return TABX_OK;
}

int tabx_import_state(tabx_handle* h, const tabx_state* src) {
  if (!h || !src) return fail(TABX_E_ARGUMENT, "tabx_import_state: bad argument");
  DeviceGuard guard(h->device);
  if (src->config) pin_all_slots(h);
  TABX_CUDA(launch_import(h->st, *src, h->cfg_dev, h->dcfg_dev, h->B, h->N, h->W, h->sm_count,
                          h->stream),
            "import");
  TABX_CUDA(cudaMemsetAsync(h->sync->refresh, 0, sizeof(h->sync->refresh), h->stream),
            "refresh clear");
  return TABX_OK;
}

int tabx_get_error(tabx_handle* h, tabx_error* err, int32_t clear) {
  if (!h || !err) return fail(TABX_E_ARGUMENT, "tabx_get_error: bad argument");
  DeviceGuard guard(h->device);
  unsigned long long idx = NO_ERROR;
  TABX_CUDA(cudaMemcpyAsync(&idx, &h->sync->err_index, 8, cudaMemcpyDeviceToHost, h->stream),
            "error read");
  TABX_CUDA(cudaStreamSynchronize(h->stream), "error sync");
  memset(err, 0, sizeof(*err));
  if (idx != NO_ERROR) {
    err->code = TABX_E_ACTION_MASK;
    err->env = (int64_t)(idx / (unsigned long long)h->N);
    err->unit = (int32_t)(idx % (unsigned long long)h->N);
    int64_t a = 0;
    if (h->last_actions) {
      TABX_CUDA(cudaMemcpy(&a, h->last_actions + idx, 8, cudaMemcpyDeviceToHost), "action read");
    }
    err->action = a;
    if (clear) {
      TABX_CUDA(cudaMemsetAsync(&h->sync->err_index, 0xFF, 8, h->stream), "error clear");
      TABX_CUDA(cudaStreamSynchronize(h->stream), "error clear sync");
    }
  }
  return TABX_OK;
}

int tabx_copy_error_word(tabx_handle* h, uint64_t* dst) {
  if (!h || !dst) return fail(TABX_E_ARGUMENT, "tabx_copy_error_word: bad argument");
  DeviceGuard guard(h->device);
  TABX_CUDA(cudaMemcpyAsync(dst, &h->sync->err_index, 8, cudaMemcpyDefault, h->stream),
            "error word copy");
  return TABX_OK;
}

int tabx_episode_stats(tabx_handle* h, double* dst_host, double* dst_device, int32_t reset) {
  if (!h) return fail(TABX_E_ARGUMENT, "null handle");
  DeviceGuard guard(h->device);
  double* out = dst_device ? dst_device : h->stats_dev;
  TABX_CUDA(cudaMemsetAsync(out, 0, 8 * TABX_NUM_STATS, h->stream), "stats clear");
  TABX_CUDA(launch_stats(h->st, h->B, out, reset, h->stream), "stats launch");
  if (dst_host) {
    TABX_CUDA(cudaMemcpyAsync(dst_host, out, 8 * TABX_NUM_STATS, cudaMemcpyDeviceToHost,
                              h->stream),
              "stats read");
    TABX_CUDA(cudaStreamSynchronize(h->stream), "stats sync");
  }
  return TABX_OK;
}

int tabx_set_profiling(tabx_handle* h, int32_t enable) {
  if (!h) return fail(TABX_E_ARGUMENT, "null handle");
  DeviceGuard guard(h->device);
  if (enable && !h->prof_ev[0][0]) {
    for (int s = 0; s < tabx_handle::PROF_SLOTS; ++s)
      for (int k = 0; k < 4; ++k) TABX_CUDA(cudaEventCreate(&h->prof_ev[s][k]), "event create");
  }
  h->profiling = enable != 0;
  h->prof_next = h->prof_pending = 0;
  h->prof_ms[0] = h->prof_ms[1] = h->prof_ms[2] = 0.0;
  h->prof_steps = 0;
  return TABX_OK;
}

int tabx_get_profile(tabx_handle* h, double* ms, int64_t* steps) {
  if (!h || !ms) return fail(TABX_E_ARGUMENT, "tabx_get_profile: bad argument");
  DeviceGuard guard(h->device);
  const int first = (h->prof_next - h->prof_pending + tabx_handle::PROF_SLOTS) %
                    tabx_handle::PROF_SLOTS;
  for (int q = 0; q < h->prof_pending; ++q) prof_collect(h, (first + q) % tabx_handle::PROF_SLOTS);
  h->prof_pending = 0;
  for (int k = 0; k < 3; ++k) ms[k] = h->prof_ms[k];
  if (steps) *steps = h->prof_steps;
  return TABX_OK;
}

int tabx_step_path(const tabx_handle* h, int32_t* fused) {
  if (!h || !fused) return fail(TABX_E_ARGUMENT, "tabx_step_path: bad argument");
  *fused = h->fused_ran;
  return TABX_OK;
}

int tabx_struct_sizes(int64_t* config, int64_t* outputs, int64_t* state, int64_t* level_spec,
                      int64_t* pcg64) {
  if (config) *config = (int64_t)sizeof(tabx_config);
  if (outputs) *outputs = (int64_t)sizeof(tabx_outputs);
  if (state) *state = (int64_t)sizeof(tabx_state);
  if (level_spec) *level_spec = (int64_t)sizeof(tabx_level_spec);
  if (pcg64) *pcg64 = (int64_t)sizeof(tabx_pcg64);
  return TABX_OK;
}

int tabx_masked_sample(const void* logits, int32_t logits_bf16, int64_t ld,
                       const uint8_t* mask, int64_t m, uint64_t seed, const uint64_t* step_ptr,
                       uint64_t step_add, int64_t* actions, float* logp, void* stream) {
  if (m < 0 || (m > 0 && (!logits || !mask || !actions || !logp)) || ld < TABX_NUM_ACTIONS)
    return fail(TABX_E_ARGUMENT, "tabx_masked_sample: bad argument");
  static int sm_count = 0;
  if (!sm_count) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sm_count = 148;
  }
  TABX_CUDA(launch_masked_sample(logits, logits_bf16, ld, mask, m, seed, step_ptr, step_add,
                                 actions, logp, sm_count, (cudaStream_t)stream),
            "masked sample");
  return TABX_OK;
}

int tabx_pack_bf16(const float* src, int64_t rows, int32_t d, int32_t dp, void* dst,
                   void* stream) {
  if (rows < 0 || d < 1 || dp < d || (dp & 7) || (rows > 0 && (!src || !dst)) ||
      ((uintptr_t)dst & 15))
    return fail(TABX_E_ARGUMENT, "tabx_pack_bf16: bad argument");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  TABX_CUDA(launch_pack_bf16(src, rows, d, dp, dst, sms, (cudaStream_t)stream), "pack bf16");
  return TABX_OK;
}

int tabx_policy_mlp(const void* x, int64_t rows, int32_t k, int64_t ldx, const void* w1,
                    const void* b1, const void* w2, const void* b2, void* logits, void* stream) {
  if (rows < 0 || k < 8 || (k & 7) || ldx < k || (ldx & 7) ||
      (rows > 0 && (!x || !w1 || !b1 || !w2 || !b2 || !logits)) ||
      (((uintptr_t)x | (uintptr_t)w1 | (uintptr_t)logits) & 15))
    return fail(TABX_E_ARGUMENT, "tabx_policy_mlp: bad argument");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const MlpSample none{nullptr, 0, nullptr, 0, nullptr, nullptr};
  TABX_CUDA(launch_mlp_policy(x, rows, k, ldx, w1, b1, w2, b2, logits, none, sms,
                              (cudaStream_t)stream),
            "policy mlp");
  return TABX_OK;
}

int tabx_policy_mlp_sample(const void* x, int64_t rows, int32_t k, int64_t ldx, const void* w1,
                           const void* b1, const void* w2, const void* b2, void* logits,
                           const uint8_t* mask, uint64_t seed, const uint64_t* step_ptr,
                           uint64_t step_add, int64_t* actions, float* logp, void* stream) {
  if (rows < 0 || k < 8 || (k & 7) || ldx < k || (ldx & 7) ||
      (rows > 0 && (!x || !w1 || !b1 || !w2 || !b2 || !mask || !actions || !logp)) ||
      (((uintptr_t)x | (uintptr_t)w1 | (uintptr_t)logits) & 15))
    return fail(TABX_E_ARGUMENT, "tabx_policy_mlp_sample: bad argument");
  if (!logits && !mlp_fused_sampling(k))
    return fail(TABX_E_ARGUMENT, "tabx_policy_mlp_sample: this k needs a logits buffer");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const MlpSample sa{mask, seed, step_ptr, step_add, actions, logp};
  TABX_CUDA(launch_mlp_policy(x, rows, k, ldx, w1, b1, w2, b2, logits, sa, sms,
                              (cudaStream_t)stream),
            "policy mlp + sample");
  return TABX_OK;
}

int tabx_debug_phase_cycles(uint64_t* host16, int32_t reset) {
  if (!host16) return fail(TABX_E_ARGUMENT, "tabx_debug_phase_cycles: bad argument");
  unsigned long long part[16];
  for (int k = 0; k < 16; ++k) host16[k] = 0;
  cudaError_t (*fns[4])(unsigned long long*, int) = {phase_cycles_w1, phase_cycles_w2,
                                                      phase_cycles_w4, phase_cycles_w8};
  for (auto fn : fns) {
    TABX_CUDA(fn(part, reset), "phase cycles");
    for (int k = 0; k < 16; ++k) host16[k] += part[k];
  }
  return TABX_OK;
}

int tabx_debug_sincos(const double* x, double* s, double* c, int64_t n, void* stream) {
  TABX_CUDA(launch_sincos_debug(x, s, c, n, (cudaStream_t)stream), "sincos launch");
  return TABX_OK;
}

}  // extern "C"
