// Device-side data structures shared by the step kernels and the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tabx.h"

namespace tabx {

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
};

// Control block: action-error latch, device step counter and the
// three-slot "some lane was refilled" flag ring (cache refresh).
struct Sync {
  unsigned long long err_index;
  uint32_t step;
  uint32_t blocks_done;
  int32_t refresh[3];
  int32_t pad;
};

enum Mode : int { MODE_STEP = 0, MODE_INIT = 1, MODE_REFRESH = 2 };

struct Params {
  DevState st;
  const tabx_config* cfgs;
  Sync* sync;
  const int64_t* actions;  // [B*N] or nullptr
  tabx_outputs out;
  int64_t B;
  int N, Z, D, G;
  int auto_reset;
  int mode;
  int stage_rows;    // observation rows per staged chunk
  int stage_floats;  // floats per stage buffer (multiple of 4)
};

}  // namespace tabx
