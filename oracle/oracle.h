/*
 * oracle.h — C-ABI of the CPU oracle for the CuLE hot path (arXiv 1907.08467).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * / --impl reference legs may load liboracle.so.  The product path (libcule.so and the Python
 * binding) never links, imports or executes anything under oracle/.
 *
 * The oracle shares no code or header with the CUDA path (not even include/cule.h): the two
 * agree only on the documented 256-byte snapshot layout and on the call
 * semantics, which is what the parity tests compare.
 *
 * What it computes: PAPER.md P:252-276 (one emulated console = 6502 CPU + TIA + 128 B RAM +
 * ROM, rendering 160x210 frames), P:280-284 (render only the frames the max needs),
 * P:290-300 (reset from a cache of random initial states), P:310-314 (the same emulator on the
 * CPU "for debugging and benchmarking").  Hardware details the paper omits follow the written
 * model of SURVEY.md §8(c) and the readings listed in DESIGN.md §2.
 */
#ifndef CULE_ORACLE_H
#define CULE_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_STATE_BYTES 256
#define ORC_FB_W 160
#define ORC_FB_H 210
#define ORC_OBS84 84

typedef struct {
  int32_t obs_mode;           /* 0 = raw 160x210 palette indices, 1 = gray 84x84          */
  int32_t reset_cache_size;   /* K (default 30)                                 */
  int32_t startup_frames;     /* default 64                                        */
  int32_t max_random_frames;  /* R, default 30                                 */
  int32_t max_episode_frames; /* 0 = no cap                                                */
  int32_t line_cap;           /* runaway-frame fault threshold in scanlines (default 1024) */
  int32_t ystart;             /* first frame-relative scanline of row 0 (default 34)        */
  uint8_t score_addr;         /* RAM bus address of the BCD score high byte                */
  uint8_t term_addr;          /* done iff RAM[term_addr] & term_mask                        */
  uint8_t term_mask;
  uint8_t tia_delays;         /* 1: delayed register effects [R#35] (default 0)              */
  uint64_t seed;              /* reset-cache construction seed                             */
  int64_t env_index_base;     /* global id of local env 0                                  */
} orc_config;

/* ---- machine-level entries (single console, packed 256 B snapshot) ---------------------- */
/* Power-on state.  Returns 0, or -1 on a bad ROM size. */
int orc_power_on(const uint8_t* rom, size_t rom_len, uint8_t* state);
/* Execute up to n_instr instructions; then catch the TIA up to the CPU clock.  A VSYNC rising
 * edge ends the frame (rebases clocks) and stops early.  Returns 0 = budget used, 1 = JAM or
 * unstable opcode (fault 1), 2 = runaway line cap (fault 2), 3 = frame ended. */
int orc_exec(const uint8_t* rom, size_t rom_len, uint8_t* state, int n_instr, int line_cap,
             int64_t* cycles_out);
/* Run one frame.  action < 0 keeps the latched inputs.  fb (160x210,
 * may be NULL) receives the palette indices when non-NULL.  Returns 0 ok, 1/2 fault.
 * *instr_out gets the number of instructions executed. */
int orc_run_frame(const uint8_t* rom, size_t rom_len, uint8_t* state, int action, int ystart,
                  int line_cap, uint8_t* fb, int64_t* instr_out, int64_t* lines_out);
/* orc_run_frame with the delayed register effects of DESIGN.md R#35 on (tia_delays = 1) or off. */
int orc_run_frame_ex(const uint8_t* rom, size_t rom_len, uint8_t* state, int action, int ystart,
                     int line_cap, uint8_t* fb, int64_t* instr_out, int64_t* lines_out, int tia_delays);
/* Gray LUT derived from an RGB palette (384 bytes) — §8(c).12 */
void orc_gray_lut(const uint8_t* rgb, uint8_t* gray128);
/* area84 of a 160x210 gray image (u8) — §8(c).12, exact area weights, round-half-even */
void orc_area84(const uint8_t* gray, uint8_t* out84);
/* splitmix64 / H / pick helpers (§8(c).11) */
uint64_t orc_splitmix64(uint64_t x);
uint64_t orc_hash2(uint64_t a, uint64_t b);

/* ---- environment-level entries (mirror of the cule_* calls) ------------------------------ */
typedef struct orc_env orc_env;
void orc_default_config(orc_config* cfg);
/* Returns NULL on error; *err gets -1 (invalid), -2 (ROM size), -3 (ROM fault in cache). */
orc_env* orc_create(const uint8_t* const* roms, const size_t* rom_lens, int n_roms, int num_envs,
                    int frameskip, const orc_config* cfg, const uint8_t* palette_rgb, int* err);
/* Override the global ids of the local envs (sampled parity at scale). */
int orc_set_env_ids(orc_env* e, const int64_t* gids);
int orc_reset(orc_env* e, uint64_t seed, uint8_t* obs);
int orc_step(orc_env* e, const uint8_t* actions, uint8_t* obs, int32_t* rewards, uint8_t* dones);
/* frame stack of the inference path (GRAY84; stack = u8[N][4][84][84]; R#32) */
int orc_reset_stacked(orc_env* e, uint64_t seed, uint8_t* stack);
int orc_step_stacked(orc_env* e, const uint8_t* actions, uint8_t* stack, int slot, int32_t* rewards,
                     uint8_t* dones);
int orc_get_state(orc_env* e, uint8_t* states);
int orc_set_state(orc_env* e, const uint8_t* states);
int orc_counters(orc_env* e, int64_t* counters4);
/* Copy the reset cache out: states [n_roms*K][256] and observations [n_roms*K][obs_bytes]. */
int orc_get_cache(orc_env* e, uint8_t* states, uint8_t* obs);
void orc_destroy(orc_env* e);

#ifdef __cplusplus
}
#endif
#endif
