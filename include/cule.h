/*
 * cule.h — C-ABI of libcule: batched Atari 2600 emulation on one B200 (sm_100a).
 *
 * The hot path of CuLE (Dalton, Frosio & Garland, arXiv 1907.08467): thousands of independent
 * consoles each step a 6502 CPU + RIOT + TIA for `frameskip` frames per action, render the
 * frames the observation needs, reduce them to an observation, decode reward and terminal from
 * RAM, and reset finished environments from a cache of random initial states.
 *
 *   PAPER.md P:252-276  one console = 6502 + TIA + 128 B RAM + ROM, 160x210 frames in GPU memory
 *   PAPER.md P:280-284  only the last two frames of an action window are rendered; pixel-wise max
 *   PAPER.md P:290-300  reset from a cache of random initial states (64 startup + up to 30 random)
 *   PAPER.md P:540-541  84x84 grayscale observations
 *   SPEC.md  S:530-573  flat create/step/reset/close API, buffer reuse, error classes
 * Hardware details the paper does not give follow the written model in DESIGN.md §2 (the same
 * model the CPU oracle implements independently).
 *
 * Conventions for every call:
 *   - returns 0 (CULE_OK) or a negative CULE_E_* code; cule_last_error() gives a message
 *     (thread-local, valid until the next call on the same thread);
 *   - "d_" pointers are DEVICE pointers on the handle's device, "h_" pointers are HOST pointers;
 *   - the caller owns all device memory (workspace, actions, observations, rewards, dones,
 *     counters) and keeps it alive while the handle uses it; the library never allocates device
 *     memory;
 *   - calls taking `cuda_stream` (a cudaStream_t, NULL = legacy default stream) are asynchronous
 *     on that stream unless stated; a sticky CUDA error surfaces as CULE_E_CUDA on a later call;
 *   - every call on a handle runs on the device that was current at cule_create (the library
 *     switches to it and restores the caller's device on return); `cuda_stream` must belong to
 *     that device;
 *   - one handle is used from one stream at a time: calls on the same handle must not be in
 *     flight on two streams at once (they share the workspace: state, staging, work tickets);
 *   - per-environment runtime faults (JAM / unstable opcode, runaway frame) are data, not call
 *     errors: the env reports done = 1 with reward 0 and an all-zero observation, is reset from
 *     the cache, and the `faults` counter is incremented.
 */
#ifndef CULE_H
#define CULE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CULE_OK 0
#define CULE_E_INVAL (-1)    /* bad argument (null pointer, size, range, workspace too small) */
#define CULE_E_ROM_SIZE (-2) /* ROM length not in {2048 (2K), 4096 (4K), 8192 (F8), 16384 (F6),
                                32768 (F4)} (2K/F6/F4: SURVEY.md §8(f) NEXT-4) */
#define CULE_E_ROM_FAULT (-3)/* the reset-cache build hit a JAM or a runaway frame             */
#define CULE_E_CUDA (-4)     /* CUDA launch / runtime failure                                  */
#define CULE_E_CLOSED (-5)   /* use after cule_destroy                             */

#define CULE_OBS_RAW 0    /* obs = u8[N][210][160] palette index (COLUxx >> 1) of the last frame */
#define CULE_OBS_GRAY84 1 /* obs = u8[N][84][84] area84(max(gray(frame fs-1), gray(frame fs)))   */

#define CULE_STATE_BYTES 256 /* packed per-env snapshot, layout in DESIGN.md §3 */
#define CULE_FRAME_W 160
#define CULE_FRAME_H 210

typedef struct cule_env cule_env; /* opaque, owned by the library */

typedef struct {
  int32_t obs_mode;           /* CULE_OBS_RAW or CULE_OBS_GRAY84 (default GRAY84)            */
  int32_t reset_cache_size;   /* K cached start states per ROM (default 30)       */
  int32_t startup_frames;     /* NOOP frames after power-on (default 64)              */
  int32_t max_random_frames;  /* R: + u_k in [0, R] extra NOOP frames (default 30)*/
  int32_t max_episode_frames; /* done when an episode reaches this many frames; 0 = no cap   */
  int32_t line_cap;           /* runaway-frame fault after this many scanlines (default 1024)*/
  int32_t ystart;             /* frame-relative scanline of observation row 0 (default 34)   */
  uint8_t score_addr;         /* RAM bus address ($80-$FE) of the BCD score high byte; low at +1 */
  uint8_t term_addr;          /* done iff (RAM[term_addr] & term_mask) != 0 ($80-$FF)        */
  uint8_t term_mask;
  uint8_t idle_skip;          /* 1: exact closed-form skip of [timer read; branch back] poll loops
                                 (results bit-identical), 0 (default): off   */
  uint64_t seed;              /* reset-cache construction seed (u_k draws)                   */
  int64_t env_index_base;     /* global id of local env 0 (multi-GPU sharding)               */
  const uint8_t* palette_rgb; /* HOST, 128 x (R,G,B) NTSC palette; read only during
                                 cule_create; required for GRAY84 (gray LUT), ignored for RAW  */
  int32_t engine;             /* CULE_ENGINE_AUTO (default) or one of the engines below; the
                                 environment variable CULE_ENGINE (simt|scalar|jit|vjit|wsvjit) overrides */
  int32_t tia_delays;         /* 1: delayed register effects (R#35):
                                 PF0/PF1/PF2 written at visible pixel x take effect at the next
                                 4-pixel playfield cell boundary 4*ceil(x/4), GRP0/GRP1 one colour
                                 clock after the write; 0 (default): every write at its clock    */
} cule_config;

/* Engines (all compute the same results, bit for bit):
 *   SIMT   batched datapath, up to 32 envs per warp;
 *   SCALAR one env per warp, record-driven interpreter + warp-cooperative TIA replay;
 *   JIT    the scalar engine with the cartridge code translated to CUDA at cule_create and
 *          compiled with NVRTC for sm_100a (static recompilation; cached on disk by content);
 *   VJIT   one env per lane running the translated code (up to 32 envs per warp), basic
 *          blocks scheduled by warp vote so lanes at the same PC run together; per-lane TIA
 *          replay (the SIMT engine's renderer);
 *   WSVJIT VJIT with warp specialization: warp pairs share 32 envs, the producer warp emulates
 *          into double-buffered TIA logs, the consumer warp replays and renders (mbarriers).
 * AUTO picks among them by env count (cule.cu choose_engine, measured); an engine that does
 * not apply (idle_skip on, translation too large) falls back to SCALAR / SIMT. */
#define CULE_ENGINE_AUTO 0
#define CULE_ENGINE_SIMT 1
#define CULE_ENGINE_SCALAR 2
#define CULE_ENGINE_JIT 3
#define CULE_ENGINE_VJIT 4
#define CULE_ENGINE_WSVJIT 5

/* Fill *cfg with the defaults above (score $80/$81, terminal $82 bit 0, seed 0, base 0). */
void cule_default_config(cule_config* cfg);

/* Bytes of device workspace cule_create needs for (num_envs, n_roms, cfg).  0 on bad input. */
size_t cule_workspace_bytes(int num_envs, int n_roms, const cule_config* cfg);

/* Create a batch of num_envs environments.  Env with global id g = env_index_base + i runs
 * ROM g % n_roms.  roms[r] / rom_lens[r] are HOST buffers (copied; may be freed afterwards);
 * 1 <= n_roms <= 4; each length must be 2048 (2K, mirrored in the 4 KB window), 4096 (4K),
 * 8192 (F8: 2 banks, hotspots $1FF8-$1FF9), 16384 (F6: 4 banks, $1FF6-$1FF9) or 32768 (F4:
 * 8 banks, $1FF4-$1FFB); any access to a hotspot switches bank (R#31, R#34).  The
 * scalar engine needs its pre-decoded records (8 B per ROM byte) in shared memory: up to
 * 20 KB of ROM in total; larger sets run on the batched engine.  d_workspace (device,
 * >= cule_workspace_bytes, 256-byte aligned) must outlive the handle.  Builds the reset cache
 * on the device (synchronous: returns after the build, CULE_E_ROM_FAULT if any entry faulted).
 * The handle uses the device current at the call.  Errors: CULE_E_INVAL, CULE_E_ROM_SIZE,
 * CULE_E_ROM_FAULT, CULE_E_CUDA. */
int cule_create(const uint8_t* const* roms, const size_t* rom_lens, int n_roms, int num_envs,
                int frameskip, const cule_config* cfg, void* d_workspace, size_t workspace_bytes,
                cule_env** out);

/* All envs <- cache[rom(g)][pick(seed, g, 0)] (pick = splitmix64 hash, DESIGN.md §2 R#22);
 * bookkeeping and the per-GPU counters are zeroed.  d_obs (device, may be NULL) receives each
 * env's cached observation in the layout of the obs mode.  Async on cuda_stream. */
int cule_reset(cule_env* env, uint64_t seed, void* d_obs, void* cuda_stream);

/* One step of every env: latch d_actions[i] (u8, ALE 18-action ids; >= 18 = NOOP), run
 * frameskip frames, write d_obs (u8, layout per obs mode), d_rewards (i32, BCD score delta),
 * d_dones (u8), then reset done envs from the cache.  All pointers are device pointers of
 * N elements.  Async on cuda_stream. */
int cule_step(cule_env* env, const uint8_t* d_actions, void* d_obs, int32_t* d_rewards,
              uint8_t* d_dones, void* cuda_stream);

/* Inference path (R#32), GRAY84 only.  d_stack is a DEVICE
 * frame stack u8[N][4][84][84]: per env a ring of the last four observations of its current
 * episode.  cule_reset_stacked: as cule_reset, with the reset observation in all four slots.
 * cule_step_stacked: as cule_step, writing each env's observation into slot `slot` (0..3; the
 * caller rotates it, so slots slot+1, slot+2, slot+3, slot (mod 4) run oldest to newest); an env
 * whose step ended the episode (d_dones[i] = 1) is reset from the cache (R#20) and gets that
 * entry's start observation in all four slots instead (its terminal observation is not
 * returned).  CULE_E_INVAL for RAW handles, a slot outside [0, 3] or NULL buffers.  Async. */
int cule_reset_stacked(cule_env* env, uint64_t seed, uint8_t* d_stack, void* cuda_stream);
int cule_step_stacked(cule_env* env, const uint8_t* d_actions, uint8_t* d_stack, int slot,
                      int32_t* d_rewards, uint8_t* d_dones, void* cuda_stream);

/* Batched V-trace targets (Eq. target.off computed
 * by the recursive form, Eqs. rho / c truncated importance weights).  All arrays are DEVICE
 * memory, time-major [T][B] (step t of trajectory b at t*B + b), fp32; d_bootstrap is [B]
 * (V(s_T)); d_dones[t][b] = 1 marks a terminal at step t, which stops bootstrapping through it
 * (gamma_t = 0; R#33).  Outputs: d_vs[T][B] = v_t, d_rho[T][B] = rho_t =
 * min(rho_bar, pi/mu), d_adv[T][B] = r_t + gamma_t v_{t+1} - V(s_t) (v_T = bootstrap).
 * CULE_E_INVAL for NULL buffers, T or B <= 0, gamma outside (0, 1] or not rho_bar >= c_bar > 0.
 * Async on cuda_stream; needs no env handle. */
int cule_vtrace(const float* d_rewards, const float* d_values, const float* d_bootstrap, const float* d_log_mu,
                const float* d_log_pi, const uint8_t* d_dones, int T, int B, float gamma, float rho_bar,
                float c_bar, float* d_vs, float* d_rho, float* d_adv, void* cuda_stream);

/* Same as cule_step but with HOST buffers: copies h_actions in, steps, copies obs/rewards/
 * dones out through the workspace's I/O staging area; synchronises cuda_stream before
 * returning.  h_obs may be NULL (observations stay on the device). */
int cule_step_host(cule_env* env, const uint8_t* h_actions, void* h_obs, int32_t* h_rewards,
                   uint8_t* h_dones, void* cuda_stream);

/* Copy the packed snapshots u8[N][256] to / from HOST memory.  Synchronous
 * with respect to cuda_stream.  cule_set_state validates every snapshot on the host before
 * anything is uploaded and returns CULE_E_INVAL (state unchanged) if any has rom_id >= n_roms,
 * a bank outside its ROM, a timer shift not in {0,3,6,10}, an object position >= 160, fc at or
 * beyond the line cap (76 * line_cap cycles) or a fault code > 2. */
int cule_get_state(cule_env* env, uint8_t* h_states, void* cuda_stream);
int cule_set_state(cule_env* env, const uint8_t* h_states, void* cuda_stream);

/* Copy the per-GPU counters int64[4] = {frames, episodes finished, sum of finished episode
 * returns, faults} to DEVICE memory d_counters4.  Async on cuda_stream. */
int cule_counters(cule_env* env, int64_t* d_counters4, void* cuda_stream);

/* Diagnostic entry for single-instruction parity tests: every env executes up to n_instr
 * instructions (no rendering; a VSYNC rise ends the frame and stops that env), then the TIA
 * is caught up to the CPU clock.  d_status (device i32[N], may be NULL) gets 0 = budget used,
 * 1 = JAM/unstable opcode, 2 = runaway, 3 = frame ended.  Async on cuda_stream. */
int cule_debug_exec(cule_env* env, int n_instr, int32_t* d_status, void* cuda_stream);

/* Number of envs / frameskip / observation bytes per env of a handle. */
int cule_num_envs(const cule_env* env);
/* Which step kernel the handle runs: CULE_ENGINE_SIMT, CULE_ENGINE_SCALAR, CULE_ENGINE_JIT,
 * CULE_ENGINE_VJIT or CULE_ENGINE_WSVJIT (see cule_config.engine).  CULE_E_CLOSED for a destroyed handle. */
int cule_engine(const cule_env* env);

/* Host only (no GPU needed): translate the ROM set (as cule_create would for the JIT engine)
 * and compile it with NVRTC for sm_100a into the on-disk kernel cache (directory jit_cache/
 * next to libcule.so, or $CULE_JIT_CACHE), so a later cule_create finds it.  obs_mode selects
 * the RAW or GRAY84 kernel.  `info` (may be NULL) receives a one-line summary.  Errors:
 * CULE_E_INVAL, CULE_E_ROM_SIZE, CULE_E_CUDA (translation or compilation failed; message in
 * cule_last_error). */
int cule_jit_prepare(const uint8_t* const* roms, const size_t* rom_lens, int n_roms, int obs_mode, char* info,
                     size_t info_len);
/* Same for a given translated engine: CULE_ENGINE_JIT (as cule_jit_prepare), CULE_ENGINE_VJIT
 * (the SIMT translation) or CULE_ENGINE_WSVJIT (its warp-specialized kernel).  CULE_E_INVAL for
 * any other engine. */
int cule_jit_prepare_engine(const uint8_t* const* roms, const size_t* rom_lens, int n_roms, int obs_mode,
                            int engine, char* info, size_t info_len);
int cule_frameskip(const cule_env* env);
size_t cule_obs_bytes(const cule_env* env);

/* Release the handle (not the caller-owned workspace).  Using it afterwards is an error. */
int cule_destroy(cule_env* env);

const char* cule_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* CULE_H */
