// cule.cu — libcule: the C-ABI boundary (include/cule.h) over the sm_100a kernels.
//
// Host code only marshals arguments, carves the caller-owned workspace and launches kernels;
// every step of the emulation path runs on the device (kernels.cuh).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <string>

#include "../../include/cule.h"
#include "decode_table.h"
#include "kernels.cuh"
#include <vector>

#include "scalar_decode.h"
#include "scalar_predecode.h"
#include "scalar_kernels.cuh"
#include "vtrace.cuh"
#include "jit.h"
#include "vjit_kernels.cuh"

namespace {

thread_local std::string g_err;
std::mutex g_live_mu;
std::set<const void*> g_live;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct Layout {
  size_t state, pack, staging, cstate, cobs, cscore, cstage, roms, decode, sdecode, srec, gray, counters, err,
      tickets, io_act, io_obs, io_rew, io_done, total;
};

size_t obs_bytes_of(int mode) { return mode == CULE_OBS_RAW ? (size_t)cule::kFrameBytes : (size_t)cule::kObs84; }

bool compute_layout(int N, int n_roms, const cule_config* c, Layout* L) {
  if (N <= 0 || n_roms < 1 || n_roms > 4 || !c || c->reset_cache_size < 1) return false;
  const size_t n = (size_t)N;
  const size_t nk = (size_t)n_roms * (size_t)c->reset_cache_size;
  const size_t ob = obs_bytes_of(c->obs_mode);
  const bool gray = c->obs_mode == CULE_OBS_GRAY84;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align256(o + bytes); return r; };
  L->state = take(256 * n);
  L->pack = take(256 * n);
  L->staging = take(gray ? 2 * n * cule::kFrameBytes : 0);  // frames fs-1 and fs per env
  L->cstate = take(256 * nk);
  L->cobs = take(nk * ob);
  L->cscore = take(2 * nk);
  L->cstage = take(gray ? 2 * nk * cule::kFrameBytes : 0);
  L->roms = take(4 * 32768);
  L->decode = take(2048);
  L->sdecode = take(2048);
  L->srec = take(cule::kRecBytes * 4 * 32768);
  L->gray = take(128);
  L->counters = take(32);
  L->err = take(16);
  L->tickets = take(16);
  L->io_act = take(n);
  L->io_obs = take(n * ob);
  L->io_rew = take(4 * n);
  L->io_done = take(n);
  L->total = o;
  return true;
}

// ROM images packed in 4 KB banks (a 2K cartridge stored twice: its mirror in the window),
// per-ROM offsets and bank counts, and the scalar engine's pre-decoded records
struct RomSet {
  std::vector<uint8_t> img;
  uint32_t rom_off[4] = {0, 0, 0, 0};
  uint32_t banks[4] = {0, 0, 0, 0};
  uint32_t rom_banks = 0;
  uint32_t bytes = 0;
  std::vector<uint64_t> recs;
};

int check_roms(const uint8_t* const* roms, const size_t* rom_lens, int n_roms) {
  if (!roms || !rom_lens) return fail(CULE_E_INVAL, "null argument");
  if (n_roms < 1 || n_roms > 4) return fail(CULE_E_INVAL, "n_roms must be in [1, 4]");
  for (int r = 0; r < n_roms; ++r) {
    if (!roms[r]) return fail(CULE_E_INVAL, "null ROM");
    const size_t n = rom_lens[r];
    if (n != 2048 && n != 4096 && n != 8192 && n != 16384 && n != 32768)
      return fail(CULE_E_ROM_SIZE, "ROM size must be 2048 (2K), 4096 (4K), 8192 (F8), 16384 (F6) or 32768 (F4), got " +
                                       std::to_string(n));
  }
  return CULE_OK;
}

RomSet make_romset(const uint8_t* const* roms, const size_t* rom_lens, int n_roms) {
  RomSet rs;
  uint32_t off = 0;
  for (int r = 0; r < n_roms; ++r) {
    rs.rom_off[r] = off;
    const uint32_t img = rom_lens[r] < 4096 ? 4096u : (uint32_t)rom_lens[r];
    off += img;
    rs.banks[r] = img / 4096u;
    rs.rom_banks |= (img / 4096u) << (8 * r);
  }
  rs.bytes = off;
  rs.img.assign(off, 0);
  for (int r = 0; r < n_roms; ++r) {
    std::memcpy(rs.img.data() + rs.rom_off[r], roms[r], rom_lens[r]);
    if (rom_lens[r] == 2048) std::memcpy(rs.img.data() + rs.rom_off[r] + 2048, roms[r], 2048);  // 2K mirror
  }
  rs.recs.resize(off);
  uint32_t lens[4] = {0, 0, 0, 0};
  for (int r = 0; r < n_roms; ++r) lens[r] = 4096u * rs.banks[r];
  cule::predecode_roms(rs.img.data(), rs.rom_off, lens, n_roms, rs.recs.data());
  return rs;
}

// translate + compile (or fetch from the caches) the JIT step kernel for a ROM set
std::vector<char> jit_cubin(const RomSet& rs, int n_roms, bool gray, bool simt, bool ws, bool delays, size_t* n_insn,
                            double* secs, bool* from_disk, std::string& err, uint32_t vlogcap = 32) {
  cule::jit::Translator tr(rs.img.data(), rs.rom_off, rs.banks, n_roms, rs.bytes, rs.recs.data());
  if (const char* v = getenv("CULE_VELIDE")) tr.vnoelide_ = !strcmp(v, "0");  // ablation switch
  cule::jit::Translation t = tr.run(gray, simt, ws);
  if (!t.ok) { err = t.why; return {}; }
  // ablation switch (measurement only): rebuild every coverage mask on every span
  if (getenv("CULE_TIA_NO_MASK_CACHE")) t.source = "#define CULE_TIA_NO_MASK_CACHE 1\n" + t.source;
  // ablation switch (measurement only): VJIT block scheduler by __match_any_sync, largest group first
  if (const char* v = getenv("CULE_VSCHED"))
    if (simt && !strcmp(v, "match")) t.source = "#define CULE_VSCHED_MATCH 1\n" + t.source;
  // the kernel is compiled for one setting of the delayed register effects (tia.cuh CULE_DELAYS_ON)
  t.source = std::string("#define CULE_TIA_DELAYS ") + (delays ? "1" : "0") + "\n" + t.source;
  if (simt && !ws && vlogcap != 32) t.source = "#define CULE_VLOGCAP " + std::to_string(vlogcap) + "\n" + t.source;
  *n_insn = t.n_insn;
  if (const char* dump = getenv("CULE_JIT_DUMP")) {
    if (FILE* f = fopen(dump, "w")) { fwrite(t.source.data(), 1, t.source.size(), f); fclose(f); }
  }
  return cule::jit::cubin_for(t.source, err, secs, from_disk);
}

}  // namespace

struct cule_env {
  cule_config cfg;
  int N, fs, n_roms, device;
  uint8_t* ws;
  Layout L;
  uint32_t rom_off[4];
  uint32_t rom_bytes;
  uint32_t rom_banks;      // 4 KB banks per ROM, 8 bits each (kernels.cuh banks_of)
  uint64_t pick_seed;
  size_t smem;
  uint32_t block;
  uint32_t epw;            // envs per warp
  int engine;              // 0 batched (SIMT datapath, epw envs per warp), 1 scalar (one env per warp)
  size_t ssmem;            // dynamic shared memory of the scalar kernels
  uint32_t use_rec;        // scalar engine: pre-decoded records fit in shared memory
  uint32_t sgrid;          // scalar engine: persistent blocks (<= one per SM)
  uint32_t slot_start[4], first_env[4];
  uint32_t grid;           // blocks of the step / debug kernels
  bool jit = false;        // engine 1 runs the translated step kernel (jit.h)
  CUmodule jit_mod = nullptr;
  CUfunction jit_fn = nullptr;
  size_t jit_smem = 0;     // dynamic shared memory of the translated kernel (no records staged)
  size_t jit_insn = 0;
  double jit_compile_s = 0.0;
  // engine 2: the SIMT translated kernel (vjit_kernels.cuh), vepw envs per warp
  uint32_t vepw = 32, vblock = 0, vgrid = 0;
  bool vws = false;        // the warp-specialized variant (producer / consumer warp pairs)
  size_t vsmem = 0;
};

static cule::Params base_params(const cule_env* e) {
  cule::Params p;
  std::memset(&p, 0, sizeof p);
  p.state = e->ws + e->L.state;
  p.N = (uint32_t)e->N;
  p.staging = e->ws + e->L.staging;
  p.roms = e->ws + e->L.roms;
  p.rom_bytes = e->rom_bytes;
  for (int r = 0; r < 4; ++r) p.rom_off[r] = e->rom_off[r];
  p.rom_banks = e->rom_banks;
  p.n_roms = (uint32_t)e->n_roms;
  p.decode = reinterpret_cast<const uint64_t*>(e->ws + e->L.decode);
  p.sdecode = reinterpret_cast<const uint64_t*>(e->ws + e->L.sdecode);
  p.gray = e->ws + e->L.gray;
  p.cache_state = e->ws + e->L.cstate;
  p.cache_score = reinterpret_cast<const uint16_t*>(e->ws + e->L.cscore);
  p.K = (uint32_t)e->cfg.reset_cache_size;
  p.counters = reinterpret_cast<unsigned long long*>(e->ws + e->L.counters);
  p.fs = (uint32_t)e->fs;
  p.line_cap = (uint32_t)e->cfg.line_cap;
  p.ystart = (uint32_t)e->cfg.ystart;
  p.score_addr = e->cfg.score_addr;
  p.term_addr = e->cfg.term_addr;
  p.term_mask = e->cfg.term_mask;
  p.max_episode_frames = (uint32_t)e->cfg.max_episode_frames;
  p.pick_seed = e->pick_seed;
  p.env_base = e->cfg.env_index_base;
  p.startup_frames = (uint32_t)e->cfg.startup_frames;
  p.max_random_frames = (uint32_t)e->cfg.max_random_frames;
  p.cache_seed = e->cfg.seed;
  p.cache_state_out = e->ws + e->L.cstate;
  p.cache_obs_out = e->ws + e->L.cobs;
  p.cache_score_out = reinterpret_cast<uint16_t*>(e->ws + e->L.cscore);
  p.cache_staging = e->ws + e->L.cstage;
  p.error_flag = reinterpret_cast<int32_t*>(e->ws + e->L.err);
  p.epw = e->epw;
  p.idle_skip = e->cfg.idle_skip ? 1u : 0u;
  p.srec = reinterpret_cast<const uint64_t*>(e->ws + e->L.srec);
  p.use_rec = e->use_rec;
  p.tickets = reinterpret_cast<unsigned int*>(e->ws + e->L.tickets);
  p.obs_stride = (uint32_t)obs_bytes_of(e->cfg.obs_mode);
  p.stacked = 0u;
  p.stack_slot = 0u;
  p.tia_delays = e->cfg.tia_delays ? 1u : 0u;
  for (int r = 0; r < 4; ++r) { p.slot_start[r] = e->slot_start[r]; p.first_env[r] = e->first_env[r]; }
  return p;
}

static bool live(const cule_env* e) {
  std::lock_guard<std::mutex> g(g_live_mu);
  return e && g_live.count(e);
}

// Every handle call runs on the handle's device (its workspace lives there), whatever device
// the calling thread has current; the previous device is restored on return.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

#define CHECK_LIVE(e) \
  do { if (!live(e)) return fail(CULE_E_CLOSED, "invalid or destroyed cule_env handle"); } while (0); \
  DeviceGuard device_guard_((e)->device)

static int cuda_check(const char* what) {
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return fail(CULE_E_CUDA, std::string(what) + ": " + cudaGetErrorString(err));
  return CULE_OK;
}

static constexpr int kMaxBlock = 128;

static int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// Engine: the scalar engine (one env per warp, compact interpreter, warp-cooperative TIA)
// wins at low env counts (the batched engine is latency-bound there: a few envs per SM
// sub-partition), the batched engine (SIMT datapath, issue-efficient) at high ones.  CULE_ENGINE
// overrides (simt | scalar).
static int requested_engine(const cule_config* c) {
  if (const char* v = getenv("CULE_ENGINE")) {
    if (!strcmp(v, "simt")) return CULE_ENGINE_SIMT;
    if (!strcmp(v, "scalar")) return CULE_ENGINE_SCALAR;
    if (!strcmp(v, "jit")) return CULE_ENGINE_JIT;
    if (!strcmp(v, "vjit")) return CULE_ENGINE_VJIT;
    if (!strcmp(v, "wsvjit")) return CULE_ENGINE_WSVJIT;
  }
  return c->engine;
}

static int choose_engine(int N) {
  // measured (profiles/r01_v6_engine_sweep.txt): 4096 envs scalar 2.81M vs SIMT 0.74M FPS;
  // 16384 (F8) 2.72M vs 2.30M; 32768 (4 ROMs) 2.09M vs 2.87M
  return N <= 16384 ? 1 : 0;
}

// Envs per warp: the per-env 6502 chain is latency-bound, so at low env counts the kernel
// uses fewer lanes per warp (more warps, less divergence) until each SM sub-partition has a
// few warps to switch between.  CULE_EPW overrides (1..32, power of two).
static uint32_t choose_epw(int N) {
  if (const char* v = getenv("CULE_EPW")) {
    int b = atoi(v);
    if (b >= 1 && b <= 32 && (b & (b - 1)) == 0) return (uint32_t)b;
  }
  // measured on B200 (profiles/r01_*): 4096 envs peak at 4-8 envs/warp, 32K envs at 32
  const uint32_t target_warps = 6u * (uint32_t)sm_count();
  uint32_t e = 32;
  while (e > 1 && ((uint32_t)N + e - 1) / e < target_warps) e /= 2;
  return e;
}

// threads per block: small blocks spread few warps over all SMs; CULE_BLOCK overrides
static uint32_t choose_block(uint32_t warps) {
  if (const char* v = getenv("CULE_BLOCK")) {
    int b = atoi(v);
    if (b == 32 || b == 64 || b == 128) return (uint32_t)b;
  }
  // measured at 32768 envs (epw 32): 128 threads 2.90M FPS, 64 2.86M, 32 2.02M
  uint32_t b = 128;
  while (b > 32 && (warps * 32u + b - 1) / b < (uint32_t)sm_count()) b /= 2;
  return b;
}

extern "C" {

void cule_default_config(cule_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof *c);
  c->obs_mode = CULE_OBS_GRAY84;
  c->reset_cache_size = 30;
  c->startup_frames = 64;
  c->max_random_frames = 30;
  c->max_episode_frames = 0;
  c->line_cap = 1024;
  c->ystart = 34;
  c->score_addr = 0x80;
  c->term_addr = 0x82;
  c->term_mask = 0x01;
  c->seed = 0;
  c->env_index_base = 0;
  c->idle_skip = 0;
  c->palette_rgb = nullptr;
  c->engine = CULE_ENGINE_AUTO;
  c->tia_delays = 0;
}

size_t cule_workspace_bytes(int num_envs, int n_roms, const cule_config* cfg) {
  Layout L;
  if (!compute_layout(num_envs, n_roms, cfg, &L)) return 0;
  return L.total;
}

int cule_create(const uint8_t* const* roms, const size_t* rom_lens, int n_roms, int num_envs,
                int frameskip, const cule_config* cfg, void* d_workspace, size_t workspace_bytes,
                cule_env** out) {
  if (!out) return fail(CULE_E_INVAL, "out is NULL");
  *out = nullptr;
  if (!roms || !rom_lens || !cfg || !d_workspace) return fail(CULE_E_INVAL, "null argument");
  if (n_roms < 1 || n_roms > 4) return fail(CULE_E_INVAL, "n_roms must be in [1, 4]");
  if (num_envs <= 0) return fail(CULE_E_INVAL, "num_envs must be > 0");
  if (frameskip < 1) return fail(CULE_E_INVAL, "frameskip must be >= 1");
  if (cfg->obs_mode != CULE_OBS_RAW && cfg->obs_mode != CULE_OBS_GRAY84)
    return fail(CULE_E_INVAL, "bad obs_mode");
  if (cfg->reset_cache_size < 1 || cfg->startup_frames < 0 || cfg->max_random_frames < 0 ||
      cfg->line_cap < 1 || cfg->ystart < 0 || cfg->ystart + cule::kFrameH > cfg->line_cap ||
      cfg->max_episode_frames < 0)
    return fail(CULE_E_INVAL, "bad config value");
  if (cfg->line_cap > 1024) return fail(CULE_E_INVAL, "line_cap must be <= 1024 (18-bit log timestamps)");
  if (cfg->score_addr < 0x80 || cfg->score_addr == 0xFF || cfg->term_addr < 0x80)
    return fail(CULE_E_INVAL, "score/terminal addresses must be RAM bus addresses $80-$FF");
  if (cfg->obs_mode == CULE_OBS_GRAY84 && !cfg->palette_rgb)
    return fail(CULE_E_INVAL, "GRAY84 needs cfg->palette_rgb (384 bytes)");
  if (((uintptr_t)d_workspace & 255) != 0) return fail(CULE_E_INVAL, "workspace must be 256-byte aligned");
  if (cfg->engine < CULE_ENGINE_AUTO || cfg->engine > CULE_ENGINE_WSVJIT) return fail(CULE_E_INVAL, "bad engine");
  for (int r = 0; r < n_roms; ++r) {
    if (!roms[r]) return fail(CULE_E_INVAL, "null ROM");
    const size_t n = rom_lens[r];
    if (n != 2048 && n != 4096 && n != 8192 && n != 16384 && n != 32768)
      return fail(CULE_E_ROM_SIZE, "ROM size must be 2048 (2K), 4096 (4K), 8192 (F8), 16384 (F6) or 32768 (F4), got " +
                                       std::to_string(n));
  }
  Layout L;
  compute_layout(num_envs, n_roms, cfg, &L);
  if (workspace_bytes < L.total)
    return fail(CULE_E_INVAL, "workspace too small: need " + std::to_string(L.total));

  cule_env* e = new cule_env;
  e->cfg = *cfg;
  e->cfg.palette_rgb = nullptr;
  e->N = num_envs;
  e->fs = frameskip;
  e->n_roms = n_roms;
  cudaGetDevice(&e->device);
  e->ws = static_cast<uint8_t*>(d_workspace);
  e->L = L;
  e->pick_seed = 0;
  e->rom_banks = 0;
  uint32_t off = 0;
  for (int r = 0; r < 4; ++r) e->rom_off[r] = 0;
  // images in 4 KB banks: a 2K cartridge is stored twice (its mirror in the 4 KB window)
  for (int r = 0; r < n_roms; ++r) {
    e->rom_off[r] = off;
    const uint32_t img = rom_lens[r] < 4096 ? 4096u : (uint32_t)rom_lens[r];
    off += img;
    e->rom_banks |= (img / 4096u) << (8 * r);
  }
  e->rom_bytes = off;
  e->epw = choose_epw(num_envs);
  const int want = requested_engine(cfg);
  e->engine = (want == CULE_ENGINE_SIMT || want == CULE_ENGINE_VJIT || want == CULE_ENGINE_WSVJIT) ? 0
                                                                    : (want == CULE_ENGINE_AUTO ? choose_engine(num_envs) : 1);
  {
    // records cost 8 B per ROM byte of shared memory: they fit for every combination up to
    // 4 x 4 KB or 2 x F8 + 1 x 4 KB (CULE_NO_REC=1 pretends they do not)
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (optin <= 0) optin = 232448;
    const char* nr = getenv("CULE_NO_REC");
    e->use_rec = (!(nr && atoi(nr) == 1) && cule::scalar_smem_bytes(e->rom_bytes, true) <= (size_t)optin) ? 1u : 0u;
    if (!e->use_rec && want != CULE_ENGINE_JIT) e->engine = 0;  // the interpreter runs from the records
    e->jit_smem = cule::scalar_smem_bytes(e->rom_bytes, false);
    e->ssmem = cule::scalar_smem_bytes(e->rom_bytes, e->use_rec != 0u);
    const uint32_t need = ((uint32_t)num_envs + cule::kSWarps - 1) / cule::kSWarps;
    const uint32_t sms = (uint32_t)sm_count();
    e->sgrid = need < sms ? need : sms;
  }
  {
    const uint32_t warps = ((uint32_t)num_envs + e->epw - 1) / e->epw;
    e->block = choose_block(warps);
    e->grid = (warps * 32u + e->block - 1) / e->block;
    uint32_t slot = 0;
    for (int r = 0; r < 4; ++r) { e->slot_start[r] = 0; e->first_env[r] = 0; }
    for (int r = 0; r < n_roms; ++r) {
      const int64_t base = cfg->env_index_base;
      const uint32_t first = (uint32_t)((((int64_t)r - base) % n_roms + n_roms) % n_roms);
      const uint32_t cnt = first < (uint32_t)num_envs ? ((uint32_t)num_envs - first + n_roms - 1) / n_roms : 0u;
      e->slot_start[r] = slot;
      e->first_env[r] = first;
      slot += cnt;
    }
  }
  e->smem = cule::smem_bytes(e->rom_bytes, e->block);
  const size_t smem_max = cule::smem_bytes(e->rom_bytes, kMaxBlock);

  // static inputs: ROM images, decode table, gray LUT (ITU-R 601 integer, half-up, §8(c).12)
  std::vector<uint8_t> romimg_v((size_t)e->rom_bytes);
  uint8_t* romimg = romimg_v.data();
  for (int r = 0; r < n_roms; ++r) {
    std::memcpy(romimg + e->rom_off[r], roms[r], rom_lens[r]);
    if (rom_lens[r] == 2048) std::memcpy(romimg + e->rom_off[r] + 2048, roms[r], 2048);  // 2K mirror
  }
  uint64_t table[256];
  cule::build_decode_table(table);
  uint64_t stable[256];
  cule::build_scalar_table(stable);
  std::vector<uint64_t> recs((size_t)e->rom_bytes);
  {
    uint32_t lens[4] = {0, 0, 0, 0};
    for (int r = 0; r < n_roms; ++r) lens[r] = 4096u * cule::banks_of(e->rom_banks, (uint32_t)r);
    cule::predecode_roms(romimg, e->rom_off, lens, n_roms, recs.data());
  }
  uint8_t gray[128] = {0};
  if (cfg->palette_rgb) {
    for (int i = 0; i < 128; ++i) {
      int R = cfg->palette_rgb[3 * i], G = cfg->palette_rgb[3 * i + 1], B = cfg->palette_rgb[3 * i + 2];
      gray[i] = (uint8_t)((299 * R + 587 * G + 114 * B + 500) / 1000);
    }
  }
  cudaMemcpy(e->ws + L.roms, romimg, e->rom_bytes, cudaMemcpyHostToDevice);
  cudaMemcpy(e->ws + L.decode, table, sizeof table, cudaMemcpyHostToDevice);
  cudaMemcpy(e->ws + L.sdecode, stable, sizeof stable, cudaMemcpyHostToDevice);
  cudaMemcpy(e->ws + L.srec, recs.data(), recs.size() * sizeof(uint64_t), cudaMemcpyHostToDevice);
  cudaMemset(e->ws + L.tickets, 0, 16);
  cudaMemcpy(e->ws + L.gray, gray, sizeof gray, cudaMemcpyHostToDevice);
  cudaMemset(e->ws + L.state, 0, 256 * (size_t)num_envs);
  cudaMemset(e->ws + L.counters, 0, 32);
  cudaMemset(e->ws + L.err, 0, 16);
  int rc = cuda_check("workspace init");
  if (rc) { delete e; return rc; }

  const bool g = cfg->obs_mode == CULE_OBS_GRAY84;
  cudaFuncSetAttribute(cule::step_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
  cudaFuncSetAttribute(cule::step_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
  cudaFuncSetAttribute(cule::cache_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
  cudaFuncSetAttribute(cule::cache_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
  cudaFuncSetAttribute(cule::debug_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
  cudaFuncSetAttribute(cule::scalar_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e->ssmem);
  cudaFuncSetAttribute(cule::scalar_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e->ssmem);
  cudaFuncSetAttribute(cule::scalar_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e->ssmem);

  // reset cache build: one thread per (rom, entry)
  cule::Params p = base_params(e);
  const uint32_t total = (uint32_t)n_roms * (uint32_t)cfg->reset_cache_size;
  const uint32_t cblock = 32;
  const size_t csmem = cule::smem_bytes(e->rom_bytes, cblock);
  const uint32_t blocks = (total + cblock - 1) / cblock;
  if (g) cule::cache_kernel<true><<<blocks, cblock, csmem>>>(p);
  else cule::cache_kernel<false><<<blocks, cblock, csmem>>>(p);
  rc = cuda_check("cache_kernel launch");
  if (rc) { delete e; return rc; }
  int32_t err_flag = 0;
  if (cudaMemcpy(&err_flag, e->ws + L.err, sizeof err_flag, cudaMemcpyDeviceToHost) != cudaSuccess) {
    rc = cuda_check("cache_kernel");
    delete e;
    return rc ? rc : fail(CULE_E_CUDA, "cache build failed");
  }
  if (err_flag) {
    delete e;
    return fail(CULE_E_ROM_FAULT, "reset-cache build hit a JAM or runaway frame");
  }
  // the translated engines: explicitly requested, or AUTO where they apply (idle skip off)
  // translated engines (measured crossover with the TIA write elision in both, R#37,
  // profiles/r02_crossover_v77.txt and profiles/r02_v78_pytest_gpu.txt): VJIT (one env per lane)
  // from 16384 envs, or from 8192 with several ROMs (8192 envs of the 4-ROM mix: 6.83M vs 5.14M
  // FPS); below that JIT (one env per warp; 8192 envs of one ROM: 9.39M vs 8.51M); neither has
  // the idle-loop skip
  const bool xlate = !cfg->idle_skip;
  const bool vjit_auto = want == CULE_ENGINE_AUTO && xlate && (num_envs >= 16384 || (n_roms > 1 && num_envs >= 8192));
  bool jit_auto = want == CULE_ENGINE_AUTO && xlate && !vjit_auto && (n_roms == 1 || num_envs <= 16384);
  if (want == CULE_ENGINE_VJIT || want == CULE_ENGINE_WSVJIT || vjit_auto) {
    const bool ws = want == CULE_ENGINE_WSVJIT;
    std::string jerr;
    auto& drv = cule::jit::driver();
    std::vector<char> cubin;
    bool from_disk = false;
    // envs per warp (CULE_VEPW overrides: power of two <= 32; measured: 32 from 16384 envs, 16
    // from 8192, else 8) and warps per block: as many warps as the envs need to cover every SM,
    // within the shared memory of one block per SM
    uint32_t vepw = num_envs >= 16384 ? 32u : (num_envs >= 8192 ? 16u : 8u);
    if (const char* v = getenv("CULE_VEPW")) {
      const int b = atoi(v);
      if (b >= 1 && b <= 32 && (b & (b - 1)) == 0) vepw = (uint32_t)b;
    }
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (optin <= 0) optin = 232448;
    // (warp-specialized: groups of envs per warp PAIR, which shares one set of lane areas)
    const uint32_t warps = ((uint32_t)num_envs + vepw - 1) / vepw;
    uint32_t wpb = (warps + (uint32_t)sm_count() - 1) / (uint32_t)sm_count();
    if (const char* v = getenv("CULE_VWPB")) wpb = (uint32_t)atoi(v);
    // TIA log entries per lane (vjit_kernels.cuh CULE_VLOGCAP): 64 up to 8 warps per SM, else 32
    uint32_t vcap = (!ws && wpb <= 8u) ? 64u : 32u;
    if (const char* v = getenv("CULE_VLOGCAP")) vcap = (!ws && atoi(v) == 64) ? 64u : 32u;
    const size_t lane_off = ws ? cule::wsvjit_lane_off(e->rom_bytes) : cule::vjit_lane_off(e->rom_bytes);
    const uint32_t fit = (uint32_t)(((size_t)optin - lane_off) /
                                    (32u * 4u * (ws ? cule::kWLaneWords : cule::vjit_lane_words(vcap))));
    wpb = std::max(1u, std::min({wpb, fit, (uint32_t)CULE_VWARPS / (ws ? 2u : 1u)}));
    // more warps than one wave of blocks holds (e.g. 65536 envs): equal waves of smaller blocks,
    // so every SM runs whole waves instead of a short second one, with the log capacity they allow
    if (!ws && !getenv("CULE_VWPB") && !getenv("CULE_VLOGCAP")) {
      const uint32_t sm = (uint32_t)sm_count(), per_wave = wpb * sm;
      if (warps > per_wave) {
        const uint32_t waves = (warps + per_wave - 1) / per_wave;
        const uint32_t w2 = (warps + waves * sm - 1) / (waves * sm);
        const uint32_t cap2 = w2 <= 8u ? 64u : 32u;
        const uint32_t fit2 = (uint32_t)(((size_t)optin - lane_off) / (32u * 4u * cule::vjit_lane_words(cap2)));
        if (w2 >= 1u && w2 <= fit2) { wpb = w2; vcap = cap2; }
      }
    }
    e->vepw = vepw;
    e->vws = ws;
    e->vblock = (ws ? 64u : 32u) * wpb;
    e->vgrid = (warps + wpb - 1) / wpb;
    e->vsmem = ws ? cule::wsvjit_smem_bytes(e->rom_bytes, wpb) : cule::vjit_smem_bytes(e->rom_bytes, e->vblock, vcap);
    if (!drv.ok) jerr = "CUDA driver entry points unavailable";
    else if (cfg->idle_skip) jerr = "the translated engine has no idle-loop skip";
    else {
      RomSet rs = make_romset(roms, rom_lens, n_roms);
      cubin = jit_cubin(rs, n_roms, g, true, ws, cfg->tia_delays != 0, &e->jit_insn, &e->jit_compile_s, &from_disk, jerr,
                        vcap);
    }
    CUresult cr = CUDA_SUCCESS;
    if (!cubin.empty()) {
      cr = drv.moduleLoadData(&e->jit_mod, cubin.data());
      if (cr == CUDA_SUCCESS) cr = drv.moduleGetFunction(&e->jit_fn, e->jit_mod, ws ? "cule_vjit_ws_step" : "cule_vjit_step");
      if (cr == CUDA_SUCCESS)
        cr = drv.funcSetAttribute(e->jit_fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)e->vsmem);
      if (cr != CUDA_SUCCESS) jerr = "loading the SIMT translated kernel failed (CUresult " + std::to_string((int)cr) + ")";
    }
    if (jerr.empty() && e->jit_fn) {
      e->jit = true;
      e->engine = 2;
    } else if (want == CULE_ENGINE_VJIT || want == CULE_ENGINE_WSVJIT) {
      if (e->jit_mod) drv.moduleUnload(e->jit_mod);
      delete e;
      return fail(CULE_E_CUDA, std::string(ws ? "WSVJIT" : "VJIT") + " engine: " + jerr);
    } else {  // AUTO: the interpreter engines (the translation did not apply)
      if (e->jit_mod) drv.moduleUnload(e->jit_mod);
      e->jit_mod = nullptr;
      e->jit_fn = nullptr;
      jit_auto = false;
    }
  }
  if (e->engine == 2) {
    // the SIMT translated engine runs
  } else if (want == CULE_ENGINE_JIT || jit_auto) {
    std::string jerr;
    bool from_disk = false;
    std::vector<char> cubin;
    auto& drv = cule::jit::driver();
    if (!drv.ok) jerr = "CUDA driver entry points unavailable";
    else if (cfg->idle_skip) jerr = "the translated engine has no idle-loop skip";
    else {
      RomSet rs = make_romset(roms, rom_lens, n_roms);
      cubin = jit_cubin(rs, n_roms, g, false, false, cfg->tia_delays != 0, &e->jit_insn, &e->jit_compile_s, &from_disk,
                        jerr);
    }
    CUresult cr = CUDA_SUCCESS;
    if (!cubin.empty()) {
      cr = drv.moduleLoadData(&e->jit_mod, cubin.data());
      if (cr == CUDA_SUCCESS) cr = drv.moduleGetFunction(&e->jit_fn, e->jit_mod, "cule_jit_step");
      if (cr == CUDA_SUCCESS)
        cr = drv.funcSetAttribute(e->jit_fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)e->jit_smem);
      if (cr != CUDA_SUCCESS) jerr = "loading the translated kernel failed (CUresult " + std::to_string((int)cr) + ")";
    }
    if (jerr.empty() && e->jit_fn) {
      e->jit = true;
      e->engine = 1;
    } else if (want == CULE_ENGINE_JIT) {
      if (e->jit_mod) drv.moduleUnload(e->jit_mod);
      delete e;
      return fail(CULE_E_CUDA, "JIT engine: " + jerr);
    } else if (e->jit_mod) {
      drv.moduleUnload(e->jit_mod);
      e->jit_mod = nullptr;
    }
  }
  {
    std::lock_guard<std::mutex> lk(g_live_mu);
    g_live.insert(e);
  }
  *out = e;
  return CULE_OK;
}

int cule_reset(cule_env* e, uint64_t seed, void* d_obs, void* stream) {
  CHECK_LIVE(e);
  e->pick_seed = seed;
  cule::Params p = base_params(e);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint32_t blocks = ((uint32_t)e->N + 255) / 256;
  cule::reset_kernel<<<blocks, 256, 0, s>>>(p, (uint32_t)obs_bytes_of(e->cfg.obs_mode),
                                            static_cast<uint8_t*>(d_obs), e->ws + e->L.cobs, 1u);
  cudaMemsetAsync(e->ws + e->L.counters, 0, 32, s);
  return cuda_check("reset_kernel");
}

int cule_reset_stacked(cule_env* e, uint64_t seed, uint8_t* d_stack, void* stream) {
  CHECK_LIVE(e);
  if (e->cfg.obs_mode != CULE_OBS_GRAY84) return fail(CULE_E_INVAL, "frame stacks need GRAY84 observations");
  if (!d_stack) return fail(CULE_E_INVAL, "null buffer");
  e->pick_seed = seed;
  cule::Params p = base_params(e);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint32_t blocks = ((uint32_t)e->N + 255) / 256;
  cule::reset_kernel<<<blocks, 256, 0, s>>>(p, (uint32_t)cule::kObs84, d_stack, e->ws + e->L.cobs, 4u);
  cudaMemsetAsync(e->ws + e->L.counters, 0, 32, s);
  return cuda_check("reset_kernel");
}

static int launch_step(cule_env* e, const uint8_t* d_actions, void* d_obs, int32_t* d_rewards,
                       uint8_t* d_dones, cudaStream_t s, int stack_slot = -1) {
  cule::Params p = base_params(e);
  p.actions = d_actions;
  p.obs = static_cast<uint8_t*>(d_obs);
  if (stack_slot >= 0) {  // frame stack: observation into slot `stack_slot` of u8[N][4][84][84]
    p.stacked = 1u;
    p.stack_slot = (uint32_t)stack_slot;
    p.obs_stride = 4u * cule::kObs84;
    p.obs += (size_t)stack_slot * cule::kObs84;
  }
  p.rewards = d_rewards;
  p.dones = d_dones;
  if (e->engine == 2) {
    p.use_rec = 0u;
    p.epw = e->vepw;
    void* args[] = {&p};
    const CUresult cr = cule::jit::driver().launchKernel(e->jit_fn, e->vgrid, 1, 1, e->vblock, 1, 1, (unsigned)e->vsmem,
                                                         (CUstream)s, args, nullptr);
    if (cr != CUDA_SUCCESS) return fail(CULE_E_CUDA, "cule_vjit_step launch failed (CUresult " + std::to_string((int)cr) + ")");
    return cuda_check("cule_vjit_step");
  }
  if (e->engine == 1) {
    const uint32_t sg = e->sgrid;
    // the persistent kernel's work tickets start from zero on the launch stream (the kernel also
    // re-zeroes them when it finishes; this covers an aborted launch)
    cudaMemsetAsync(e->ws + e->L.tickets, 0, 16, s);
    if (e->jit) {
      p.use_rec = 0u;  // the translated kernel stages no records
      void* args[] = {&p};
      const CUresult cr = cule::jit::driver().launchKernel(e->jit_fn, sg, 1, 1, 32 * cule::kSWarps, 1, 1,
                                                           (unsigned)e->jit_smem, (CUstream)s, args, nullptr);
      if (cr != CUDA_SUCCESS) return fail(CULE_E_CUDA, "cule_jit_step launch failed (CUresult " + std::to_string((int)cr) + ")");
      return cuda_check("cule_jit_step");
    }
    if (e->cfg.obs_mode == CULE_OBS_GRAY84) cule::scalar_kernel<true, false><<<sg, 32 * cule::kSWarps, e->ssmem, s>>>(p);
    else cule::scalar_kernel<false, false><<<sg, 32 * cule::kSWarps, e->ssmem, s>>>(p);
  } else if (e->cfg.obs_mode == CULE_OBS_GRAY84) {
    cule::step_kernel<true><<<e->grid, e->block, e->smem, s>>>(p);
  } else {
    cule::step_kernel<false><<<e->grid, e->block, e->smem, s>>>(p);
  }
  return cuda_check("step_kernel");
}

int cule_step(cule_env* e, const uint8_t* d_actions, void* d_obs, int32_t* d_rewards,
              uint8_t* d_dones, void* stream) {
  CHECK_LIVE(e);
  if (!d_actions || !d_obs || !d_rewards || !d_dones) return fail(CULE_E_INVAL, "null buffer");
  return launch_step(e, d_actions, d_obs, d_rewards, d_dones, static_cast<cudaStream_t>(stream));
}

int cule_step_stacked(cule_env* e, const uint8_t* d_actions, uint8_t* d_stack, int slot, int32_t* d_rewards,
                      uint8_t* d_dones, void* stream) {
  CHECK_LIVE(e);
  if (e->cfg.obs_mode != CULE_OBS_GRAY84) return fail(CULE_E_INVAL, "frame stacks need GRAY84 observations");
  if (!d_actions || !d_stack || !d_rewards || !d_dones) return fail(CULE_E_INVAL, "null buffer");
  if (slot < 0 || slot > 3) return fail(CULE_E_INVAL, "stack slot must be in [0, 3]");
  return launch_step(e, d_actions, d_stack, d_rewards, d_dones, static_cast<cudaStream_t>(stream), slot);
}

int cule_step_host(cule_env* e, const uint8_t* h_actions, void* h_obs, int32_t* h_rewards,
                   uint8_t* h_dones, void* stream) {
  CHECK_LIVE(e);
  if (!h_actions || !h_rewards || !h_dones) return fail(CULE_E_INVAL, "null buffer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t n = (size_t)e->N, ob = obs_bytes_of(e->cfg.obs_mode);
  uint8_t* act = e->ws + e->L.io_act;
  uint8_t* obs = e->ws + e->L.io_obs;
  int32_t* rew = reinterpret_cast<int32_t*>(e->ws + e->L.io_rew);
  uint8_t* done = e->ws + e->L.io_done;
  cudaMemcpyAsync(act, h_actions, n, cudaMemcpyHostToDevice, s);
  int rc = launch_step(e, act, obs, rew, done, s);
  if (rc) return rc;
  if (h_obs) cudaMemcpyAsync(h_obs, obs, n * ob, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(h_rewards, rew, 4 * n, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(h_dones, done, n, cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_check("cule_step_host");
  return cuda_check("cule_step_host");
}

int cule_get_state(cule_env* e, uint8_t* h_states, void* stream) {
  CHECK_LIVE(e);
  if (!h_states) return fail(CULE_E_INVAL, "null buffer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t n = (size_t)e->N;
  cule::pack_kernel<<<(unsigned)((n * 16 + 255) / 256), 256, 0, s>>>(e->ws + e->L.state, e->ws + e->L.pack, (uint32_t)n);
  cudaMemcpyAsync(h_states, e->ws + e->L.pack, 256 * n, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  return cuda_check("cule_get_state");
}

// A snapshot indexes shared-memory ROM/record images (rom_id, bank) and the reset cache
// (rom_id), and the renderer assumes positions in [0, 160): reject anything outside the model
// before it reaches the device.
static int validate_snapshot(const cule_env* e, const uint8_t* s, size_t i) {
  // rom_id must name one of this handle's ROMs (a get_state snapshot carries rom (env_index_base+i)
  // % n_roms; the single-instruction tests load other valid ids on purpose)
  const uint32_t rom = s[61];
  const std::string at = "snapshot of env " + std::to_string(i) + ": ";
  if (rom >= (uint32_t)e->n_roms) return fail(CULE_E_INVAL, at + "rom_id " + std::to_string(rom) + " >= n_roms");
  if (s[5] >= cule::banks_of(e->rom_banks, rom)) return fail(CULE_E_INVAL, at + "bank out of range for its ROM");
  if (s[17] != 0 && s[17] != 3 && s[17] != 6 && s[17] != 10) return fail(CULE_E_INVAL, at + "timer shift not in {0,3,6,10}");
  for (int k = 56; k <= 60; ++k)
    if (s[k] >= 160) return fail(CULE_E_INVAL, at + "object position >= 160");
  const uint32_t fc = (uint32_t)s[8] | ((uint32_t)s[9] << 8) | ((uint32_t)s[10] << 16) | ((uint32_t)s[11] << 24);
  if (fc >= 76u * (uint32_t)e->cfg.line_cap) return fail(CULE_E_INVAL, at + "fc beyond the line cap");
  if (s[62] > 2) return fail(CULE_E_INVAL, at + "fault code not in {0,1,2}");
  if (s[63] > 15) return fail(CULE_E_INVAL, at + "start-delay bits (byte 63) not in [0, 15]");
  if (s[63] && !e->cfg.tia_delays) return fail(CULE_E_INVAL, at + "start-delay bits (byte 63) need tia_delays = 1");
  return CULE_OK;
}

int cule_set_state(cule_env* e, const uint8_t* h_states, void* stream) {
  CHECK_LIVE(e);
  if (!h_states) return fail(CULE_E_INVAL, "null buffer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t n = (size_t)e->N;
  for (size_t i = 0; i < n; ++i) {
    const int rc = validate_snapshot(e, h_states + 256 * i, i);
    if (rc) return rc;
  }
  cudaMemcpyAsync(e->ws + e->L.pack, h_states, 256 * n, cudaMemcpyHostToDevice, s);
  cule::unpack_kernel<<<(unsigned)((n * 16 + 255) / 256), 256, 0, s>>>(e->ws + e->L.state, e->ws + e->L.pack, (uint32_t)n);
  cudaStreamSynchronize(s);
  return cuda_check("cule_set_state");
}

int cule_counters(cule_env* e, int64_t* d_counters4, void* stream) {
  CHECK_LIVE(e);
  if (!d_counters4) return fail(CULE_E_INVAL, "null buffer");
  cudaMemcpyAsync(d_counters4, e->ws + e->L.counters, 32, cudaMemcpyDeviceToDevice,
                  static_cast<cudaStream_t>(stream));
  return cuda_check("cule_counters");
}

int cule_debug_exec(cule_env* e, int n_instr, int32_t* d_status, void* stream) {
  CHECK_LIVE(e);
  if (n_instr < 0) return fail(CULE_E_INVAL, "n_instr must be >= 0");
  cule::Params p = base_params(e);
  p.debug_instr = n_instr;
  p.debug_status = d_status;
  if (e->engine == 1 && e->use_rec) {  // the translated engine has no debug entry: the interpreter's
    const uint32_t sg = e->sgrid;
    cudaMemsetAsync(e->ws + e->L.tickets, 0, 16, static_cast<cudaStream_t>(stream));
    cule::scalar_kernel<false, true><<<sg, 32 * cule::kSWarps, e->ssmem, static_cast<cudaStream_t>(stream)>>>(p);
  } else {
    cule::debug_kernel<<<e->grid, e->block, e->smem, static_cast<cudaStream_t>(stream)>>>(p);
  }
  return cuda_check("debug_kernel");
}

int cule_vtrace(const float* d_rewards, const float* d_values, const float* d_bootstrap, const float* d_log_mu,
                const float* d_log_pi, const uint8_t* d_dones, int T, int B, float gamma, float rho_bar, float c_bar,
                float* d_vs, float* d_rho, float* d_adv, void* stream) {
  if (!d_rewards || !d_values || !d_bootstrap || !d_log_mu || !d_log_pi || !d_dones || !d_vs || !d_rho || !d_adv)
    return fail(CULE_E_INVAL, "null buffer");
  if (T <= 0 || B <= 0) return fail(CULE_E_INVAL, "T and B must be > 0");
  if (!(gamma > 0.0f && gamma <= 1.0f)) return fail(CULE_E_INVAL, "gamma must be in (0, 1]");
  if (!(c_bar > 0.0f && rho_bar >= c_bar)) return fail(CULE_E_INVAL, "need rho_bar >= c_bar > 0");
  // 64-thread blocks: a training-sized batch (thousands of trajectories) still spreads over
  // the SMs, and each SM keeps many trajectories' loads in flight
  const uint32_t blocks = ((uint32_t)B + 63u) / 64u;
  cule::vtrace_kernel<<<blocks, 64, 0, static_cast<cudaStream_t>(stream)>>>(
      d_rewards, d_values, d_bootstrap, d_log_mu, d_log_pi, d_dones, (uint32_t)T, (uint32_t)B, gamma, rho_bar, c_bar,
      d_vs, d_rho, d_adv);
  return cuda_check("vtrace_kernel");
}

int cule_num_envs(const cule_env* e) { return live(e) ? e->N : CULE_E_CLOSED; }
int cule_frameskip(const cule_env* e) { return live(e) ? e->fs : CULE_E_CLOSED; }
int cule_engine(const cule_env* e) {
  if (!live(e)) return CULE_E_CLOSED;
  if (e->engine == 2) return e->vws ? CULE_ENGINE_WSVJIT : CULE_ENGINE_VJIT;
  return e->engine == 0 ? CULE_ENGINE_SIMT : (e->jit ? CULE_ENGINE_JIT : CULE_ENGINE_SCALAR);
}

int cule_jit_prepare(const uint8_t* const* roms, const size_t* rom_lens, int n_roms, int obs_mode, char* info,
                     size_t info_len) {
  return cule_jit_prepare_engine(roms, rom_lens, n_roms, obs_mode, CULE_ENGINE_JIT, info, info_len);
}

int cule_jit_prepare_engine(const uint8_t* const* roms, const size_t* rom_lens, int n_roms, int obs_mode,
                            int engine, char* info, size_t info_len) {
  int rc = check_roms(roms, rom_lens, n_roms);
  if (rc) return rc;
  if (obs_mode != CULE_OBS_RAW && obs_mode != CULE_OBS_GRAY84) return fail(CULE_E_INVAL, "bad obs_mode");
  if (engine != CULE_ENGINE_JIT && engine != CULE_ENGINE_VJIT && engine != CULE_ENGINE_WSVJIT)
    return fail(CULE_E_INVAL, "engine must be JIT, VJIT or WSVJIT");
  RomSet rs = make_romset(roms, rom_lens, n_roms);
  size_t n_insn = 0;
  double secs = 0.0;
  bool from_disk = false;
  std::string err;
  std::vector<char> cubin =
      jit_cubin(rs, n_roms, obs_mode == CULE_OBS_GRAY84, engine != CULE_ENGINE_JIT, engine == CULE_ENGINE_WSVJIT, false,
                &n_insn, &secs, &from_disk, err);
  if (cubin.empty()) return fail(CULE_E_CUDA, "JIT: " + err);
  if (engine == CULE_ENGINE_VJIT) {  // both log capacities (cule_create picks by warps per SM)
    double s2 = 0.0;
    bool d2 = false;
    if (jit_cubin(rs, n_roms, obs_mode == CULE_OBS_GRAY84, true, false, false, &n_insn, &s2, &d2, err, 64).empty())
      return fail(CULE_E_CUDA, "JIT: " + err);
    secs += s2;
  }
  if (info && info_len) {
    snprintf(info, info_len, "%zu instructions translated, cubin %zu bytes, %s %.1f s, cache %s", n_insn,
             cubin.size(), from_disk ? "loaded from disk" : "compiled in", secs, cule::jit::cache_dir().c_str());
  }
  return CULE_OK;
}
size_t cule_obs_bytes(const cule_env* e) { return live(e) ? obs_bytes_of(e->cfg.obs_mode) : 0; }

int cule_destroy(cule_env* e) {
  {
    std::lock_guard<std::mutex> lk(g_live_mu);
    if (!e || !g_live.count(e)) return fail(CULE_E_CLOSED, "invalid or destroyed cule_env handle");
    g_live.erase(e);
  }
  if (e->jit_mod) cule::jit::driver().moduleUnload(e->jit_mod);
  delete e;
  return CULE_OK;
}

const char* cule_last_error(void) { return g_err.c_str(); }

}  // extern "C"
