// kernels.cuh — the step kernel and its companions (cache build, reset, pack/unpack, debug).
//
// Step kernel (one launch per cule_step, one thread per environment):
//   a0  the block stages ROM(s), the micro-coded decode table and the gray LUT into shared
//       memory with TMA bulk copies (cp.async.bulk + mbarrier); every thread gets interleaved
//       (bank-conflict-free) RAM, TIA-register, pixel-writer and write-log slots
//   a1  SoA state load with 16-byte vector loads; action -> SWCHA / INPT4 latches
//   a2  6502 loop with the CPU in registers; a3 TIA writes go to the on-chip log
//   a4  warp-synchronous log replay: collisions every frame, pixels on rendered frames only
//   a6  reward (BCD score delta) and done (terminal flag, episode cap, fault)
//   a7  done envs are overwritten from the reset cache
//   a8  SoA state store; per-GPU counters with warp-aggregated atomics
//   a5  warp-cooperative epilogue: 32 lanes reduce each env's max-pooled gray frame to 84x84
//       (coalesced), or zero a faulted env's observation
#pragma once
#include "cpu.cuh"

namespace cule {

// min resident blocks of 128 threads per SM for the step/debug kernels (register budget)
#ifndef CULE_MINB
#define CULE_MINB 1
#endif

enum RunStatus : int32_t { RUN_BUDGET = 0, RUN_JAM = 1, RUN_RUNAWAY = 2, RUN_FRAME = 3 };
constexpr uint32_t EV_BUDGET = 4;
constexpr uint32_t kFull = 0xFFFFFFFFu;

struct Params {
  uint8_t* state;            // SoA chunks [16][N][16]
  uint32_t N;
  const uint8_t* actions;    // [N]
  uint8_t* obs;              // RAW [N][210][160] / GRAY [N][84][84]
  int32_t* rewards;          // [N]
  uint8_t* dones;            // [N]
  uint8_t* staging;          // GRAY: [N][210][160] max-pooled gray frame
  const uint8_t* roms;       // packed ROM images (global)
  uint32_t rom_bytes;
  uint32_t rom_off[4];
  uint32_t rom_banks;        // 4 KB banks per ROM, packed 8 bits per ROM: 1 (2K/4K), 2 (F8), 4 (F6), 8 (F4)
  uint32_t n_roms;
  const uint64_t* decode;    // [256] batched-engine decode table
  const uint64_t* sdecode;   // [256] scalar-engine decode table
  const uint8_t* gray;       // [128]
  const uint8_t* cache_state;// [n_roms*K][256] packed
  const uint16_t* cache_score;
  uint32_t K;
  unsigned long long* counters;
  uint32_t fs, line_cap, ystart, score_addr, term_addr, term_mask, max_episode_frames;
  uint64_t pick_seed;
  int64_t env_base;
  int32_t debug_instr;
  int32_t* debug_status;
  uint32_t startup_frames, max_random_frames;
  uint64_t cache_seed;
  uint8_t* cache_state_out;
  uint8_t* cache_obs_out;
  uint16_t* cache_score_out;
  uint8_t* cache_staging;
  int32_t* error_flag;
  // thread -> env mapping: `epw` envs per warp (lanes >= epw idle), slots grouped by ROM
  uint32_t epw;
  uint32_t slot_start[4];   // first slot of ROM r
  uint32_t first_env[4];    // first local env of ROM r (envs of ROM r are first_env[r] + n_roms*k)
  uint32_t idle_skip;       // exact idle-loop skip (cule_config.idle_skip; off by default)
  // scalar engine
  const uint64_t* srec;     // pre-decoded cartridge records, one per ROM image byte (scalar_predecode.h)
  uint32_t use_rec;         // records staged into shared memory (they fit)
  unsigned int* tickets;    // [2] env-slot ticket counter and finished-warp counter (self-resetting)
  // GRAY84 observation placement: env i's observation at obs + i * obs_stride.  Frame stack
  // (inference path, R#32): obs = stack + slot * 7056, obs_stride = 4 * 7056, and an
  // env whose step ended the episode gets its new start observation in all four slots
  uint32_t obs_stride;
  uint32_t stacked, stack_slot;
  uint32_t tia_delays;      // delayed register effects (cule_config.tia_delays; R#35)
};

// cartridge bank switching (F8 / F6 / F4; DESIGN.md §2 R#31, R#34): banks of ROM r, and the
// window offset of its first hotspot ($FF8 / $FF6 / $FF4; 0x1000 = none).  An access to window
// offset o switches to bank o - hs_lo when that is below the bank count.
__host__ __device__ __forceinline__ uint32_t banks_of(uint32_t rom_banks, uint32_t r) {
  return (rom_banks >> (8u * r)) & 0xFFu;
}
__host__ __device__ __forceinline__ uint32_t hs_lo_of(uint32_t banks) {
  return banks == 2u ? 0xFF8u : (banks == 4u ? 0xFF6u : (banks == 8u ? 0xFF4u : 0x1000u));
}

// frame stack: all four slots of env i <- the cached start observation of entry ent
__device__ __forceinline__ void stack_fill(const Params& p, uint32_t i, uint32_t ent, uint32_t lane) {
  constexpr uint32_t kQ = (uint32_t)kObs84 / 16u;  // 441 16-byte chunks per observation
  uint8_t* base = p.obs - (size_t)p.stack_slot * kObs84 + (size_t)i * p.obs_stride;
  const uint4* src = reinterpret_cast<const uint4*>(p.cache_obs_out + (size_t)ent * kObs84);
  for (uint32_t q = lane; q < 4u * kQ; q += 32u)
    reinterpret_cast<uint4*>(base + (q / kQ) * kObs84)[q % kQ] = src[q % kQ];
}

// The env a thread emulates.  Envs are laid out so that the lanes of a warp run the same ROM
// (g % n_roms), and at most `epw` lanes of a warp are used: at low env counts fewer envs per
// warp means more warps to hide latency and less divergence per warp.
__device__ __forceinline__ bool env_of_thread(const Params& p, uint32_t& i) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t l = t & 31u;
  if (l >= p.epw) return false;
  const uint32_t s = (t >> 5) * p.epw + l;
  if (s >= p.N) return false;
  uint32_t r = 0;
  while (r + 1 < p.n_roms && s >= p.slot_start[r + 1]) ++r;
  i = p.first_env[r] + p.n_roms * (s - p.slot_start[r]);
  return true;
}

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t hash2(uint64_t a, uint64_t b) { return splitmix64(a ^ splitmix64(b)); }

// ---- TMA bulk staging (cp.async.bulk -> SASS UBLKCP) --------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n"
               ::"r"(smem_addr(bar)), "r"(parity) : "memory");
}

// dynamic shared memory: [mbarrier 16][decode 2048][gray 128][roms][ram 128*B][thread words 4*W*B]
constexpr uint32_t kSmDecode = 16, kSmGray = 16 + 2048, kSmRom = 16 + 2048 + 128;
__host__ __device__ __forceinline__ size_t smem_bytes(uint32_t rom_bytes, uint32_t block) {
  return kSmRom + rom_bytes + 128u * block + 4u * (uint32_t)kThreadWords * block;
}

__device__ __forceinline__ Ctx stage_block(const Params& p, uint8_t* smem, bool gray) {
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_expect_tx(bar, 2048u + 128u + p.rom_bytes);
    bulk_g2s(smem + kSmDecode, p.decode, 2048u, bar);
    bulk_g2s(smem + kSmGray, p.gray, 128u, bar);
    for (uint32_t r = 0; r < p.n_roms; ++r) {
      const uint32_t len = 4096u * banks_of(p.rom_banks, r);
      bulk_g2s(smem + kSmRom + p.rom_off[r], p.roms + p.rom_off[r], len, bar);
    }
  }
  __syncthreads();
  mbar_wait(bar, 0);
  Ctx c;
  c.smem = smem;
  c.decode = reinterpret_cast<const uint64_t*>(smem + kSmDecode);
  c.gray = gray ? smem + kSmGray : nullptr;
  c.rom0 = kSmRom;
  c.s = blockDim.x;
  c.ram0 = kSmRom + p.rom_bytes + 4u * threadIdx.x;
  c.ram_stride = 4u * blockDim.x;
  uint32_t* words = reinterpret_cast<uint32_t*>(smem + kSmRom + p.rom_bytes + 128u * blockDim.x);
  c.tw = words + threadIdx.x;
  c.pw = words + kTiaWords * blockDim.x + threadIdx.x;
  c.lg = words + (kTiaWords + kPwWords) * blockDim.x + threadIdx.x;
  c.ystart = p.ystart;
  c.line_cap = p.line_cap;
  c.cap_cycles = 76u * p.line_cap;
  c.idle_skip = p.idle_skip;
  c.tia_delays = p.tia_delays;
  return c;
}

// ---- snapshot <-> machine (layout DESIGN.md §3) ------------------------------------------------
struct Hdr { uint4 c[4]; };
__device__ __forceinline__ uint32_t hw(const Hdr& h, int w) {
  const uint4& q = h.c[w >> 2];
  return (w & 3) == 0 ? q.x : (w & 3) == 1 ? q.y : (w & 3) == 2 ? q.z : q.w;
}
__device__ __forceinline__ uint32_t hb(const Hdr& h, int o) { return (hw(h, o >> 2) >> (8 * (o & 3))) & 0xFFu; }
__device__ __forceinline__ uint32_t pk(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return (a & 0xFFu) | ((b & 0xFFu) << 8) | ((c & 0xFFu) << 16) | ((d & 0xFFu) << 24);
}

__device__ __forceinline__ void load_machine(Cpu& m, const Ctx& c, const Hdr& h, const Params& p) {
  m.A = hb(h, 0); m.X = hb(h, 1); m.Y = hb(h, 2); m.SP = hb(h, 3); m.setP(hb(h, 4));
  m.bank = hb(h, 5);
  m.PC = hb(h, 6) | (hb(h, 7) << 8);
  m.fc = hw(h, 2);
  m.tW = (int32_t)hw(h, 3);
  m.tV = hb(h, 16); m.tS = hb(h, 17); m.swcha = hb(h, 18); m.inpt4 = hb(h, 19);
  m.vsync = hb(h, 24);
  const uint32_t rom_id = hb(h, 61);
  m.rom_off = p.rom_off[rom_id];
  m.nbank = banks_of(p.rom_banks, rom_id);
  m.hs_lo = hs_lo_of(m.nbank);
  m.flim = m.nbank > 1u ? m.hs_lo - 3u : 0xFFDu;  // fast fetch: pc..pc+2 clear of the hotspots
  m.fault = hb(h, 62);
  m.log_len = 0;
  m.t_phaseA = 3u * m.fc;
  m.now = m.fc;
  m.pff = 0u;
  m.ppc = 0xFFFFFFFFu;
  m.pn = 0u;
  // TIA words (tia.cuh Tia::load layout)
  const uint32_t s = c.s;
  uint32_t* w = c.tw;
  w[0] = hw(h, 7);                                                      // colup0..colubk (28..31)
  w[s] = pk(hb(h, 35), hb(h, 36), hb(h, 37), hb(h, 32));                // pf0 pf1 pf2 ctrlpf
  w[2 * s] = pk(hb(h, 26), hb(h, 27), hb(h, 38), hb(h, 39));            // nusiz0 nusiz1 grp0n grp0o
  w[3 * s] = pk(hb(h, 40), hb(h, 41), hb(h, 46), hb(h, 47));            // grp1n grp1o hmp0 hmp1
  w[4 * s] = pk(hb(h, 48), hb(h, 49), hb(h, 50), hb(h, 63) & 0x0Fu);     // hmm0 hmm1 hmbl, start delay (R#36)
  const uint32_t flags = (hb(h, 25) & 1u) | ((hb(h, 33) & 1u) << 1) | ((hb(h, 34) & 1u) << 2) |
                         ((hb(h, 42) & 1u) << 3) | ((hb(h, 43) & 1u) << 4) | ((hb(h, 44) & 1u) << 5) |
                         ((hb(h, 45) & 1u) << 6) | ((hb(h, 51) & 1u) << 7) | ((hb(h, 52) & 1u) << 8) |
                         ((hb(h, 53) & 1u) << 9) | ((hb(h, 54) & 1u) << 10) | ((hb(h, 55) & 1u) << 11);
  w[5 * s] = flags | (hw(h, 5) & 0xFFFF0000u);                          // comb_line (22..23)
  w[6 * s] = hw(h, 14);                                                 // posP0 posP1 posM0 posM1
  w[7 * s] = hb(h, 60) | ((hw(h, 5) & 0xFFFFu) << 16);                  // posBL, coll (20..21)
  w[8 * s] = 3u * m.fc;                                                 // t_tia
  c.pw[8 * s] = 0u;                                                     // writer idle
}

__device__ __forceinline__ Hdr pack_machine(const Cpu& m, const Ctx& c, uint32_t rom_id) {
  const uint32_t s = c.s;
  const uint32_t* w = c.tw;
  const uint32_t w1 = w[s], w2 = w[2 * s], w3 = w[3 * s], w4 = w[4 * s], w5 = w[5 * s], w6 = w[6 * s],
                 w7 = w[7 * s];
  const uint32_t fl = w5 & 0xFFFFu;
  auto F = [&](int b) { return (fl >> b) & 1u; };
  Hdr h;
  h.c[0] = make_uint4(pk(m.A, m.X, m.Y, m.SP), pk(m.getP(), m.bank, m.PC, m.PC >> 8), m.fc, (uint32_t)m.tW);
  h.c[1] = make_uint4(pk(m.tV, m.tS, m.swcha, m.inpt4), (w7 >> 16) | (w5 & 0xFFFF0000u),
                      pk(m.vsync, F(0), w2, w2 >> 8), w[0]);
  h.c[2] = make_uint4(pk(w1 >> 24, F(1), F(2), w1), pk(w1 >> 8, w1 >> 16, w2 >> 16, w2 >> 24),
                      pk(w3, w3 >> 8, F(3), F(4)), pk(F(5), F(6), w3 >> 16, w3 >> 24));
  h.c[3] = make_uint4(pk(w4, w4 >> 8, w4 >> 16, F(7)), pk(F(8), F(9), F(10), F(11)), w6,
                      pk(w7, rom_id, m.fault, (w4 >> 24) & 0x0Fu));
  return h;
}

__device__ __forceinline__ void ram_from_chunks(const Ctx& c, const uint4* src, size_t stride_chunks) {
  uint32_t* w = reinterpret_cast<uint32_t*>(c.smem + c.ram0);
  const uint32_t s = c.ram_stride >> 2;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    uint4 v = src[k * stride_chunks];
    w[(4 * k + 0) * s] = v.x; w[(4 * k + 1) * s] = v.y; w[(4 * k + 2) * s] = v.z; w[(4 * k + 3) * s] = v.w;
  }
}
__device__ __forceinline__ void ram_to_chunks(const Ctx& c, uint4* dst, size_t stride_chunks) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(c.smem + c.ram0);
  const uint32_t s = c.ram_stride >> 2;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    dst[k * stride_chunks] = make_uint4(w[(4 * k + 0) * s], w[(4 * k + 1) * s], w[(4 * k + 2) * s], w[(4 * k + 3) * s]);
}

__device__ __forceinline__ void set_inputs(Cpu& m, uint32_t a) {
  // ALE action ids: bits 0 up 1 down 2 left 3 right 4 fire; >= 18 = NOOP (DESIGN.md §2 R#7)
  // 5-bit codes of actions 0..11 and 12..17 packed into two constants (no local-memory table)
  constexpr uint64_t kLo = (0ull) | (16ull << 5) | (1ull << 10) | (8ull << 15) | (4ull << 20) | (2ull << 25) |
                           (9ull << 30) | (5ull << 35) | (10ull << 40) | (6ull << 45) | (17ull << 50) | (24ull << 55);
  constexpr uint64_t kHi = (20ull) | (18ull << 5) | (25ull << 10) | (21ull << 15) | (26ull << 20) | (22ull << 25);
  const uint32_t b = a < 12u ? (uint32_t)(kLo >> (5 * a)) & 31u : (a < 18u ? (uint32_t)(kHi >> (5 * (a - 12))) & 31u : 0u);
  uint32_t sw = 0xFFu;
  if (b & 8u) sw &= 0x7Fu;
  if (b & 4u) sw &= 0xBFu;
  if (b & 2u) sw &= 0xDFu;
  if (b & 1u) sw &= 0xEFu;
  m.swcha = sw;
  m.inpt4 = (b & 16u) ? 0u : 0x80u;
}

__device__ __forceinline__ uint32_t bcd(uint32_t b) { return 10u * (b >> 4) + (b & 0xFu); }

// frame end at the VSYNC edge (after the warp flush caught the TIA up to 3 fc): rebase clocks
// to the VSYNC line, canonical timer stamp (DESIGN.md §2 R#6, R#24)
__device__ __forceinline__ void end_frame(Cpu& m, const Ctx& c) {
  const uint32_t L = m.fc / 76u;
  m.fc -= 76u * L;
  m.tW -= (int32_t)(76u * L);
  const uint32_t s = c.s;
  c.tw[8 * s] -= 228u * L;
  const uint32_t w5 = c.tw[5 * s];
  int32_t cl = (int32_t)(int16_t)(w5 >> 16) - (int32_t)L;
  if (cl < 0) cl = -1;
  c.tw[5 * s] = (w5 & 0xFFFFu) | ((uint32_t)(cl & 0xFFFF) << 16);
  const int32_t e = (int32_t)m.fc - m.tW;
  const int32_t VI = (int32_t)(m.tV << m.tS);
  if (e > VI) m.tW = (int32_t)m.fc - (VI + 1 + ((e - VI - 1) & 0xFF));
  m.t_phaseA = 3u * m.fc;
  m.now = m.fc;
}

// Run frames (or an instruction budget) for the envs of one warp.  Must be called by all 32
// lanes together; `active` lanes own an env.  nframes: frames this lane runs; render policy:
// RAW renders the last frame, GRAY the last two.  Returns the RunStatus of this
// lane (RUN_FRAME when all frames completed).
template <bool kGray, bool kDebug>
__device__ __forceinline__ int32_t simulate(Cpu& m, const Ctx& c, bool active, uint32_t nframes,
                                            uint8_t* frame_out, uint32_t* episode_frames, int32_t budget) {
  const uint32_t fill = kGray ? (uint32_t)c.smem[kSmGray] * 0x01010101u : 0u;
  bool running = active && (kDebug || nframes > 0);
  uint32_t f = 0;
  bool render = false;
  int32_t status = RUN_FRAME;
  int32_t count = 0;
  auto begin_frame = [&]() {
    ++f;
    render = !kDebug && (kGray ? (f + 1 >= nframes) : (f == nframes));
    // GRAY: frame fs-1 -> first half of the env's staging pair, frame fs -> second half
    if (render) pw_begin(c.pw, c.s, (kGray && f == nframes) ? frame_out + kFrameBytes : frame_out, fill);
    if (episode_frames) ++*episode_frames;
  };
  if (running) begin_frame();
  while (__any_sync(kFull, running)) {
    uint32_t ev = EV_NONE;
    if (running) {
      if (kDebug && count >= budget) {
        ev = EV_BUDGET;
      } else {
        ev = m.template exec<!kDebug>(c);
        ++count;
      }
    }
    if (__any_sync(kFull, ev != EV_NONE)) {
      const bool fin = ev == EV_FRAME || ev == EV_FAULT || ev == EV_BUDGET;
      if (m.log_len || fin)
        flush_call(c.tw, c.pw, c.lg, c.s, m.log_len, fin ? 1u : 0u, 3u * m.fc, c.ystart, c.gray, c.tia_delays);
      m.log_len = 0;
      if (ev == EV_FRAME) {
        end_frame(m, c);
        if (render) pw_end(c.pw, c.s);
        if (kDebug) { status = RUN_FRAME; running = false; }
        else if (f >= nframes) running = false;
        else begin_frame();
      } else if (ev == EV_FAULT) {
        pw_stop(c.pw, c.s);
        status = (int32_t)m.fault;
        running = false;
      } else if (ev == EV_BUDGET) {
        status = RUN_BUDGET;
        running = false;
      }
    }
  }
  return status;
}

// ---- warp-cooperative area84 ------------------------------------------------------------------
// out[i][j] = round_half_even(sum wr(i,r) wc(j,c) f[r][c] / 200): exact overlap weights of
// 210->84 rows (units 2 vs 5) and 160->84 columns (units 21 vs 40) (§8(c).12)
// m = max(fa, fb) pixel-wise (fb may be null: single frame)
__device__ __forceinline__ uint32_t px_max(const uint8_t* fa, const uint8_t* fb, uint32_t o) {
  const uint32_t a = fa[o];
  return fb ? max(a, (uint32_t)fb[o]) : a;
}
__device__ __forceinline__ void warp_area84(const uint8_t* fa, const uint8_t* fb, uint8_t* out, uint32_t lane) {
  for (uint32_t j = lane; j < 84u; j += 32u) {
    const uint32_t a = 40u * j, b = a + 40u;
    const uint32_t c0 = a / 21u;
    const uint32_t wc0 = min(b, 21u * (c0 + 1)) - a;
    const uint32_t wc1 = min(b, 21u * (c0 + 2)) - 21u * (c0 + 1);
    const uint32_t wc2 = b > 21u * (c0 + 2) ? b - 21u * (c0 + 2) : 0u;
    for (uint32_t i = 0; i < 84u; ++i) {
      const uint32_t r0 = (i >> 1) * 5u + ((i & 1u) ? 2u : 0u);
      const uint32_t w0 = (i & 1u) ? 1u : 2u, w2 = (i & 1u) ? 2u : 1u;
      uint32_t o = r0 * 160u + c0;
      uint32_t s0 = wc0 * px_max(fa, fb, o) + wc1 * px_max(fa, fb, o + 1) + (wc2 ? wc2 * px_max(fa, fb, o + 2) : 0u);
      o += 160;
      uint32_t s1 = wc0 * px_max(fa, fb, o) + wc1 * px_max(fa, fb, o + 1) + (wc2 ? wc2 * px_max(fa, fb, o + 2) : 0u);
      o += 160;
      uint32_t s2 = wc0 * px_max(fa, fb, o) + wc1 * px_max(fa, fb, o + 1) + (wc2 ? wc2 * px_max(fa, fb, o + 2) : 0u);
      const uint32_t S = w0 * s0 + 2u * s1 + w2 * s2;
      uint32_t q = S / 200u;
      const uint32_t r = S - 200u * q;
      q += (r > 100u || (r == 100u && (q & 1u))) ? 1u : 0u;
      out[i * 84u + j] = (uint8_t)q;
    }
  }
}

__device__ __forceinline__ void warp_zero(uint8_t* p, uint32_t bytes, uint32_t lane) {
  uint4* q = reinterpret_cast<uint4*>(p);
  for (uint32_t k = lane; k < bytes / 16u; k += 32u) q[k] = make_uint4(0, 0, 0, 0);
}

template <bool kGray>
__global__ void __launch_bounds__(128, CULE_MINB) step_kernel(Params p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const Ctx c = stage_block(p, smem, kGray);
  uint32_t i = 0;
  const bool active = env_of_thread(p, i);
  const uint32_t lane = threadIdx.x & 31u;
  const size_t N = p.N;
  uint4* st = reinterpret_cast<uint4*>(p.state);
  Cpu m{};
  Hdr h;
  uint32_t rom_id = 0, episode_frames = 0, episode_index = 0, prev_score = 0;
  int32_t episode_return = 0;
  uint8_t* frame_out = nullptr;
  if (active) {
#pragma unroll
    for (int k = 0; k < 4; ++k) h.c[k] = st[k * N + i];
    load_machine(m, c, h, p);
    rom_id = hb(h, 61);
    ram_from_chunks(c, st + 4 * N + i, N);
    const uint4 bk = st[12 * N + i];
    episode_frames = bk.x; episode_index = bk.y; episode_return = (int32_t)bk.z; prev_score = bk.w & 0xFFFFu;
    set_inputs(m, p.actions[i]);
    frame_out = kGray ? p.staging + (size_t)i * (2 * kFrameBytes) : p.obs + (size_t)i * kFrameBytes;
  }
  const int32_t status = simulate<kGray, false>(m, c, active, p.fs, frame_out, &episode_frames, 0);
  uint32_t fault = 0, done = 0, ep_ret_done = 0, ent_done = 0;
  if (active) {
    fault = status == RUN_FRAME ? 0u : (uint32_t)status;
    m.fault = fault;
    // a6: reward and done, once at step end (DESIGN.md §2 R#19)
    const uint32_t score = 100u * bcd(m.ram_rd(c, p.score_addr)) + bcd(m.ram_rd(c, p.score_addr + 1));
    const int32_t reward = fault ? 0 : (int32_t)score - (int32_t)prev_score;
    prev_score = score;
    episode_return += reward;
    done = (fault != 0) || (m.ram_rd(c, p.term_addr) & p.term_mask) != 0 ||
           (p.max_episode_frames > 0 && episode_frames >= p.max_episode_frames);
    p.rewards[i] = reward;
    p.dones[i] = (uint8_t)done;
    if (!done) {
      const Hdr o = pack_machine(m, c, rom_id);
#pragma unroll
      for (int k = 0; k < 4; ++k) st[k * N + i] = o.c[k];
      ram_to_chunks(c, st + 4 * N + i, N);
      st[12 * N + i] = make_uint4(episode_frames, episode_index, (uint32_t)episode_return, prev_score);
    } else {
      // a7: reset from the cache entry picked by (seed, global id, next episode) (R#22)
      ep_ret_done = (uint32_t)episode_return;
      const uint64_t g = (uint64_t)(p.env_base + (int64_t)i);
      const uint32_t e = episode_index + 1u;
      const uint32_t k = (uint32_t)(hash2(hash2(p.pick_seed, g), e) % p.K);
      const uint32_t ent = rom_id * p.K + k;
      const uint4* src = reinterpret_cast<const uint4*>(p.cache_state + (size_t)ent * 256u);
#pragma unroll
      for (int q = 0; q < 12; ++q) {
        uint4 v = src[q];
        if (q == 3) v.w = (v.w & 0xFF0000FFu) | (rom_id << 8);  // rom_id, fault 0, byte 63 kept (R#36)
        st[q * N + i] = v;
      }
      st[12 * N + i] = make_uint4(0u, e, 0u, (uint32_t)p.cache_score[ent]);
      ent_done = ent;
    }
  }
  // a8: counters (warp-aggregated)
  const uint32_t amask = __ballot_sync(kFull, active);
  const uint32_t n_done = __popc(__ballot_sync(kFull, active && done));
  const uint32_t n_fault = __popc(__ballot_sync(kFull, active && fault));
  const int32_t ret_sum = (int32_t)__reduce_add_sync(kFull, active && done ? ep_ret_done : 0u);
  if (lane == 0 && amask) {
    atomicAdd(&p.counters[0], (unsigned long long)__popc(amask) * p.fs);
    if (n_done) atomicAdd(&p.counters[1], (unsigned long long)n_done);
    if (n_done) atomicAdd(&p.counters[2], (unsigned long long)(long long)ret_sum);
    if (n_fault) atomicAdd(&p.counters[3], (unsigned long long)n_fault);
  }
  // a5: warp-cooperative observation epilogue
  for (uint32_t l = 0; l < 32u; ++l) {
    if (!((amask >> l) & 1u)) continue;
    const uint32_t env = __shfl_sync(kFull, i, l);
    const uint32_t f = __shfl_sync(kFull, fault, l);
    const uint32_t dn = __shfl_sync(kFull, done, l), en = __shfl_sync(kFull, ent_done, l);
    if (kGray && p.stacked && dn) {
      stack_fill(p, env, en, lane);
    } else if (kGray) {
      uint8_t* o = p.obs + (size_t)env * p.obs_stride;
      if (f) warp_zero(o, kObs84, lane);
      else {
        const uint8_t* pair = p.staging + (size_t)env * (2 * kFrameBytes);
        // fs >= 2: max of frames fs-1 (first half) and fs (second half); fs == 1: frame fs only
        warp_area84(pair + kFrameBytes, p.fs >= 2 ? pair : nullptr, o, lane);
      }
    } else if (f) {
      warp_zero(p.obs + (size_t)env * kFrameBytes, kFrameBytes, lane);
    }
  }
}

#ifndef CULE_JIT  // the jit module (jit.h) holds only the translated step kernel
// ---- debug: n instructions per env, no rendering ------------------------------------------------
__global__ void __launch_bounds__(128) debug_kernel(Params p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const Ctx c = stage_block(p, smem, false);
  uint32_t i = 0;
  const bool active = env_of_thread(p, i);
  const size_t N = p.N;
  uint4* st = reinterpret_cast<uint4*>(p.state);
  Cpu m{};
  Hdr h;
  uint32_t rom_id = 0;
  if (active) {
#pragma unroll
    for (int k = 0; k < 4; ++k) h.c[k] = st[k * N + i];
    load_machine(m, c, h, p);
    rom_id = hb(h, 61);
    ram_from_chunks(c, st + 4 * N + i, N);
  }
  const int32_t s = simulate<false, true>(m, c, active, 1, nullptr, nullptr, p.debug_instr);
  if (!active) return;
  const Hdr o = pack_machine(m, c, rom_id);
#pragma unroll
  for (int k = 0; k < 4; ++k) st[k * N + i] = o.c[k];
  ram_to_chunks(c, st + 4 * N + i, N);
  if (p.debug_status) p.debug_status[i] = s;
}

// ---- reset cache build: power-on, startup + u_k NOOP frames --------------------------
template <bool kGray>
__global__ void __launch_bounds__(128) cache_kernel(Params p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const Ctx c = stage_block(p, smem, kGray);
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t total = p.n_roms * p.K;
  const bool active = j < total;
  Cpu m{};
  uint32_t nframes = 0, r = 0;
  uint8_t* frame_out = nullptr;
  if (active) {
    r = j / p.K;
    const uint32_t k = j - r * p.K;
    const uint64_t u = hash2(p.cache_seed ^ 0x5245534554434143ull, ((uint64_t)r << 32) | k) %
                       (uint64_t)(p.max_random_frames + 1u);
    nframes = p.startup_frames + (uint32_t)u;
    // power-on (DESIGN.md §2 R#3, R#23): everything zero, SP=$FD, P=$24, last bank, timer s=10
    Hdr h;
    for (int q = 0; q < 4; ++q) h.c[q] = make_uint4(0, 0, 0, 0);
    h.c[0].x = pk(0, 0, 0, 0xFD);
    h.c[0].y = pk(0x24, banks_of(p.rom_banks, r) - 1u, 0, 0);
    h.c[1].x = pk(0, 10, 0xFF, 0x80);
    h.c[1].y = 0xFFFF0000u;  // coll 0, comb_line -1
    h.c[3].w = pk(0, r, 0, 0);
    load_machine(m, c, h, p);
    uint32_t* rw = reinterpret_cast<uint32_t*>(c.smem + c.ram0);
    for (uint32_t a = 0; a < 32u; ++a) rw[a * (c.ram_stride >> 2)] = 0u;
    const uint32_t lo = m.rd<false>(c, 0x1FFCu), hi = m.rd<false>(c, 0x1FFDu);
    m.PC = lo | (hi << 8);
    set_inputs(m, 0);
    frame_out = kGray ? p.cache_staging + (size_t)j * (2 * kFrameBytes) : p.cache_obs_out + (size_t)j * kFrameBytes;
    if (nframes == 0)
      for (uint32_t q = 0; q < (uint32_t)kFrameChunks; ++q) reinterpret_cast<uint4*>(frame_out)[q] = make_uint4(0, 0, 0, 0);
  }
  const int32_t status = simulate<kGray, false>(m, c, active, nframes, frame_out, nullptr, 0);
  uint32_t zero_obs = 0;
  if (active) {
    if (status != RUN_FRAME) atomicOr(p.error_flag, 1);
    const uint32_t score = 100u * bcd(m.ram_rd(c, p.score_addr)) + bcd(m.ram_rd(c, p.score_addr + 1));
    p.cache_score_out[j] = (uint16_t)score;
    m.fault = 0;
    const Hdr o = pack_machine(m, c, 0);
    uint4* dst = reinterpret_cast<uint4*>(p.cache_state_out + (size_t)j * 256u);
#pragma unroll
    for (int q = 0; q < 4; ++q) dst[q] = o.c[q];
    ram_to_chunks(c, dst + 4, 1);
    for (int q = 12; q < 16; ++q) dst[q] = make_uint4(0, 0, 0, 0);
    zero_obs = (status != RUN_FRAME || nframes == 0) ? 1u : 0u;
  }
  if (kGray) {
    const uint32_t amask = __ballot_sync(kFull, active);
    const uint32_t warp_base = j - lane;
    for (uint32_t l = 0; l < 32u; ++l) {
      if (!((amask >> l) & 1u)) continue;
      const uint32_t ent = warp_base + l;
      const uint32_t zf = __shfl_sync(kFull, zero_obs, l);
      uint8_t* o = p.cache_obs_out + (size_t)ent * kObs84;
      if (zf) warp_zero(o, kObs84, lane);
      else {
        const uint8_t* pair = p.cache_staging + (size_t)ent * (2 * kFrameBytes);
        const uint32_t nf = __shfl_sync(kFull, nframes, l);
        warp_area84(pair + kFrameBytes, nf >= 2 ? pair : nullptr, o, lane);
      }
    }
  }
}

// ---- reset: every env <- cache[rom(g)][pick(seed, g, 0)] ----------------------------------------
__global__ void reset_kernel(Params p, uint32_t obs_bytes, uint8_t* d_obs, const uint8_t* cache_obs, uint32_t copies) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.N) return;
  const size_t N = p.N;
  uint4* st = reinterpret_cast<uint4*>(p.state);
  const uint64_t g = (uint64_t)(p.env_base + (int64_t)i);
  const uint32_t rom_id = (uint32_t)(g % p.n_roms);
  const uint32_t k = (uint32_t)(hash2(hash2(p.pick_seed, g), 0) % p.K);
  const uint32_t ent = rom_id * p.K + k;
  const uint4* c = reinterpret_cast<const uint4*>(p.cache_state + (size_t)ent * 256u);
  for (int q = 0; q < 12; ++q) {
    uint4 v = c[q];
    if (q == 3) v.w = (v.w & 0xFF0000FFu) | (rom_id << 8);  // rom_id, fault 0, byte 63 kept (R#36)
    st[q * N + i] = v;
  }
  st[12 * N + i] = make_uint4(0u, 0u, 0u, (uint32_t)p.cache_score[ent]);
  for (int q = 13; q < 16; ++q) st[q * N + i] = make_uint4(0, 0, 0, 0);
  if (d_obs) {  // `copies` consecutive copies per env (4: every slot of a frame stack)
    const uint4* src = reinterpret_cast<const uint4*>(cache_obs + (size_t)ent * obs_bytes);
    for (uint32_t k = 0; k < copies; ++k) {
      uint4* dst = reinterpret_cast<uint4*>(d_obs + ((size_t)i * copies + k) * obs_bytes);
      for (uint32_t q = 0; q < obs_bytes / 16u; ++q) dst[q] = src[q];
    }
  }
}

// ---- SoA <-> packed snapshots -------------------------------------------------------------------
__global__ void pack_kernel(const uint8_t* state, uint8_t* packed, uint32_t N) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t >= (size_t)N * 16u) return;
  const size_t i = t >> 4, k = t & 15u;
  reinterpret_cast<uint4*>(packed)[i * 16u + k] = reinterpret_cast<const uint4*>(state)[k * N + i];
}
__global__ void unpack_kernel(uint8_t* state, const uint8_t* packed, uint32_t N) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t >= (size_t)N * 16u) return;
  const size_t i = t >> 4, k = t & 15u;
  uint4 v = reinterpret_cast<const uint4*>(packed)[i * 16u + k];
  if (k == 3) v.w &= 0x0FFFFFFFu;          // byte 63: RESxx start-delay bits 0-3 (R#36)
  if (k == 12) v.w &= 0x0000FFFFu;         // bytes 206-207 reserved
  if (k >= 13) v = make_uint4(0, 0, 0, 0); // bytes 208-255 reserved
  reinterpret_cast<uint4*>(state)[k * N + i] = v;
}

#endif  // CULE_JIT

}  // namespace cule
