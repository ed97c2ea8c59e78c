// kernels.cuh — the step kernel and its companions (cache build, reset, pack/unpack, debug).
//
// Step kernel (one launch per cule_step, one thread per environment):
//   a0  block stages ROM(s), the decode table and the gray LUT into shared memory with one
//       TMA bulk copy each (cp.async.bulk + mbarrier), RAM gets a conflict-free interleaved slot
//   a1  SoA state load with 16-byte vector loads; action -> SWCHA / INPT4 latches
//   a2-a4  frameskip frames of 6502 + RIOT + TIA; only the frames the observation needs render
//   a6  reward (BCD score delta) and done (terminal flag, episode cap, fault)
//   a7  done envs are overwritten from the reset cache
//   a8  SoA state store; per-GPU counters with warp-aggregated atomics
//   a5  warp-cooperative epilogue: the 32 lanes of a warp reduce each env's max-pooled gray
//       frame to 84x84 (coalesced), or zero a faulted env's observation
#pragma once
#include "cpu.cuh"

namespace cule {

struct Params {
  uint8_t* state;            // SoA chunks [16][N][16]
  uint32_t N;
  const uint8_t* actions;    // [N]
  uint8_t* obs;              // RAW [N][210][160] / GRAY [N][84][84]
  int32_t* rewards;          // [N]
  uint8_t* dones;            // [N]
  uint8_t* staging;          // GRAY: [N][210][160] max-pooled gray frame
  const uint8_t* roms;       // packed ROM images (global)
  uint32_t rom_bytes;        // total bytes of all ROMs
  uint32_t rom_off[4];
  uint32_t f8_mask;          // bit r: ROM r is F8 (8 KB)
  uint32_t n_roms;
  const uint32_t* decode;    // [256]
  const uint8_t* gray;       // [128]
  const uint8_t* cache_state;// [n_roms*K][256] packed
  const uint16_t* cache_score;
  uint32_t K;
  unsigned long long* counters;  // [4]
  uint32_t fs, line_cap, ystart, score_addr, term_addr, term_mask, max_episode_frames;
  uint64_t pick_seed;
  int64_t env_base;
  int32_t debug_instr;       // debug kernel: instruction budget
  int32_t* debug_status;
  // cache build
  uint32_t startup_frames, max_random_frames;
  uint64_t cache_seed;
  uint8_t* cache_state_out;
  uint8_t* cache_obs_out;
  uint16_t* cache_score_out;
  uint8_t* cache_staging;    // [n_roms*K][33600]
  int32_t* error_flag;
};

// ---- splitmix64 counter RNG (DESIGN.md §2 R#22) ---------------------------------------------
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t hash2(uint64_t a, uint64_t b) { return splitmix64(a ^ splitmix64(b)); }

// ---- TMA bulk staging helpers (sm_90+ PTX; SASS UBLKCP) ---------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// dynamic shared memory layout: [mbarrier 16][decode 1024][gray 128][roms rom_bytes][ram 128*B]
__device__ __forceinline__ void stage_block(const Params& p, uint8_t* smem, Smem& sm) {
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  uint32_t* dec = reinterpret_cast<uint32_t*>(smem + 16);
  uint8_t* gray = smem + 16 + 1024;
  uint8_t* rom = smem + 16 + 1024 + 128;
  uint8_t* ram = rom + p.rom_bytes;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_expect_tx(bar, 1024u + 128u + p.rom_bytes);
    bulk_g2s(dec, p.decode, 1024u, bar);
    bulk_g2s(gray, p.gray, 128u, bar);
    for (uint32_t r = 0; r < p.n_roms; ++r) {
      uint32_t len = ((p.f8_mask >> r) & 1u) ? 8192u : 4096u;
      bulk_g2s(rom + p.rom_off[r], p.roms + p.rom_off[r], len, bar);
    }
  }
  __syncthreads();
  mbar_wait(bar, 0);
  sm.rom = rom;
  sm.decode = dec;
  sm.gray = gray;
  sm.ram = ram + 4u * threadIdx.x;
  sm.ram_stride = 4u * blockDim.x;
}

__host__ __device__ __forceinline__ size_t smem_bytes(uint32_t rom_bytes, uint32_t block) {
  return 16 + 1024 + 128 + rom_bytes + 128u * block;
}

// ---- snapshot <-> machine ------------------------------------------------------------------
struct Hdr { uint4 c[4]; };

__device__ __forceinline__ uint32_t hb(const Hdr& h, int o) {
  const uint4& c = h.c[o >> 4];
  uint32_t w = ((o >> 2) & 3) == 0 ? c.x : ((o >> 2) & 3) == 1 ? c.y : ((o >> 2) & 3) == 2 ? c.z : c.w;
  return (w >> (8 * (o & 3))) & 0xFFu;
}

__device__ __forceinline__ void unpack_header(Machine& m, const Hdr& h) {
  m.A = hb(h, 0); m.X = hb(h, 1); m.Y = hb(h, 2); m.SP = hb(h, 3); m.setP(hb(h, 4));
  m.bank = hb(h, 5);
  m.PC = hb(h, 6) | (hb(h, 7) << 8);
  m.fc = h.c[0].z;
  m.tW = (int32_t)h.c[0].w;
  m.tV = hb(h, 16); m.tS = hb(h, 17); m.swcha = hb(h, 18); m.inpt4 = hb(h, 19);
  m.coll = hb(h, 20) | (hb(h, 21) << 8);
  m.comb_line = (int32_t)(int16_t)(hb(h, 22) | (hb(h, 23) << 8));
  m.vsync = hb(h, 24); m.vblank = hb(h, 25); m.nusiz0 = hb(h, 26); m.nusiz1 = hb(h, 27);
  m.colup0 = hb(h, 28); m.colup1 = hb(h, 29); m.colupf = hb(h, 30); m.colubk = hb(h, 31);
  m.ctrlpf = hb(h, 32); m.refp0 = hb(h, 33); m.refp1 = hb(h, 34); m.pf0 = hb(h, 35);
  m.pf1 = hb(h, 36); m.pf2 = hb(h, 37); m.grp0n = hb(h, 38); m.grp0o = hb(h, 39);
  m.grp1n = hb(h, 40); m.grp1o = hb(h, 41); m.enam0 = hb(h, 42); m.enam1 = hb(h, 43);
  m.enbln = hb(h, 44); m.enblo = hb(h, 45); m.hmp0 = hb(h, 46); m.hmp1 = hb(h, 47);
  m.hmm0 = hb(h, 48); m.hmm1 = hb(h, 49); m.hmbl = hb(h, 50); m.vdelp0 = hb(h, 51);
  m.vdelp1 = hb(h, 52); m.vdelbl = hb(h, 53); m.resmp0 = hb(h, 54); m.resmp1 = hb(h, 55);
  m.posP0 = hb(h, 56); m.posP1 = hb(h, 57); m.posM0 = hb(h, 58); m.posM1 = hb(h, 59);
  m.posBL = hb(h, 60);
  m.t_tia = 3u * m.fc;
  m.t_phaseA = m.t_tia;
}

__device__ __forceinline__ uint32_t pk(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return (a & 0xFFu) | ((b & 0xFFu) << 8) | ((c & 0xFFu) << 16) | ((d & 0xFFu) << 24);
}

__device__ __forceinline__ Hdr pack_header(const Machine& m, uint32_t rom_id, uint32_t fault) {
  Hdr h;
  h.c[0] = make_uint4(pk(m.A, m.X, m.Y, m.SP), pk(m.getP(), m.bank, m.PC, m.PC >> 8), m.fc, (uint32_t)m.tW);
  h.c[1] = make_uint4(pk(m.tV, m.tS, m.swcha, m.inpt4),
                      (m.coll & 0xFFFFu) | ((uint32_t)(m.comb_line & 0xFFFF) << 16),
                      pk(m.vsync, m.vblank, m.nusiz0, m.nusiz1), pk(m.colup0, m.colup1, m.colupf, m.colubk));
  h.c[2] = make_uint4(pk(m.ctrlpf, m.refp0, m.refp1, m.pf0), pk(m.pf1, m.pf2, m.grp0n, m.grp0o),
                      pk(m.grp1n, m.grp1o, m.enam0, m.enam1), pk(m.enbln, m.enblo, m.hmp0, m.hmp1));
  h.c[3] = make_uint4(pk(m.hmm0, m.hmm1, m.hmbl, m.vdelp0), pk(m.vdelp1, m.vdelbl, m.resmp0, m.resmp1),
                      pk(m.posP0, m.posP1, m.posM0, m.posM1), pk(m.posBL, rom_id, fault, 0));
  return h;
}

__device__ __forceinline__ void ram_from_chunks(Machine& m, const uint4* src, size_t stride_chunks) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    uint4 v = src[k * stride_chunks];
    uint32_t* w = reinterpret_cast<uint32_t*>(m.sm->ram);
    uint32_t s = m.sm->ram_stride >> 2;
    w[(4 * k + 0) * s] = v.x; w[(4 * k + 1) * s] = v.y; w[(4 * k + 2) * s] = v.z; w[(4 * k + 3) * s] = v.w;
  }
}
__device__ __forceinline__ void ram_to_chunks(const Machine& m, uint4* dst, size_t stride_chunks) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(m.sm->ram);
    uint32_t s = m.sm->ram_stride >> 2;
    dst[k * stride_chunks] = make_uint4(w[(4 * k + 0) * s], w[(4 * k + 1) * s], w[(4 * k + 2) * s], w[(4 * k + 3) * s]);
  }
}

__device__ __forceinline__ void set_inputs(Machine& m, uint32_t a) {
  // ALE action ids: 0 NOOP 1 FIRE 2 UP 3 RIGHT 4 LEFT 5 DOWN 6 UR 7 UL 8 DR 9 DL 10 UF 11 RF
  // 12 LF 13 DF 14 URF 15 ULF 16 DRF 17 DLF; >= 18 NOOP.  Bits: 0 up 1 down 2 left 3 right 4 fire
  const uint8_t kDir[18] = {0, 16, 1, 8, 4, 2, 9, 5, 10, 6, 17, 24, 20, 18, 25, 21, 26, 22};
  uint32_t b = a < 18u ? kDir[a] : 0u;
  uint32_t sw = 0xFFu;
  if (b & 8u) sw &= 0x7Fu;
  if (b & 4u) sw &= 0xBFu;
  if (b & 2u) sw &= 0xDFu;
  if (b & 1u) sw &= 0xEFu;
  m.swcha = sw;
  m.inpt4 = (b & 16u) ? 0u : 0x80u;
}

__device__ __forceinline__ uint32_t bcd(uint32_t b) { return 10u * (b >> 4) + (b & 0xFu); }

// ---- warp-cooperative area84 ---------------------------------------------------------------
// out[i][j] = round_half_even(sum_rc wr(i,r) wc(j,c) f[r][c] / 200) with the exact overlap
// weights of 210->84 rows (units 2 vs 5) and 160->84 columns (units 21 vs 40).
__device__ __forceinline__ void warp_area84(const uint8_t* f, uint8_t* out, uint32_t lane) {
  for (uint32_t j = lane; j < 84u; j += 32u) {
    uint32_t a = 40u * j, b = a + 40u;
    uint32_t c0 = a / 21u;
    uint32_t wc0 = min(b, 21u * (c0 + 1)) - a;
    uint32_t wc1 = c0 + 1 < 160u ? min(b, 21u * (c0 + 2)) - max(a, 21u * (c0 + 1)) : 0u;
    uint32_t wc2 = (c0 + 2 < 160u && b > 21u * (c0 + 2)) ? b - 21u * (c0 + 2) : 0u;
    if (wc1 > 40u) wc1 = 0u;
    for (uint32_t i = 0; i < 84u; ++i) {
      uint32_t m5 = (i >> 1) * 5u;
      uint32_t r0 = (i & 1u) ? m5 + 2u : m5;
      uint32_t w0 = (i & 1u) ? 1u : 2u, w1 = 2u, w2 = (i & 1u) ? 2u : 1u;
      const uint8_t* p = f + r0 * 160u + c0;
      uint32_t s0 = wc0 * p[0] + wc1 * (wc1 ? p[1] : 0u) + wc2 * (wc2 ? p[2] : 0u);
      p += 160;
      uint32_t s1 = wc0 * p[0] + wc1 * (wc1 ? p[1] : 0u) + wc2 * (wc2 ? p[2] : 0u);
      p += 160;
      uint32_t s2 = wc0 * p[0] + wc1 * (wc1 ? p[1] : 0u) + wc2 * (wc2 ? p[2] : 0u);
      uint32_t S = w0 * s0 + w1 * s1 + w2 * s2;
      uint32_t q = S / 200u, r = S - 200u * q;
      q += (r > 100u || (r == 100u && (q & 1u))) ? 1u : 0u;
      out[i * 84u + j] = (uint8_t)q;
    }
  }
}

__device__ __forceinline__ void warp_zero(uint8_t* p, uint32_t bytes, uint32_t lane) {
  uint4* q = reinterpret_cast<uint4*>(p);
  for (uint32_t k = lane; k < bytes / 16u; k += 32u) q[k] = make_uint4(0, 0, 0, 0);
}

// ---- one environment's frames for one step ---------------------------------------------------
// Returns 0 or the fault code (1 JAM, 2 runaway).  frame_out: where the rendered frame(s) go
// (RAW: palette frame; GRAY: max-pooled gray frame).
template <bool kGray>
__device__ __forceinline__ uint32_t run_frames(Machine& m, uint32_t nframes, uint8_t* frame_out,
                                               uint32_t line_cap, uint32_t ystart,
                                               uint32_t* episode_frames) {
  const uint32_t fill = kGray ? (uint32_t)m.sm->gray[0] * 0x01010101u : 0u;
  for (uint32_t f = 1; f <= nframes; ++f) {
    bool render = kGray ? (f + 1 >= nframes) : (f == nframes);
    m.render = render;
    m.ystart = ystart;
    if (render) m.pw.begin(frame_out, fill, kGray && f == nframes && nframes >= 2);
    if (episode_frames) ++*episode_frames;
    int32_t st = run_frame<kGray>(m, line_cap, -1);
    if (st != RUN_FRAME) { m.render = 0; return (uint32_t)st; }
    if (render) m.pw.finish();
    m.render = 0;
  }
  return 0;
}

template <bool kGray>
__global__ void __launch_bounds__(128) step_kernel(Params p) {
  extern __shared__ __align__(16) uint8_t smem[];
  Smem sm;
  stage_block(p, smem, sm);
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u;
  const bool active = i < p.N;
  const size_t N = p.N;
  uint4* st = reinterpret_cast<uint4*>(p.state);
  uint32_t fault = 0, done = 0, ep_ret_done = 0;
  int32_t reward = 0;
  uint8_t* frame_out = nullptr;
  if (active) {
    Machine m;
    m.sm = &sm;
    Hdr h;
#pragma unroll
    for (int k = 0; k < 4; ++k) h.c[k] = st[k * N + i];
    unpack_header(m, h);
    const uint32_t rom_id = hb(h, 61);
    m.rom_off = p.rom_off[rom_id];
    m.is_f8 = (p.f8_mask >> rom_id) & 1u;
    ram_from_chunks(m, st + kRamChunk0 * N + i, N);
    uint4 bk = st[kBookChunk * N + i];
    uint32_t episode_frames = bk.x, episode_index = bk.y;
    int32_t episode_return = (int32_t)bk.z;
    uint32_t prev_score = bk.w & 0xFFFFu;
    set_inputs(m, p.actions[i]);
    frame_out = kGray ? p.staging + (size_t)i * kFrameBytes : p.obs + (size_t)i * kFrameBytes;
    fault = run_frames<kGray>(m, p.fs, frame_out, p.line_cap, p.ystart, &episode_frames);
    // a6: reward and done, evaluated once at step end (DESIGN.md §2 R#19)
    uint32_t score = 100u * bcd(m.ram_rd(p.score_addr & 0x7Fu)) + bcd(m.ram_rd((p.score_addr + 1) & 0x7Fu));
    reward = fault ? 0 : (int32_t)score - (int32_t)prev_score;
    prev_score = score;
    episode_return += reward;
    done = (fault != 0) || (m.ram_rd(p.term_addr & 0x7Fu) & p.term_mask) != 0 ||
           (p.max_episode_frames > 0 && episode_frames >= p.max_episode_frames);
    p.rewards[i] = reward;
    p.dones[i] = (uint8_t)done;
    if (!done) {
      Hdr o = pack_header(m, rom_id, fault);
#pragma unroll
      for (int k = 0; k < 4; ++k) st[k * N + i] = o.c[k];
      ram_to_chunks(m, st + kRamChunk0 * N + i, N);
      st[kBookChunk * N + i] = make_uint4(episode_frames, episode_index, (uint32_t)episode_return, prev_score);
    } else {
      // a7: reset from the cache entry picked by (seed, global id, next episode)
      ep_ret_done = (uint32_t)episode_return;
      const uint64_t g = (uint64_t)(p.env_base + (int64_t)i);
      const uint32_t e = episode_index + 1u;
      const uint32_t k = (uint32_t)(hash2(hash2(p.pick_seed, g), e) % p.K);
      const uint32_t ent = rom_id * p.K + k;
      const uint4* c = reinterpret_cast<const uint4*>(p.cache_state + (size_t)ent * 256u);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 v = c[q];
        if (q == 3) v.w = (v.w & 0x000000FFu) | (rom_id << 8);  // rom_id, fault = 0, reserved 0
        st[q * N + i] = v;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) st[(kRamChunk0 + q) * N + i] = c[kRamChunk0 + q];
      st[kBookChunk * N + i] = make_uint4(0u, e, 0u, (uint32_t)p.cache_score[ent]);
    }
  }
  // a8: counters (warp-aggregated)
  const uint32_t amask = __ballot_sync(0xFFFFFFFFu, active);
  const uint32_t n_done = __popc(__ballot_sync(0xFFFFFFFFu, active && done));
  const uint32_t n_fault = __popc(__ballot_sync(0xFFFFFFFFu, active && fault));
  const int32_t ret_sum = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)(active && done ? ep_ret_done : 0u));
  if (lane == 0 && amask) {
    atomicAdd(&p.counters[0], (unsigned long long)__popc(amask) * p.fs);
    if (n_done) atomicAdd(&p.counters[1], (unsigned long long)n_done);
    if (n_done) atomicAdd(&p.counters[2], (unsigned long long)(long long)ret_sum);
    if (n_fault) atomicAdd(&p.counters[3], (unsigned long long)n_fault);
  }
  // a5: warp-cooperative observation epilogue
  const uint32_t warp_base = i - lane;
  for (uint32_t l = 0; l < 32u; ++l) {
    if (!((amask >> l) & 1u)) continue;
    const uint32_t env = warp_base + l;
    const uint32_t f = __shfl_sync(0xFFFFFFFFu, fault, l);
    if (kGray) {
      uint8_t* o = p.obs + (size_t)env * kObs84;
      if (f) warp_zero(o, kObs84, lane);
      else warp_area84(p.staging + (size_t)env * kFrameBytes, o, lane);
    } else if (f) {
      warp_zero(p.obs + (size_t)env * kFrameBytes, kFrameBytes, lane);
    }
  }
}

// ---- debug: n instructions per env, no rendering ------------------------------------------------
__global__ void __launch_bounds__(128) debug_kernel(Params p) {
  extern __shared__ __align__(16) uint8_t smem[];
  Smem sm;
  stage_block(p, smem, sm);
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.N) return;
  const size_t N = p.N;
  uint4* st = reinterpret_cast<uint4*>(p.state);
  Machine m;
  m.sm = &sm;
  Hdr h;
#pragma unroll
  for (int k = 0; k < 4; ++k) h.c[k] = st[k * N + i];
  unpack_header(m, h);
  const uint32_t rom_id = hb(h, 61);
  m.rom_off = p.rom_off[rom_id];
  m.is_f8 = (p.f8_mask >> rom_id) & 1u;
  ram_from_chunks(m, st + kRamChunk0 * N + i, N);
  m.render = 0;
  m.ystart = p.ystart;
  int32_t s = run_frame<false>(m, p.line_cap, p.debug_instr);
  uint32_t fault = hb(h, 62);
  if (s == RUN_JAM) fault = 1;
  if (s == RUN_RUNAWAY) fault = 2;
  Hdr o = pack_header(m, rom_id, fault);
#pragma unroll
  for (int k = 0; k < 4; ++k) st[k * N + i] = o.c[k];
  ram_to_chunks(m, st + kRamChunk0 * N + i, N);
  if (p.debug_status) p.debug_status[i] = s;
}

// ---- reset cache build: power-on, startup + u_k NOOP frames ------------------------
template <bool kGray>
__global__ void __launch_bounds__(128) cache_kernel(Params p) {
  extern __shared__ __align__(16) uint8_t smem[];
  Smem sm;
  stage_block(p, smem, sm);
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t total = p.n_roms * p.K;
  const bool active = j < total;
  uint32_t fault = 0;
  if (active) {
    const uint32_t r = j / p.K, k = j - r * p.K;
    const uint64_t u = hash2(p.cache_seed ^ 0x5245534554434143ull, ((uint64_t)r << 32) | k) %
                       (uint64_t)(p.max_random_frames + 1u);
    const uint32_t nframes = p.startup_frames + (uint32_t)u;
    Machine m;
    m.sm = &sm;
    // power-on (DESIGN.md §2 R#3, R#23): everything zero, SP=$FD, P=$24, last bank, timer s=10
    m.A = m.X = m.Y = 0; m.SP = 0xFD; m.setP(0x24);
    m.fc = 0; m.tV = 0; m.tS = 10; m.tW = 0;
    m.colup0 = m.colup1 = m.colupf = m.colubk = m.ctrlpf = m.pf0 = m.pf1 = m.pf2 = 0;
    m.nusiz0 = m.nusiz1 = m.grp0n = m.grp0o = m.grp1n = m.grp1o = 0;
    m.hmp0 = m.hmp1 = m.hmm0 = m.hmm1 = m.hmbl = 0;
    m.vsync = m.vblank = m.refp0 = m.refp1 = m.enam0 = m.enam1 = m.enbln = m.enblo = 0;
    m.vdelp0 = m.vdelp1 = m.vdelbl = m.resmp0 = m.resmp1 = 0;
    m.posP0 = m.posP1 = m.posM0 = m.posM1 = m.posBL = 0;
    m.coll = 0; m.comb_line = -1;
    m.t_tia = 0; m.t_phaseA = 0;
    m.rom_off = p.rom_off[r];
    m.is_f8 = (p.f8_mask >> r) & 1u;
    m.bank = m.is_f8 ? 1u : 0u;
    for (uint32_t a = 0; a < 128u; a += 4u)
      *reinterpret_cast<uint32_t*>(&sm.ram[(a >> 2) * sm.ram_stride]) = 0u;
    m.now = 0;
    uint32_t lo = m.cart_rd(0x1FFCu), hi = m.cart_rd(0x1FFDu);
    m.PC = lo | (hi << 8);
    set_inputs(m, 0);
    uint8_t* frame_out = kGray ? p.cache_staging + (size_t)j * kFrameBytes : p.cache_obs_out + (size_t)j * kFrameBytes;
    if (nframes == 0) {
      for (uint32_t q = 0; q < (uint32_t)kFrameChunks; ++q)
        reinterpret_cast<uint4*>(frame_out)[q] = make_uint4(0, 0, 0, 0);
    }
    fault = run_frames<kGray>(m, nframes, frame_out, p.line_cap, p.ystart, nullptr);
    if (fault) atomicOr(p.error_flag, 1);
    uint32_t score = 100u * bcd(m.ram_rd(p.score_addr & 0x7Fu)) + bcd(m.ram_rd((p.score_addr + 1) & 0x7Fu));
    p.cache_score_out[j] = (uint16_t)score;
    Hdr o = pack_header(m, 0, 0);
    uint4* dst = reinterpret_cast<uint4*>(p.cache_state_out + (size_t)j * 256u);
#pragma unroll
    for (int q = 0; q < 4; ++q) dst[q] = o.c[q];
    ram_to_chunks(m, dst + kRamChunk0, 1);
    for (int q = kBookChunk; q < 16; ++q) dst[q] = make_uint4(0, 0, 0, 0);
    if (kGray && nframes == 0) fault = 1;  // no frame: observation stays zero
  }
  if (kGray) {
    const uint32_t amask = __ballot_sync(0xFFFFFFFFu, active);
    const uint32_t warp_base = j - lane;
    for (uint32_t l = 0; l < 32u; ++l) {
      if (!((amask >> l) & 1u)) continue;
      const uint32_t ent = warp_base + l;
      const uint32_t f = __shfl_sync(0xFFFFFFFFu, fault, l);
      uint8_t* o = p.cache_obs_out + (size_t)ent * kObs84;
      if (f) warp_zero(o, kObs84, lane);
      else warp_area84(p.cache_staging + (size_t)ent * kFrameBytes, o, lane);
    }
  }
}

// ---- reset: every env <- cache[rom(g)][pick(seed, g, 0)] ----------------------------------------
__global__ void reset_kernel(Params p, uint32_t obs_bytes, uint8_t* d_obs, const uint8_t* cache_obs) {
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
    if (q == 3) v.w = (v.w & 0x000000FFu) | (rom_id << 8);
    st[q * N + i] = v;
  }
  st[kBookChunk * N + i] = make_uint4(0u, 0u, 0u, (uint32_t)p.cache_score[ent]);
  for (int q = 13; q < 16; ++q) st[q * N + i] = make_uint4(0, 0, 0, 0);
  if (d_obs) {
    const uint4* src = reinterpret_cast<const uint4*>(cache_obs + (size_t)ent * obs_bytes);
    uint4* dst = reinterpret_cast<uint4*>(d_obs + (size_t)i * obs_bytes);
    for (uint32_t q = 0; q < obs_bytes / 16u; ++q) dst[q] = src[q];
  }
}

// ---- SoA <-> packed snapshots ----------------------------------------------------------------
__global__ void pack_kernel(const uint8_t* state, uint8_t* packed, uint32_t N) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;  // (env, chunk)
  if (t >= (size_t)N * 16u) return;
  const size_t i = t >> 4, k = t & 15u;
  reinterpret_cast<uint4*>(packed)[i * 16u + k] = reinterpret_cast<const uint4*>(state)[k * N + i];
}
__global__ void unpack_kernel(uint8_t* state, const uint8_t* packed, uint32_t N) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t >= (size_t)N * 16u) return;
  const size_t i = t >> 4, k = t & 15u;
  uint4 v = reinterpret_cast<const uint4*>(packed)[i * 16u + k];
  if (k == 3) v.w &= 0x00FFFFFFu;          // byte 63 reserved
  if (k == 12) v.w &= 0x0000FFFFu;         // bytes 206-207 reserved
  if (k >= 13) v = make_uint4(0, 0, 0, 0); // bytes 208-255 reserved
  reinterpret_cast<uint4*>(state)[k * N + i] = v;
}

}  // namespace cule
