// scalar_kernels.cuh — the scalar engine: one environment per warp.
//
// Lane 0 runs the per-opcode interpreter (scalar_cpu.cuh) in registers, appending TIA writes to
// the warp's on-chip log; when the log fills, a frame ends, the env faults, or a collision latch
// is read, all 32 lanes replay the log together (scalar_tia.cuh).  At low env counts this keeps
// thousands of independent warps in flight (the batched engine has a few envs per warp, and
// its datapath pays for every opcode's fields on every instruction).  Same state layout, same
// cache, same epilogue as the batched engine (kernels.cuh).
#pragma once
#include "kernels.cuh"
#include "scalar_cpu.cuh"
#include "scalar_tia.cuh"

// warps per block of the scalar kernel: one block of 28 warps per SM (<= 72 registers per thread)
#ifndef CULE_SWARPS
#define CULE_SWARPS 28
#endif

namespace cule {

// per-warp shared memory: [RAM 128][TIA words 48][SMach 128][state staging 80][log 4*kSLogCap]
// [fused-observation ring 3 x 160][shaded colours 16][TIA write shadow 64 x u16 (R#37)]
constexpr uint32_t kSLogCap = 128;
constexpr uint32_t kSOffTia = 128, kSOffMach = 176, kSOffStg = 304, kSOffLog = 384;
constexpr uint32_t kSOffRing = kSOffLog + 4 * kSLogCap;
constexpr uint32_t kSOffShd = kSOffRing + 480 + 16;     // after the ring and the shaded colour cache
constexpr uint32_t kSWarpBytes = kSOffShd + 2 * kShdEntries;
constexpr uint32_t kSWarps = CULE_SWARPS;  // warps per block (each warp emulates one env at a time)
constexpr uint32_t kSmSDecode = kSmRom;  // scalar decode table [256] u64 right after the gray LUT
constexpr uint32_t kSDecBytes = 2048;
constexpr uint32_t kSmCols = kSmDecode;  // 84 packed area-average column weights (the batched
                                         // engine's decode-table slot, unused by this kernel)

// [header + gray][decode table][ROM images][records: 8 B per ROM byte, if staged][per-warp areas]
__host__ __device__ __forceinline__ size_t scalar_rec_off(uint32_t rom_bytes) { return kSmSDecode + kSDecBytes + rom_bytes; }
__host__ __device__ __forceinline__ size_t scalar_smem_bytes(uint32_t rom_bytes, bool use_rec) {
  return scalar_rec_off(rom_bytes) + (use_rec ? (size_t)kRecBytes * rom_bytes : 0) + (size_t)kSWarps * kSWarpBytes;
}

__device__ __forceinline__ bool env_of_slot(const Params& p, uint32_t s, uint32_t& i) {
  if (s >= p.N) return false;
  uint32_t r = 0;
  while (r + 1 < p.n_roms && s >= p.slot_start[r + 1]) ++r;
  i = p.first_env[r] + p.n_roms * (s - p.slot_start[r]);
  return true;
}

// snapshot header -> machine record + TIA words (tia.cuh Tia::load layout, stride 1)
__device__ __forceinline__ void load_smach(SMach* M, const Hdr& h, const Params& p, uint32_t* tw) {
  M->A = hb(h, 0); M->X = hb(h, 1); M->Y = hb(h, 2); M->SP = hb(h, 3);
  const uint32_t P = hb(h, 4);
  M->nreg = P & 0x80u; M->V = (P >> 6) & 1u; M->D = (P >> 3) & 1u; M->I = (P >> 2) & 1u;
  M->zreg = (P & 2u) ? 0u : 1u; M->C = P & 1u;
  M->bank = hb(h, 5);
  M->PC = hb(h, 6) | (hb(h, 7) << 8);
  M->fc = hw(h, 2);
  M->tW = (int32_t)hw(h, 3);
  M->tV = hb(h, 16); M->tS = hb(h, 17); M->swcha = hb(h, 18); M->inpt4 = hb(h, 19);
  M->vsync = hb(h, 24);
  const uint32_t rom_id = hb(h, 61);
  M->rom0 = p.rom_off[rom_id];
  M->cart = hs_lo_of(banks_of(p.rom_banks, rom_id)) | (banks_of(p.rom_banks, rom_id) << 16);
  M->fault = hb(h, 62);
  M->log_len = 0u;
  M->t_phaseA = 3u * M->fc;
  M->tia_done = 3u * M->fc;
  M->coll = hw(h, 5) & 0xFFFFu;
  M->pa_T = 0xFFFFFFFFu;
  M->idle_skip = p.idle_skip;
  M->shd = 0u;  // no write elision unless the engine sets up a shadow (R#37)
  tw[0] = hw(h, 7);
  tw[1] = pk(hb(h, 35), hb(h, 36), hb(h, 37), hb(h, 32));
  tw[2] = pk(hb(h, 26), hb(h, 27), hb(h, 38), hb(h, 39));
  tw[3] = pk(hb(h, 40), hb(h, 41), hb(h, 46), hb(h, 47));
  tw[4] = pk(hb(h, 48), hb(h, 49), hb(h, 50), hb(h, 63) & 0x0Fu);  // + RESxx start delay (R#36)
  const uint32_t flags = (hb(h, 25) & 1u) | ((hb(h, 33) & 1u) << 1) | ((hb(h, 34) & 1u) << 2) |
                         ((hb(h, 42) & 1u) << 3) | ((hb(h, 43) & 1u) << 4) | ((hb(h, 44) & 1u) << 5) |
                         ((hb(h, 45) & 1u) << 6) | ((hb(h, 51) & 1u) << 7) | ((hb(h, 52) & 1u) << 8) |
                         ((hb(h, 53) & 1u) << 9) | ((hb(h, 54) & 1u) << 10) | ((hb(h, 55) & 1u) << 11);
  tw[5] = flags | (hw(h, 5) & 0xFFFF0000u);
  tw[6] = hw(h, 14);
  tw[7] = hb(h, 60) | ((hw(h, 5) & 0xFFFFu) << 16);
  tw[8] = 3u * M->fc;
}

__device__ __forceinline__ Hdr pack_smach(const SMach* M, const uint32_t* tw, uint32_t rom_id) {
  const uint32_t w1 = tw[1], w2 = tw[2], w3 = tw[3], w4 = tw[4], w5 = tw[5], w6 = tw[6], w7 = tw[7];
  const uint32_t fl = w5 & 0xFFFFu;
  auto F = [&](int b) { return (fl >> b) & 1u; };
  const uint32_t P = (M->nreg & 0x80u) | (M->V << 6) | 0x20u | (M->D << 3) | (M->I << 2) |
                     ((M->zreg & 0xFFu) == 0u ? 2u : 0u) | M->C;
  Hdr h;
  h.c[0] = make_uint4(pk(M->A, M->X, M->Y, M->SP), pk(P, M->bank, M->PC, M->PC >> 8), M->fc, (uint32_t)M->tW);
  h.c[1] = make_uint4(pk(M->tV, M->tS, M->swcha, M->inpt4), (w7 >> 16) | (w5 & 0xFFFF0000u),
                      pk(M->vsync, F(0), w2, w2 >> 8), tw[0]);
  h.c[2] = make_uint4(pk(w1 >> 24, F(1), F(2), w1), pk(w1 >> 8, w1 >> 16, w2 >> 16, w2 >> 24),
                      pk(w3, w3 >> 8, F(3), F(4)), pk(F(5), F(6), w3 >> 16, w3 >> 24));
  h.c[3] = make_uint4(pk(w4, w4 >> 8, w4 >> 16, F(7)), pk(F(8), F(9), F(10), F(11)), w6,
                      pk(w7, rom_id, M->fault, (w4 >> 24) & 0x0Fu));
  return h;
}

__device__ __forceinline__ void set_inputs_s(SMach* M, uint32_t a) {
  constexpr uint64_t kLo = (0ull) | (16ull << 5) | (1ull << 10) | (8ull << 15) | (4ull << 20) | (2ull << 25) |
                           (9ull << 30) | (5ull << 35) | (10ull << 40) | (6ull << 45) | (17ull << 50) | (24ull << 55);
  constexpr uint64_t kHi = (20ull) | (18ull << 5) | (25ull << 10) | (21ull << 15) | (26ull << 20) | (22ull << 25);
  const uint32_t b = a < 12u ? (uint32_t)(kLo >> (5 * a)) & 31u : (a < 18u ? (uint32_t)(kHi >> (5 * (a - 12))) & 31u : 0u);
  uint32_t sw = 0xFFu;
  if (b & 8u) sw &= 0x7Fu;
  if (b & 4u) sw &= 0xBFu;
  if (b & 2u) sw &= 0xDFu;
  if (b & 1u) sw &= 0xEFu;
  M->swcha = sw;
  M->inpt4 = (b & 16u) ? 0u : 0x80u;
}

// frame end at the VSYNC edge, after the warp caught the TIA up to 3 fc (R#6, R#24)
__device__ __forceinline__ void end_frame_s(SMach* M, uint32_t* tw) {
  const uint32_t L = M->fc / 76u;
  M->fc -= 76u * L;
  M->tW -= (int32_t)(76u * L);
  tw[8] -= 228u * L;
  const uint32_t w5 = tw[5];
  int32_t cl = (int32_t)(int16_t)(w5 >> 16) - (int32_t)L;
  if (cl < 0) cl = -1;
  tw[5] = (w5 & 0xFFFFu) | ((uint32_t)(cl & 0xFFFF) << 16);
  const int32_t e = (int32_t)M->fc - M->tW;
  const int32_t VI = (int32_t)(M->tV << M->tS);
  if (e > VI) M->tW = (int32_t)M->fc - (VI + 1 + ((e - VI - 1) & 0xFF));
  M->t_phaseA = 3u * M->fc;
  M->tia_done = 3u * M->fc;
  M->pa_T = 0xFFFFFFFFu;
}

// one env for one step (or one debug budget); all 32 lanes of the warp call it together
template <bool kGray, bool kDebug>
__device__ __forceinline__ int32_t simulate_s(SMach* M, const uint8_t* rom_all, const uint64_t* dtab, uint8_t* ram,
                                              uint32_t* lg, uint32_t* tw, uint32_t cap_cycles, uint32_t lane,
                                              uint32_t nframes, uint8_t* frame_out, uint32_t& episode_frames,
                                              int32_t budget, uint32_t ystart, const uint8_t* gray,
                                              uint32_t rec_s, uint8_t* obs84, uint8_t* ring, const uint8_t* cols,
                                              uint32_t tia_delays) {
  const uint32_t fill = kGray ? (uint32_t)gray[0] * 0x01010101u : 0u;
  RowBuf rb;
  rb.fill = fill;
  rb.render = false;
  rb.row = 0u;
  rb.frame = nullptr;
  rb.obs84 = nullptr;
  rb.prev = (kGray && nframes >= 2u) ? frame_out : nullptr;  // frame fs-1, staged by this step
  rb.ring_s = smem_addr(ring);
  rb.cols_s = smem_addr(cols);
  shade_init(rb.ring_s + kShadeOff, tw[0], gray);  // colours as loaded (all lanes, same values)
  __syncwarp();
  rb.r0 = rb.r1 = rb.r2 = rb.r3 = fill;
  uint32_t f = 0;
  int32_t status = RUN_FRAME;
  auto begin_frame = [&]() {
    ++f;
    rb.render = !kDebug && (kGray ? (f + 1 >= nframes) : (f == nframes));
    rb.row = 0u;
    rb.r0 = rb.r1 = rb.r2 = rb.r3 = fill;
    rb.frame = frame_out;                               // GRAY84: frame fs-1; RAW: frame fs
    rb.obs84 = (kGray && !kDebug && f == nframes) ? obs84 : nullptr;  // GRAY84 frame fs: fused
    ++episode_frames;
  };
  if (!kDebug && nframes == 0) return RUN_FRAME;
  begin_frame();
  const uint32_t rom_s = smem_addr(rom_all), dtab_s = smem_addr(dtab), ram_s = smem_addr(ram),
                 lg_s = smem_addr(lg);
  for (;;) {
    uint32_t ev = SE_NONE;
    if (lane == 0u) {
#if defined(CULE_JIT) && !defined(CULE_VJIT)
      // the translated engine (jit.h): the ROMs' code compiled into run_cpu_jit (no debug entry)
      ev = run_cpu_jit(M, rom_s, dtab_s, ram_s, lg_s, kSLogCap - 3u, cap_cycles);
      (void)budget;
      (void)rec_s;
#else
      ev = (!kDebug && M->idle_skip)
               ? run_cpu<kDebug, !kDebug>(M, rom_s, dtab_s, ram_s, lg_s, kSLogCap - 3u, cap_cycles, budget, rec_s)
               : run_cpu<kDebug, false>(M, rom_s, dtab_s, ram_s, lg_s, kSLogCap - 3u, cap_cycles, budget, rec_s);
#endif
    }
    ev = __shfl_sync(kFull, ev, 0);
    __syncwarp();
    const uint32_t n = M->log_len;
    const bool fin = ev == SE_FRAME || ev == SE_FAULT || ev == SE_BUDGET;
    const bool tgt = fin || ev == SE_COLL;
    const uint32_t target = fin ? 3u * M->fc : M->abort_T;
    const uint32_t coll = flush_coop(tw, lg, n, tgt, target, rb, lane, ystart, gray, tia_delays);
    if (lane == 0u) {
      M->log_len = 0u;
      M->coll = coll;
      M->tia_done = tgt ? target : tw[8];
      if (ev == SE_COLL && M->abort_pa) { M->pa_T = target; M->pa_coll = coll; }
    }
    __syncwarp();
    if (ev == SE_FRAME) {
      finish_frame_coop(rb, lane);
      if (lane == 0u) end_frame_s(M, tw);
      __syncwarp();
      if (kDebug) { status = RUN_FRAME; break; }
      if (f >= nframes) break;
      begin_frame();
    } else if (ev == SE_FAULT) {
      status = (int32_t)M->fault;
      break;
    } else if (ev == SE_BUDGET) {
      status = RUN_BUDGET;
      break;
    }
  }
  return status;
}

// block staging for the scalar engine (same ROM / decode / gray offsets as the batched engine)
__device__ __forceinline__ void stage_block_s(const Params& p, uint8_t* smem) {
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_expect_tx(bar, kSDecBytes + 128u + p.rom_bytes * (p.use_rec ? 1u + kRecBytes : 1u));
    bulk_g2s(smem + kSmSDecode, p.sdecode, kSDecBytes, bar);
    bulk_g2s(smem + kSmGray, p.gray, 128u, bar);
    uint8_t* rec = smem + scalar_rec_off(p.rom_bytes);
    for (uint32_t r = 0; r < p.n_roms; ++r) {
      const uint32_t len = 4096u * banks_of(p.rom_banks, r);
      bulk_g2s(smem + kSmSDecode + kSDecBytes + p.rom_off[r], p.roms + p.rom_off[r], len, bar);
      if (p.use_rec) bulk_g2s(rec + kRecBytes * p.rom_off[r], p.srec + p.rom_off[r], kRecBytes * len, bar);
    }
  }
  for (uint32_t j = threadIdx.x; j < 84u; j += blockDim.x)
    reinterpret_cast<uint32_t*>(smem + kSmCols)[j] = area84_col(j);
  __syncthreads();
  mbar_wait(bar, 0);
}

// one env for one step (or one debug budget), run by the whole warp
template <bool kGray, bool kDebug>
__device__ __forceinline__ void scalar_env(const Params& p, uint32_t i, uint32_t lane, const uint8_t* smem,
                                           uint8_t* wb) {
  const uint8_t* rom_all = smem + kSmSDecode + kSDecBytes;
  const uint64_t* dtab = reinterpret_cast<const uint64_t*>(smem + kSmSDecode);
  const uint32_t rec_s = smem_addr(smem + scalar_rec_off(p.rom_bytes));  // records (always staged)
  uint8_t* ram = wb;
  uint32_t* tw = reinterpret_cast<uint32_t*>(wb + kSOffTia);
  SMach* M = reinterpret_cast<SMach*>(wb + kSOffMach);
  uint8_t* stg = wb + kSOffStg;
  uint32_t* lg = reinterpret_cast<uint32_t*>(wb + kSOffLog);
  const uint8_t* gray = kGray ? smem + kSmGray : nullptr;
  const size_t N = p.N;
  uint4* st = reinterpret_cast<uint4*>(p.state);
  // state load: lane k < 13 fetches chunk k (header 0-3, RAM 4-11, bookkeeping 12)
  if (lane < 13u) {
    const uint4 v = st[lane * N + i];
    if (lane >= 4u && lane < 12u) reinterpret_cast<uint4*>(ram)[lane - 4u] = v;
    else reinterpret_cast<uint4*>(stg)[lane < 4u ? lane : 4u] = v;
  }
  __syncwarp();
  const Hdr h = *reinterpret_cast<const Hdr*>(stg);
  const uint32_t rom_id = hb(h, 61);
  uint32_t episode_frames = 0, episode_index = 0, prev_score = 0;
  int32_t episode_return = 0;
  if (lane == 0u) {
    load_smach(M, h, p, tw);
    if (!kDebug) {
      const uint4 bk = reinterpret_cast<const uint4*>(stg)[4];
      episode_frames = bk.x; episode_index = bk.y; episode_return = (int32_t)bk.z; prev_score = bk.w & 0xFFFFu;
      set_inputs_s(M, p.actions[i]);
    }
  }
#if defined(CULE_JIT) && !defined(CULE_VJIT)
  // the translated engine drops TIA writes that change nothing (R#37): shadow unknown at step start
  shd_init_warp(smem_addr(wb + kSOffShd), lane);
  if (lane == 0u) M->shd = smem_addr(wb + kSOffShd);
#endif
  __syncwarp();
  uint8_t* frame_out = kDebug ? nullptr
                              : (kGray ? p.staging + (size_t)i * (2 * kFrameBytes) : p.obs + (size_t)i * kFrameBytes);
  uint8_t* obs84 = (kGray && !kDebug) ? p.obs + (size_t)i * p.obs_stride : nullptr;
  const int32_t status = simulate_s<kGray, kDebug>(M, rom_all, dtab, ram, lg, tw, 76u * p.line_cap, lane,
                                                   kDebug ? 1u : p.fs, frame_out, episode_frames, p.debug_instr,
                                                   p.ystart, gray, rec_s, obs84, wb + kSOffRing,
                                                   smem + kSmCols, p.tia_delays);
  if (kDebug) {
    if (lane == 0u) {
      if (status == RUN_JAM) M->fault = 1u;
      if (status == RUN_RUNAWAY) M->fault = 2u;
      const Hdr o = pack_smach(M, tw, rom_id);
      for (int k = 0; k < 4; ++k) reinterpret_cast<uint4*>(stg)[k] = o.c[k];
      if (p.debug_status) p.debug_status[i] = status;
    }
    __syncwarp();
    if (lane < 12u) st[lane * N + i] = lane < 4u ? reinterpret_cast<const uint4*>(stg)[lane]
                                                 : reinterpret_cast<const uint4*>(ram)[lane - 4u];
    __syncwarp();
    return;
  }
  // a6: reward and done, once at step end (R#19); a7: reset from the cache
  uint32_t fault = 0, done = 0, ent = 0;
  if (lane == 0u) {
    fault = status == RUN_FRAME ? 0u : (uint32_t)status;
    M->fault = fault;
    const uint32_t score = 100u * bcd(ram[p.score_addr & 0x7Fu]) + bcd(ram[(p.score_addr + 1) & 0x7Fu]);
    const int32_t reward = fault ? 0 : (int32_t)score - (int32_t)prev_score;
    prev_score = score;
    episode_return += reward;
    done = (fault != 0) || (ram[p.term_addr & 0x7Fu] & p.term_mask) != 0 ||
           (p.max_episode_frames > 0 && episode_frames >= p.max_episode_frames);
    p.rewards[i] = reward;
    p.dones[i] = (uint8_t)done;
    if (!done) {
      const Hdr o = pack_smach(M, tw, rom_id);
      for (int k = 0; k < 4; ++k) reinterpret_cast<uint4*>(stg)[k] = o.c[k];
      reinterpret_cast<uint4*>(stg)[4] = make_uint4(episode_frames, episode_index, (uint32_t)episode_return, prev_score);
    } else {
      const uint64_t g = (uint64_t)(p.env_base + (int64_t)i);
      const uint32_t e_next = episode_index + 1u;
      ent = rom_id * p.K + (uint32_t)(hash2(hash2(p.pick_seed, g), e_next) % p.K);
      reinterpret_cast<uint4*>(stg)[4] = make_uint4(0u, e_next, 0u, (uint32_t)p.cache_score[ent]);
      atomicAdd(&p.counters[1], 1ull);
      atomicAdd(&p.counters[2], (unsigned long long)(long long)episode_return);
      if (fault) atomicAdd(&p.counters[3], 1ull);
    }
    atomicAdd(&p.counters[0], (unsigned long long)p.fs);
  }
  done = __shfl_sync(kFull, done, 0);
  fault = __shfl_sync(kFull, fault, 0);
  ent = __shfl_sync(kFull, ent, 0);
  __syncwarp();
  // a8: state store, lanes 0..12 one chunk each (a done env takes the cache entry's machine part)
  if (lane < 13u) {
    uint4 v;
    if (lane == 12u) v = reinterpret_cast<const uint4*>(stg)[4];
    else if (done) {
      v = reinterpret_cast<const uint4*>(p.cache_state + (size_t)ent * 256u)[lane];
      if (lane == 3u) v.w = (v.w & 0xFF0000FFu) | (rom_id << 8);  // byte 63 kept (R#36)
    } else {
      v = lane < 4u ? reinterpret_cast<const uint4*>(stg)[lane] : reinterpret_cast<const uint4*>(ram)[lane - 4u];
    }
    st[lane * N + i] = v;
  }
  // a5: observation (GRAY84: already reduced row by row while frame fs was drawn; a faulted
  // env's is zero; frame stack: an env that ended its episode gets its new start observation
  // in all four slots)
  if (kGray) {
    if (p.stacked && done) stack_fill(p, i, ent, lane);
    else if (fault) warp_zero(p.obs + (size_t)i * p.obs_stride, kObs84, lane);
  } else if (fault) {
    warp_zero(p.obs + (size_t)i * kFrameBytes, kFrameBytes, lane);
  }
  __syncwarp();
}

// Persistent blocks: every warp takes env slots from a ticket counter until they run out, so
// envs of different lengths balance across the SMs and the staged ROM/record images are reused.
// The last warp to finish resets the counters for the next launch on the stream.
template <bool kGray, bool kDebug>
__device__ __forceinline__ void scalar_kernel_body(const Params& p) {
  extern __shared__ __align__(16) uint8_t smem[];
  stage_block_s(p, smem);
  const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
  const size_t wb_off = scalar_smem_bytes(p.rom_bytes, p.use_rec != 0u) - (size_t)(kSWarps - wib) * kSWarpBytes;
  uint8_t* wb = smem + wb_off;
  for (;;) {
    uint32_t s = 0;
    if (lane == 0u) s = atomicAdd(&p.tickets[0], 1u);
    s = __shfl_sync(kFull, s, 0);
    uint32_t i = 0;
    if (!env_of_slot(p, s, i)) break;
    scalar_env<kGray, kDebug>(p, i, lane, smem, wb);
  }
  if (lane == 0u) {
    const uint32_t total = gridDim.x * kSWarps;
    if (atomicAdd(&p.tickets[1], 1u) == total - 1u) {
      atomicExch(&p.tickets[0], 0u);
      atomicExch(&p.tickets[1], 0u);
    }
  }
}

#ifndef CULE_JIT
template <bool kGray, bool kDebug>
__global__ void __launch_bounds__(32 * kSWarps, 1) scalar_kernel(Params p) {
  scalar_kernel_body<kGray, kDebug>(p);
}
#endif

}  // namespace cule
