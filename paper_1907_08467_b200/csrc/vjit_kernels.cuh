// vjit_kernels.cuh — the SIMT translated engine ("vjit"): one environment per LANE running the
// translated code of its ROM (jit.h emit_simt), the paper's one-thread-per-game mapping
// with the per-instruction decode compiled away.
//
// Lanes of a warp run envs of the same ROM (the ROM-grouped env -> lane map of env_of_thread).
// run_cpu_vjit() (generated) schedules basic blocks: each round the warp picks the lowest block
// id any lane waits at (__reduce_min_sync) and the lanes at that block run it together, so
// lanes that branched apart re-converge where their paths meet (P:452-465 measures up to 30%
// lost to divergence; this is north_star's warp vote to group envs sharing a PC).  A lane stops
// ("parks") on an event — TIA log full, frame end, collision-latch read, fault — and once every
// lane is parked or idle, each lane replays its own TIA write log (tia.cuh flush_lane: the
// batched engine's per-lane renderer), then the lanes resume.
//
// Shared memory per lane, 131 words (odd, so the same field of the 32 lanes falls in 32
// different banks): TIA words 9 | pixel writer 9 | SMach 32 | RAM 32 | TIA log 32 + 1 | TIA write
// shadow 16 (R#37; log capacity 64: 163 words).
#pragma once

namespace cule {

#ifndef CULE_VWARPS
#define CULE_VWARPS 16  // most warps per block (launch bound); the host picks the block size
#endif
// TIA log entries per lane: 64 while the warps of an SM fit one block (fewer flushes, and each
// flush reloads the TIA and rebuilds its coverage masks), 32 when more warps per SM are needed;
// the host compiles the kernel for one of them (CULE_VLOGCAP) and sizes shared memory to match
#ifndef CULE_VLOGCAP
#define CULE_VLOGCAP 32
#endif
constexpr uint32_t kVLogCap = CULE_VLOGCAP;
constexpr uint32_t kWLogCap = 32;  // per buffer, warp-specialized variant
constexpr uint32_t kVOffTw = 0, kVOffPw = 9, kVOffM = 18, kVOffRam = 50, kVOffLog = 82;
// + the TIA write shadow (R#37: kShdEntries u16, 16 words) after the log
__host__ __device__ constexpr uint32_t vjit_lane_words(uint32_t cap) { return kVOffLog + cap + 1u + kShdEntries / 2u; }
constexpr uint32_t kVOffShd = kVOffLog + kVLogCap + 1u;
constexpr uint32_t kVLaneWords = vjit_lane_words(kVLogCap);
static_assert(kVLaneWords % 2 == 1 && vjit_lane_words(64u) % 2 == 1, "odd lane stride: conflict-free fields");
static_assert(sizeof(SMach) == 4 * (kVOffRam - kVOffM), "SMach slot");

// [mbarrier][area84 column weights][gray LUT][scalar decode table][ROM images][lanes]
__host__ __device__ __forceinline__ size_t vjit_lane_off(uint32_t rom_bytes) { return scalar_rec_off(rom_bytes); }
__host__ __device__ __forceinline__ size_t vjit_smem_bytes(uint32_t rom_bytes, uint32_t threads, uint32_t cap) {
  return vjit_lane_off(rom_bytes) + (size_t)threads * vjit_lane_words(cap) * 4u;
}

// ---- warp-specialized variant (NEXT-2): producer warps emulate, consumer warps render
//
// The paper's two-kernel split (a CPU kernel fills a TIA instruction buffer, a TIA
// kernel renders from it) redone on chip: warps come in pairs that share 32 envs.  The producer
// warp runs the translated CPUs of the 32 envs (run_cpu_vjit) into one of two TIA-log buffers
// per lane; the consumer warp replays the other buffer's logs (flush_lane) and renders.  The
// buffers change hands through mbarriers (FULL: producer -> consumer, EMPTY: consumer ->
// producer), so emulation of round k+1 overlaps the replay of round k.  The producer's view of
// the TIA (collision latches and the clock they hold at) is only valid right after it waited for
// the consumer to drain; between such points M->tia_done is "unknown", so a collision-latch
// read aborts (SE_COLL) and the producer waits for the replay up to the read's clock, as the
// alternating engine does.  A frame end splits in two: the producer rebases the CPU and timer
// clocks at once, the consumer rebases the TIA clock when it replays that frame's last buffer.
//
// Per lane, 151 words (odd): TIA words 9 | pixel writer 9 | SMach 32 | RAM 32 | log buffer 0
// 32 | log buffer 1 32 | per-buffer meta 2 x (n | event << 8, target clock) | pad.
constexpr uint32_t kWOffTw = 0, kWOffPw = 9, kWOffM = 18, kWOffRam = 50, kWOffL0 = 82, kWOffL1 = 114,
                   kWOffMeta = 146;
constexpr uint32_t kWLaneWords = 151;
static_assert(kWLaneWords % 2 == 1 && kWOffMeta + 4 < kWLaneWords, "ws lane layout");
constexpr uint32_t kWBarBytes = 16u * 4u * 8u;  // 4 mbarriers per pair, up to 16 pairs
__host__ __device__ __forceinline__ size_t wsvjit_lane_off(uint32_t rom_bytes) {
  return scalar_rec_off(rom_bytes) + kWBarBytes;
}
__host__ __device__ __forceinline__ size_t wsvjit_smem_bytes(uint32_t rom_bytes, uint32_t pairs) {
  return wsvjit_lane_off(rom_bytes) + (size_t)pairs * 32u * 4u * kWLaneWords;  // a pair shares 32 lane areas
}

#ifdef CULE_VJIT  // the device code lives in the generated module (it calls run_cpu_vjit)
// GRAY84 observation of one env from its staged gray frames fs (fa) and fs-1 (fb; null for
// fs = 1), by the whole warp, in groups of five rows (group g closes output rows 2g and 2g+1):
// both frames' 800-byte row groups stream HBM -> shared memory with cp.async, three groups
// ahead of the one being reduced (a 4-slot ring of 1600 bytes); the group is max-pooled in place
// (__vmaxu4), then each lane takes output columns j: the five rows' horizontal sums with the
// packed column weights (area84_col), rows weighted 2:2:1 / 1:2:2 (total 200, round half to even;
// R#16, R#17 — the arithmetic of kernels.cuh warp_area84).
__device__ __forceinline__ void cp_async16(uint32_t dst_s, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst_s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int kN>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(kN) : "memory"); }

constexpr uint32_t kA84Slot = 1600u, kA84Bytes = 4u * kA84Slot;  // per-warp ring (shared memory)
static_assert(kA84Bytes <= 32u * 4u * vjit_lane_words(32u), "the epilogue ring fits in the warp's lane areas");

__device__ __forceinline__ void warp_area84_staged(const uint8_t* fa, const uint8_t* fb, uint8_t* out, uint32_t lane,
                                                   uint32_t ring_s, uint32_t cols_s) {
  const uint32_t nq = fb ? 100u : 50u;  // 16-byte chunks per group: frame fs, then frame fs-1
  // group g's copies (one call site in the loop below: the prologue runs it for groups 0-2)
  // the lane's output columns (lane, lane + 32, lane + 64): first source column and the packed
  // byte weights wc0 | wc1 << 8 | wc2 << 16, once per env
  uint32_t cs[3], wpk[3];
#pragma unroll
  for (uint32_t u = 0; u < 3u; ++u) {
    const uint32_t j = lane + 32u * u;
    uint32_t cw = 0u;
    if (j < 84u) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cw) : "r"(cols_s + 4u * j) : "memory");
    cs[u] = cw & 0xFFu;
    wpk[u] = cw >> 8;
  }
  auto issue = [&](uint32_t g) {
    if (g < 42u) {
      const uint32_t slot = ring_s + (g & 3u) * kA84Slot;
#pragma unroll 1
      for (uint32_t q = lane; q < nq; q += 32u)
        cp_async16(slot + 16u * q, (q < 50u ? fa : fb) + 800u * g + 16u * (q < 50u ? q : q - 50u));
    }
    cp_async_commit();  // (an empty group past the end keeps the wait count uniform)
  };
#pragma unroll 1
  for (uint32_t g = 0; g < 3u; ++g) issue(g);
#pragma unroll 1
  for (uint32_t g = 0; g < 42u; ++g) {
    cp_async_wait<2>();  // group g has landed (groups g+1, g+2 may be in flight)
    __syncwarp();
    const uint32_t slot = ring_s + (g & 3u) * kA84Slot;
    if (fb) {
      for (uint32_t q = lane; q < 50u; q += 32u) {
        uint32_t a0, a1, a2, a3, b0, b1, b2, b3;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(slot + 16u * q) : "memory");
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3) : "r"(slot + 800u + 16u * q) : "memory");
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(slot + 16u * q), "r"(__vmaxu4(a0, b0)),
                     "r"(__vmaxu4(a1, b1)), "r"(__vmaxu4(a2, b2)), "r"(__vmaxu4(a3, b3)) : "memory");
      }
      __syncwarp();
    }
#pragma unroll
    for (uint32_t u = 0; u < 3u; ++u) {  // output columns lane, lane + 32, lane + 64 (< 84)
      const uint32_t j = lane + 32u * u;
      if (j >= 84u) break;
      // the five rows' weighted sums: bytes c0 .. c0+3 of each row by two aligned 32-bit loads
      // and a funnel shift, weighted by one byte dot product (the 4th weight is 0; reading one
      // byte past a row stays inside the ring slot)
      const uint32_t q = slot + cs[u];
      const uint32_t qa = q & ~3u, sh = 8u * (q & 3u);
      uint32_t h[5];
#pragma unroll
      for (int r = 0; r < 5; ++r) {
        uint32_t lo, hi;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(lo) : "r"(qa + 160u * r) : "memory");
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(hi) : "r"(qa + 160u * r + 4u) : "memory");
        h[r] = __dp4a(__funnelshift_r(lo, hi, sh), wpk[u], 0u);
      }
      const uint32_t S0 = 2u * h[0] + 2u * h[1] + h[2], S1 = h[2] + 2u * h[3] + 2u * h[4];
      uint32_t q0 = S0 / 200u, q1 = S1 / 200u;
      const uint32_t r0 = S0 - 200u * q0, r1 = S1 - 200u * q1;
      q0 += (r0 > 100u || (r0 == 100u && (q0 & 1u))) ? 1u : 0u;
      q1 += (r1 > 100u || (r1 == 100u && (q1 & 1u))) ? 1u : 0u;
      out[2u * g * 84u + j] = (uint8_t)q0;
      out[(2u * g + 1u) * 84u + j] = (uint8_t)q1;
    }
    __syncwarp();  // slot g & 3 is free again
    issue(g + 3u);
  }
  cp_async_wait<0>();
  __syncwarp();
}

// frames of one step for the lanes of a warp (all 32 lanes call it together)
template <bool kGray>
__device__ __forceinline__ int32_t simulate_v(SMach* M, uint32_t* tw, uint32_t* pw, const uint32_t* lg, bool active,
                                              uint32_t nframes, uint8_t* frame_out, uint32_t& episode_frames,
                                              const Params& p, uint32_t rom_all0, uint32_t dtab0, uint32_t ram0,
                                              uint32_t lg0, const uint8_t* gray) {
  const uint32_t fill = kGray ? (uint32_t)gray[0] * 0x01010101u : 0u;
  bool running = active && nframes > 0;
  uint32_t f = 0;
  bool render = false;
  int32_t status = RUN_FRAME;
  auto begin_frame = [&]() {
    ++f;
    render = kGray ? (f + 1 >= nframes) : (f == nframes);
    // GRAY: frame fs-1 -> first half of the env's staging pair, frame fs -> second half
    if (render) pw_begin(pw, 1u, (kGray && f == nframes) ? frame_out + kFrameBytes : frame_out, fill);
    ++episode_frames;
  };
  if (running) begin_frame();
  const uint32_t cap_cycles = 76u * p.line_cap;
  while (__any_sync(kFull, running)) {
    const uint32_t ev = run_cpu_vjit(M, rom_all0, dtab0, ram0, lg0, kVLogCap - 3u, cap_cycles, running);
    if (running) {
      const uint32_t n = M->log_len;
      const bool fin = ev == SE_FRAME || ev == SE_FAULT;
      const bool tgt = fin || ev == SE_COLL;
      const uint32_t target = fin ? 3u * M->fc : M->abort_T;
      if (n || tgt) flush_lane(tw, pw, lg, 1u, n, tgt, target, p.ystart, gray, p.tia_delays);
      const uint32_t coll = tw[7] >> 16;
      M->log_len = 0u;
      M->coll = coll;
      M->tia_done = tgt ? target : tw[8];
      if (ev == SE_COLL && M->abort_pa) { M->pa_T = target; M->pa_coll = coll; }
      if (ev == SE_FRAME) {
        end_frame_s(M, tw);
        if (render) pw_end(pw, 1u);
        if (f >= nframes) running = false;
        else begin_frame();
      } else if (ev == SE_FAULT) {
        pw_stop(pw, 1u);
        status = (int32_t)M->fault;
        running = false;
      }
    }
  }
  return status;
}

template <bool kGray>
__device__ __forceinline__ void vjit_kernel_body(const Params& p) {
  extern __shared__ __align__(16) uint8_t smem[];
  stage_block_s(p, smem);  // decode table, gray LUT, ROM images (no records: p.use_rec == 0)
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t* lw = reinterpret_cast<uint32_t*>(smem + vjit_lane_off(p.rom_bytes)) + threadIdx.x * kVLaneWords;
  uint32_t* tw = lw + kVOffTw;
  uint32_t* pw = lw + kVOffPw;
  SMach* M = reinterpret_cast<SMach*>(lw + kVOffM);
  uint32_t* ramw = lw + kVOffRam;
  const uint8_t* ram = reinterpret_cast<const uint8_t*>(ramw);
  uint32_t* lg = lw + kVOffLog;
  const uint8_t* gray = kGray ? smem + kSmGray : nullptr;
  uint32_t i = 0;
  const bool active = env_of_thread(p, i);
  const size_t N = p.N;
  uint4* st = reinterpret_cast<uint4*>(p.state);
  uint32_t rom_id = 0, episode_frames = 0, episode_index = 0, prev_score = 0;
  int32_t episode_return = 0;
  uint8_t* frame_out = nullptr;
  // a1: SoA state load (16-byte chunks), machine record, RAM, bookkeeping, input latch
  if (active) {
    Hdr h;
#pragma unroll
    for (int k = 0; k < 4; ++k) h.c[k] = st[k * N + i];
    rom_id = hb(h, 61);
    load_smach(M, h, p, tw);
    M->shd = smem_addr(lw + kVOffShd);  // TIA write elision (R#37): every entry unknown at step start
    shd_init_lane(M->shd);
    pw[8] = 0u;  // pixel writer idle until a rendered frame begins
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint4 v = st[(4 + k) * N + i];
      ramw[4 * k] = v.x; ramw[4 * k + 1] = v.y; ramw[4 * k + 2] = v.z; ramw[4 * k + 3] = v.w;
    }
    const uint4 bk = st[12 * N + i];
    episode_frames = bk.x; episode_index = bk.y; episode_return = (int32_t)bk.z; prev_score = bk.w & 0xFFFFu;
    set_inputs_s(M, p.actions[i]);
    frame_out = kGray ? p.staging + (size_t)i * (2 * kFrameBytes) : p.obs + (size_t)i * kFrameBytes;
  }
  const uint8_t* smem_c = smem;
  const int32_t status =
      simulate_v<kGray>(M, tw, pw, lg, active, p.fs, frame_out, episode_frames, p,
                        smem_addr(smem_c + kSmSDecode + kSDecBytes), smem_addr(smem_c + kSmSDecode), smem_addr(ramw),
                        smem_addr(lg), gray);
  uint32_t fault = 0, done = 0, ep_ret_done = 0, ent_done = 0;
  if (active) {
    fault = status == RUN_FRAME ? 0u : (uint32_t)status;
    M->fault = fault;
    // a6: reward and done, once at step end (R#19)
    const uint32_t score = 100u * bcd(ram[p.score_addr & 0x7Fu]) + bcd(ram[(p.score_addr + 1) & 0x7Fu]);
    const int32_t reward = fault ? 0 : (int32_t)score - (int32_t)prev_score;
    prev_score = score;
    episode_return += reward;
    done = (fault != 0) || (ram[p.term_addr & 0x7Fu] & p.term_mask) != 0 ||
           (p.max_episode_frames > 0 && episode_frames >= p.max_episode_frames);
    p.rewards[i] = reward;
    p.dones[i] = (uint8_t)done;
    if (!done) {  // a8: SoA state store
      const Hdr o = pack_smach(M, tw, rom_id);
#pragma unroll
      for (int k = 0; k < 4; ++k) st[k * N + i] = o.c[k];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        st[(4 + k) * N + i] = make_uint4(ramw[4 * k], ramw[4 * k + 1], ramw[4 * k + 2], ramw[4 * k + 3]);
      st[12 * N + i] = make_uint4(episode_frames, episode_index, (uint32_t)episode_return, prev_score);
    } else {  // a7: reset from the cache entry picked by (seed, global id, next episode) (R#22)
      ep_ret_done = (uint32_t)episode_return;
      const uint64_t g = (uint64_t)(p.env_base + (int64_t)i);
      const uint32_t e = episode_index + 1u;
      const uint32_t ent = rom_id * p.K + (uint32_t)(hash2(hash2(p.pick_seed, g), e) % p.K);
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
  // a5: warp-cooperative observation epilogue, one env at a time; the warp's lane areas are
  // free now (state stored) and hold the epilogue's 6.4 KB ring
  __syncwarp();
  const uint32_t buf_s = smem_addr(lw - threadIdx.x * kVLaneWords + (threadIdx.x & ~31u) * kVLaneWords);
  const uint32_t cols_s = smem_addr(smem + kSmCols);
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
        warp_area84_staged(pair + kFrameBytes, p.fs >= 2 ? pair : nullptr, o, lane, buf_s, cols_s);
      }
    } else if (f) {
      warp_zero(p.obs + (size_t)env * kFrameBytes, kFrameBytes, lane);
    }
  }
}

// ---- warp-specialized variant: device code ------------------------------------------------------
__device__ __forceinline__ void mbar_arrive1(uint32_t bar_s) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar_s) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t bar_s, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n WS_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WS_WAIT_%=;\n}\n"
               ::"r"(bar_s), "r"(parity) : "memory");
}
// the two warps of a pair (named barrier 1 + pair; the non-aligned form: the warps arrive from
// different code)
__device__ __forceinline__ void pair_sync(uint32_t pair) {
  __syncwarp();
  asm volatile("barrier.sync %0, 64;" ::"r"(1u + pair) : "memory");
}

// CPU half of a frame end (R#6, R#24): clocks rebased to the VSYNC line, canonical timer stamp;
// the TIA half (its clock, the HMOVE comb line) is rebased by the consumer (end_frame_tia)
__device__ __forceinline__ void end_frame_cpu(SMach* M) {
  const uint32_t L = M->fc / 76u;
  M->fc -= 76u * L;
  M->tW -= (int32_t)(76u * L);
  const int32_t e = (int32_t)M->fc - M->tW;
  const int32_t VI = (int32_t)(M->tV << M->tS);
  if (e > VI) M->tW = (int32_t)M->fc - (VI + 1 + ((e - VI - 1) & 0xFF));
  M->t_phaseA = 3u * M->fc;
  M->pa_T = 0xFFFFFFFFu;
}
__device__ __forceinline__ void end_frame_tia(uint32_t* tw, uint32_t L) {
  tw[8] -= 228u * L;
  const uint32_t w5 = tw[5];
  int32_t cl = (int32_t)(int16_t)(w5 >> 16) - (int32_t)L;
  if (cl < 0) cl = -1;
  tw[5] = (w5 & 0xFFFFu) | ((uint32_t)(cl & 0xFFFF) << 16);
}

template <bool kGray>
__device__ __forceinline__ void wsvjit_kernel_body(const Params& p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, pair = warp >> 1;
  const bool producer = (warp & 1u) == 0u;
  const uint32_t pairs = blockDim.x >> 6;
  const uint32_t bar0 = smem_addr(smem + scalar_rec_off(p.rom_bytes)) + 32u * pair;  // FULL0 FULL1 EMPTY0 EMPTY1
  if (producer && lane == 0u) {
    for (uint32_t k = 0; k < 4u; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8u * k) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  stage_block_s(p, smem);  // (its __syncthreads also publishes the mbarrier initialisation)
  uint32_t* pw_base = reinterpret_cast<uint32_t*>(smem + wsvjit_lane_off(p.rom_bytes)) + pair * 32u * kWLaneWords;
  uint32_t* lw = pw_base + lane * kWLaneWords;
  uint32_t* tw = lw + kWOffTw;
  uint32_t* pw = lw + kWOffPw;
  SMach* M = reinterpret_cast<SMach*>(lw + kWOffM);
  uint32_t* ramw = lw + kWOffRam;
  const uint8_t* ram = reinterpret_cast<const uint8_t*>(ramw);
  uint32_t* meta = lw + kWOffMeta;
  const uint8_t* gray = kGray ? smem + kSmGray : nullptr;
  uint32_t i = 0;
  const bool active = env_of_slot(p, (blockIdx.x * pairs + pair) * p.epw + lane, i) && lane < p.epw;
  const size_t N = p.N;
  uint4* st = reinterpret_cast<uint4*>(p.state);
  const uint32_t nframes = p.fs;
  uint32_t rom_id = 0, episode_frames = 0, episode_index = 0, prev_score = 0;
  int32_t episode_return = 0, status = RUN_FRAME;
  if (producer) {
    // a1: state load by the producer (machine record, RAM, TIA words)
    if (active) {
      Hdr h;
#pragma unroll
      for (int k = 0; k < 4; ++k) h.c[k] = st[k * N + i];
      rom_id = hb(h, 61);
      load_smach(M, h, p, tw);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint4 v = st[(4 + k) * N + i];
        ramw[4 * k] = v.x; ramw[4 * k + 1] = v.y; ramw[4 * k + 2] = v.z; ramw[4 * k + 3] = v.w;
      }
      const uint4 bk = st[12 * N + i];
      episode_frames = bk.x; episode_index = bk.y; episode_return = (int32_t)bk.z; prev_score = bk.w & 0xFFFFu;
      set_inputs_s(M, p.actions[i]);
    }
    pair_sync(pair);
    const uint32_t rom_all0 = smem_addr(smem + kSmSDecode + kSDecBytes), dtab0 = smem_addr(smem + kSmSDecode);
    const uint32_t ram0 = smem_addr(ramw), cap_cycles = 76u * p.line_cap;
    bool running = active && nframes > 0;
    uint32_t f = running ? 1u : 0u;
    if (running) ++episode_frames;
    uint32_t buf = 0, pending0 = 0, pending1 = 0, waited0 = 0, waited1 = 0;
    auto wait_empty = [&](uint32_t b) {
      if (b == 0u) { mbar_wait_s(bar0 + 16u, waited0 & 1u); ++waited0; pending0 = 0u; }
      else { mbar_wait_s(bar0 + 24u, waited1 & 1u); ++waited1; pending1 = 0u; }
    };
    while (__any_sync(kFull, running)) {
      if (buf == 0u ? pending0 : pending1) wait_empty(buf);  // the consumer is done with this buffer
      M->log_len = 0u;
      const uint32_t ev = run_cpu_vjit(M, rom_all0, dtab0, ram0, smem_addr(lw + (buf ? kWOffL1 : kWOffL0)),
                                       kWLogCap - 3u, cap_cycles, running);
      bool need_sync = false;
      uint32_t tgt = 0u;
      if (running) {
        const bool fin = ev == SE_FRAME || ev == SE_FAULT;
        tgt = fin ? 3u * M->fc : (ev == SE_COLL ? M->abort_T : 0u);
        meta[2u * buf] = M->log_len | (ev << 8);
        meta[2u * buf + 1u] = tgt;
        if (ev == SE_FRAME) {
          end_frame_cpu(M);
          if (f >= nframes) running = false;
          else { ++f; ++episode_frames; }
        } else if (ev == SE_FAULT) {
          status = (int32_t)M->fault;
          running = false;
        } else if (ev == SE_COLL) {
          need_sync = true;
        }
        M->tia_done = 0xFFFFFFFFu;  // the TIA view is unknown until the next drain
      } else {
        meta[2u * buf] = 0u;
        meta[2u * buf + 1u] = 0u;
      }
      __syncwarp();
      if (lane == 0u) mbar_arrive1(bar0 + 8u * buf);  // FULL[buf]
      if (buf == 0u) pending0 = 1u; else pending1 = 1u;
      if (__any_sync(kFull, need_sync)) {
        wait_empty(buf);  // replayed up to every lane's target: take the TIA's view
        if (active) {
          const uint32_t coll = tw[7] >> 16;
          M->coll = coll;
          M->tia_done = ev == SE_COLL ? tgt : tw[8];
          if (ev == SE_COLL && M->abort_pa) { M->pa_T = tgt; M->pa_coll = coll; }
        }
      }
      buf ^= 1u;
    }
    if (pending0) wait_empty(0u);
    if (pending1) wait_empty(1u);
  } else {
    // consumer: replay each buffer the producer hands over, render, rebase the TIA at frame ends
    pair_sync(pair);
    uint8_t* frame_out = nullptr;
    if (active) frame_out = kGray ? p.staging + (size_t)i * (2 * kFrameBytes) : p.obs + (size_t)i * kFrameBytes;
    const uint32_t fill = kGray ? (uint32_t)gray[0] * 0x01010101u : 0u;
    bool done = !(active && nframes > 0);
    uint32_t f = 0;
    bool render = false;
    auto begin_frame = [&]() {
      ++f;
      render = kGray ? (f + 1 >= nframes) : (f == nframes);
      if (render) pw_begin(pw, 1u, (kGray && f == nframes) ? frame_out + kFrameBytes : frame_out, fill);
    };
    pw[8] = 0u;
    if (!done) begin_frame();
    uint32_t buf = 0, full0 = 0, full1 = 0;
    while (!__all_sync(kFull, done)) {
      if (buf == 0u) { mbar_wait_s(bar0, full0 & 1u); ++full0; }
      else { mbar_wait_s(bar0 + 8u, full1 & 1u); ++full1; }
      if (!done) {
        const uint32_t m0 = meta[2u * buf], T = meta[2u * buf + 1u];
        const uint32_t n = m0 & 0xFFu, ev = m0 >> 8;
        const bool fin = ev == SE_FRAME || ev == SE_FAULT;
        const bool tg = fin || ev == SE_COLL;
        if (n || tg) flush_lane(tw, pw, lw + (buf ? kWOffL1 : kWOffL0), 1u, n, tg, T, p.ystart, gray, p.tia_delays);
        if (ev == SE_FRAME) {
          end_frame_tia(tw, T / 228u);
          if (render) pw_end(pw, 1u);
          if (f >= nframes) done = true;
          else begin_frame();
        } else if (ev == SE_FAULT) {
          pw_stop(pw, 1u);
          done = true;
        }
      }
      __syncwarp();
      if (lane == 0u) mbar_arrive1(bar0 + 16u + 8u * buf);  // EMPTY[buf]
      buf ^= 1u;
    }
  }
  pair_sync(pair);  // both loops are over: M, RAM (producer) and the TIA words (consumer) are final
  uint32_t* info = pw_base + 32u * kWLaneWords - 128u;  // 32 x (env, fault | done << 1, entry, -)
  if (producer) {
    uint32_t fault = 0, done = 0, ep_ret_done = 0, ent_done = 0;
    if (active) {
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
#pragma unroll
        for (int k = 0; k < 4; ++k) st[k * N + i] = o.c[k];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          st[(4 + k) * N + i] = make_uint4(ramw[4 * k], ramw[4 * k + 1], ramw[4 * k + 2], ramw[4 * k + 3]);
        st[12 * N + i] = make_uint4(episode_frames, episode_index, (uint32_t)episode_return, prev_score);
      } else {
        ep_ret_done = (uint32_t)episode_return;
        const uint64_t g = (uint64_t)(p.env_base + (int64_t)i);
        const uint32_t e = episode_index + 1u;
        const uint32_t ent = rom_id * p.K + (uint32_t)(hash2(hash2(p.pick_seed, g), e) % p.K);
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
    __syncwarp();
    info[4u * lane] = active ? i : 0xFFFFFFFFu;
    info[4u * lane + 1u] = fault | (done << 1);
    info[4u * lane + 2u] = ent_done;
  }
  pair_sync(pair);
  // a5: observation epilogue, the producer warp for lanes 0-15, the consumer warp for 16-31,
  // each with its own ring in the pair's (now free) lane areas
  const uint32_t ring_s = smem_addr(pw_base) + (producer ? 0u : kA84Bytes);
  const uint32_t cols_s = smem_addr(smem + kSmCols);
  for (uint32_t l = producer ? 0u : 16u; l < (producer ? 16u : 32u); ++l) {
    const uint32_t env = info[4u * l];
    if (env == 0xFFFFFFFFu) continue;
    const uint32_t fl = info[4u * l + 1u], en = info[4u * l + 2u];
    const uint32_t f = fl & 1u, dn = fl >> 1;
    if (kGray && p.stacked && dn) {
      stack_fill(p, env, en, lane);
    } else if (kGray) {
      uint8_t* o = p.obs + (size_t)env * p.obs_stride;
      if (f) warp_zero(o, kObs84, lane);
      else {
        const uint8_t* pr = p.staging + (size_t)env * (2 * kFrameBytes);
        warp_area84_staged(pr + kFrameBytes, p.fs >= 2 ? pr : nullptr, o, lane, ring_s, cols_s);
      }
    } else if (f) {
      warp_zero(p.obs + (size_t)env * kFrameBytes, kFrameBytes, lane);
    }
  }
}

#endif  // CULE_VJIT

}  // namespace cule
