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
// Shared memory per lane, 115 words (odd, so the same field of the 32 lanes falls in 32
// different banks): TIA words 9 | pixel writer 9 | SMach 32 | RAM 32 | TIA log 32 + 1.
#pragma once

namespace cule {

#ifndef CULE_VWARPS
#define CULE_VWARPS 16  // most warps per block (launch bound); the host picks the block size
#endif
constexpr uint32_t kVLogCap = 32;
constexpr uint32_t kVOffTw = 0, kVOffPw = 9, kVOffM = 18, kVOffRam = 50, kVOffLog = 82;
constexpr uint32_t kVLaneWords = kVOffLog + kVLogCap + 1;
static_assert(kVLaneWords % 2 == 1, "odd lane stride: conflict-free shared-memory fields");
static_assert(sizeof(SMach) == 4 * (kVOffRam - kVOffM), "SMach slot");

// [mbarrier][area84 column weights][gray LUT][scalar decode table][ROM images][lanes]
__host__ __device__ __forceinline__ size_t vjit_lane_off(uint32_t rom_bytes) { return scalar_rec_off(rom_bytes); }
__host__ __device__ __forceinline__ size_t vjit_smem_bytes(uint32_t rom_bytes, uint32_t threads) {
  return vjit_lane_off(rom_bytes) + (size_t)threads * kVLaneWords * 4u;
}

#ifdef CULE_VJIT  // the device code lives in the generated module (it calls run_cpu_vjit)
// GRAY84 observation of one env from its staged gray frames fs (fa) and fs-1 (fb; null for
// fs = 1), by the whole warp: rows in groups of five (group g closes output rows 2g and 2g+1),
// 16-byte loads of both frames (the next group's loads in flight while this one is reduced),
// byte max into an 800-byte shared buffer, then the exact area weights — packed per column
// (area84_col) and 2:2:1 / 1:2:2 over rows, total 200, round half to even (R#16, R#17; the
// same arithmetic as kernels.cuh warp_area84, which reads single bytes from HBM).
__device__ __forceinline__ void warp_area84_staged(const uint8_t* fa, const uint8_t* fb, uint8_t* out, uint32_t lane,
                                                   uint32_t buf_s, uint32_t cols_s) {
  const uint4* A = reinterpret_cast<const uint4*>(fa);
  const uint4* B = reinterpret_cast<const uint4*>(fb);
  constexpr uint32_t kG = 50u;  // 16-byte chunks per five rows
  uint4 a0, b0, a1 = make_uint4(0, 0, 0, 0), b1 = a1;
  auto load = [&](uint32_t g) {
    const uint32_t q = g * kG + lane;
    a0 = A[q];
    b0 = fb ? B[q] : a0;
    if (lane < kG - 32u) {
      a1 = A[q + 32u];
      b1 = fb ? B[q + 32u] : a1;
    }
  };
  auto vmax = [](uint4 x, uint4 y) {
    return make_uint4(__vmaxu4(x.x, y.x), __vmaxu4(x.y, y.y), __vmaxu4(x.z, y.z), __vmaxu4(x.w, y.w));
  };
  load(0);
  for (uint32_t g = 0; g < 42u; ++g) {
    const uint4 m0 = vmax(a0, b0), m1 = vmax(a1, b1);
    __syncwarp();  // the previous group's reads of the buffer are done
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(buf_s + 16u * lane), "r"(m0.x), "r"(m0.y),
                 "r"(m0.z), "r"(m0.w) : "memory");
    if (lane < kG - 32u)
      asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(buf_s + 16u * (lane + 32u)), "r"(m1.x),
                   "r"(m1.y), "r"(m1.z), "r"(m1.w) : "memory");
    if (g + 1u < 42u) load(g + 1u);
    __syncwarp();
    for (uint32_t o = lane; o < 168u; o += 32u) {
      const uint32_t odd = o >= 84u ? 1u : 0u, j = o - 84u * odd;
      uint32_t cw;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cw) : "r"(cols_s + 4u * j) : "memory");
      const uint32_t c0 = cw & 0xFFu, wc0 = (cw >> 8) & 0xFFu, wc1 = (cw >> 16) & 0xFFu, wc2 = cw >> 24;
      const uint32_t c2 = wc2 ? c0 + 2u : c0;
      const uint32_t q0 = buf_s + (odd ? 320u : 0u) + c0;
      const uint32_t s0 = wc0 * lds_u8(q0) + wc1 * lds_u8(q0 + 1u) + wc2 * lds_u8(q0 + (c2 - c0));
      const uint32_t s1 = wc0 * lds_u8(q0 + 160u) + wc1 * lds_u8(q0 + 161u) + wc2 * lds_u8(q0 + 160u + (c2 - c0));
      const uint32_t s2 = wc0 * lds_u8(q0 + 320u) + wc1 * lds_u8(q0 + 321u) + wc2 * lds_u8(q0 + 320u + (c2 - c0));
      const uint32_t S = (odd ? 1u : 2u) * s0 + 2u * s1 + (odd ? 2u : 1u) * s2;
      uint32_t q = S / 200u;
      const uint32_t r = S - 200u * q;
      q += (r > 100u || (r == 100u && (q & 1u))) ? 1u : 0u;
      out[(2u * g + odd) * 84u + j] = (uint8_t)q;
    }
  }
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
      if (n || tgt) flush_lane(tw, pw, lg, 1u, n, tgt, target, p.ystart, gray);
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
        if (q == 3) v.w = (v.w & 0x000000FFu) | (rom_id << 8);
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
  // free now (state stored) and serve as the 800-byte reduction buffer
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

#endif  // CULE_VJIT

}  // namespace cule
