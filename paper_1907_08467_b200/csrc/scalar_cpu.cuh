// scalar_cpu.cuh — the 6502/6507 + RIOT + bus interpreter of the scalar engine (one env per
// warp, run by lane 0).
//
// Same written machine model as cpu.cuh (R#1 fetch/JAM, R#4 bus phases, R#5
// WSYNC, R#6 VSYNC frame end, R#24 RIOT timer), written for a single thread: an instruction
// costs only its own work.  The loop body is kept small so that the hot loop of every warp on
// an SM fits the instruction cache:
//   fetch (3 shared-memory bytes) -> decode word (scalar_decode.h) -> branch-free effective
//   address (pointer modes branch) -> data read (RAM/ROM: one load; I/O: out-of-line path) ->
//   one jump-table case per operation kind -> data write (RAM: one store; TIA: log append).
//
// The machine's registers live in registers only inside run_cpu(); between calls they sit in
// the warp's shared-memory SMach record, so the warp-cooperative TIA replay that runs between
// two calls does not have to keep them live (register budget: 28 warps per SM).
//
// A collision-latch read needs the TIA replayed up to the read's colour clock, which only the
// whole warp can do.  Such a read aborts the instruction before it commits anything (PC, SP and
// the bank are restored, nothing was written), run_cpu() returns SE_COLL with the clock to
// replay to, and the instruction re-executes after the replay with the latches in SMach.
#pragma once
#include <stdint.h>

#include "scalar_decode.h"
#include "scalar_predecode.h"

namespace cule {

enum SEvent : uint32_t { SE_NONE = 0, SE_LOGFULL = 1, SE_FRAME = 2, SE_FAULT = 3, SE_COLL = 4, SE_BUDGET = 5 };

// per-warp machine record in shared memory (lane 0 reads and writes it)
struct SMach {
  // registers (copied into registers by run_cpu)
  uint32_t PC, A, X, Y, SP, C, V, D, I, nreg, zreg, fc, bank, log_len, t_phaseA;
  // rarely used state (accessed in place)
  uint32_t tV, tS, swcha, inpt4, vsync, fault;
  int32_t tW;
  uint32_t rom0;      // shared-memory offset of this env's ROM image
  uint32_t cart;      // bank switching: first hotspot window offset | banks << 16 (kernels.cuh hs_lo_of)
  uint32_t coll;      // collision latches at colour clock tia_done
  uint32_t tia_done;  // the TIA has been replayed to this colour clock
  uint32_t pa_T, pa_coll;  // latches kept for a phase-A read at pa_T (see run_cpu)
  uint32_t abort_T, abort_pa;
  uint32_t idle_skip;  // exact idle-loop skip enabled (cule_config.idle_skip)
  uint32_t shd;        // shared address of the TIA write shadow (R#37), 0 = no write elision
};
static_assert(sizeof(SMach) == 32 * 4, "SMach is 32 words");

// TIA write registers with an effect on the picture (VSYNC and WSYNC are handled by the CPU;
// RSYNC, audio and the unused range never reach the log): 0x01, 0x04-0x14, 0x1B-0x2C
constexpr uint64_t kTiaEffect = (1ull << 0x01) | (((1ull << 0x15) - 1) & ~((1ull << 0x04) - 1)) |
                                (((1ull << 0x2D) - 1) & ~((1ull << 0x1B) - 1));

// ---- TIA write elision (DESIGN.md §2 R#37) ---------------------------------------------------
// A logged write whose register already holds the written value leaves the TIA state exactly as
// it was, so the replay would only split a span of constant registers in two.  The producer keeps
// a shadow of what the log has written this step and drops such writes.  Shadow entry shd_idx(r)
// (u16; scalar_predecode.h) is the last raw byte logged for register r, or a token 0x100 + k
// (unknown: unequal to every byte and to every other entry); entries kShdG0o / kShdG1o / kShdEbo
// shadow the VDEL copies GRP0 old, GRP1 old and ENABL old.  Registers whose write is a pure store
// of the value (kTiaPure): NUSIZ0 ... PF2 (0x04-0x0F) and ENAM0 ... RESMP1 (0x1D-0x29; a RESMP
// write acts only on a change of D1).  GRP0 / GRP1 also copy the other player's (and the ball's)
// new value into its old one, so they are dropped only when both are unchanged; HMCLR zeroes the
// five motion registers; the strobes (RESxx, HMOVE, CXCLR) and VBLANK always reach the log.
__device__ __forceinline__ uint32_t ld_shd(uint32_t shd, uint32_t k) {
  uint32_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(shd + 2u * k) : "memory");
  return v;
}
__device__ __forceinline__ void st_shd(uint32_t shd, uint32_t k, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(shd + 2u * k), "r"(v) : "memory");
}
// every entry unknown: by the whole warp (one entry per lane) ...
__device__ __forceinline__ void shd_init_warp(uint32_t shd, uint32_t lane) { st_shd(shd, lane, 0x100u + lane); }
// ... or by one lane (its own shadow; 4-byte aligned)
__device__ __forceinline__ void shd_init_lane(uint32_t shd) {
#pragma unroll 1
  for (uint32_t k = 0; k < kShdEntries; k += 2u)
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(shd + 2u * k), "r"((0x100u + k) | ((0x101u + k) << 16)) : "memory");
}
// the shadow after a write of byte v to TIA effect register r; false when the write changes
// nothing (drop it), true when it must reach the log
__device__ __forceinline__ bool shd_write(uint32_t shd, uint32_t r, uint32_t v) {
  if ((kTiaPure >> r) & 1ull) {
    if (ld_shd(shd, shd_idx(r)) == v) return false;
    st_shd(shd, shd_idx(r), v);
    return true;
  }
  constexpr uint32_t G0 = shd_idx(0x1Bu), G1 = shd_idx(0x1Cu), EB = shd_idx(0x1Fu);
  if (r == 0x1Bu) {  // GRP0; GRP1 old <- GRP1 new
    const uint32_t g1n = ld_shd(shd, G1);
    if (ld_shd(shd, G0) == v && ld_shd(shd, kShdG1o) == g1n) return false;
    st_shd(shd, G0, v);
    st_shd(shd, kShdG1o, g1n);
    return true;
  }
  if (r == 0x1Cu) {  // GRP1; GRP0 old <- GRP0 new; ENABL old <- ENABL new
    const uint32_t g0n = ld_shd(shd, G0), ebn = ld_shd(shd, EB);
    if (ld_shd(shd, G1) == v && ld_shd(shd, kShdG0o) == g0n && ld_shd(shd, kShdEbo) == ebn) return false;
    st_shd(shd, G1, v);
    st_shd(shd, kShdG0o, g0n);
    st_shd(shd, kShdEbo, ebn);
    return true;
  }
  if (r == 0x2Bu) {  // HMCLR: HMP0 ... HMBL read as written with 0
#pragma unroll 1
    for (uint32_t k = shd_idx(0x20u); k <= shd_idx(0x24u); ++k) st_shd(shd, k, 0u);
  }
  return true;
}

// (out of line: the per-lane engine's translated code calls it from many sites)
__device__ __noinline__ bool shd_write_ool(uint32_t shd, uint32_t r, uint32_t v) { return shd_write(shd, r, v); }

__device__ __forceinline__ uint32_t s_coll_bits(uint32_t coll, uint32_t r) {
  return (((coll >> (2 * r)) & 1u) << 7) | (((coll >> (2 * r + 1)) & 1u) << 6);
}

// I/O read (TIA read registers, RIOT), out of the hot path; T = colour clock of the access
__device__ __noinline__ uint32_t s_rd_io(SMach* M, uint32_t a, uint32_t T, uint32_t now, uint32_t pa) {
  if (!(a & 0x80u)) {
    const uint32_t r = a & 0x0Fu;
    if (r < 8u) {
      // a phase-A read keeps its latches in pa_*: if a later read of the same instruction
      // aborts and the TIA moves on, the re-execution must see the same phase-A values
      if (pa && M->pa_T == T) return s_coll_bits(M->pa_coll, r);
      if (M->tia_done == T) {
        if (pa) { M->pa_T = T; M->pa_coll = M->coll; }
        return s_coll_bits(M->coll, r);
      }
      M->abort_T = T;  // abort: replay to T, then re-execute
      M->abort_pa = pa;
      return 0x100u;
    }
    return r == 0x0Cu ? M->inpt4 : (r == 0x0Du ? 0x80u : 0u);
  }
  if (!(a & 0x04u)) {
    const uint32_t k = a & 3u;
    return k == 0 ? M->swcha : (k == 2 ? 0x0Bu : 0u);
  }
  const int32_t e = (int32_t)now - M->tW;  // RIOT timer, closed form (R#24)
  const uint32_t tV = M->tV, tS = M->tS;
  const int32_t VI = (int32_t)(tV << tS);
  if (a & 1u) return e > VI ? 0x80u : 0u;
  if (e <= VI) return (tV - (uint32_t)((e + (1 << tS) - 1) >> tS)) & 0xFFu;
  return (uint32_t)(0xFF - (e - VI - 1)) & 0xFFu;
}

// shared-memory accesses by 32-bit shared address (no generic-pointer conversions in the loop);
// RAM accesses are volatile so they keep program order, ROM / decode loads may be scheduled freely
__device__ __forceinline__ uint32_t ld_ro8(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t ld_ro32(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t ld_ram(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_ram(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

__device__ __forceinline__ void st_log(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// VSYNC and RIOT writes (rare, out of line); returns 2 when VSYNC rose (R#6)
__device__ __noinline__ uint32_t s_wr_slow(SMach* M, uint32_t a, uint32_t v, uint32_t now) {
  if (!(a & 0x80u)) {  // TIA VSYNC
    const uint32_t nv = (v >> 1) & 1u;
    const uint32_t rose = (!M->vsync && nv) ? 2u : 0u;
    M->vsync = nv;
    return rose;
  }
  if ((a & 0x14u) == 0x14u) {  // timer write: interval 1 / 8 / 64 / 1024
    M->tV = v & 0xFFu;
    M->tS = (0xA630u >> (4 * (a & 3u))) & 0xFu;
    M->tW = (int32_t)now;
  }
  return 0u;
}

// Fetch through the bus (PC outside the fast window): fetches have side effects (bank switches,
// TIA reads at phase A).  Returns op | b1 << 8 | b2 << 16, bit 24 = abort, bits 25.. = new bank.
__device__ __noinline__ uint32_t s_fetch_slow(SMach* M, uint32_t rom0, uint32_t ram0, uint32_t dtab0, uint32_t pc0,
                                              uint32_t bank, uint32_t tpa, uint32_t now) {
  uint32_t out = 0u, bad = 0u;
  uint32_t nbytes = 1u;
  for (uint32_t k = 0; k < nbytes; ++k) {
    const uint32_t a = (pc0 + k) & 0x1FFFu;
    uint32_t v;
    if (a & 0x1000u) {
      if (((a & 0xFFFu) - (M->cart & 0xFFFFu)) < (M->cart >> 16)) bank = (a & 0xFFFu) - (M->cart & 0xFFFFu);
      v = ld_ro8(rom0 + (bank << 12) + (a & 0xFFFu));
    } else if ((a & 0x0280u) == 0x0080u) {
      v = ld_ram(ram0 + (a & 0x7Fu));
    } else {
      v = s_rd_io(M, a, tpa, now, 1u);
      bad |= v;
      v &= 0xFFu;
    }
    out |= v << (8 * k);
    if (k == 0) nbytes = (ld_ro32(dtab0 + 8u * v) >> sk::LEN) & 3u;
  }
  return out | ((bad & 0x100u) ? (1u << 24) : 0u) | (bank << 25);
}

constexpr uint32_t kGenCommitted = 0x100u;

// One instruction through the general interpreter (the full machine model), on the machine
// record in shared memory: registers and clocks in M, M->t_phaseA = 3 x the cycle at which the
// instruction's phase A samples.  Out of line, so the fast loop of run_cpu() keeps its
// registers to itself.  Returns the event (SEvent), | kGenCommitted if the instruction completed
// (a collision-latch read that must wait for the TIA commits nothing; JAM faults uncommitted).
// The idle-loop skip is not applied here (skipping is optional and exact either way).
__device__ __noinline__ uint32_t s_gen_one(SMach* M, uint32_t rom_all0, uint32_t dtab0, uint32_t ram0, uint32_t lg0,
                                           uint32_t log_lim, uint32_t cap_cycles) {
  uint32_t PC = M->PC, A = M->A, X = M->X, Y = M->Y, SP = M->SP;
  uint32_t C = M->C, V = M->V, D = M->D, I = M->I, nreg = M->nreg, zreg = M->zreg;
  uint32_t fc = M->fc, bank = M->bank, log_len = M->log_len;
  const uint32_t pend = M->t_phaseA / 3u;  // end cycle of the previous instruction
  uint32_t pnext = pend;
  const uint32_t rom0 = rom_all0 + M->rom0;
  const uint32_t hs_lo = M->cart & 0xFFFFu, nbank = M->cart >> 16;
  const uint32_t flim = nbank > 1u ? hs_lo - 3u : 0xFFDu;  // fast fetch: pc..pc+2 inside the page, no hotspot
  const uint32_t hlim = nbank > 1u ? hs_lo - 1u : 0xFFFu;  // fast data read: no hotspot
  uint32_t ev = SE_NONE, committed = 0u;
  auto nz = [&](uint32_t x) { nreg = x; zreg = x; };
  auto adc = [&](uint32_t m) {
    if (!D) {
      const uint32_t t = A + m + C;
      V = ((~(A ^ m) & (A ^ t)) >> 7) & 1u;
      C = t >> 8;
      A = t & 0xFFu;
      nz(A);
    } else {  // NMOS decimal (R#2)
      uint32_t lo = (A & 0xFu) + (m & 0xFu) + C;
      if (lo >= 0xAu) lo = ((lo + 6u) & 0xFu) + 0x10u;
      uint32_t s = (A & 0xF0u) + (m & 0xF0u) + lo;
      const int32_t sv = (int32_t)(int8_t)(A & 0xF0u) + (int32_t)(int8_t)(m & 0xF0u) + (int32_t)lo;
      zreg = (A + m + C) & 0xFFu;
      nreg = s;
      V = (sv < -128 || sv > 127) ? 1u : 0u;
      if (s >= 0xA0u) s += 0x60u;
      C = s >= 0x100u ? 1u : 0u;
      A = s & 0xFFu;
    }
  };
  auto sbc = [&](uint32_t m) {
    const uint32_t t = A + (m ^ 0xFFu) + C;
    const uint32_t r = t & 0xFFu;
    V = ((~(A ^ (m ^ 0xFFu)) & (A ^ t)) >> 7) & 1u;
    if (D) {  // NMOS decimal: binary flags, BCD result (R#2)
      int32_t lo = (int32_t)(A & 0xFu) - (int32_t)(m & 0xFu) + (int32_t)C - 1;
      if (lo < 0) lo = ((lo - 6) & 0xF) - 0x10;
      int32_t s = (int32_t)(A & 0xF0u) - (int32_t)(m & 0xF0u) + lo;
      if (s < 0) s -= 0x60;
      A = (uint32_t)s & 0xFFu;
    } else {
      A = r;
    }
    C = t >> 8;
    nz(r);
  };
  auto cmp = [&](uint32_t r, uint32_t m) { C = r >= m ? 1u : 0u; nz((r - m) & 0xFFu); };
  auto getP = [&]() {
    return (nreg & 0x80u) | (V << 6) | 0x30u | (D << 3) | (I << 2) | ((zreg & 0xFFu) == 0u ? 2u : 0u) | C;
  };
  // branch condition of K_BR / C_BR: flag (0 N 1 V 2 C 3 Z) == taken-when bit
  auto br_taken = [&](uint32_t aux) {
    const uint32_t f = aux & 3u;
    const uint32_t fl = f == 0u ? (nreg >> 7) & 1u : (f == 1u ? V : (f == 2u ? C : ((zreg & 0xFFu) == 0u ? 1u : 0u)));
    return fl == ((aux >> 2) & 1u);
  };
  const uint32_t pc0 = PC;
  {
    const uint32_t bank0 = bank;
    uint32_t now = fc;
    uint32_t bad = 0u;  // bit 8 set: a collision read must wait for the TIA (abort)
    // full bus read (phase A: T = 3 pend; phase C: T = 3 now)
    auto rd = [&](uint32_t addr, uint32_t T, uint32_t pa) -> uint32_t {
      const uint32_t a = addr & 0x1FFFu;
      if (a & 0x1000u) {
        if (((a & 0xFFFu) - hs_lo) < nbank) bank = (a & 0xFFFu) - hs_lo;
        return ld_ro8(rom0 + (bank << 12) + (a & 0xFFFu));
      }
      if ((a & 0x0280u) == 0x0080u) return ld_ram(ram0 + (a & 0x7Fu));
      const uint32_t r = s_rd_io(M, a, T, now, pa);
      bad |= r;
      return r & 0xFFu;
    };
    uint32_t op, b1, b2;
    if ((pc0 & 0x1000u) && (pc0 & 0xFFFu) <= flim) {
      const uint32_t p = rom0 + (bank << 12) + (pc0 & 0xFFFu);
      op = ld_ro8(p); b1 = ld_ro8(p + 1u); b2 = ld_ro8(p + 2u);
    } else {
      const uint32_t f = s_fetch_slow(M, rom0, ram0, dtab0, pc0, bank, 3u * pend, now);
      bank = f >> 25;
      if (f & (1u << 24)) goto coll;
      op = f & 0xFFu; b1 = (f >> 8) & 0xFFu; b2 = (f >> 16) & 0xFFu;
    }
    {
      uint32_t d, e;  // decode entry (scalar_decode.h): d = mode/flags word, e = kind/aux word
      asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(d), "=r"(e) : "r"(dtab0 + 8u * op));
      const uint32_t kind = e & 0xFFu, aux = e >> sk::AUX;
      uint32_t n = (d >> sk::CYC) & 0xFu;
      uint32_t nPC = pc0 + ((d >> sk::LEN) & 3u);
      // ---- phase A: effective address ------------------------------------------------------
      const uint32_t ix = __byte_perm(X | (Y << 8), 0u, d);  // X, Y or 0
      uint32_t base = b1 | (b2 << 8), ea;
      if (!(d & (sk::PTRZ | sk::PTRA))) {
        ea = (base + ix) & ((d & sk::ZP) ? 0xFFu : 0xFFFFu);
      } else {  // (zp,X): index before the pointer; (zp),Y: after; JMP (abs): page-wrap bug
        const bool pa = (d & sk::PTRA) != 0u, pre = (d & sk::ZP) != 0u;
        const uint32_t z = (b1 + (pre ? ix : 0u)) & 0xFFu;
        const uint32_t p0 = pa ? base : z;
        const uint32_t p1 = pa ? ((base & 0xFF00u) | ((base + 1u) & 0xFFu)) : ((z + 1u) & 0xFFu);
        const uint32_t lo = rd(p0, 3u * pend, 1u);
        const uint32_t hi = rd(p1, 3u * pend, 1u);
        if (bad & 0x100u) goto coll;
        base = lo | (hi << 8);
        ea = (base + (pre ? 0u : ix)) & 0xFFFFu;
      }
      n += ((d & sk::PEN) && ((ea ^ base) & 0x100u)) ? 1u : 0u;
      now = fc + n;
      // ---- phase C: data read ------------------------------------------------------------
      uint32_t v = (d & sk::ACC) ? A : b1;
      uint32_t ff = 0u;  // timer reads: cycles over which the value read stays the same
      if (d & sk::RD) {
        const uint32_t a = ea & 0x1FFFu;
        const bool cart = (a & 0x1000u) != 0u;
        if (cart ? (a & 0xFFFu) <= hlim : (a & 0x0280u) == 0x0080u) {
          v = cart ? ld_ro8(rom0 + (bank << 12) + (a & 0xFFFu)) : ld_ram(ram0 + (a & 0x7Fu));
        } else if ((a & 0x1284u) == 0x0284u) {  // RIOT timer, closed form (R#24)
          const int32_t et = (int32_t)now - M->tW;
          const uint32_t tV = M->tV, tS = M->tS;
          const int32_t VI = (int32_t)(tV << tS);
          if (a & 1u) {  // TIMINT: 0 up to the expiry, 0x80 after it
            v = et > VI ? 0x80u : 0u;
            ff = et > VI ? 0x7FFFFFFFu : (uint32_t)(VI - et);
          } else if (et <= VI) {  // INTIM while counting: constant up to the next interval edge
            const int32_t q = (et + (1 << tS) - 1) >> tS;
            v = (tV - (uint32_t)q) & 0xFFu;
            ff = (uint32_t)((q << tS) - et);
          } else {  // INTIM after the expiry: counts down every cycle
            v = (uint32_t)(0xFF - (et - VI - 1)) & 0xFFu;
          }
        } else {
          v = rd(a, 3u * now, 0u);
          if (bad & 0x100u) goto coll;
        }
      }
      uint32_t wv = 0u, xf = 0u;  // xf: exit flags (2 VSYNC rose); fw: cycle after a WSYNC stall
      uint32_t fw = 0xFFFFFFFFu;
      auto wr = [&](uint32_t addr, uint32_t val) {
        const uint32_t a = addr & 0x1FFFu;
        if ((a & 0x1280u) == 0x0080u) {
          st_ram(ram0 + (a & 0x7Fu), val & 0xFFu);
        } else if (!(a & 0x1080u)) {  // TIA: effect registers go to the log (R#4)
          const uint32_t r = a & 0x3Fu;
          // R#37: the shadow follows every logged write; the one-env-per-warp engine drops a
          // write that changes nothing, the per-lane engines log it (their lanes' logs stay
          // aligned; the translated code drops by warp vote, jit.h emit_simt)
#ifdef CULE_VJIT
          if ((kTiaEffect >> r) & 1ull) {
            if (M->shd) (void)shd_write(M->shd, r, val & 0xFFu);
#else
          if (((kTiaEffect >> r) & 1ull) && (!M->shd || shd_write(M->shd, r, val & 0xFFu))) {
#endif
            st_log(lg0 + 4u * log_len, ((3u * now) << 14) | (r << 8) | (val & 0xFFu));
            ++log_len;
          } else if (r == 0x02u) {
            fw = ((now + 75u) / 76u) * 76u;  // WSYNC: stall to the next line start (R#5)
          } else if (r == 0x00u) {
            xf |= s_wr_slow(M, a, val, now);
          }
        } else if (a & 0x1000u) {
          if (((a & 0xFFFu) - hs_lo) < nbank) bank = (a & 0xFFFu) - hs_lo;
        } else {
          s_wr_slow(M, a, val, now);  // RIOT
        }
      };
      // ---- operation ---------------------------------------------------------------------
      switch (kind) {
        case K_NOP: break;
        case K_ORA: A |= v; nz(A); break;
        case K_AND: A &= v; nz(A); break;
        case K_EOR: A ^= v; nz(A); break;
        case K_ADC: adc(v); break;
        case K_SBC: sbc(v); break;
        case K_CMP: cmp(aux == 0u ? A : (aux == 1u ? X : Y), v); break;
        case K_BIT: nreg = v; zreg = A & v; V = (v >> 6) & 1u; break;
        case K_LD:
          A = (aux & 1u) ? v : A;
          X = (aux & 2u) ? v : X;
          Y = (aux & 4u) ? v : Y;
          nz(v);
          break;
        case K_ST: wv = aux == 0u ? A : (aux == 1u ? X : (aux == 2u ? Y : (A & X))); break;
        case K_ASL: C = v >> 7; wv = (v << 1) & 0xFFu; nz(wv); break;
        case K_LSR: C = v & 1u; wv = v >> 1; nz(wv); break;
        case K_ROL: wv = ((v << 1) | C) & 0xFFu; C = v >> 7; nz(wv); break;
        case K_ROR: wv = (v >> 1) | (C << 7); C = v & 1u; nz(wv); break;
        case K_ASLA: C = A >> 7; A = (A << 1) & 0xFFu; nz(A); break;
        case K_LSRA: C = A & 1u; A >>= 1; nz(A); break;
        case K_ROLA: { const uint32_t c = C; C = A >> 7; A = ((A << 1) | c) & 0xFFu; nz(A); } break;
        case K_RORA: { const uint32_t c = C; C = A & 1u; A = (A >> 1) | (c << 7); nz(A); } break;
        case K_INC: wv = (v + 1u) & 0xFFu; nz(wv); break;
        case K_DEC: wv = (v - 1u) & 0xFFu; nz(wv); break;
        case K_SLO: C = v >> 7; wv = (v << 1) & 0xFFu; A |= wv; nz(A); break;
        case K_RLA: wv = ((v << 1) | C) & 0xFFu; C = v >> 7; A &= wv; nz(A); break;
        case K_SRE: C = v & 1u; wv = v >> 1; A ^= wv; nz(A); break;
        case K_RRA: wv = (v >> 1) | (C << 7); C = v & 1u; adc(wv); break;
        case K_DCP: wv = (v - 1u) & 0xFFu; cmp(A, wv); break;
        case K_ISB: wv = (v + 1u) & 0xFFu; sbc(wv); break;
        case K_INR: {
          const uint32_t r = (((aux & 1u) ? Y : X) + ((aux & 2u) ? 0xFFu : 1u)) & 0xFFu;
          X = (aux & 1u) ? X : r;
          Y = (aux & 1u) ? r : Y;
          nz(r);
        } break;
        case K_TR: {
          const uint32_t s = aux & 3u, t = (aux >> 2) & 3u;
          const uint32_t r = s == 0u ? A : (s == 1u ? X : (s == 2u ? Y : SP));
          A = t == 0u ? r : A;
          X = t == 1u ? r : X;
          Y = t == 2u ? r : Y;
          SP = t == 3u ? r : SP;
          if (aux & 16u) nz(r);
        } break;
        case K_FLAG: {
          const uint32_t f = aux & 3u, b = (aux >> 2) & 1u;
          C = f == 0u ? b : C;
          I = f == 1u ? b : I;
          D = f == 2u ? b : D;
          V = f == 3u ? b : V;
        } break;
        case K_BR: {
          if (br_taken(aux)) {
            const uint32_t from = nPC & 0xFFFFu;
            const uint32_t tgt = (from + (uint32_t)(int32_t)(int8_t)b1) & 0xFFFFu;
            now += 1u + (((tgt ^ from) >> 8) & 1u);
            nPC = tgt;
          }
        } break;
        case K_JMP: nPC = ea; break;
        case K_JSR: {
          const uint32_t ret = (pc0 + 2u) & 0xFFFFu;
          wr(0x100u | SP, ret >> 8); SP = (SP - 1u) & 0xFFu;
          wr(0x100u | SP, ret & 0xFFu); SP = (SP - 1u) & 0xFFu;
          nPC = ea;
        } break;
        case K_RTS: {
          const uint32_t s1 = (SP + 1u) & 0xFFu, s2 = (SP + 2u) & 0xFFu;
          const uint32_t lo = rd(0x100u | s1, 3u * now, 0u);
          const uint32_t hi = rd(0x100u | s2, 3u * now, 0u);
          if (bad & 0x100u) goto coll;
          SP = s2;
          nPC = (lo | (hi << 8)) + 1u;
        } break;
        case K_RTI: {
          const uint32_t s1 = (SP + 1u) & 0xFFu, s2 = (SP + 2u) & 0xFFu, s3 = (SP + 3u) & 0xFFu;
          const uint32_t p = rd(0x100u | s1, 3u * now, 0u);
          const uint32_t lo = rd(0x100u | s2, 3u * now, 0u);
          const uint32_t hi = rd(0x100u | s3, 3u * now, 0u);
          if (bad & 0x100u) goto coll;
          SP = s3;
          nreg = p & 0x80u; V = (p >> 6) & 1u; D = (p >> 3) & 1u; I = (p >> 2) & 1u;
          zreg = (p & 2u) ? 0u : 1u; C = p & 1u;
          nPC = lo | (hi << 8);
        } break;
        case K_BRK: {
          const uint32_t ret = (pc0 + 2u) & 0xFFFFu;
          wr(0x100u | SP, ret >> 8); SP = (SP - 1u) & 0xFFu;
          wr(0x100u | SP, ret & 0xFFu); SP = (SP - 1u) & 0xFFu;
          wr(0x100u | SP, getP()); SP = (SP - 1u) & 0xFFu;
          I = 1u;
          const uint32_t lo = rd(0x1FFEu, 3u * now, 0u);
          const uint32_t hi = rd(0x1FFFu, 3u * now, 0u);
          nPC = lo | (hi << 8);
        } break;
        case K_PHA: wr(0x100u | SP, A); SP = (SP - 1u) & 0xFFu; break;
        case K_PHP: wr(0x100u | SP, getP()); SP = (SP - 1u) & 0xFFu; break;
        case K_PLA: {
          const uint32_t s1 = (SP + 1u) & 0xFFu;
          const uint32_t x = rd(0x100u | s1, 3u * now, 0u);
          if (bad & 0x100u) goto coll;
          SP = s1; A = x; nz(A);
        } break;
        case K_PLP: {
          const uint32_t s1 = (SP + 1u) & 0xFFu;
          const uint32_t p = rd(0x100u | s1, 3u * now, 0u);
          if (bad & 0x100u) goto coll;
          SP = s1;
          nreg = p & 0x80u; V = (p >> 6) & 1u; D = (p >> 3) & 1u; I = (p >> 2) & 1u;
          zreg = (p & 2u) ? 0u : 1u; C = p & 1u;
        } break;
        case K_ANC: A &= v; nz(A); C = A >> 7; break;
        case K_ALR: { const uint32_t t = A & v; C = t & 1u; A = t >> 1; nz(A); } break;
        case K_ARR: {
          const uint32_t t = A & v;
          A = (t >> 1) | (C << 7);
          nz(A);
          C = (A >> 6) & 1u;
          V = ((A >> 6) ^ (A >> 5)) & 1u;
        } break;
        case K_SBX: { const uint32_t t = A & X; C = t >= v ? 1u : 0u; X = (t - v) & 0xFFu; nz(X); } break;
        default:  // K_JAM: the opcode fetch happened, then the env faults, fc unchanged (R#1)
          PC = (pc0 + 1u) & 0xFFFFu;
          M->fault = 1u;
          ev = SE_FAULT;
          goto out;
      }
      if (d & sk::WR) wr(ea, wv);
      (void)ff;
      // ---- end of instruction (R#4, R#5) --------------------------------------------------
      committed = kGenCommitted;
      PC = nPC & 0xFFFFu;
      pnext = now;  // phase A of the next instruction: this one's end, before any WSYNC stall
      fc = fw != 0xFFFFFFFFu ? fw : now;
      if (fc >= cap_cycles || xf != 0u || log_len > log_lim) {
        if (fc >= cap_cycles) { M->fault = 2u; ev = SE_FAULT; }  // runaway: fc / 76 >= line_cap
        else ev = xf ? SE_FRAME : SE_LOGFULL;
      }
    }
    goto out;
  coll:  // a collision-latch read must wait for the TIA: nothing was committed
    bank = bank0;
    ev = SE_COLL;
  }
out:
  M->PC = PC; M->A = A; M->X = X; M->Y = Y; M->SP = SP;
  M->C = C; M->V = V; M->D = D; M->I = I; M->nreg = nreg; M->zreg = zreg;
  M->fc = fc; M->bank = bank; M->log_len = log_len; M->t_phaseA = 3u * pnext;
  return ev | committed;
}

// Run lane 0's machine until an event; `budget` (debug) counts instructions.
//
// Every instruction whose pre-decoded record (scalar_predecode.h) has a fast class runs a short
// specialised case; everything else goes through s_gen_one().  While in the fast loop the PC is
// in a cartridge window and is kept split: pcw = PC & 0xF000, pco = PC & 0xFFF (fast classes
// never leave the window except C_JMP, which sets both; the general path re-enters the fast loop
// only with PC in a cartridge window).  Phase A of an instruction samples at the end of the
// previous one: that is fc, except right after a WSYNC stall, recorded as (ws_fc, ws_now) — fc
// strictly increases within a call, so fc == ws_fc identifies the instruction after the stall.
// kSkip: the exact idle-loop skip is enabled (cule_config.idle_skip); compiled separately so
// the headline path (skip off) carries none of its bookkeeping.
template <bool kDebug, bool kSkip>
__device__ __forceinline__ uint32_t run_cpu(SMach* M, uint32_t rom_all0, uint32_t dtab0, uint32_t ram0, uint32_t lg0,
                                            uint32_t log_lim, uint32_t cap_cycles, int32_t& budget,
                                            uint32_t rec_all0) {
  uint32_t A = M->A, X = M->X, Y = M->Y, SP = M->SP;
  uint32_t C = M->C, V = M->V, D = M->D, I = M->I;
  // N and Z packed in one register: the Z byte in bits 0-7 (Z = it is 0), N at bit 15; an
  // ordinary result x sets nz = x * 257 (one multiply-add, no second register copy)
  uint32_t nz = (M->zreg & 0xFFu) | ((M->nreg & 0x80u) << 8);
  uint32_t fc = M->fc, bank = M->bank, log_len = M->log_len;
  uint32_t pcw = M->PC & 0xF000u, pco = M->PC & 0xFFFu;
  uint32_t ws_fc = fc, ws_now = M->t_phaseA / 3u;  // phase A of the first instruction
  const uint32_t rec0 = rec_all0 + 8u * M->rom0;  // pre-decoded records of this env's ROM
  const uint32_t rom0 = rom_all0 + M->rom0;       // its raw image (data reads)
  uint32_t recb = rec0 + (bank << 15), romb = rom0 + (bank << 12);
  uint32_t ev = SE_NONE;
  // idle-loop skip (exact): the last plain timer read (offset, cycles, cycles its value holds, end)
  uint32_t ppc = 0xFFFFFFFFu, pn = 0u, pff = 0u, pfe = 0xFFFFFFFFu;
  // the RIOT timer's parameters stay in registers (only RIOT writes, in the general path, change them)
  int32_t tW = M->tW;
  uint32_t tVS = M->tV | (M->tS << 8) | (((1u << M->tS) - 1u) << 16);  // V | shift << 8 | (2^shift - 1) << 16
  auto setnz = [&](uint32_t x) { nz = x * 257u; };  // x <= 0xFF
  auto adc = [&](uint32_t m) {
    if (!D) {
      const uint32_t t = A + m + C;
      V = ((~(A ^ m) & (A ^ t)) >> 7) & 1u;
      C = t >> 8;
      A = t & 0xFFu;
      setnz(A);
    } else {  // NMOS decimal (R#2)
      uint32_t lo = (A & 0xFu) + (m & 0xFu) + C;
      if (lo >= 0xAu) lo = ((lo + 6u) & 0xFu) + 0x10u;
      uint32_t s = (A & 0xF0u) + (m & 0xF0u) + lo;
      const int32_t sv = (int32_t)(int8_t)(A & 0xF0u) + (int32_t)(int8_t)(m & 0xF0u) + (int32_t)lo;
      nz = ((A + m + C) & 0xFFu) | ((s & 0x80u) << 8);  // Z from the binary sum, N from s
      V = (sv < -128 || sv > 127) ? 1u : 0u;
      if (s >= 0xA0u) s += 0x60u;
      C = s >= 0x100u ? 1u : 0u;
      A = s & 0xFFu;
    }
  };
  auto sbc = [&](uint32_t m) {
    const uint32_t t = A + (m ^ 0xFFu) + C;
    const uint32_t r = t & 0xFFu;
    V = ((~(A ^ (m ^ 0xFFu)) & (A ^ t)) >> 7) & 1u;
    if (D) {  // NMOS decimal: binary flags, BCD result (R#2)
      int32_t lo = (int32_t)(A & 0xFu) - (int32_t)(m & 0xFu) + (int32_t)C - 1;
      if (lo < 0) lo = ((lo - 6) & 0xF) - 0x10;
      int32_t s = (int32_t)(A & 0xF0u) - (int32_t)(m & 0xF0u) + lo;
      if (s < 0) s -= 0x60;
      A = (uint32_t)s & 0xFFu;
    } else {
      A = r;
    }
    C = t >> 8;
    setnz(r);
  };
  auto cmp = [&](uint32_t r, uint32_t m) { C = r >= m ? 1u : 0u; setnz((r - m) & 0xFFu); };
  auto prmt = [](uint32_t a, uint32_t b, uint32_t sel) {  // raw PRMT: selector bits used as stored
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
  };
  if (kDebug && budget <= 0) { ev = SE_BUDGET; goto out; }
  if (!(pcw & 0x1000u)) goto general;  // entered outside the cartridge (code in RAM)
  for (;;) {
    if (kDebug && budget <= 0) { ev = SE_BUDGET; break; }
    {
      uint32_t lo, hi;
      asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(recb + 8u * pco));
      // back to the instruction's start for the general path: nothing was committed, and
      // pco / fc are recovered from the record, so they need not stay live across the switch
#define CULE_FALLBACK() do { pco = (lo >> pd::NXT) - ((lo >> pd::LENF) & 3u); fc = now - ((lo >> pd::CYC) & 0xFu); goto general; } while (0)
      const uint32_t cls = lo & 31u;
      uint32_t now = fc + ((lo >> pd::CYC) & 0xFu);
      uint32_t npco = lo >> pd::NXT;
      if (cls == C_BR) {  // the most frequent class, tested before the switch
        const uint32_t aux = lo >> pd::AUX;
        const uint32_t src = (aux & 2u) ? ((aux & 1u) ? nz : C) : ((aux & 1u) ? V : nz);
        if (((src & (hi >> 16)) != 0u) == ((aux & 4u) != 0u)) {
          npco = hi & 0xFFFu;
          // idle-loop skip: [timer read; branch back to it] — later iterations whose read falls
          // in the same constant interval repeat this one exactly, so only time advances
          // (stopping short of the runaway cap, which the loop then reaches normally).
          // pfe == fc: the read was the instruction right before this branch.
          if (kSkip && pff != 0u && pfe == fc && npco == ppc && now < cap_cycles) {
            const uint32_t P = pn + (now - fc);
            const uint32_t j = min(pff / P, (cap_cycles - 1u - now) / P);
            now += j * P;
          }
          // a runaway frame can only spin through a taken branch, a jump or the general path:
          // the step kernel checks the cap there (a faulted env's state is replaced by the
          // reset cache, so only the step of the fault matters); the debug entry checks it
          // after every instruction
          if (!kDebug && now >= cap_cycles) { pco = npco; fc = now; M->fault = 2u; ev = SE_FAULT; break; }
        } else {
          now -= ((lo >> pd::CYC) & 0xFu) - 2u;  // not taken: 2 cycles
        }
        goto fast_done;
      }
      {
        const uint32_t aux = (lo >> pd::AUX) & 7u;
        // data operand: RAM[(opnd + ix) & 0x7F] (needs bit 7 of opnd + ix, else the general
        // path: zp,X into the TIA) or the cartridge byte (opnd + ix) & 0xFFF of the bank
        const uint32_t opnd = hi >> pd::OPND;
        auto ea_t = [&]() { return opnd + prmt(X + Y * 256u, 0u, hi); };  // computed per case
        uint32_t v = 0u;
        auto rd_operand = [&]() -> bool {
          const uint32_t t = ea_t();
          if (hi & pd::RAM) {
            if (!(t & 0x80u)) return false;
            v = ld_ram(ram0 + (t & 0x7Fu));
          } else {
            v = ld_ro8(romb + (t & 0xFFFu));
          }
          now += ((t ^ opnd) & hi & pd::PEN) >> 8;
          return true;
        };
        if (cls <= C_HOT_LAST) {
          switch (cls) {
          case C_SBC: if (!rd_operand()) CULE_FALLBACK(); sbc(v); break;
          case C_CMP: if (!rd_operand()) CULE_FALLBACK(); cmp(aux == 0u ? A : (aux == 1u ? X : Y), v); break;
          case C_LD:
            if (!rd_operand()) CULE_FALLBACK();
          ld_v:
            A = (aux & 1u) ? v : A;
            X = (aux & 2u) ? v : X;
            Y = (aux & 4u) ? v : Y;
            setnz(v);
            break;
          case C_TLD: case C_TBIT: {  // RIOT timer, closed form (R#24); an idle-loop head candidate
            const int32_t et = (int32_t)now - tW;
            const uint32_t tV = tVS & 0xFFu, tS = (tVS >> 8) & 0xFFu, tm = tVS >> 16;  // tm = 2^tS - 1
            const int32_t VI = (int32_t)(tV << tS);
            // branch-free: INTIM while counting / after expiry (0xFF - (e - VI - 1) = VI - e mod 256), TIMINT
            const bool expired = et > VI;
            const uint32_t counting = (tV - (uint32_t)((et + (int32_t)tm) >> tS)) & 0xFFu;
            const uint32_t intim = expired ? ((uint32_t)(VI - et) & 0xFFu) : counting;
            v = (hi & 1u) ? (expired ? 0x80u : 0u) : intim;
            if (kSkip) {  // cycles over which the value read stays the same
              uint32_t ff = 0u;
              if (hi & 1u) ff = et > VI ? 0x7FFFFFFFu : (uint32_t)(VI - et);
              else if (et <= VI) ff = (uint32_t)((((et + (int32_t)tm) >> tS) << tS) - et);
              pff = ff;
              ppc = pco;
              pn = now - fc;
              pfe = now;
            }
            if (cls == C_TLD) goto ld_v;
            nz = (A & v) | ((v & 0x80u) << 8);  // C_TBIT
            V = (v >> 6) & 1u;
          } break;
          case C_LDA: if (!rd_operand()) CULE_FALLBACK(); A = v; setnz(v); break;
          case C_STATIA: case C_STTIA: {
            const uint32_t wv = cls == C_STATIA ? A : (aux == 0u ? A : (aux == 1u ? X : (aux == 2u ? Y : (A & X))));
            st_log(lg0 + 4u * log_len, ((3u * now) << 14) | hi | wv);
            ++log_len;
            if (log_len > log_lim) {
              pco = npco;
              fc = now;
              if (kDebug) --budget;
              if (fc >= cap_cycles) { M->fault = 2u; ev = SE_FAULT; }
              else ev = SE_LOGFULL;
              goto out;
            }
          } break;
          case C_WSYNC:  // stall to the next line start (R#5)
            ws_now = now;
            now = ((now + 75u) / 76u) * 76u;
            ws_fc = now;
            break;
          case C_TR: {
            const uint32_t s = aux & 3u, d = hi;
            const uint32_t r = s == 0u ? A : (s == 1u ? X : (s == 2u ? Y : SP));
            A = d == 0u ? r : A;
            X = d == 1u ? r : X;
            Y = d == 2u ? r : Y;
            SP = d == 3u ? r : SP;
            if (aux & 4u) setnz(r);
          } break;
          case C_FLAG: {
            const uint32_t f = aux & 3u, b = (aux >> 2) & 1u;
            C = f == 0u ? b : C;
            I = f == 1u ? b : I;
            D = f == 2u ? b : D;
            V = f == 3u ? b : V;
          } break;
          default: CULE_FALLBACK();
          }
        } else {
          switch (cls) {
          case C_ORA: if (!rd_operand()) CULE_FALLBACK(); A |= v; setnz(A); break;
          case C_AND: if (!rd_operand()) CULE_FALLBACK(); A &= v; setnz(A); break;
          case C_EOR: if (!rd_operand()) CULE_FALLBACK(); A ^= v; setnz(A); break;
          case C_ADC: if (!rd_operand()) CULE_FALLBACK(); adc(v); break;
          case C_BIT: if (!rd_operand()) CULE_FALLBACK(); nz = (A & v) | ((v & 0x80u) << 8); V = (v >> 6) & 1u; break;
          case C_STRAM: {
            const uint32_t t = ea_t();
            if (!(t & 0x80u)) CULE_FALLBACK();
            st_ram(ram0 + (t & 0x7Fu), aux == 0u ? A : (aux == 1u ? X : (aux == 2u ? Y : (A & X))));
          } break;
          case C_INC: case C_DEC: case C_ASL: case C_LSR: case C_ROL: case C_ROR: {
            const uint32_t t = ea_t();
            if (!(t & 0x80u)) CULE_FALLBACK();
            const uint32_t a = ram0 + (t & 0x7Fu);
            const uint32_t m = ld_ram(a);
            uint32_t r;
            if (cls == C_INC) r = (m + 1u) & 0xFFu;
            else if (cls == C_DEC) r = (m - 1u) & 0xFFu;
            else if (cls == C_ASL) { C = m >> 7; r = (m << 1) & 0xFFu; }
            else if (cls == C_LSR) { C = m & 1u; r = m >> 1; }
            else if (cls == C_ROL) { r = ((m << 1) | C) & 0xFFu; C = m >> 7; }
            else { r = (m >> 1) | (C << 7); C = m & 1u; }
            setnz(r);
            st_ram(a, r);
          } break;
          case C_INR: {
            const uint32_t r = (((aux & 1u) ? Y : X) + ((aux & 2u) ? 0xFFu : 1u)) & 0xFFu;
            X = (aux & 1u) ? X : r;
            Y = (aux & 1u) ? r : Y;
            setnz(r);
          } break;
          case C_ASLA: C = A >> 7; A = (A << 1) & 0xFFu; setnz(A); break;
          case C_LSRA: C = A & 1u; A >>= 1; setnz(A); break;
          case C_ROLA: { const uint32_t c = C; C = A >> 7; A = ((A << 1) | c) & 0xFFu; setnz(A); } break;
          case C_RORA: { const uint32_t c = C; C = A & 1u; A = (A >> 1) | (c << 7); setnz(A); } break;
          case C_NOP: break;
          case C_JMP:
            pcw = hi & 0xF000u;
            npco = hi & 0xFFFu;
            if (!kDebug && now >= cap_cycles) { pco = npco; fc = now; M->fault = 2u; ev = SE_FAULT; goto out; }
            break;
          default: CULE_FALLBACK();
          }
        }
      }
#undef CULE_FALLBACK
    fast_done:
      pco = npco;
      fc = now;
      if (kDebug) {
        --budget;
        if (fc >= cap_cycles) { M->fault = 2u; ev = SE_FAULT; break; }  // runaway: fc / 76 >= line_cap
      }
      continue;
    }
  general:  // everything else: the general interpreter, out of line, until the PC is back in a
            // cartridge window
    for (;;) {
      M->PC = pcw | pco; M->A = A; M->X = X; M->Y = Y; M->SP = SP;
      M->C = C; M->V = V; M->D = D; M->I = I; M->nreg = nz >> 8; M->zreg = nz & 0xFFu;
      M->fc = fc; M->bank = bank; M->log_len = log_len; M->t_phaseA = 3u * (fc == ws_fc ? ws_now : fc);
      const uint32_t r = s_gen_one(M, rom_all0, dtab0, ram0, lg0, log_lim, cap_cycles);
      const uint32_t PC = M->PC;
      pcw = PC & 0xF000u; pco = PC & 0xFFFu;
      A = M->A; X = M->X; Y = M->Y; SP = M->SP;
      C = M->C; V = M->V; D = M->D; I = M->I;
      nz = (M->zreg & 0xFFu) | ((M->nreg & 0x80u) << 8);
      fc = M->fc; bank = M->bank; log_len = M->log_len;
      ws_fc = fc; ws_now = M->t_phaseA / 3u;
      tW = M->tW; tVS = M->tV | (M->tS << 8) | (((1u << M->tS) - 1u) << 16);
      if (kDebug && (r & kGenCommitted)) --budget;
      ev = r & 0xFFu;
      if (ev != SE_NONE) goto out;
      if (PC & 0x1000u) break;
      if (kDebug && budget <= 0) { ev = SE_BUDGET; goto out; }
    }
    recb = rec0 + (bank << 15);
    romb = rom0 + (bank << 12);
  }
out:
  M->PC = pcw | pco; M->A = A; M->X = X; M->Y = Y; M->SP = SP;
  M->C = C; M->V = V; M->D = D; M->I = I; M->nreg = nz >> 8; M->zreg = nz & 0xFFu;
  M->fc = fc; M->bank = bank; M->log_len = log_len; M->t_phaseA = 3u * (fc == ws_fc ? ws_now : fc);
  return ev;
}

}  // namespace cule
