// cpu.cuh — the 6502/6507 + RIOT + bus of one environment, registers-resident.
//
// One instruction (DESIGN.md §2 R#4): (A) opcode/operand fetches and pointer reads fix the
// cycle count n; (B) the instruction ends at T = 3(fc+n) colour clocks; (C) data read, data
// write and stack accesses all sample at T.  Ordinary instructions run through one branch-free
// micro-coded datapath (decode_table.h); the data read of RAM or ROM is a single shared-memory
// load whose address is selected arithmetically, so only TIA/RIOT/bank-switch accesses, stack
// and control instructions, and decimal arithmetic leave the common path.
#pragma once
#include "decode_table.h"
#include "tia.cuh"

namespace cule {

enum Event : uint32_t { EV_NONE = 0, EV_LOGFULL = 1, EV_FRAME = 2, EV_FAULT = 3 };

// out-of-line so the rare collision-read path does not bloat the hot loop; scalar arguments
// only, so no caller state is forced into local memory
__device__ __noinline__ uint32_t flush_call(uint32_t* tw, uint32_t* pw, const uint32_t* lg, uint32_t s,
                                            uint32_t n, uint32_t fin, uint32_t t, uint32_t ystart,
                                            const uint8_t* gray, uint32_t delays) {
  flush_lane(tw, pw, lg, s, n, fin != 0, t, ystart, gray, delays);
  return tw[7 * s] >> 16;  // collision latches
}
__device__ __forceinline__ uint32_t coll_read_flush(uint32_t* tw, uint32_t* pw, const uint32_t* lg, uint32_t s,
                                                    uint32_t n, uint32_t t, uint32_t ystart, const uint8_t* gray,
                                                    uint32_t delays) {
  return flush_call(tw, pw, lg, s, n, 1u, t, ystart, gray, delays);
}

struct Ctx {
  uint8_t* smem;          // dynamic shared memory base
  const uint64_t* decode; // [256]
  const uint8_t* gray;    // GRAY84: gray LUT in smem; RAW: nullptr
  uint32_t rom0;          // smem offset of the ROM images
  uint32_t ram0;          // smem offset of this thread's RAM word 0 (stride ram_stride)
  uint32_t ram_stride;    // bytes between RAM words of one thread (4 * blockDim)
  uint32_t* tw;           // this thread's TIA words        (stride s)
  uint32_t* pw;           // this thread's pixel-writer words
  uint32_t* lg;           // this thread's TIA write log
  uint32_t s;             // word stride = blockDim
  uint32_t ystart, line_cap;
  uint32_t cap_cycles;    // 76 * line_cap
  uint32_t idle_skip;     // exact idle-loop skip enabled (cule_config.idle_skip)
  uint32_t tia_delays;    // delayed register effects (cule_config.tia_delays, R#35)
};

struct Cpu {
  uint32_t PC, A, X, Y, SP, C, V, D, I, nreg, zreg;
  uint32_t fc, now, t_phaseA;
  uint32_t bank, rom_off, hs_lo, nbank, flim;
  uint32_t tV, tS, swcha, inpt4;
  int32_t tW;
  uint32_t vsync, log_len, fault;
  // idle-loop skip (exact): timer-read constancy (cycles) of this instruction's data read, and
  // the previous instruction when it was a plain timer read (its PC and cycles)
  uint32_t ff, ppc, pn, pff;

  __device__ __forceinline__ uint32_t getP() const {
    return (nreg & 0x80u) | (V << 6) | 0x20u | (D << 3) | (I << 2) | ((zreg & 0xFFu) == 0 ? 2u : 0u) | C;
  }
  __device__ __forceinline__ void setP(uint32_t p) {
    nreg = p & 0x80u; V = (p >> 6) & 1u; D = (p >> 3) & 1u; I = (p >> 2) & 1u;
    zreg = (p & 2u) ? 0u : 1u; C = p & 1u;
  }

  __device__ __forceinline__ uint32_t ram_addr(const Ctx& c, uint32_t a) const {
    return c.ram0 + (a >> 2) * c.ram_stride + (a & 3u);
  }
  __device__ __forceinline__ uint32_t ram_rd(const Ctx& c, uint32_t a) const { return c.smem[ram_addr(c, a & 0x7Fu)]; }

  // RIOT interval timer, closed form from the write stamp (DESIGN.md §2 R#24)
  __device__ __forceinline__ uint32_t riot_read(uint32_t a) const {
    if (!(a & 0x04u)) {
      uint32_t k = a & 3u;
      return k == 0 ? swcha : (k == 2 ? 0x0Bu : 0u);
    }
    int32_t e = (int32_t)now - tW;
    int32_t VI = (int32_t)(tV << tS);
    if (a & 1u) return e > VI ? 0x80u : 0u;
    if (e <= VI) return (tV - (uint32_t)((e + (1 << tS) - 1) >> tS)) & 0xFFu;
    return (uint32_t)(0xFF - (e - VI - 1)) & 0xFFu;
  }
  // the same read, also noting for how many more cycles the value read stays the same
  __device__ __forceinline__ uint32_t riot_read_ff(uint32_t a) {
    if (!(a & 0x04u)) return riot_read(a);
    const int32_t e = (int32_t)now - tW;
    const int32_t VI = (int32_t)(tV << tS);
    if (a & 1u) {
      ff = e > VI ? 0x7FFFFFFFu : (uint32_t)(VI - e);
      return e > VI ? 0x80u : 0u;
    }
    if (e <= VI) {
      const int32_t q = (e + (1 << tS) - 1) >> tS;
      ff = (uint32_t)((q << tS) - e);
      return (tV - (uint32_t)q) & 0xFFu;
    }
    return (uint32_t)(0xFF - (e - VI - 1)) & 0xFFu;
  }

  // collision-latch read: flush this lane's log (divergent but rare) and advance to t
  __device__ __forceinline__ uint32_t tia_coll_read(const Ctx& c, uint32_t r, uint32_t t) {
    const uint32_t coll = coll_read_flush(c.tw, c.pw, c.lg, c.s, log_len, t, c.ystart, c.gray, c.tia_delays);
    log_len = 0;
    return (((coll >> (2 * r)) & 1u) << 7) | (((coll >> (2 * r + 1)) & 1u) << 6);
  }

  // full bus read; phase A (fetch / pointer) or phase C (data) — DESIGN.md §2 R#4
  template <bool kPhaseA>
  __device__ __forceinline__ uint32_t rd(const Ctx& c, uint32_t addr) {
    const uint32_t a = addr & 0x1FFFu;
    const bool cart = (a & 0x1000u) != 0;
    const bool hot = cart && ((a & 0xFFFu) - hs_lo) < nbank;
    const bool ram = !cart && ((a & 0x0280u) == 0x0080u);
    if (cart | ram) {
      if (hot) bank = (a & 0xFFFu) - hs_lo;
      const uint32_t off = cart ? c.rom0 + rom_off + (bank << 12) + (a & 0xFFFu) : ram_addr(c, a & 0x7Fu);
      return c.smem[off];
    }
    if (!(a & 0x80u)) {  // TIA read registers
      const uint32_t r = a & 0x0Fu;
      if (r < 8u) return tia_coll_read(c, r, kPhaseA ? t_phaseA : 3u * now);
      return r == 0x0Cu ? inpt4 : (r == 0x0Du ? 0x80u : 0u);
    }
    return kPhaseA ? riot_read(a) : riot_read_ff(a);
  }

  __device__ __forceinline__ void wr(const Ctx& c, uint32_t addr, uint32_t v) {
    const uint32_t a = addr & 0x1FFFu;
    if ((a & 0x1280u) == 0x0080u) { c.smem[ram_addr(c, a & 0x7Fu)] = (uint8_t)v; return; }
    if (a & 0x1000u) {
      if (((a & 0xFFFu) - hs_lo) < nbank) bank = (a & 0xFFFu) - hs_lo;
      return;
    }
    if (!(a & 0x80u)) {
      const uint32_t r = a & 0x3Fu;
      if (r == 0x02u) { wsync_pending = 1; return; }
      if (r == 0x00u) {
        uint32_t nv = (v >> 1) & 1u;
        if (!vsync && nv) vsync_rose = 1;
        vsync = nv;
        return;
      }
      if (r == 0x03u || (r >= 0x15u && r <= 0x1Au) || r >= 0x2Du) return;  // no TIA effect
      c.lg[log_len * c.s] = log_entry(3u * now, r, v);
      ++log_len;
      return;
    }
    if ((a & 0x14u) == 0x14u) {  // timer write: interval 1 / 8 / 64 / 1024
      tV = v & 0xFFu;
      tS = (0xA630u >> (4 * (a & 3u))) & 0xFu;
      tW = (int32_t)now;
    }
  }
  uint32_t wsync_pending, vsync_rose;

  __device__ __forceinline__ void push(const Ctx& c, uint32_t v) { wr(c, 0x100u | SP, v); SP = (SP - 1) & 0xFFu; }
  __device__ __forceinline__ uint32_t pull(const Ctx& c) { SP = (SP + 1) & 0xFFu; return rd<false>(c, 0x100u | SP); }

  // ---- one instruction; returns an Event ------------------------------------------------------
  template <bool kSkip>
  __device__ __forceinline__ uint32_t exec(const Ctx& c) {
    now = fc;
    wsync_pending = 0;
    vsync_rose = 0;
    const uint32_t pc = PC;
    uint32_t op, b1, b2;
    uint64_t d;
    if ((pc & 0x1000u) && (pc & 0xFFFu) <= flim) {
      const uint8_t* p = c.smem + c.rom0 + rom_off + (bank << 12) + (pc & 0xFFFu);
      op = p[0]; b1 = p[1]; b2 = p[2];
      d = c.decode[op];
    } else {
      op = rd<true>(c, pc);
      d = c.decode[op];
      const uint32_t len = (uint32_t)d & 3u;
      b1 = len > 1 ? rd<true>(c, pc + 1) : 0u;
      b2 = len > 2 ? rd<true>(c, pc + 2) : 0u;
    }
    const uint32_t lo = (uint32_t)d, hi = (uint32_t)(d >> 32);
    const uint32_t spc = (hi >> dk::SPC) & 0xFu;
    uint32_t n = (lo >> dk::CYC) & 0xFu;  // JAM entries: 1 byte, 0 cycles, no effects (R#1)
    PC = (pc + (lo & 3u)) & 0xFFFFu;

    // ---- phase A: effective address --------------------------------------------------------------
    const uint32_t zpa = (b1 + ((lo & dk::ZIX) ? X : 0u) + ((lo & dk::ZIY) ? Y : 0u)) & 0xFFu;
    uint32_t base = b1 | (b2 << 8);
    if (lo & (dk::PTRZ | dk::PTRA)) {
      const bool pa = (lo & dk::PTRA) != 0;
      const uint32_t p0 = pa ? base : zpa;
      const uint32_t p1 = pa ? ((base & 0xFF00u) | ((base + 1) & 0xFFu)) : ((zpa + 1) & 0xFFu);
      const uint32_t plo = rd<true>(c, p0);
      const uint32_t phi = rd<true>(c, p1);
      base = plo | (phi << 8);
    }
    const uint32_t ea16 = (base + ((lo & dk::AIX) ? X : 0u) + ((lo & dk::AIY) ? Y : 0u)) & 0xFFFFu;
    const uint32_t ea = (lo & dk::ZP) ? zpa : ea16;
    if ((lo & dk::PEN) && ((ea16 ^ base) & 0x100u)) ++n;
    if (lo & dk::BR) {
      const uint32_t flags4 = ((nreg >> 7) & 1u) | (V << 1) | (C << 2) | ((zreg & 0xFFu) == 0 ? 8u : 0u);
      const uint32_t taken = ((flags4 >> ((hi >> dk::BRF) & 3u)) ^ ((hi & dk::BRT) ? 0u : 1u)) & 1u;
      const uint32_t tgt = (PC + (uint32_t)(int32_t)(int8_t)b1) & 0xFFFFu;
      n += taken ? 1u + (((tgt ^ PC) >> 8) & 1u) : 0u;
      PC = taken ? tgt : PC;
      // idle-loop skip: [plain timer read; branch back to it] — the iterations whose read falls
      // in the same constant interval repeat this one exactly, so only time advances (stopping
      // short of the runaway cap, which the loop then reaches normally).  Same rule as the
      // scalar engine (scalar_cpu.cuh).
      if (kSkip && taken && pff != 0u && tgt == ppc && (pc & 0x1000u) && fc + n < c.cap_cycles) {
        const uint32_t P = pn + n;
        n += min(pff / P, (c.cap_cycles - 1u - (fc + n)) / P) * P;
      }
    }
    if (lo & dk::JMP) PC = ea;

    // ---- phase C ---------------------------------------------------------------------------------
    now = fc + n;
    ff = 0u;
    uint32_t v = b1;  // immediate operand
    if (lo & dk::RD) v = rd<false>(c, ea);

    {
      // register operand and unit1 (shift / rotate / increment); special ops have no unit bits,
      // so this datapath leaves their state unchanged and the special switch runs after it
      const uint32_t R = ((lo & dk::RA) ? A : 0u) | ((lo & dk::RX) ? X : 0u) | ((lo & dk::RY) ? Y : 0u) |
                         ((lo & dk::RS) ? SP : 0u);
      const uint32_t M = (lo & dk::OPR) ? R : v;
      const uint32_t cr = (lo & dk::ROT) ? C : 0u;
      const uint32_t idc = (M + ((lo & dk::INC) ? 1u : 0u) + ((lo & dk::DEC) ? 0xFFu : 0u)) & 0xFFu;
      const uint32_t r1 = (lo & dk::SHL) ? (((M << 1) | cr) & 0xFFu) : ((lo & dk::SHR) ? ((M >> 1) | (cr << 7)) : idc);
      const uint32_t c1 = (lo & dk::SHL) ? (M >> 7) : ((lo & dk::SHR) ? (M & 1u) : C);
      // unit2: logic / adder (ADC, SBC, CMP) / BIT
      const uint32_t lhs = (hi & dk::CMP) ? R : A;
      const uint32_t add = (hi & dk::INV) ? (r1 ^ 0xFFu) : r1;
      const uint32_t sum = lhs + add + ((hi & dk::CMP) ? 1u : c1);
      const uint32_t rlog = (hi & dk::OR) ? (A | r1) : ((hi & dk::AND) ? (A & r1) : (A ^ r1));
      uint32_t r2 = (hi & dk::LOGIC) ? rlog : ((hi & dk::ARITH) ? (sum & 0xFFu) : r1);
      uint32_t nC = (hi & dk::ARITH) ? (sum >> 8) : c1;
      uint32_t nV = (hi & dk::ADDV) ? (((~(lhs ^ add) & (lhs ^ sum)) >> 7) & 1u)
                                    : ((hi & dk::BIT) ? ((r1 >> 6) & 1u) : V);
      uint32_t nn = (hi & dk::BIT) ? r1 : r2;
      uint32_t nz_ = (hi & dk::BIT) ? (A & r1) : r2;
      if (D && (hi & dk::ADDV)) decimal((hi & dk::INV) == 0, r1, c1, r2, nC, nV, nn, nz_);
      if (lo & dk::WR) wr(c, ea, (lo & dk::WSEL) ? ((lo & dk::SAX) ? (A & X) : R) : r1);
      A = (hi & dk::DA) ? r2 : A;
      X = (hi & dk::DX) ? r2 : X;
      Y = (hi & dk::DY) ? r2 : Y;
      SP = (hi & dk::DS) ? r2 : SP;
      nreg = (lo & dk::NZ) ? nn : nreg;
      zreg = (lo & dk::NZ) ? (nz_ & 0xFFu) : zreg;
      C = nC;
      V = nV;
      if (lo & dk::FOP) {
        const uint32_t fi = (hi >> dk::FIDX) & 3u, fv = (hi & dk::FVAL) ? 1u : 0u;
        C = fi == 0 ? fv : C;
        I = fi == 1 ? fv : I;
        D = fi == 2 ? fv : D;
        V = fi == 3 ? fv : V;
      }
    }
    if (spc) special(c, spc, v, ea);

    // ---- end of instruction ------------------------------------------------------------------------
    // a plain timer read (cartridge code, abs, read-only, idempotent effect) can head an idle loop
    const bool plain = (pc & 0x1000u) && (lo & dk::RD) && !(lo & dk::WR) && spc == 0u &&
                       !(lo & (dk::ZP | dk::ZIX | dk::ZIY | dk::AIX | dk::AIY | dk::PTRZ | dk::PTRA)) &&
                       !(hi & (dk::LOGIC | dk::ADDV));
    pff = (plain && c.idle_skip) ? ff : 0u;
    ppc = pc;
    pn = now - fc;
    fc = now;
    t_phaseA = 3u * now;
    if (wsync_pending) fc = ((fc + 75u) / 76u) * 76u;  // stall to the next line start (R#5)
    fault = (fc >= c.cap_cycles && !fault) ? 2u : fault;  // runaway: fc / 76 >= line_cap
    return fault ? EV_FAULT
                 : (vsync_rose ? EV_FRAME : (log_len > (uint32_t)(kLogCap - kLogMargin) ? EV_LOGFULL : EV_NONE));
  }

  // NMOS decimal ADC / SBC (Bruce Clark's sequences, DESIGN.md §2 R#2)
  __device__ __forceinline__ void decimal(bool is_adc, uint32_t m, uint32_t cin, uint32_t& r2, uint32_t& nC,
                                       uint32_t& nV, uint32_t& nn, uint32_t& nz_) const {
    if (is_adc) {
      uint32_t lo = (A & 0xFu) + (m & 0xFu) + cin;
      if (lo >= 0xAu) lo = ((lo + 6u) & 0xFu) + 0x10u;
      uint32_t s = (A & 0xF0u) + (m & 0xF0u) + lo;
      int32_t sv = (int32_t)(int8_t)(A & 0xF0u) + (int32_t)(int8_t)(m & 0xF0u) + (int32_t)lo;
      nz_ = (A + m + cin) & 0xFFu;
      nn = s;
      nV = (sv < -128 || sv > 127) ? 1u : 0u;
      if (s >= 0xA0u) s += 0x60u;
      nC = s >= 0x100u ? 1u : 0u;
      r2 = s & 0xFFu;
    } else {
      int32_t lo = (int32_t)(A & 0xFu) - (int32_t)(m & 0xFu) + (int32_t)cin - 1;
      if (lo < 0) lo = ((lo - 6) & 0xF) - 0x10;
      int32_t s = (int32_t)(A & 0xF0u) - (int32_t)(m & 0xF0u) + lo;
      if (s < 0) s -= 0x60;
      r2 = (uint32_t)s & 0xFFu;  // flags stay binary
    }
  }

  // stack / control flow / immediate undocumented ops
  __device__ __forceinline__ void special(const Ctx& c, uint32_t spc, uint32_t v, uint32_t ea) {
    switch (spc) {
      case SP_PHA: push(c, A); break;
      case SP_PHP: push(c, getP() | 0x30u); break;
      case SP_PLA: A = pull(c); nreg = A; zreg = A; break;
      case SP_PLP: setP(pull(c)); break;
      case SP_JSR: {
        const uint32_t ret = (PC - 1) & 0xFFFFu;
        push(c, ret >> 8);
        push(c, ret & 0xFFu);
        PC = ea;
      } break;
      case SP_RTS: {
        const uint32_t lo = pull(c);
        const uint32_t hi = pull(c);
        PC = ((lo | (hi << 8)) + 1) & 0xFFFFu;
      } break;
      case SP_RTI: {
        setP(pull(c));
        const uint32_t lo = pull(c);
        const uint32_t hi = pull(c);
        PC = lo | (hi << 8);
      } break;
      case SP_BRK: {
        const uint32_t ret = (PC + 1) & 0xFFFFu;
        push(c, ret >> 8);
        push(c, ret & 0xFFu);
        push(c, getP() | 0x30u);
        I = 1;
        const uint32_t lo = rd<false>(c, 0x1FFEu);
        const uint32_t hi = rd<false>(c, 0x1FFFu);
        PC = lo | (hi << 8);
      } break;
      case SP_ANC: A &= v; nreg = A; zreg = A; C = A >> 7; break;
      case SP_ALR: { uint32_t t = A & v; C = t & 1u; A = t >> 1; nreg = A; zreg = A; } break;
      case SP_ARR: {
        uint32_t t = A & v;
        A = (t >> 1) | (C << 7);
        nreg = A; zreg = A;
        C = (A >> 6) & 1u;
        V = ((A >> 6) ^ (A >> 5)) & 1u;
      } break;
      case SP_SBX: { uint32_t t = A & X; C = t >= v ? 1u : 0u; X = (t - v) & 0xFFu; nreg = X; zreg = X; } break;
      case SP_JAM: fault = 1; break;
      default: break;
    }
  }
};

}  // namespace cule
