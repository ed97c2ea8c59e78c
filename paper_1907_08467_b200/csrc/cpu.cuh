// cpu.cuh — 6502 instruction execution and the frame loop on top of emu.cuh.
//
// One instruction = (A) opcode/operand fetches and pointer reads, which fix the cycle count n;
// (B) the instruction's end T = 3(fc+n) colour clocks; (C) data read, data write and stack
// accesses, all sampling at T (DESIGN.md §2 R#4; SURVEY.md §8(c).4 "bus timing model").
// The TIA is only caught up when an access touches it (or the frame ends).
#pragma once
#include "emu.cuh"

namespace cule {

enum RunStatus : int32_t { RUN_BUDGET = 0, RUN_JAM = 1, RUN_RUNAWAY = 2, RUN_FRAME = 3 };

template <bool kGray>
__device__ __forceinline__ uint32_t exec_one(Machine& m, bool& jam) {
  m.now = m.fc;
  m.wsync_req = 0;
  m.vsync_rose = 0;
  const uint32_t op = m.fetch<kGray>();
  const uint32_t d = m.sm->decode[op];
  const uint32_t mode = d & 0xFu;
  const uint32_t oper = (d >> 4) & 0x7Fu;
  uint32_t n = (d >> 11) & 0xFu;
  if (oper == OP_JAM) { jam = true; return 0; }

  // ---- phase A: effective address -------------------------------------------------------
  uint32_t ea = 0, v = 0;
  switch (mode) {
    case AM_IMM: v = m.fetch<kGray>(); break;
    case AM_ZP: ea = m.fetch<kGray>(); break;
    case AM_ZPX: ea = (m.fetch<kGray>() + m.X) & 0xFFu; break;
    case AM_ZPY: ea = (m.fetch<kGray>() + m.Y) & 0xFFu; break;
    case AM_ABS: case AM_IND: case AM_ABSX: case AM_ABSY: {
      uint32_t lo = m.fetch<kGray>();
      uint32_t hi = m.fetch<kGray>();
      uint32_t base = lo | (hi << 8);
      if (mode == AM_ABS) { ea = base; break; }
      if (mode == AM_IND) {
        uint32_t tl = m.rd<kGray, true>(base);
        uint32_t th = m.rd<kGray, true>((base & 0xFF00u) | ((base + 1) & 0xFFu));
        ea = tl | (th << 8);
        break;
      }
      ea = (base + (mode == AM_ABSX ? m.X : m.Y)) & 0xFFFFu;
      if ((d >> 15) & 1u) n += ((ea ^ base) >> 8) & 1u ? 1u : 0u;
    } break;
    case AM_INDX: {
      uint32_t p = (m.fetch<kGray>() + m.X) & 0xFFu;
      uint32_t lo = m.rd<kGray, true>(p);
      uint32_t hi = m.rd<kGray, true>((p + 1) & 0xFFu);
      ea = lo | (hi << 8);
    } break;
    case AM_INDY: {
      uint32_t p = m.fetch<kGray>();
      uint32_t lo = m.rd<kGray, true>(p);
      uint32_t hi = m.rd<kGray, true>((p + 1) & 0xFFu);
      uint32_t base = lo | (hi << 8);
      ea = (base + m.Y) & 0xFFFFu;
      if ((d >> 15) & 1u) n += ((ea ^ base) >> 8) & 1u ? 1u : 0u;
    } break;
    case AM_REL: {
      uint32_t off = m.fetch<kGray>();
      uint32_t sel = (d >> 17) & 3u;
      uint32_t flag = sel == 0 ? (m.nreg >> 7) & 1u
                    : sel == 1 ? m.fV
                    : sel == 2 ? m.fC
                               : ((m.zreg & 0xFFu) == 0 ? 1u : 0u);
      if (flag == ((d >> 19) & 1u)) {
        uint32_t tgt = (m.PC + (uint32_t)(int32_t)(int8_t)off) & 0xFFFFu;
        n += 1u + (((tgt ^ m.PC) >> 8) & 1u ? 1u : 0u);
        m.PC = tgt;
      }
    } break;
    default: break;  // implied / accumulator
  }

  // ---- phase B/C: accesses at the instruction's end -------------------------------------
  m.now = m.fc + n;
  if ((d >> 16) & 1u) v = m.rd<kGray, false>(ea);

  switch (oper) {
    case OP_LDA: m.A = v; m.nz(v); break;
    case OP_LDX: m.X = v; m.nz(v); break;
    case OP_LDY: m.Y = v; m.nz(v); break;
    case OP_LAX: m.A = m.X = v; m.nz(v); break;
    case OP_STA: m.wr<kGray>(ea, m.A); break;
    case OP_STX: m.wr<kGray>(ea, m.X); break;
    case OP_STY: m.wr<kGray>(ea, m.Y); break;
    case OP_SAX: m.wr<kGray>(ea, m.A & m.X); break;
    case OP_ORA: m.A |= v; m.nz(m.A); break;
    case OP_AND: m.A &= v; m.nz(m.A); break;
    case OP_EOR: m.A ^= v; m.nz(m.A); break;
    case OP_ADC: m.adc(v); break;
    case OP_SBC: m.sbc(v); break;
    case OP_CMP: m.cmp(m.A, v); break;
    case OP_CPX: m.cmp(m.X, v); break;
    case OP_CPY: m.cmp(m.Y, v); break;
    case OP_BIT: m.nreg = v; m.fV = (v >> 6) & 1u; m.zreg = m.A & v; break;
    case OP_ASL: case OP_LSR: case OP_ROL: case OP_ROR: case OP_INC: case OP_DEC:
    case OP_SLO: case OP_RLA: case OP_SRE: case OP_RRA: case OP_DCP: case OP_ISB: {
      const bool acc = mode == AM_ACC;
      uint32_t x = acc ? m.A : v;
      uint32_t r;
      switch (oper) {
        case OP_ASL: case OP_SLO: m.fC = x >> 7; r = (x << 1) & 0xFFu; break;
        case OP_LSR: case OP_SRE: m.fC = x & 1u; r = x >> 1; break;
        case OP_ROL: case OP_RLA: r = ((x << 1) | m.fC) & 0xFFu; m.fC = x >> 7; break;
        case OP_ROR: case OP_RRA: r = (x >> 1) | (m.fC << 7); m.fC = x & 1u; break;
        case OP_INC: case OP_ISB: r = (x + 1) & 0xFFu; break;
        default: r = (x - 1) & 0xFFu; break;  // DEC, DCP
      }
      switch (oper) {
        case OP_SLO: m.A |= r; m.nz(m.A); break;
        case OP_RLA: m.A &= r; m.nz(m.A); break;
        case OP_SRE: m.A ^= r; m.nz(m.A); break;
        case OP_RRA: m.adc(r); break;
        case OP_DCP: m.cmp(m.A, r); break;
        case OP_ISB: m.sbc(r); break;
        default: m.nz(r); break;
      }
      if (acc) m.A = r; else m.wr<kGray>(ea, r);
    } break;
    case OP_ANC: m.A &= v; m.nz(m.A); m.fC = m.A >> 7; break;
    case OP_ALR: { uint32_t t = m.A & v; m.fC = t & 1u; m.A = t >> 1; m.nz(m.A); } break;
    case OP_ARR: {
      uint32_t t = m.A & v;
      m.A = (t >> 1) | (m.fC << 7);
      m.nz(m.A);
      m.fC = (m.A >> 6) & 1u;
      m.fV = ((m.A >> 6) ^ (m.A >> 5)) & 1u;
    } break;
    case OP_SBX: { uint32_t t = m.A & m.X; m.fC = t >= v ? 1u : 0u; m.X = (t - v) & 0xFFu; m.nz(m.X); } break;
    case OP_NOP: break;
    case OP_INX: m.X = (m.X + 1) & 0xFFu; m.nz(m.X); break;
    case OP_INY: m.Y = (m.Y + 1) & 0xFFu; m.nz(m.Y); break;
    case OP_DEX: m.X = (m.X - 1) & 0xFFu; m.nz(m.X); break;
    case OP_DEY: m.Y = (m.Y - 1) & 0xFFu; m.nz(m.Y); break;
    case OP_TAX: m.X = m.A; m.nz(m.X); break;
    case OP_TAY: m.Y = m.A; m.nz(m.Y); break;
    case OP_TXA: m.A = m.X; m.nz(m.A); break;
    case OP_TYA: m.A = m.Y; m.nz(m.A); break;
    case OP_TSX: m.X = m.SP; m.nz(m.X); break;
    case OP_TXS: m.SP = m.X; break;
    case OP_CLC: m.fC = 0; break;
    case OP_SEC: m.fC = 1; break;
    case OP_CLI: m.fI = 0; break;
    case OP_SEI: m.fI = 1; break;
    case OP_CLV: m.fV = 0; break;
    case OP_CLD: m.fD = 0; break;
    case OP_SED: m.fD = 1; break;
    case OP_PHA: m.push<kGray>(m.A); break;
    case OP_PHP: m.push<kGray>(m.getP() | 0x30u); break;
    case OP_PLA: m.A = m.pull<kGray>(); m.nz(m.A); break;
    case OP_PLP: m.setP(m.pull<kGray>()); break;
    case OP_JMP: m.PC = ea; break;
    case OP_JSR: {
      uint32_t ret = (m.PC - 1) & 0xFFFFu;  // address of the JSR's last byte
      m.push<kGray>(ret >> 8);
      m.push<kGray>(ret & 0xFFu);
      m.PC = ea;
    } break;
    case OP_RTS: {
      uint32_t lo = m.pull<kGray>();
      uint32_t hi = m.pull<kGray>();
      m.PC = ((lo | (hi << 8)) + 1) & 0xFFFFu;
    } break;
    case OP_RTI: {
      m.setP(m.pull<kGray>());
      uint32_t lo = m.pull<kGray>();
      uint32_t hi = m.pull<kGray>();
      m.PC = lo | (hi << 8);
    } break;
    case OP_BRK: {
      uint32_t ret = (m.PC + 1) & 0xFFFFu;
      m.push<kGray>(ret >> 8);
      m.push<kGray>(ret & 0xFFu);
      m.push<kGray>(m.getP() | 0x30u);
      m.fI = 1;
      uint32_t lo = m.rd<kGray, false>(0x1FFEu);
      uint32_t hi = m.rd<kGray, false>(0x1FFFu);
      m.PC = lo | (hi << 8);
    } break;
    default: break;  // OP_BRANCH handled in phase A
  }
  return n;
}

// End the frame at the VSYNC edge: finish the TIA, rebase clocks to the VSYNC line, canonical
// timer stamp (DESIGN.md §2 R#6, R#24).
template <bool kGray>
__device__ __forceinline__ void end_frame(Machine& m) {
  m.catch_up<kGray>(3u * m.fc);
  uint32_t L = m.fc / 76u;
  m.last_lines = L;
  m.fc -= 76u * L;
  m.tW -= (int32_t)(76u * L);
  m.t_tia -= 228u * L;
  m.t_phaseA = m.t_tia;
  int32_t cl = m.comb_line - (int32_t)L;
  m.comb_line = cl < 0 ? -1 : cl;
  int32_t e = (int32_t)m.fc - m.tW;
  int32_t VI = (int32_t)(m.tV << m.tS);
  if (e > VI) m.tW = (int32_t)m.fc - (VI + 1 + ((e - VI - 1) & 0xFF));
}

// Run until the frame ends (VSYNC rise), a fault, or max_instr instructions (<0: unlimited).
template <bool kGray>
__device__ int32_t run_frame(Machine& m, uint32_t line_cap, int32_t max_instr) {
  int32_t count = 0;
  for (;;) {
    if (max_instr >= 0 && count >= max_instr) {
      m.catch_up<kGray>(3u * m.fc);
      m.t_phaseA = m.t_tia;
      return RUN_BUDGET;
    }
    bool jam = false;
    uint32_t n = exec_one<kGray>(m, jam);
    if (jam) {
      m.catch_up<kGray>(3u * m.fc);
      return RUN_JAM;
    }
    ++count;
    m.fc += n;
    m.t_phaseA = 3u * m.fc;
    if (m.wsync_req) m.fc = ((m.fc + 75u) / 76u) * 76u;
    if (m.fc / 76u >= line_cap) {
      m.catch_up<kGray>(3u * m.fc);
      return RUN_RUNAWAY;
    }
    if (m.vsync_rose) {
      end_frame<kGray>(m);
      return RUN_FRAME;
    }
  }
}

}  // namespace cule
