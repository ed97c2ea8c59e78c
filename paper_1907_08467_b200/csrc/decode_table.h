// decode_table.h — host-side construction of the 6502 micro-coded decode table used by the
// step kernel (one 64-bit entry per opcode, staged into shared memory once per block).
// Product code; independent of the oracle (which executes a per-opcode switch).
//
// The kernel runs every ordinary instruction through ONE branch-free datapath:
//   R  = register operand (A/X/Y/SP);  M = memory/immediate byte, or R for implied forms
//   u1 = unit1(M): pass | ASL | LSR | ROL | ROR | INC | DEC   (carry c1)
//   r2 = unit2(u1): pass | OR | AND | EOR | ADC | SBC | CMP(R) | BIT  (8-bit adder shared)
//   then destination register, memory write value, N/Z/C/V updates — all selected by fields
// so lanes executing different opcodes still share instructions.  Stack/control and the
// rare undocumented immediates take a small "special" switch.
//
// Cycle counts derive from the addressing-mode x access-class rules of the NMOS 6502
// (bottom table), not from a per-opcode list.
#pragma once
#include <stdint.h>

#include <initializer_list>
#include <utility>

namespace cule {

enum AddrMode : uint32_t {
  AM_IMP = 0, AM_ACC, AM_IMM, AM_ZP, AM_ZPX, AM_ZPY, AM_ABS, AM_ABSX, AM_ABSY, AM_IND,
  AM_INDX, AM_INDY, AM_REL
};
enum Unit1 : uint32_t { U1_PASS = 0, U1_ASL, U1_LSR, U1_ROL, U1_ROR, U1_INC, U1_DEC };
enum Unit2 : uint32_t { U2_PASS = 0, U2_OR, U2_AND, U2_EOR, U2_ADC, U2_SBC, U2_CMP, U2_BIT };
enum Reg : uint32_t { RG_A = 0, RG_X, RG_Y, RG_SP };
enum Dst : uint32_t { DS_NONE = 0, DS_A, DS_X, DS_Y, DS_SP, DS_AX };
enum Special : uint32_t {
  SP_NONE = 0, SP_PHA, SP_PHP, SP_PLA, SP_PLP, SP_JSR, SP_RTS, SP_RTI, SP_BRK, SP_ANC, SP_ALR,
  SP_ARR, SP_SBX, SP_JAM
};

// bit fields of an entry
namespace dk {
constexpr int MODE = 0;     // 4 bits
constexpr int LEN = 4;      // 2 bits: instruction length 1..3
constexpr int CYC = 6;      // 4 bits: base cycles
constexpr int PEN = 10;     // 1: +1 on page cross
constexpr int RD = 11;      // 1: data read at EA
constexpr int WR = 12;      // 1: data write at EA
constexpr int RSRC = 13;    // 2: register operand R
constexpr int OPR = 15;     // 1: M = R (implied/accumulator forms)
constexpr int U1 = 16;      // 3
constexpr int U2 = 19;      // 3
constexpr int DST = 22;     // 3
constexpr int WSEL = 25;    // 1: write value = store value (R, or A&X) instead of u1
constexpr int SAX = 26;     // 1: store value A&X
constexpr int NZ = 27;      // 1: update N/Z
constexpr int FOP = 28;     // 1: flag set/clear op
constexpr int FIDX = 29;    // 2: 0 C, 1 I, 2 D, 3 V
constexpr int FVAL = 31;    // 1
constexpr int SPC = 32;     // 4: special op
constexpr int BR = 36;      // 1: conditional branch
constexpr int BRF = 37;     // 2: branch flag 0 N 1 V 2 C 3 Z
constexpr int BRT = 39;     // 1: taken when flag set
constexpr int JMP = 40;     // 1: PC <- EA
}  // namespace dk

inline uint32_t mode_len(uint32_t mode) {
  switch (mode) {
    case AM_IMP: case AM_ACC: return 1;
    case AM_ABS: case AM_ABSX: case AM_ABSY: case AM_IND: return 3;
    default: return 2;
  }
}

enum AccessClass { CL_READ, CL_WRITE, CL_RMW };

inline uint32_t mode_cycles(uint32_t mode, AccessClass cl, bool* pen) {
  *pen = false;
  switch (mode) {
    case AM_IMP: case AM_ACC: case AM_IMM: return 2;
    case AM_ZP: return cl == CL_RMW ? 5 : 3;
    case AM_ZPX: case AM_ZPY: return cl == CL_RMW ? 6 : 4;
    case AM_ABS: return cl == CL_RMW ? 6 : 4;
    case AM_ABSX: case AM_ABSY:
      if (cl == CL_READ) { *pen = true; return 4; }
      return cl == CL_RMW ? 7 : 5;
    case AM_INDX: return cl == CL_RMW ? 8 : 6;
    case AM_INDY:
      if (cl == CL_READ) { *pen = true; return 5; }
      return cl == CL_RMW ? 8 : 6;
    default: return 2;
  }
}

struct Micro {
  uint32_t u1 = U1_PASS, u2 = U2_PASS, rsrc = RG_A, dst = DS_NONE;
  bool opr = false, wsel = false, sax = false, nz = false;
};

inline uint64_t entry(uint32_t mode, uint32_t cyc, bool pen, bool rd, bool wr, const Micro& u) {
  uint64_t e = 0;
  e |= (uint64_t)mode << dk::MODE;
  e |= (uint64_t)mode_len(mode) << dk::LEN;
  e |= (uint64_t)cyc << dk::CYC;
  e |= (uint64_t)(pen ? 1 : 0) << dk::PEN;
  e |= (uint64_t)(rd ? 1 : 0) << dk::RD;
  e |= (uint64_t)(wr ? 1 : 0) << dk::WR;
  e |= (uint64_t)u.rsrc << dk::RSRC;
  e |= (uint64_t)(u.opr ? 1 : 0) << dk::OPR;
  e |= (uint64_t)u.u1 << dk::U1;
  e |= (uint64_t)u.u2 << dk::U2;
  e |= (uint64_t)u.dst << dk::DST;
  e |= (uint64_t)(u.wsel ? 1 : 0) << dk::WSEL;
  e |= (uint64_t)(u.sax ? 1 : 0) << dk::SAX;
  e |= (uint64_t)(u.nz ? 1 : 0) << dk::NZ;
  return e;
}

inline void build_decode_table(uint64_t* table) {
  for (int i = 0; i < 256; i++) table[i] = ((uint64_t)SP_JAM << dk::SPC) | (1ull << dk::LEN);
  auto group = [&](const Micro& u, AccessClass cl, std::initializer_list<std::pair<uint32_t, uint32_t>> ms) {
    for (auto& p : ms) {
      bool pen;
      uint32_t cyc = mode_cycles(p.first, cl, &pen);
      bool rd = (cl == CL_READ && p.first != AM_IMM) || cl == CL_RMW;
      bool wr = cl != CL_READ;
      table[p.second] = entry(p.first, cyc, pen, rd, wr, u);
    }
  };
  auto mk = [](uint32_t u1, uint32_t u2, uint32_t rsrc, uint32_t dst, bool nz) {
    Micro m;
    m.u1 = u1; m.u2 = u2; m.rsrc = rsrc; m.dst = dst; m.nz = nz;
    return m;
  };
  // eight-mode ALU group aaa bbb 01
  const uint32_t alu8[7][3] = {{U2_OR, 0x00, DS_A}, {U2_AND, 0x20, DS_A}, {U2_EOR, 0x40, DS_A},
                               {U2_ADC, 0x60, DS_A}, {U2_PASS, 0xA0, DS_A}, {U2_CMP, 0xC0, DS_NONE},
                               {U2_SBC, 0xE0, DS_A}};
  for (auto& g : alu8) {
    uint32_t b = g[1];
    group(mk(U1_PASS, g[0], RG_A, g[2], true), CL_READ,
          {{AM_INDX, b + 0x01}, {AM_ZP, b + 0x05}, {AM_IMM, b + 0x09}, {AM_ABS, b + 0x0D},
           {AM_INDY, b + 0x11}, {AM_ZPX, b + 0x15}, {AM_ABSY, b + 0x19}, {AM_ABSX, b + 0x1D}});
  }
  group(mk(U1_PASS, U2_SBC, RG_A, DS_A, true), CL_READ, {{AM_IMM, 0xEB}});
  auto store = [&](uint32_t rsrc, bool sax) {
    Micro m;
    m.rsrc = rsrc; m.wsel = true; m.sax = sax;
    return m;
  };
  group(store(RG_A, false), CL_WRITE, {{AM_INDX, 0x81}, {AM_ZP, 0x85}, {AM_ABS, 0x8D}, {AM_INDY, 0x91},
                                       {AM_ZPX, 0x95}, {AM_ABSY, 0x99}, {AM_ABSX, 0x9D}});
  group(store(RG_X, false), CL_WRITE, {{AM_ZP, 0x86}, {AM_ABS, 0x8E}, {AM_ZPY, 0x96}});
  group(store(RG_Y, false), CL_WRITE, {{AM_ZP, 0x84}, {AM_ABS, 0x8C}, {AM_ZPX, 0x94}});
  group(store(RG_A, true), CL_WRITE, {{AM_INDX, 0x83}, {AM_ZP, 0x87}, {AM_ABS, 0x8F}, {AM_ZPY, 0x97}});
  group(mk(U1_PASS, U2_PASS, RG_A, DS_X, true), CL_READ,
        {{AM_IMM, 0xA2}, {AM_ZP, 0xA6}, {AM_ABS, 0xAE}, {AM_ZPY, 0xB6}, {AM_ABSY, 0xBE}});
  group(mk(U1_PASS, U2_PASS, RG_A, DS_Y, true), CL_READ,
        {{AM_IMM, 0xA0}, {AM_ZP, 0xA4}, {AM_ABS, 0xAC}, {AM_ZPX, 0xB4}, {AM_ABSX, 0xBC}});
  group(mk(U1_PASS, U2_PASS, RG_A, DS_AX, true), CL_READ,
        {{AM_INDX, 0xA3}, {AM_ZP, 0xA7}, {AM_ABS, 0xAF}, {AM_INDY, 0xB3}, {AM_ZPY, 0xB7}, {AM_ABSY, 0xBF}});
  group(mk(U1_PASS, U2_CMP, RG_X, DS_NONE, true), CL_READ, {{AM_IMM, 0xE0}, {AM_ZP, 0xE4}, {AM_ABS, 0xEC}});
  group(mk(U1_PASS, U2_CMP, RG_Y, DS_NONE, true), CL_READ, {{AM_IMM, 0xC0}, {AM_ZP, 0xC4}, {AM_ABS, 0xCC}});
  group(mk(U1_PASS, U2_BIT, RG_A, DS_NONE, true), CL_READ, {{AM_ZP, 0x24}, {AM_ABS, 0x2C}});
  // shifts / rotates / inc / dec on memory, and the accumulator forms
  const uint32_t rmw[6][2] = {{U1_ASL, 0x00}, {U1_ROL, 0x20}, {U1_LSR, 0x40}, {U1_ROR, 0x60},
                              {U1_DEC, 0xC0}, {U1_INC, 0xE0}};
  for (auto& g : rmw) {
    uint32_t b = g[1];
    group(mk(g[0], U2_PASS, RG_A, DS_NONE, true), CL_RMW,
          {{AM_ZP, b + 0x06}, {AM_ABS, b + 0x0E}, {AM_ZPX, b + 0x16}, {AM_ABSX, b + 0x1E}});
    if (g[0] != U1_DEC && g[0] != U1_INC) {
      Micro m = mk(g[0], U2_PASS, RG_A, DS_A, true);
      m.opr = true;
      table[b + 0x0A] = entry(AM_ACC, 2, false, false, false, m);
    }
  }
  // undocumented RMW combinations (unit1 on memory, unit2 into A)
  const uint32_t urmw[6][4] = {{U1_ASL, U2_OR, 0x00, DS_A}, {U1_ROL, U2_AND, 0x20, DS_A},
                               {U1_LSR, U2_EOR, 0x40, DS_A}, {U1_ROR, U2_ADC, 0x60, DS_A},
                               {U1_DEC, U2_CMP, 0xC0, DS_NONE}, {U1_INC, U2_SBC, 0xE0, DS_A}};
  for (auto& g : urmw) {
    uint32_t b = g[2];
    group(mk(g[0], g[1], RG_A, g[3], true), CL_RMW,
          {{AM_INDX, b + 0x03}, {AM_ZP, b + 0x07}, {AM_ABS, b + 0x0F}, {AM_INDY, b + 0x13},
           {AM_ZPX, b + 0x17}, {AM_ABSY, b + 0x1B}, {AM_ABSX, b + 0x1F}});
  }
  // NOPs (the reading forms perform their data read)
  Micro nop;
  for (uint32_t o : {0xEAu, 0x1Au, 0x3Au, 0x5Au, 0x7Au, 0xDAu, 0xFAu}) table[o] = entry(AM_IMP, 2, false, false, false, nop);
  group(nop, CL_READ, {{AM_IMM, 0x80}, {AM_IMM, 0x82}, {AM_IMM, 0x89}, {AM_IMM, 0xC2}, {AM_IMM, 0xE2},
                       {AM_ZP, 0x04}, {AM_ZP, 0x44}, {AM_ZP, 0x64}, {AM_ABS, 0x0C},
                       {AM_ZPX, 0x14}, {AM_ZPX, 0x34}, {AM_ZPX, 0x54}, {AM_ZPX, 0x74}, {AM_ZPX, 0xD4},
                       {AM_ZPX, 0xF4}, {AM_ABSX, 0x1C}, {AM_ABSX, 0x3C}, {AM_ABSX, 0x5C},
                       {AM_ABSX, 0x7C}, {AM_ABSX, 0xDC}, {AM_ABSX, 0xFC}});
  // register increments / transfers: M = R
  auto reg = [&](uint32_t opc, uint32_t u1, uint32_t rsrc, uint32_t dst, bool nz) {
    Micro m = mk(u1, U2_PASS, rsrc, dst, nz);
    m.opr = true;
    table[opc] = entry(AM_IMP, 2, false, false, false, m);
  };
  reg(0xE8, U1_INC, RG_X, DS_X, true);   // INX
  reg(0xC8, U1_INC, RG_Y, DS_Y, true);   // INY
  reg(0xCA, U1_DEC, RG_X, DS_X, true);   // DEX
  reg(0x88, U1_DEC, RG_Y, DS_Y, true);   // DEY
  reg(0xAA, U1_PASS, RG_A, DS_X, true);  // TAX
  reg(0xA8, U1_PASS, RG_A, DS_Y, true);  // TAY
  reg(0x8A, U1_PASS, RG_X, DS_A, true);  // TXA
  reg(0x98, U1_PASS, RG_Y, DS_A, true);  // TYA
  reg(0xBA, U1_PASS, RG_SP, DS_X, true); // TSX
  reg(0x9A, U1_PASS, RG_X, DS_SP, false);// TXS
  // flag set/clear: (opcode, flag index C=0 I=1 D=2 V=3, value)
  const uint32_t fl[7][3] = {{0x18, 0, 0}, {0x38, 0, 1}, {0x58, 1, 0}, {0x78, 1, 1},
                             {0xB8, 3, 0}, {0xD8, 2, 0}, {0xF8, 2, 1}};
  for (auto& f : fl)
    table[f[0]] = entry(AM_IMP, 2, false, false, false, nop) | (1ull << dk::FOP) |
                  ((uint64_t)f[1] << dk::FIDX) | ((uint64_t)f[2] << dk::FVAL);
  // control flow
  table[0x4C] = entry(AM_ABS, 3, false, false, false, nop) | (1ull << dk::JMP);
  table[0x6C] = entry(AM_IND, 5, false, false, false, nop) | (1ull << dk::JMP);
  const uint32_t br[8][3] = {{0x10, 0, 0}, {0x30, 0, 1}, {0x50, 1, 0}, {0x70, 1, 1},
                             {0x90, 2, 0}, {0xB0, 2, 1}, {0xD0, 3, 0}, {0xF0, 3, 1}};
  for (auto& b : br)
    table[b[0]] = entry(AM_REL, 2, false, false, false, nop) | (1ull << dk::BR) |
                  ((uint64_t)b[1] << dk::BRF) | ((uint64_t)b[2] << dk::BRT);
  // specials: stack/control and the immediate-only undocumented ops
  auto spc = [&](uint32_t opc, uint32_t mode, uint32_t cyc, uint32_t s) {
    table[opc] = entry(mode, cyc, false, false, false, nop) | ((uint64_t)s << dk::SPC);
  };
  spc(0x48, AM_IMP, 3, SP_PHA);
  spc(0x08, AM_IMP, 3, SP_PHP);
  spc(0x68, AM_IMP, 4, SP_PLA);
  spc(0x28, AM_IMP, 4, SP_PLP);
  spc(0x20, AM_ABS, 6, SP_JSR);
  spc(0x60, AM_IMP, 6, SP_RTS);
  spc(0x40, AM_IMP, 6, SP_RTI);
  spc(0x00, AM_IMP, 7, SP_BRK);
  spc(0x0B, AM_IMM, 2, SP_ANC);
  spc(0x2B, AM_IMM, 2, SP_ANC);
  spc(0x4B, AM_IMM, 2, SP_ALR);
  spc(0x6B, AM_IMM, 2, SP_ARR);
  spc(0xCB, AM_IMM, 2, SP_SBX);
}

}  // namespace cule
