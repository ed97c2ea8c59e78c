// decode_table.h — host-side construction of the 6502 micro-coded decode table used by the
// step kernel (one 64-bit entry per opcode, staged into shared memory once per block).
// Product code; independent of the oracle (which executes a per-opcode switch).
//
// The kernel runs every ordinary instruction through ONE branch-free datapath:
//   R  = register operand (A/X/Y/SP);  M = memory/immediate byte, or R for implied forms
//   r1 = unit1(M): pass | shift left | shift right (rotate: carry in) | +1 | -1   (carry c1)
//   r2 = unit2(r1): pass | OR | AND | EOR | adder (ADC, SBC, CMP share it) | BIT
//   then destination register(s), memory write value, N/Z/C/V updates.
// Every control field is a one-hot flag bit, so each select compiles to a single predicate
// test + SEL/LOP3 (multi-bit codes make the compiler emit compare-and-branch trees).
// Stack/control and the rare undocumented immediates take a small "special" switch.
//
// Cycle counts derive from the addressing-mode x access-class rules of the NMOS 6502
// (bottom table), not from a per-opcode list.
#pragma once
#include <stdint.h>

#ifndef __CUDACC_RTC__  // host-only table builders (not compiled by NVRTC, jit.h)
#include <initializer_list>
#include <utility>
#endif

namespace cule {

enum AddrMode : uint32_t {
  AM_IMP = 0, AM_ACC, AM_IMM, AM_ZP, AM_ZPX, AM_ZPY, AM_ABS, AM_ABSX, AM_ABSY, AM_IND,
  AM_INDX, AM_INDY, AM_REL
};
enum Special : uint32_t {
  SP_NONE = 0, SP_PHA, SP_PHP, SP_PLA, SP_PLP, SP_JSR, SP_RTS, SP_RTI, SP_BRK, SP_ANC, SP_ALR,
  SP_ARR, SP_SBX, SP_JAM
};

// ---- bit layout of an entry: low word (front end + unit1), high word (unit2 + write-back) ----
namespace dk {
// low 32 bits
constexpr uint32_t LEN = 0;      // 2 bits: instruction length 1..3
constexpr uint32_t CYC = 2;      // 4 bits: base cycles
constexpr uint32_t PEN = 1u << 6;   // +1 cycle on a page cross
constexpr uint32_t RD = 1u << 7;    // data read at EA (phase C)
constexpr uint32_t WR = 1u << 8;    // data write at EA (phase C)
constexpr uint32_t ZP = 1u << 9;    // EA = zero-page address (zp, zp,X, zp,Y)
constexpr uint32_t ZIX = 1u << 10;  // zero-page index X (zp,X and (zp,X))
constexpr uint32_t ZIY = 1u << 11;  // zero-page index Y (zp,Y)
constexpr uint32_t AIX = 1u << 12;  // 16-bit index X (abs,X)
constexpr uint32_t AIY = 1u << 13;  // 16-bit index Y (abs,Y and (zp),Y)
constexpr uint32_t PTRZ = 1u << 14; // pointer read from zero page ((zp,X), (zp),Y)
constexpr uint32_t PTRA = 1u << 15; // pointer read with the page-wrap bug (JMP (abs))
constexpr uint32_t BR = 1u << 16;   // conditional branch
constexpr uint32_t JMP = 1u << 17;  // PC <- EA
constexpr uint32_t RA = 1u << 18;   // register operand R = A
constexpr uint32_t RX = 1u << 19;   // R = X
constexpr uint32_t RY = 1u << 20;   // R = Y
constexpr uint32_t RS = 1u << 21;   // R = SP
constexpr uint32_t OPR = 1u << 22;  // M = R (implied / accumulator forms)
constexpr uint32_t SHL = 1u << 23;  // unit1 shift left (ASL, ROL)
constexpr uint32_t SHR = 1u << 24;  // unit1 shift right (LSR, ROR)
constexpr uint32_t ROT = 1u << 25;  // carry into the vacated bit (ROL, ROR)
constexpr uint32_t INC = 1u << 26;  // unit1 +1
constexpr uint32_t DEC = 1u << 27;  // unit1 -1
constexpr uint32_t NZ = 1u << 28;   // update N and Z
constexpr uint32_t WSEL = 1u << 29; // write value = store value (R, or A&X) instead of r1
constexpr uint32_t SAX = 1u << 30;  // store value A & X
constexpr uint32_t FOP = 1u << 31;  // flag set/clear
// high 32 bits
constexpr uint32_t OR = 1u << 0;
constexpr uint32_t AND = 1u << 1;
constexpr uint32_t EOR = 1u << 2;
constexpr uint32_t LOGIC = 1u << 3; // any of OR/AND/EOR
constexpr uint32_t ADDV = 1u << 4;  // ADC or SBC: adder result to A, carry and overflow
constexpr uint32_t INV = 1u << 5;   // adder operand inverted (SBC, CMP)
constexpr uint32_t CMP = 1u << 6;   // adder: R - M with carry-in 1, result only to flags
constexpr uint32_t BIT = 1u << 7;
constexpr uint32_t ARITH = 1u << 8; // ADC, SBC or CMP
constexpr uint32_t DA = 1u << 9;    // write r2 to A
constexpr uint32_t DX = 1u << 10;
constexpr uint32_t DY = 1u << 11;
constexpr uint32_t DS = 1u << 12;
constexpr uint32_t FIDX = 13;       // 2 bits: flag op target 0 C, 1 I, 2 D, 3 V
constexpr uint32_t FVAL = 1u << 15;
constexpr uint32_t SPC = 16;        // 4 bits: special op
constexpr uint32_t BRF = 20;        // 2 bits: branch flag 0 N, 1 V, 2 C, 3 Z
constexpr uint32_t BRT = 1u << 22;  // branch taken when the flag is set
}  // namespace dk

inline uint32_t mode_len(uint32_t mode) {
  switch (mode) {
    case AM_IMP: case AM_ACC: return 1;
    case AM_ABS: case AM_ABSX: case AM_ABSY: case AM_IND: return 3;
    default: return 2;
  }
}

inline uint32_t mode_bits(uint32_t mode) {
  switch (mode) {
    case AM_ZP: return dk::ZP;
    case AM_ZPX: return dk::ZP | dk::ZIX;
    case AM_ZPY: return dk::ZP | dk::ZIY;
    case AM_ABSX: return dk::AIX;
    case AM_ABSY: return dk::AIY;
    case AM_IND: return dk::PTRA;
    case AM_INDX: return dk::PTRZ | dk::ZIX;
    case AM_INDY: return dk::PTRZ | dk::AIY;
    default: return 0;
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

// datapath fields of one operation (independent of the addressing mode)
struct Micro {
  uint32_t lo = 0;  // register operand / unit1 / NZ / write-value bits
  uint32_t hi = 0;  // unit2 / destination bits
};

inline uint64_t entry(uint32_t mode, uint32_t cyc, bool pen, bool rd, bool wr, const Micro& u) {
  uint32_t lo = u.lo | mode_bits(mode) | (mode_len(mode) << dk::LEN) | (cyc << dk::CYC);
  if (pen) lo |= dk::PEN;
  if (rd) lo |= dk::RD;
  if (wr) lo |= dk::WR;
  return (uint64_t)lo | ((uint64_t)u.hi << 32);
}

#ifndef __CUDACC_RTC__
inline void build_decode_table(uint64_t* table) {
  using namespace dk;
  Micro nop;
  // JAM / unstable: the opcode fetch happens (1 byte), then the env faults with fc unchanged
  for (int i = 0; i < 256; i++) table[i] = entry(AM_IMP, 0, false, false, false, nop) | ((uint64_t)SP_JAM << (32 + SPC));
  auto group = [&](const Micro& u, AccessClass cl, std::initializer_list<std::pair<uint32_t, uint32_t>> ms) {
    for (auto& p : ms) {
      bool pen;
      uint32_t cyc = mode_cycles(p.first, cl, &pen);
      bool rd = (cl == CL_READ && p.first != AM_IMM) || cl == CL_RMW;
      bool wr = cl != CL_READ;
      table[p.second] = entry(p.first, cyc, pen, rd, wr, u);
    }
  };
  auto mk = [](uint32_t lo, uint32_t hi) {
    Micro m;
    m.lo = lo;
    m.hi = hi;
    return m;
  };
  const uint32_t adc = ADDV | ARITH, sbc = ADDV | INV | ARITH, cmp = CMP | INV | ARITH;
  // eight-mode ALU group aaa bbb 01: ORA AND EOR ADC LDA CMP SBC
  const uint32_t alu8[7][2] = {{OR | LOGIC | DA, 0x00}, {AND | LOGIC | DA, 0x20}, {EOR | LOGIC | DA, 0x40},
                               {adc | DA, 0x60}, {DA, 0xA0}, {cmp, 0xC0}, {sbc | DA, 0xE0}};
  for (auto& g : alu8) {
    uint32_t b = g[1];
    group(mk(RA | NZ, g[0]), CL_READ,
          {{AM_INDX, b + 0x01}, {AM_ZP, b + 0x05}, {AM_IMM, b + 0x09}, {AM_ABS, b + 0x0D},
           {AM_INDY, b + 0x11}, {AM_ZPX, b + 0x15}, {AM_ABSY, b + 0x19}, {AM_ABSX, b + 0x1D}});
  }
  group(mk(RA | NZ, sbc | DA), CL_READ, {{AM_IMM, 0xEB}});
  group(mk(RA | WSEL, 0), CL_WRITE, {{AM_INDX, 0x81}, {AM_ZP, 0x85}, {AM_ABS, 0x8D}, {AM_INDY, 0x91},
                                     {AM_ZPX, 0x95}, {AM_ABSY, 0x99}, {AM_ABSX, 0x9D}});
  group(mk(RX | WSEL, 0), CL_WRITE, {{AM_ZP, 0x86}, {AM_ABS, 0x8E}, {AM_ZPY, 0x96}});
  group(mk(RY | WSEL, 0), CL_WRITE, {{AM_ZP, 0x84}, {AM_ABS, 0x8C}, {AM_ZPX, 0x94}});
  group(mk(RA | WSEL | SAX, 0), CL_WRITE, {{AM_INDX, 0x83}, {AM_ZP, 0x87}, {AM_ABS, 0x8F}, {AM_ZPY, 0x97}});
  group(mk(NZ, DX), CL_READ, {{AM_IMM, 0xA2}, {AM_ZP, 0xA6}, {AM_ABS, 0xAE}, {AM_ZPY, 0xB6}, {AM_ABSY, 0xBE}});
  group(mk(NZ, DY), CL_READ, {{AM_IMM, 0xA0}, {AM_ZP, 0xA4}, {AM_ABS, 0xAC}, {AM_ZPX, 0xB4}, {AM_ABSX, 0xBC}});
  group(mk(NZ, DA | DX), CL_READ,
        {{AM_INDX, 0xA3}, {AM_ZP, 0xA7}, {AM_ABS, 0xAF}, {AM_INDY, 0xB3}, {AM_ZPY, 0xB7}, {AM_ABSY, 0xBF}});
  group(mk(RX | NZ, cmp), CL_READ, {{AM_IMM, 0xE0}, {AM_ZP, 0xE4}, {AM_ABS, 0xEC}});
  group(mk(RY | NZ, cmp), CL_READ, {{AM_IMM, 0xC0}, {AM_ZP, 0xC4}, {AM_ABS, 0xCC}});
  group(mk(RA | NZ, BIT), CL_READ, {{AM_ZP, 0x24}, {AM_ABS, 0x2C}});
  // shifts / rotates / inc / dec on memory, and the accumulator forms
  const uint32_t rmw[6][2] = {{SHL, 0x00}, {SHL | ROT, 0x20}, {SHR, 0x40}, {SHR | ROT, 0x60},
                              {DEC, 0xC0}, {INC, 0xE0}};
  for (auto& g : rmw) {
    uint32_t b = g[1];
    group(mk(g[0] | NZ, 0), CL_RMW, {{AM_ZP, b + 0x06}, {AM_ABS, b + 0x0E}, {AM_ZPX, b + 0x16}, {AM_ABSX, b + 0x1E}});
    if (!(g[0] & (INC | DEC))) table[b + 0x0A] = entry(AM_ACC, 2, false, false, false, mk(g[0] | RA | OPR | NZ, DA));
  }
  // undocumented RMW combinations: unit1 on memory, unit2 into A (DCP compares)
  const uint32_t urmw[6][3] = {{SHL, OR | LOGIC | DA, 0x00}, {SHL | ROT, AND | LOGIC | DA, 0x20},
                               {SHR, EOR | LOGIC | DA, 0x40}, {SHR | ROT, adc | DA, 0x60},
                               {DEC, cmp, 0xC0}, {INC, sbc | DA, 0xE0}};
  for (auto& g : urmw) {
    uint32_t b = g[2];
    group(mk(g[0] | RA | NZ, g[1]), CL_RMW,
          {{AM_INDX, b + 0x03}, {AM_ZP, b + 0x07}, {AM_ABS, b + 0x0F}, {AM_INDY, b + 0x13},
           {AM_ZPX, b + 0x17}, {AM_ABSY, b + 0x1B}, {AM_ABSX, b + 0x1F}});
  }
  // NOPs (the reading forms perform their data read)
  for (uint32_t o : {0xEAu, 0x1Au, 0x3Au, 0x5Au, 0x7Au, 0xDAu, 0xFAu}) table[o] = entry(AM_IMP, 2, false, false, false, nop);
  group(nop, CL_READ, {{AM_IMM, 0x80}, {AM_IMM, 0x82}, {AM_IMM, 0x89}, {AM_IMM, 0xC2}, {AM_IMM, 0xE2},
                       {AM_ZP, 0x04}, {AM_ZP, 0x44}, {AM_ZP, 0x64}, {AM_ABS, 0x0C},
                       {AM_ZPX, 0x14}, {AM_ZPX, 0x34}, {AM_ZPX, 0x54}, {AM_ZPX, 0x74}, {AM_ZPX, 0xD4},
                       {AM_ZPX, 0xF4}, {AM_ABSX, 0x1C}, {AM_ABSX, 0x3C}, {AM_ABSX, 0x5C},
                       {AM_ABSX, 0x7C}, {AM_ABSX, 0xDC}, {AM_ABSX, 0xFC}});
  // register increments / transfers: M = R
  auto reg = [&](uint32_t opc, uint32_t lo, uint32_t hi) {
    table[opc] = entry(AM_IMP, 2, false, false, false, mk(lo | OPR, hi));
  };
  reg(0xE8, RX | INC | NZ, DX);  // INX
  reg(0xC8, RY | INC | NZ, DY);  // INY
  reg(0xCA, RX | DEC | NZ, DX);  // DEX
  reg(0x88, RY | DEC | NZ, DY);  // DEY
  reg(0xAA, RA | NZ, DX);        // TAX
  reg(0xA8, RA | NZ, DY);        // TAY
  reg(0x8A, RX | NZ, DA);        // TXA
  reg(0x98, RY | NZ, DA);        // TYA
  reg(0xBA, RS | NZ, DX);        // TSX
  reg(0x9A, RX, DS);             // TXS
  // flag set/clear: (opcode, flag index C=0 I=1 D=2 V=3, value)
  const uint32_t fl[7][3] = {{0x18, 0, 0}, {0x38, 0, 1}, {0x58, 1, 0}, {0x78, 1, 1},
                             {0xB8, 3, 0}, {0xD8, 2, 0}, {0xF8, 2, 1}};
  for (auto& f : fl)
    table[f[0]] = entry(AM_IMP, 2, false, false, false, mk(FOP, (f[1] << FIDX) | (f[2] ? FVAL : 0u)));
  // control flow
  table[0x4C] = entry(AM_ABS, 3, false, false, false, mk(JMP, 0));
  table[0x6C] = entry(AM_IND, 5, false, false, false, mk(JMP, 0));
  const uint32_t br[8][3] = {{0x10, 0, 0}, {0x30, 0, 1}, {0x50, 1, 0}, {0x70, 1, 1},
                             {0x90, 2, 0}, {0xB0, 2, 1}, {0xD0, 3, 0}, {0xF0, 3, 1}};
  for (auto& b : br)
    table[b[0]] = entry(AM_REL, 2, false, false, false, mk(BR, (b[1] << BRF) | (b[2] ? BRT : 0u)));
  // specials: stack/control and the immediate-only undocumented ops
  auto spc = [&](uint32_t opc, uint32_t mode, uint32_t cyc, uint32_t s) {
    table[opc] = entry(mode, cyc, false, false, false, nop) | ((uint64_t)s << (32 + SPC));
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
#endif  // __CUDACC_RTC__

}  // namespace cule
