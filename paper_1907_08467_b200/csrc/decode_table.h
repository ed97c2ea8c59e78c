// decode_table.h — host-side construction of the 6502 decode/cycle table used by the step
// kernel (staged into shared memory once per block).  Product code; independent of the oracle.
//
// Entry layout (u32):
//   bits 0-3   addressing mode (AM_*)
//   bits 4-10  operation (OP_*)
//   bits 11-14 base cycle count
//   bit  15    +1 cycle when the effective address crosses a page (read-class abs,X/abs,Y/(zp),Y)
//   bit  16    the operation reads its operand from memory (phase-C data read)
//   bits 17-18 branch flag selector (0 N, 1 V, 2 C, 3 Z), bit 19 = branch taken when flag set
//
// Cycle counts are derived from the addressing-mode / access-class rules of the NMOS 6502
// (bottom table), not copied per opcode.
#pragma once
#include <stdint.h>

#include <initializer_list>
#include <utility>

namespace cule {

enum AddrMode : uint32_t {
  AM_IMP = 0, AM_ACC, AM_IMM, AM_ZP, AM_ZPX, AM_ZPY, AM_ABS, AM_ABSX, AM_ABSY, AM_IND,
  AM_INDX, AM_INDY, AM_REL
};

enum Op : uint32_t {
  OP_JAM = 0,
  OP_LDA, OP_LDX, OP_LDY, OP_LAX,
  OP_STA, OP_STX, OP_STY, OP_SAX,
  OP_ORA, OP_AND, OP_EOR, OP_ADC, OP_SBC, OP_CMP, OP_CPX, OP_CPY, OP_BIT,
  OP_ASL, OP_LSR, OP_ROL, OP_ROR, OP_INC, OP_DEC,
  OP_SLO, OP_RLA, OP_SRE, OP_RRA, OP_DCP, OP_ISB,
  OP_ANC, OP_ALR, OP_ARR, OP_SBX,
  OP_NOP,
  OP_INX, OP_INY, OP_DEX, OP_DEY, OP_TAX, OP_TAY, OP_TXA, OP_TYA, OP_TSX, OP_TXS,
  OP_CLC, OP_SEC, OP_CLI, OP_SEI, OP_CLV, OP_CLD, OP_SED,
  OP_PHA, OP_PHP, OP_PLA, OP_PLP,
  OP_JMP, OP_JSR, OP_RTS, OP_RTI, OP_BRK,
  OP_BRANCH,
  OP_COUNT
};

enum AccessClass { CL_READ, CL_WRITE, CL_RMW, CL_FIXED };

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

struct OpModes { uint32_t op; AccessClass cl; struct { uint32_t mode; uint8_t opc; } m[8]; int n; };

inline void build_decode_table(uint32_t* table) {
  for (int i = 0; i < 256; i++) table[i] = OP_JAM << 4; /* JAM and unstable opcodes fault */
  auto put = [&](uint32_t opc, uint32_t mode, uint32_t op, uint32_t cyc, bool pen, bool rd) {
    table[opc] = mode | (op << 4) | (cyc << 11) | ((pen ? 1u : 0u) << 15) | ((rd ? 1u : 0u) << 16);
  };
  auto group = [&](uint32_t op, AccessClass cl, std::initializer_list<std::pair<uint32_t, uint32_t>> ms) {
    for (auto& p : ms) {
      bool pen;
      uint32_t cyc = mode_cycles(p.first, cl, &pen);
      bool rd = (cl == CL_READ && p.first != AM_IMM) || cl == CL_RMW;
      put(p.second, p.first, op, cyc, pen, rd);
    }
  };
  // the eight-mode ALU group (ORA AND EOR ADC LDA CMP SBC): aaa bbb 01
  const uint32_t alu8[7][2] = {{OP_ORA, 0x00}, {OP_AND, 0x20}, {OP_EOR, 0x40}, {OP_ADC, 0x60},
                               {OP_LDA, 0xA0}, {OP_CMP, 0xC0}, {OP_SBC, 0xE0}};
  for (auto& g : alu8) {
    uint32_t b = g[1];
    group(g[0], CL_READ, {{AM_INDX, b + 0x01}, {AM_ZP, b + 0x05}, {AM_IMM, b + 0x09},
                          {AM_ABS, b + 0x0D}, {AM_INDY, b + 0x11}, {AM_ZPX, b + 0x15},
                          {AM_ABSY, b + 0x19}, {AM_ABSX, b + 0x1D}});
  }
  group(OP_STA, CL_WRITE, {{AM_INDX, 0x81}, {AM_ZP, 0x85}, {AM_ABS, 0x8D}, {AM_INDY, 0x91},
                           {AM_ZPX, 0x95}, {AM_ABSY, 0x99}, {AM_ABSX, 0x9D}});
  group(OP_LDX, CL_READ, {{AM_IMM, 0xA2}, {AM_ZP, 0xA6}, {AM_ABS, 0xAE}, {AM_ZPY, 0xB6}, {AM_ABSY, 0xBE}});
  group(OP_LDY, CL_READ, {{AM_IMM, 0xA0}, {AM_ZP, 0xA4}, {AM_ABS, 0xAC}, {AM_ZPX, 0xB4}, {AM_ABSX, 0xBC}});
  group(OP_STX, CL_WRITE, {{AM_ZP, 0x86}, {AM_ABS, 0x8E}, {AM_ZPY, 0x96}});
  group(OP_STY, CL_WRITE, {{AM_ZP, 0x84}, {AM_ABS, 0x8C}, {AM_ZPX, 0x94}});
  group(OP_CPX, CL_READ, {{AM_IMM, 0xE0}, {AM_ZP, 0xE4}, {AM_ABS, 0xEC}});
  group(OP_CPY, CL_READ, {{AM_IMM, 0xC0}, {AM_ZP, 0xC4}, {AM_ABS, 0xCC}});
  group(OP_BIT, CL_READ, {{AM_ZP, 0x24}, {AM_ABS, 0x2C}});
  // shifts/rotates/inc/dec: aaa bbb 10
  const uint32_t rmw[6][2] = {{OP_ASL, 0x00}, {OP_ROL, 0x20}, {OP_LSR, 0x40}, {OP_ROR, 0x60},
                              {OP_DEC, 0xC0}, {OP_INC, 0xE0}};
  for (auto& g : rmw) {
    uint32_t b = g[1];
    group(g[0], CL_RMW, {{AM_ZP, b + 0x06}, {AM_ABS, b + 0x0E}, {AM_ZPX, b + 0x16}, {AM_ABSX, b + 0x1E}});
    if (g[0] != OP_DEC && g[0] != OP_INC) put(b + 0x0A, AM_ACC, g[0], 2, false, false);
  }
  // stable undocumented read-modify-write combinations: aaa bbb 11
  const uint32_t urmw[6][2] = {{OP_SLO, 0x00}, {OP_RLA, 0x20}, {OP_SRE, 0x40}, {OP_RRA, 0x60},
                               {OP_DCP, 0xC0}, {OP_ISB, 0xE0}};
  for (auto& g : urmw) {
    uint32_t b = g[1];
    group(g[0], CL_RMW, {{AM_INDX, b + 0x03}, {AM_ZP, b + 0x07}, {AM_ABS, b + 0x0F}, {AM_INDY, b + 0x13},
                         {AM_ZPX, b + 0x17}, {AM_ABSY, b + 0x1B}, {AM_ABSX, b + 0x1F}});
  }
  group(OP_LAX, CL_READ, {{AM_INDX, 0xA3}, {AM_ZP, 0xA7}, {AM_ABS, 0xAF}, {AM_INDY, 0xB3},
                          {AM_ZPY, 0xB7}, {AM_ABSY, 0xBF}});
  group(OP_SAX, CL_WRITE, {{AM_INDX, 0x83}, {AM_ZP, 0x87}, {AM_ABS, 0x8F}, {AM_ZPY, 0x97}});
  group(OP_ANC, CL_READ, {{AM_IMM, 0x0B}, {AM_IMM, 0x2B}});
  group(OP_ALR, CL_READ, {{AM_IMM, 0x4B}});
  group(OP_ARR, CL_READ, {{AM_IMM, 0x6B}});
  group(OP_SBX, CL_READ, {{AM_IMM, 0xCB}});
  group(OP_SBC, CL_READ, {{AM_IMM, 0xEB}});
  // NOPs: implied, and the reading NOPs (they perform their data read)
  for (uint32_t o : {0xEAu, 0x1Au, 0x3Au, 0x5Au, 0x7Au, 0xDAu, 0xFAu}) put(o, AM_IMP, OP_NOP, 2, false, false);
  group(OP_NOP, CL_READ, {{AM_IMM, 0x80}, {AM_IMM, 0x82}, {AM_IMM, 0x89}, {AM_IMM, 0xC2}, {AM_IMM, 0xE2}});
  group(OP_NOP, CL_READ, {{AM_ZP, 0x04}, {AM_ZP, 0x44}, {AM_ZP, 0x64}, {AM_ABS, 0x0C}});
  group(OP_NOP, CL_READ, {{AM_ZPX, 0x14}, {AM_ZPX, 0x34}, {AM_ZPX, 0x54}, {AM_ZPX, 0x74}, {AM_ZPX, 0xD4}, {AM_ZPX, 0xF4}});
  group(OP_NOP, CL_READ, {{AM_ABSX, 0x1C}, {AM_ABSX, 0x3C}, {AM_ABSX, 0x5C}, {AM_ABSX, 0x7C}, {AM_ABSX, 0xDC}, {AM_ABSX, 0xFC}});
  // implied register / flag operations
  const uint32_t impl[][2] = {{0xE8, OP_INX}, {0xC8, OP_INY}, {0xCA, OP_DEX}, {0x88, OP_DEY},
                              {0xAA, OP_TAX}, {0xA8, OP_TAY}, {0x8A, OP_TXA}, {0x98, OP_TYA},
                              {0xBA, OP_TSX}, {0x9A, OP_TXS}, {0x18, OP_CLC}, {0x38, OP_SEC},
                              {0x58, OP_CLI}, {0x78, OP_SEI}, {0xB8, OP_CLV}, {0xD8, OP_CLD},
                              {0xF8, OP_SED}};
  for (auto& e : impl) put(e[0], AM_IMP, e[1], 2, false, false);
  // stack and control flow: fixed counts
  put(0x48, AM_IMP, OP_PHA, 3, false, false);
  put(0x08, AM_IMP, OP_PHP, 3, false, false);
  put(0x68, AM_IMP, OP_PLA, 4, false, false);
  put(0x28, AM_IMP, OP_PLP, 4, false, false);
  put(0x4C, AM_ABS, OP_JMP, 3, false, false);
  put(0x6C, AM_IND, OP_JMP, 5, false, false);
  put(0x20, AM_ABS, OP_JSR, 6, false, false);
  put(0x60, AM_IMP, OP_RTS, 6, false, false);
  put(0x40, AM_IMP, OP_RTI, 6, false, false);
  put(0x00, AM_IMP, OP_BRK, 7, false, false);
  // branches: condition flag (N V C Z) in bits 17-18, taken-when-set in bit 19
  const uint32_t br[8][3] = {{0x10, 0, 0}, {0x30, 0, 1}, {0x50, 1, 0}, {0x70, 1, 1},
                             {0x90, 2, 0}, {0xB0, 2, 1}, {0xD0, 3, 0}, {0xF0, 3, 1}};
  for (auto& b : br) table[b[0]] = AM_REL | (OP_BRANCH << 4) | (2u << 11) | (b[1] << 17) | (b[2] << 19);
}

}  // namespace cule
