// scalar_decode.h — host-side construction of the decode table of the scalar engine
// (one 64-bit entry per opcode, staged into shared memory once per block).
//
// The scalar engine runs one env per warp, so an instruction pays only for its own work.  Its
// entry therefore names an operation ("kind", one case of a small jump table) and carries the
// addressing-mode fields as single bits, so the effective address is computed branch-free
// and only the pointer modes branch.  Kinds that differ only in a register (LDA/LDX/LDY/LAX,
// STA/STX/STY/SAX, CMP/CPX/CPY, INX/INY/DEX/DEY, the transfers, flag set/clear, the eight
// branches) share one case and read that register from the AUX field, which keeps the jump
// table — and the instruction-cache footprint of the hot loop — small.  The index operand of
// indexed modes comes from a byte-permute selector stored in the entry (one instruction).
// Cycle counts come from the same addressing-mode x access-class rules as decode_table.h
// (SURVEY.md Appendix A), not from a per-opcode list.
#pragma once
#include <stdint.h>

#ifndef __CUDACC_RTC__  // host-only table builders (not compiled by NVRTC, jit.h)
#include <initializer_list>
#include <utility>
#endif

#include "decode_table.h"

namespace cule {

namespace sk {
// low word: bits 0-15 = byte selector for the index operand: __byte_perm(X | Y << 8, 0, lo)
// yields X, Y or 0 in one instruction (no selects); then single-bit flags
constexpr uint32_t SEL_NONE = 0x4444, SEL_X = 0x4440, SEL_Y = 0x4441;
constexpr uint32_t LEN = 16;        // 2 bits: instruction length 1..3
constexpr uint32_t CYC = 18;        // 4 bits: base cycles
constexpr uint32_t PEN = 1u << 22;  // +1 cycle on a page cross (reads through abs,X / abs,Y / (zp),Y)
constexpr uint32_t RD = 1u << 23;   // data read at EA (phase C)
constexpr uint32_t WR = 1u << 24;   // data write at EA (phase C)
constexpr uint32_t ZP = 1u << 25;   // zero page: EA (or, with PTRZ, the pointer address) wraps at 8 bits
constexpr uint32_t PTRZ = 1u << 26; // pointer read from zero page ((zp,X): index before, (zp),Y: after)
constexpr uint32_t PTRA = 1u << 27; // pointer read with the page-wrap bug (JMP (abs))
constexpr uint32_t ACC = 1u << 28;  // operand = A (accumulator shifts)
constexpr uint32_t PLAIN = 1u << 29;// plain absolute read of an idempotent kind (idle-loop head)
// high word
constexpr uint32_t KIND = 0;        // 8 bits
constexpr uint32_t AUX = 8;         // 7 bits, kind-specific
}  // namespace sk

enum Kind : uint32_t {
  K_JAM = 0, K_NOP, K_ORA, K_AND, K_EOR, K_ADC, K_SBC, K_CMP, K_BIT, K_LD, K_ST,
  K_ASL, K_LSR, K_ROL, K_ROR, K_INC, K_DEC, K_SLO, K_RLA, K_SRE, K_RRA, K_DCP, K_ISB,
  K_INR, K_TR, K_FLAG, K_BR, K_JMP, K_JSR, K_RTS, K_RTI, K_BRK, K_PHA, K_PHP, K_PLA, K_PLP,
  K_ANC, K_ALR, K_ARR, K_SBX, K_ASLA, K_LSRA, K_ROLA, K_RORA, K_COUNT
};
// AUX encodings
//   K_CMP: register 0 A, 1 X, 2 Y          K_LD: destination bits 1 A, 2 X, 4 Y
//   K_ST : source 0 A, 1 X, 2 Y, 3 A&X     K_INR: bit0 0 X / 1 Y, bit1 decrement
//   K_TR : source (bits 0-1) and destination (bits 2-3) 0 A 1 X 2 Y 3 SP; bit 4 set N,Z
//   K_FLAG: flag (bits 0-1) 0 C 1 I 2 D 3 V, bit 2 value
//   K_BR : flag (bits 0-1) 0 N 1 V 2 C 3 Z, bit 2 taken when set

inline uint32_t s_mode_bits(uint32_t mode) {
  switch (mode) {
    case AM_ZP: return sk::ZP | sk::SEL_NONE;
    case AM_ZPX: return sk::ZP | sk::SEL_X;
    case AM_ZPY: return sk::ZP | sk::SEL_Y;
    case AM_ABSX: return sk::SEL_X;
    case AM_ABSY: return sk::SEL_Y;
    case AM_IND: return sk::PTRA | sk::SEL_NONE;
    case AM_INDX: return sk::PTRZ | sk::ZP | sk::SEL_X;
    case AM_INDY: return sk::PTRZ | sk::SEL_Y;
    default: return sk::SEL_NONE;
  }
}

inline uint64_t s_entry(uint32_t mode, uint32_t cyc, bool pen, bool rd, bool wr, uint32_t kind, uint32_t aux) {
  uint32_t lo = s_mode_bits(mode) | (mode_len(mode) << sk::LEN) | (cyc << sk::CYC);
  if (pen) lo |= sk::PEN;
  if (rd) lo |= sk::RD;
  if (wr) lo |= sk::WR;
  if (mode == AM_ACC) lo |= sk::ACC;
  if (mode == AM_ABS && rd && !wr && (kind == K_LD || kind == K_BIT || kind == K_CMP || kind == K_NOP)) lo |= sk::PLAIN;
  const uint32_t hi = (kind << sk::KIND) | (aux << sk::AUX);
  return (uint64_t)lo | ((uint64_t)hi << 32);
}

#ifndef __CUDACC_RTC__
inline void build_scalar_table(uint64_t* t) {
  // JAM and the unstable opcodes: 1-byte fetch, 0 cycles, fault (DESIGN.md §2 R#1)
  for (int i = 0; i < 256; i++) t[i] = s_entry(AM_IMP, 0, false, false, false, K_JAM, 0);
  auto group = [&](uint32_t kind, uint32_t aux, AccessClass cl,
                   std::initializer_list<std::pair<uint32_t, uint32_t>> ms) {
    for (auto& p : ms) {
      bool pen;
      const uint32_t cyc = mode_cycles(p.first, cl, &pen);
      const bool rd = (cl == CL_READ && p.first != AM_IMM) || cl == CL_RMW;
      t[p.second] = s_entry(p.first, cyc, pen, rd, cl != CL_READ, kind, aux);
    }
  };
  auto all8 = [&](uint32_t kind, uint32_t aux, uint32_t b) {
    group(kind, aux, CL_READ, {{AM_INDX, b + 0x01}, {AM_ZP, b + 0x05}, {AM_IMM, b + 0x09}, {AM_ABS, b + 0x0D},
                               {AM_INDY, b + 0x11}, {AM_ZPX, b + 0x15}, {AM_ABSY, b + 0x19}, {AM_ABSX, b + 0x1D}});
  };
  all8(K_ORA, 0, 0x00);
  all8(K_AND, 0, 0x20);
  all8(K_EOR, 0, 0x40);
  all8(K_ADC, 0, 0x60);
  all8(K_LD, 1, 0xA0);
  all8(K_CMP, 0, 0xC0);
  all8(K_SBC, 0, 0xE0);
  group(K_SBC, 0, CL_READ, {{AM_IMM, 0xEB}});
  group(K_ST, 0, CL_WRITE, {{AM_INDX, 0x81}, {AM_ZP, 0x85}, {AM_ABS, 0x8D}, {AM_INDY, 0x91},
                            {AM_ZPX, 0x95}, {AM_ABSY, 0x99}, {AM_ABSX, 0x9D}});
  group(K_ST, 1, CL_WRITE, {{AM_ZP, 0x86}, {AM_ABS, 0x8E}, {AM_ZPY, 0x96}});
  group(K_ST, 2, CL_WRITE, {{AM_ZP, 0x84}, {AM_ABS, 0x8C}, {AM_ZPX, 0x94}});
  group(K_ST, 3, CL_WRITE, {{AM_INDX, 0x83}, {AM_ZP, 0x87}, {AM_ABS, 0x8F}, {AM_ZPY, 0x97}});
  group(K_LD, 2, CL_READ, {{AM_IMM, 0xA2}, {AM_ZP, 0xA6}, {AM_ABS, 0xAE}, {AM_ZPY, 0xB6}, {AM_ABSY, 0xBE}});
  group(K_LD, 4, CL_READ, {{AM_IMM, 0xA0}, {AM_ZP, 0xA4}, {AM_ABS, 0xAC}, {AM_ZPX, 0xB4}, {AM_ABSX, 0xBC}});
  group(K_LD, 3, CL_READ, {{AM_INDX, 0xA3}, {AM_ZP, 0xA7}, {AM_ABS, 0xAF}, {AM_INDY, 0xB3}, {AM_ZPY, 0xB7},
                           {AM_ABSY, 0xBF}});
  group(K_CMP, 1, CL_READ, {{AM_IMM, 0xE0}, {AM_ZP, 0xE4}, {AM_ABS, 0xEC}});
  group(K_CMP, 2, CL_READ, {{AM_IMM, 0xC0}, {AM_ZP, 0xC4}, {AM_ABS, 0xCC}});
  group(K_BIT, 0, CL_READ, {{AM_ZP, 0x24}, {AM_ABS, 0x2C}});
  const uint32_t rmw[6][2] = {{K_ASL, 0x00}, {K_ROL, 0x20}, {K_LSR, 0x40}, {K_ROR, 0x60}, {K_DEC, 0xC0}, {K_INC, 0xE0}};
  for (auto& g : rmw) {
    const uint32_t b = g[1];
    group(g[0], 0, CL_RMW, {{AM_ZP, b + 0x06}, {AM_ABS, b + 0x0E}, {AM_ZPX, b + 0x16}, {AM_ABSX, b + 0x1E}});
    if (g[0] != K_DEC && g[0] != K_INC)
      t[b + 0x0A] = s_entry(AM_ACC, 2, false, false, false, g[0] - K_ASL + K_ASLA, 0);
  }
  const uint32_t urmw[6][2] = {{K_SLO, 0x00}, {K_RLA, 0x20}, {K_SRE, 0x40}, {K_RRA, 0x60}, {K_DCP, 0xC0}, {K_ISB, 0xE0}};
  for (auto& g : urmw) {
    const uint32_t b = g[1];
    group(g[0], 0, CL_RMW, {{AM_INDX, b + 0x03}, {AM_ZP, b + 0x07}, {AM_ABS, b + 0x0F}, {AM_INDY, b + 0x13},
                            {AM_ZPX, b + 0x17}, {AM_ABSY, b + 0x1B}, {AM_ABSX, b + 0x1F}});
  }
  for (uint32_t o : {0xEAu, 0x1Au, 0x3Au, 0x5Au, 0x7Au, 0xDAu, 0xFAu}) t[o] = s_entry(AM_IMP, 2, false, false, false, K_NOP, 0);
  group(K_NOP, 0, CL_READ, {{AM_IMM, 0x80}, {AM_IMM, 0x82}, {AM_IMM, 0x89}, {AM_IMM, 0xC2}, {AM_IMM, 0xE2},
                            {AM_ZP, 0x04}, {AM_ZP, 0x44}, {AM_ZP, 0x64}, {AM_ABS, 0x0C},
                            {AM_ZPX, 0x14}, {AM_ZPX, 0x34}, {AM_ZPX, 0x54}, {AM_ZPX, 0x74}, {AM_ZPX, 0xD4},
                            {AM_ZPX, 0xF4}, {AM_ABSX, 0x1C}, {AM_ABSX, 0x3C}, {AM_ABSX, 0x5C},
                            {AM_ABSX, 0x7C}, {AM_ABSX, 0xDC}, {AM_ABSX, 0xFC}});
  auto imp = [&](uint32_t opc, uint32_t cyc, uint32_t kind, uint32_t aux) {
    t[opc] = s_entry(AM_IMP, cyc, false, false, false, kind, aux);
  };
  imp(0xE8, 2, K_INR, 0);  // INX
  imp(0xC8, 2, K_INR, 1);  // INY
  imp(0xCA, 2, K_INR, 2);  // DEX
  imp(0x88, 2, K_INR, 3);  // DEY
  auto tr = [](uint32_t src, uint32_t dst, bool nz) { return src | (dst << 2) | (nz ? 16u : 0u); };
  imp(0xAA, 2, K_TR, tr(0, 1, true));   // TAX
  imp(0xA8, 2, K_TR, tr(0, 2, true));   // TAY
  imp(0x8A, 2, K_TR, tr(1, 0, true));   // TXA
  imp(0x98, 2, K_TR, tr(2, 0, true));   // TYA
  imp(0xBA, 2, K_TR, tr(3, 1, true));   // TSX
  imp(0x9A, 2, K_TR, tr(1, 3, false));  // TXS
  const uint32_t fl[7][3] = {{0x18, 0, 0}, {0x38, 0, 1}, {0x58, 1, 0}, {0x78, 1, 1},
                             {0xB8, 3, 0}, {0xD8, 2, 0}, {0xF8, 2, 1}};
  for (auto& f : fl) imp(f[0], 2, K_FLAG, f[1] | (f[2] << 2));
  const uint32_t br[8][3] = {{0x10, 0, 0}, {0x30, 0, 1}, {0x50, 1, 0}, {0x70, 1, 1},
                             {0x90, 2, 0}, {0xB0, 2, 1}, {0xD0, 3, 0}, {0xF0, 3, 1}};
  for (auto& b : br) t[b[0]] = s_entry(AM_REL, 2, false, false, false, K_BR, b[1] | (b[2] << 2));
  t[0x4C] = s_entry(AM_ABS, 3, false, false, false, K_JMP, 0);
  t[0x6C] = s_entry(AM_IND, 5, false, false, false, K_JMP, 0);
  t[0x20] = s_entry(AM_ABS, 6, false, false, false, K_JSR, 0);
  imp(0x60, 6, K_RTS, 0);
  imp(0x40, 6, K_RTI, 0);
  imp(0x00, 7, K_BRK, 0);
  imp(0x48, 3, K_PHA, 0);
  imp(0x08, 3, K_PHP, 0);
  imp(0x68, 4, K_PLA, 0);
  imp(0x28, 4, K_PLP, 0);
  t[0x0B] = s_entry(AM_IMM, 2, false, false, false, K_ANC, 0);
  t[0x2B] = s_entry(AM_IMM, 2, false, false, false, K_ANC, 0);
  t[0x4B] = s_entry(AM_IMM, 2, false, false, false, K_ALR, 0);
  t[0x6B] = s_entry(AM_IMM, 2, false, false, false, K_ARR, 0);
  t[0xCB] = s_entry(AM_IMM, 2, false, false, false, K_SBX, 0);
}
#endif  // __CUDACC_RTC__

}  // namespace cule
