// scalar_predecode.h — host-side pre-decoding of the cartridge for the scalar engine's fast path.
//
// The ROM is constant (PAPER.md P:266-267 keeps it in constant memory for the same reason), so
// every byte offset of every 4 KB bank can be decoded once, at cule_create, as if an instruction
// started there.  One 8-byte record per ROM byte holds everything the interpreter needs to run
// that instruction without touching the decode table: the operation class (one case of the
// fast-path switch), base cycles, the fall-through PC, page-cross rule, register selector, the
// operand and the index selector — laid out so that the fields every instruction needs come out
// of the record in one or two integer operations.
//
// The class also folds in what the address alone decides: a direct (zero-page or absolute)
// operand is statically RAM, cartridge, TIA or RIOT, so the fast path never decodes the bus for
// it.  Anything the fast path does not cover — pointer modes, stack and interrupt operations,
// TIA reads (collision latches), bank-switch hotspots, fetches that cross the end of the 4 KB
// window, JAM — is class GEN and runs through the general interpreter (scalar_cpu.cuh), which
// implements the full machine model of DESIGN.md §2.  The records change no semantics: they are
// a cache of the decode of constant bytes.
#pragma once
#include <stdint.h>

#include "decode_table.h"
#include "scalar_decode.h"

namespace cule {

// TIA registers whose write is a pure store of the value (DESIGN.md §2 R#37): NUSIZ0 ... PF2
// (0x04-0x0F) and ENAM0 ... RESMP1 (0x1D-0x29); scalar_cpu.cuh shd_write, jit.h
constexpr uint64_t kTiaPure = (0xFFFull << 0x04) | (0x1FFFull << 0x1D);
// shadow entry of TIA register r in 0x04-0x0F / 0x1B-0x29 (0..26); 27-29 the VDEL copies GRP0
// old, GRP1 old, ENABL old; 32 u16 entries in all (scalar_cpu.cuh shd_write)
#if defined(__CUDACC__) || defined(__CUDACC_RTC__)
__host__ __device__
#endif
constexpr uint32_t shd_idx(uint32_t r) { return r <= 0x0Fu ? r - 0x04u : r - 0x1Bu + 12u; }
constexpr uint32_t kShdG0o = 27u, kShdG1o = 28u, kShdEbo = 29u, kShdEntries = 32u;

namespace pd {
// Record word lo: [0:5) class, [5:8) aux, [8:12) base cycles (C_BR: cycles when taken),
// [12:14) length, [20:32) low 12 bits of the fall-through PC (the instruction ends inside the
// 4 KB window).  A class-0 (general path) record has cycles 0, length 0 and its own offset in
// the NXT field, so the fast loop recovers PC and cycle of any record as nxt - len, now - cyc.
constexpr uint32_t AUX = 5, CYC = 8, LENF = 12, NXT = 20;
// Record word hi, by class:
//   reads / stores / read-modify-writes: [0:16) byte-permute selector of the index (sk::SEL_*;
//     bit 8 = page-cross penalty, which turns selector nibble 2 from 4 into 5: both pick a zero
//     byte of the permute's second operand), [16:28) operand (RAM: zero-page address;
//     cartridge: offset in the bank; immediates: the offset of the operand byte), bit 31 RAM
//   C_STTIA: TIA register << 8 (the log entry's register field); C_TLD/C_TBIT: address bit 0
//   C_TR: destination register; C_JMP: target
//   C_BR: [0:12) low bits of the taken target (same window), [16:32) flag mask (nz packs N at
//     bit 15 and the Z byte in bits 0-7, see scalar_cpu.cuh)
constexpr uint32_t OPND = 16;
constexpr uint32_t PEN = 1u << 8, RAM = 1u << 31;
}  // namespace pd

// fast-path classes; 0 = general interpreter
enum PClass : uint32_t {
  C_GEN = 0,
  // reads: v = RAM[(opnd + ix) & 0x7F] (RAM; needs bit 7 of opnd + ix, else GEN) or the
  // cartridge byte at offset (opnd + ix) & 0xFFF of the current bank (immediates: opnd = the
  // offset of the operand byte); AUX = register (C_CMP: 0 A 1 X 2 Y, C_LD: bit mask 1 A 2 X 4 Y)
  // -- the classes most frequent after C_BR come first (1..C_HOT_LAST): the kernel dispatches
  //    them through a separate, smaller switch
  C_LDA,    // LDA (C_LD with AUX = 1): A only
  C_STATIA, // STA to a TIA effect register (C_STTIA with AUX = 0)
  C_LD, C_STTIA, C_TLD, C_TBIT, C_TR, C_CMP, C_FLAG, C_SBC, C_WSYNC,
  C_ORA, C_AND, C_EOR, C_ADC, C_BIT,
  C_STRAM,  // store to RAM (zero page, zp indexed, or absolute RAM); AUX 0 A 1 X 2 Y 3 A&X
  C_INC, C_DEC, C_ASL, C_LSR, C_ROL, C_ROR,  // read-modify-write of RAM
  C_INR,    // INX/INY/DEX/DEY, AUX as K_INR
  C_ASLA, C_LSRA, C_ROLA, C_RORA,
  C_NOP,    // implied NOP
  C_BR,     // conditional branch inside the window: AUX bits 0-1 source (0 nz, 1 V, 2 C,
            // 3 nz), bit 2 = taken when (source & mask) != 0
  C_JMP,    // JMP absolute into cartridge space
  // C_TLD / C_TBIT: LDA/LDX/LDY/LAX / BIT of INTIM/TIMINT (absolute, RIOT timer closed form)
  // C_STTIA: store to a TIA register with a picture effect (direct): log append
  // C_WSYNC: store to WSYNC (direct); C_TR: transfers, AUX bits 0-1 source, bit 2 (set N,Z),
  //   destination in hi; C_FLAG: flag set/clear, AUX as K_FLAG
  C_COUNT
};
static_assert(C_COUNT <= 32, "class field is 5 bits");
constexpr uint32_t C_HOT_LAST = C_WSYNC;

constexpr uint32_t kRecBytes = 8;

#ifndef __CUDACC_RTC__  // host only (the jit compiles the device headers with NVRTC)
// decode the record for an instruction starting at bank offset o of a 4 KB bank image
inline uint64_t predecode_one(const uint8_t* bank, uint32_t o, uint32_t nbanks, const uint64_t* stab) {
  // hotspots of the bank-switching scheme: window offsets [hs, hs + nbanks) (F8 $FF8, F6 $FF6,
  // F4 $FF4); none for one-bank cartridges
  const uint32_t hs = nbanks == 2u ? 0xFF8u : (nbanks == 4u ? 0xFF6u : (nbanks == 8u ? 0xFF4u : 0x1000u));
  auto hot = [&](uint32_t off) { return nbanks > 1u && off >= hs && off < hs + nbanks; };
  const uint32_t op = bank[o];
  const uint64_t ent = stab[op];
  const uint32_t d = (uint32_t)ent, e = (uint32_t)(ent >> 32);
  const uint32_t kind = e & 0xFFu, aux = (e >> sk::AUX) & 0x7Fu;
  const uint32_t len = (d >> sk::LEN) & 3u;
  uint32_t cyc = (d >> sk::CYC) & 0xFu;
  const uint32_t sel = d & 0xFFFFu;
  const uint32_t b1 = o + 1 <= 0xFFFu ? bank[o + 1] : 0u, b2 = o + 2 <= 0xFFFu ? bank[o + 2] : 0u;
  const uint32_t base = b1 | (b2 << 8);
  uint32_t cls = C_GEN, raux = 0;
  const bool pen = (d & sk::PEN) != 0u;
  // the whole instruction must be fetched from this bank window without touching a hotspot
  bool fast = kind != K_JAM && o + len - 1 <= 0xFFFu;
  for (uint32_t k = 0; k < len; ++k)
    if (hot(o + k)) fast = false;
  const bool zp = (d & sk::ZP) != 0u, ptr = (d & (sk::PTRZ | sk::PTRA)) != 0u;
  const bool imm = len == 2 && !zp && !ptr && kind != K_BR && !(d & sk::RD) && !(d & sk::WR);
  const bool indexed = sel != sk::SEL_NONE;
  // classify the operand of a data access: 0 none/GEN, 1 RAM, 2 cartridge, 3 TIA (direct),
  // 4 RIOT timer (direct)
  auto where = [&]() -> int {
    if (ptr) return 0;
    if (zp) {
      if (indexed) return 1;  // zp,X / zp,Y: RAM decided at run time (bit 7 of b1 + index)
      return (b1 & 0x80u) ? 1 : 3;
    }
    const uint32_t a = base & 0x1FFFu;
    if (!indexed) {
      if ((a & 0x1280u) == 0x0080u) return 1;
      if (a & 0x1000u) return hot(a & 0xFFFu) ? 0 : 2;
      if (!(a & 0x1080u)) return 3;
      if ((a & 0x1284u) == 0x0284u) return 4;
      return 0;
    }
    // abs,X / abs,Y based in zero-page RAM ($80-$FF): RAM decided at run time like zp,X (the
    // sum stays below $200, so bit 7 alone separates RAM from the TIA mirror at $100-$17F)
    if (a >= 0x80u && a <= 0xFFu) return 1;
    // abs,X / abs,Y: every index 0..255 must stay in the window of this bank, clear of hotspots
    if (!(a & 0x1000u)) return 0;
    const uint32_t lo = a & 0xFFFu;
    if (lo + 255u > 0xFFFu) return 0;
    if (nbanks > 1u && lo + 255u >= hs) return 0;
    return 2;
  };
  // the fall-through PC must stay inside the window (its low 12 bits are stored)
  if (o + len > 0xFFFu) fast = false;
  uint32_t hi = 0;
  if (fast) {
    auto mem = [&](uint32_t cl, uint32_t off, bool is_ram) {
      cls = cl;
      hi = sel | ((off & 0xFFFu) << pd::OPND) | (pen ? pd::PEN : 0u) | (is_ram ? pd::RAM : 0u);
    };
    switch (kind) {
      case K_ORA: case K_AND: case K_EOR: case K_ADC: case K_SBC: case K_CMP: case K_BIT: case K_LD:
      case K_NOP: {
        if (kind == K_NOP && len == 1) { cls = C_NOP; break; }
        const uint32_t rcls = kind == K_ORA ? C_ORA : kind == K_AND ? C_AND : kind == K_EOR ? C_EOR :
                              kind == K_ADC ? C_ADC : kind == K_SBC ? C_SBC : kind == K_CMP ? C_CMP :
                              kind == K_BIT ? C_BIT : kind == K_LD ? ((aux & 7u) == 1u ? C_LDA : C_LD) : C_GEN;
        if (rcls == C_GEN) break;  // NOP reads: general path (rare)
        raux = aux & 7u;
        if (imm) { mem(rcls, o + 1, false); break; }
        const int w = where();
        if (w == 1) mem(rcls, zp ? b1 : (base & 0x7Fu) | 0x80u, true);  // = base if indexed
        else if (w == 2) mem(rcls, base, false);
        else if (w == 4 && kind == K_LD) { cls = C_TLD; hi = base & 1u; }
        else if (w == 4 && kind == K_BIT) { cls = C_TBIT; hi = base & 1u; }
        break;
      }
      case K_ST: {
        const int w = where();
        raux = aux & 3u;
        if (w == 1) mem(C_STRAM, zp ? b1 : (base & 0x7Fu) | 0x80u, true);
        else if (w == 3 && !indexed) {
          const uint32_t r = (zp ? b1 : base) & 0x3Fu;
          // TIA writes with a picture effect: 0x01, 0x04-0x14, 0x1B-0x2C (scalar_cpu.cuh kTiaEffect)
          const bool eff = r == 0x01u || (r >= 0x04u && r <= 0x14u) || (r >= 0x1Bu && r <= 0x2Cu);
          if (eff) { cls = raux == 0u ? C_STATIA : C_STTIA; hi = r << 8; }
          else if (r == 0x02u) cls = C_WSYNC;
        }
        break;
      }
      case K_INC: case K_DEC: case K_ASL: case K_LSR: case K_ROL: case K_ROR: {
        if (where() == 1)
          mem(kind == K_INC ? C_INC : kind == K_DEC ? C_DEC : kind == K_ASL ? C_ASL :
              kind == K_LSR ? C_LSR : kind == K_ROL ? C_ROL : C_ROR, zp ? b1 : (base & 0x7Fu) | 0x80u, true);
        break;
      }
      case K_INR: cls = C_INR; raux = aux & 3u; break;
      case K_TR: cls = C_TR; raux = (aux & 3u) | ((aux & 16u) ? 4u : 0u); hi = (aux >> 2) & 3u; break;
      case K_FLAG: cls = C_FLAG; raux = aux & 7u; break;
      case K_ASLA: cls = C_ASLA; break;
      case K_LSRA: cls = C_LSRA; break;
      case K_ROLA: cls = C_ROLA; break;
      case K_RORA: cls = C_RORA; break;
      case K_BR: {  // taken iff ((flag source & mask) != 0) == AUX bit 2 (see C_BR)
        const int32_t from = (int32_t)o + 2, tgt = from + (int32_t)(int8_t)b1;
        if (tgt < 0 || tgt > 0xFFF) break;  // the target leaves the window: general path
        const uint32_t f = aux & 3u, want = (aux >> 2) & 1u;
        const uint32_t mask = f == 0u ? 0x8000u : (f == 3u ? 0xFFu : 0x01u);  // N: bit 15 of nz; Z: nz & 0xFF
        cls = C_BR;
        raux = f | ((want ^ (f == 3u ? 1u : 0u)) << 2);
        cyc = 3u + ((((uint32_t)from ^ (uint32_t)tgt) >> 8) & 1u);
        hi = (uint32_t)tgt | (mask << 16);
      } break;
      case K_JMP:
        if (!ptr && (base & 0x1000u)) { cls = C_JMP; hi = base; }  // the target is cartridge space
        break;
      default: break;
    }
  }
  const uint32_t lo = cls == C_GEN ? (o << pd::NXT)
                                   : cls | (raux << pd::AUX) | (cyc << pd::CYC) | (len << pd::LENF) | ((o + len) << pd::NXT);
  return (uint64_t)lo | ((uint64_t)hi << 32);
}

// records for a packed ROM image: rec[i] describes an instruction starting at image byte i
// (bank = i / 4096 within its ROM)
inline void predecode_roms(const uint8_t* img, const uint32_t* rom_off, const uint32_t* rom_len, int n_roms,
                           uint64_t* rec) {
  uint64_t stab[256];
  build_scalar_table(stab);
  for (int r = 0; r < n_roms; ++r) {
    const uint32_t nb = rom_len[r] / 4096u;
    for (uint32_t b = 0; b < nb; ++b) {
      const uint8_t* bank = img + rom_off[r] + 4096u * b;
      for (uint32_t o = 0; o < 4096u; ++o) rec[rom_off[r] + 4096u * b + o] = predecode_one(bank, o, nb, stab);
    }
  }
}

#endif  // __CUDACC_RTC__

}  // namespace cule
