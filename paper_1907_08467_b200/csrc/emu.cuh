// emu.cuh — the per-environment Atari 2600 machine as sm_100a device code.
//
// One thread emulates one console: 6502 + RIOT + TIA + ROM,
// rendering 160x210 frames straight into device memory.  The machine model is the
// written model of DESIGN.md §2; this file implements it independently of
// the CPU oracle, with a GPU-oriented structure:
//   * table-driven 6502 (decode table in shared memory): addressing mode -> one effective-address
//     path, operation -> one ALU path, so lanes running different opcodes of the same mode or
//     class share instructions;
//   * lazy TIA: the video chip is only advanced ("caught up") when the CPU touches a TIA
//     register or the frame ends, over a whole span of colour clocks at once;
//   * spans are rendered from 160-bit coverage masks (5 x u32 per object) — playfield, players
//     with copies/scaling/reflection, missiles and ball — and collisions are 15 AND-reductions
//     over the same masks; pixels are emitted 4 at a time (byte-select from class masks);
//   * a streaming pixel writer packs each thread's pixels into 16-byte stores;
//   * RAM lives in shared memory, word-interleaved across threads (bank = lane, conflict-free).
#pragma once
#include <stdint.h>

#include "decode_table.h"

namespace cule {

constexpr int kFrameW = 160;
constexpr int kFrameH = 210;
constexpr int kFrameBytes = kFrameW * kFrameH;       // 33,600
constexpr int kFrameChunks = kFrameBytes / 16;       // 2,100
constexpr int kObs84 = 84 * 84;                      // 7,056

// ---- snapshot layout: 16 chunks of 16 bytes -------------------------------
// chunk 0..3  bytes   0..63  CPU, clock, timer, inputs, collisions, TIA registers, positions
// chunk 4..11 bytes  64..191 RAM
// chunk 12    bytes 192..207 bookkeeping (episode_frames, episode_index, episode_return, prev_score)
constexpr int kHdrChunks = 4;
constexpr int kRamChunk0 = 4;
constexpr int kBookChunk = 12;
constexpr int kUsedChunks = 13;

// ---- small bit utilities -------------------------------------------------------------------
__device__ __forceinline__ uint32_t rev8(uint32_t v) { return __brev(v) >> 24; }

// spread bit k of an 8-bit value to bits 4k..4k+3
__device__ __forceinline__ uint32_t spread4(uint32_t b) {
  uint32_t x = b & 0xFFu;
  x = (x | (x << 12)) & 0x000F000Fu;
  x = (x | (x << 6)) & 0x03030303u;
  x = (x | (x << 3)) & 0x11111111u;
  return x * 0xFu;
}
// spread bit k of an 8-bit value to bits 2k..2k+1
__device__ __forceinline__ uint32_t spread2(uint32_t b) {
  uint32_t x = b & 0xFFu;
  x = (x | (x << 4)) & 0x0F0Fu;
  x = (x | (x << 2)) & 0x3333u;
  x = (x | (x << 1)) & 0x5555u;
  return x * 3u;
}
// nibble -> 4 byte lanes of 0x00/0xFF
__device__ __forceinline__ uint32_t nib_bytes(uint32_t n) {
  return ((((n & 0xFu) * 0x00204081u) & 0x01010101u) * 0xFFu);
}

// ---- launch-wide constants ---------------------------------------------------------------
struct Smem {
  const uint8_t* rom;       // n_roms x 8192 bytes (4K ROMs occupy the first 4096)
  const uint32_t* decode;   // 256 entries
  const uint8_t* gray;      // 128-entry gray LUT
  uint8_t* ram;             // [32 words][blockDim][4 bytes], this thread's base applied
  uint32_t ram_stride;      // bytes between consecutive RAM words of one thread (= 4*blockDim)
};

// ---- streaming pixel writer ----------------------------------------------------------------
// Pixels of a frame are produced strictly in raster order (catch-up is monotone in time), so
// each thread accumulates 16 pixels and issues one aligned 16-byte store per chunk.
struct PixWriter {
  uint8_t* base;     // 33,600-byte frame of this env (global)
  int32_t chunk;     // chunk being assembled, -1 before the first pixel
  uint32_t w0, w1, w2, w3;
  uint32_t fill;     // "black" replicated into 4 bytes (palette 0, or gray[0])
  bool max_mode;     // merge with max() into what is already there (second frame of the pair)
  bool active;

  __device__ __forceinline__ void begin(uint8_t* b, uint32_t fill4, bool mx) {
    base = b; chunk = -1; w0 = w1 = w2 = w3 = fill4; fill = fill4; max_mode = mx; active = true;
  }
  __device__ __forceinline__ void store_chunk(int32_t c, uint32_t a, uint32_t b, uint32_t d, uint32_t e) {
    uint4* p = reinterpret_cast<uint4*>(base) + c;
    if (max_mode) {
      uint4 o = *p;
      a = __vmaxu4(a, o.x); b = __vmaxu4(b, o.y); d = __vmaxu4(d, o.z); e = __vmaxu4(e, o.w);
    }
    *p = make_uint4(a, b, d, e);
  }
  // emit everything up to (not including) chunk c as black / pending
  __device__ __forceinline__ void advance_to(int32_t c) {
    if (chunk >= 0) store_chunk(chunk, w0, w1, w2, w3);
    int32_t first = chunk + 1;
    if (!(max_mode && fill == 0)) {
      for (int32_t k = first; k < c; ++k) store_chunk(k, fill, fill, fill, fill);
    }
    chunk = c;
    w0 = w1 = w2 = w3 = fill;
  }
  // put 4 pixels of group g (pixel index 4g..4g+3), byte mask selects which bytes are written
  __device__ __forceinline__ void put(int32_t g, uint32_t px, uint32_t bmask) {
    int32_t c = g >> 2;
    if (c != chunk) advance_to(c);
    uint32_t k = g & 3;
    uint32_t* w = k == 0 ? &w0 : k == 1 ? &w1 : k == 2 ? &w2 : &w3;
    *w = (*w & ~bmask) | (px & bmask);
  }
  __device__ __forceinline__ void finish() {
    advance_to(kFrameChunks);
    chunk = -1;
    active = false;
  }
};

// ---- the machine --------------------------------------------------------------------------
struct Machine {
  // CPU (flags kept unpacked; N from nreg bit 7, Z from zreg == 0)
  uint32_t PC, A, X, Y, SP;
  uint32_t fC, fV, fD, fI, nreg, zreg;
  uint32_t fc;          // CPU cycle within the frame
  uint32_t now;         // cycle at which the current access samples
  uint32_t bank;
  uint32_t rom_off;     // byte offset of this env's ROM in shared memory
  uint32_t is_f8;
  // RIOT
  uint32_t tV, tS, swcha, inpt4;
  int32_t tW;
  // TIA registers
  uint32_t colup0, colup1, colupf, colubk, ctrlpf, pf0, pf1, pf2;
  uint32_t nusiz0, nusiz1, grp0n, grp0o, grp1n, grp1o;
  uint32_t hmp0, hmp1, hmm0, hmm1, hmbl;
  uint32_t vsync, vblank, refp0, refp1, enam0, enam1, enbln, enblo, vdelp0, vdelp1, vdelbl,
      resmp0, resmp1;
  uint32_t posP0, posP1, posM0, posM1, posBL;
  uint32_t coll;
  int32_t comb_line;
  // TIA catch-up bookkeeping (not in the snapshot)
  uint32_t t_tia;       // colour clock the TIA has been advanced to
  uint32_t t_phaseA;    // colour clock that operand/pointer fetches from TIA space observe
  uint32_t wsync_req, vsync_rose;
  // frame context
  uint32_t render, ystart;
  uint32_t last_lines;
  PixWriter pw;
  const Smem* sm;

  // ------------------------------------------------------------------ RAM (shared memory)
  __device__ __forceinline__ uint32_t ram_rd(uint32_t a) const {
    return sm->ram[(a >> 2) * sm->ram_stride + (a & 3)];
  }
  __device__ __forceinline__ void ram_wr(uint32_t a, uint32_t v) {
    sm->ram[(a >> 2) * sm->ram_stride + (a & 3)] = (uint8_t)v;
  }

  // ------------------------------------------------------------------ TIA coverage masks
  struct Masks { uint32_t p0[5], p1[5], m0[5], m1[5], bl[5], pf[5]; };

  __device__ __forceinline__ static void place(uint32_t* m, uint32_t pat, uint32_t p) {
    // OR a <=32-bit pattern starting at pixel p (0..159) into a circular 160-bit line
    uint32_t w = p >> 5, s = p & 31;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      if (k == (int)w) m[k] |= pat << s;
      if (s && k == (int)(w == 4 ? 0 : w + 1)) m[k] |= pat >> (32 - s);
    }
  }
  // copy-offset set per NUSIZ mode: bit0 -> +0, bit1 -> +16, bit2 -> +32, bit3 -> +64
  __device__ __forceinline__ static uint32_t copies(uint32_t mode) { return (0x1D197531u >> (4 * mode)) & 0xF; }

  __device__ __forceinline__ static void player_mask(uint32_t* m, uint32_t pos, uint32_t nusiz,
                                                     uint32_t g, uint32_t refl) {
#pragma unroll
    for (int k = 0; k < 5; ++k) m[k] = 0;
    if (g == 0) return;
    uint32_t mode = nusiz & 7;
    uint32_t pat = refl ? g : rev8(g);            // pixel d shows graphic bit 7-d (or d if reflected)
    if (mode == 5) pat = spread2(pat);
    else if (mode == 7) pat = spread4(pat);
    uint32_t cp = copies(mode);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (cp & (1u << c)) {
        uint32_t p = pos + (c == 0 ? 0u : (8u << c));
        if (p >= 160) p -= 160;
        place(m, pat, p);
      }
    }
  }
  __device__ __forceinline__ static void missile_mask(uint32_t* m, uint32_t pos, uint32_t nusiz,
                                                      uint32_t en) {
#pragma unroll
    for (int k = 0; k < 5; ++k) m[k] = 0;
    if (!en) return;
    uint32_t mode = nusiz & 7;
    uint32_t pat = (1u << (1u << ((nusiz >> 4) & 3))) - 1u;
    uint32_t cp = (mode == 5 || mode == 7) ? 1u : copies(mode);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (cp & (1u << c)) {
        uint32_t p = pos + (c == 0 ? 0u : (8u << c));
        if (p >= 160) p -= 160;
        place(m, pat, p);
      }
    }
  }
  __device__ __forceinline__ void build_masks(Masks& M) const {
    player_mask(M.p0, posP0, nusiz0, vdelp0 ? grp0o : grp0n, refp0);
    player_mask(M.p1, posP1, nusiz1, vdelp1 ? grp1o : grp1n, refp1);
    missile_mask(M.m0, posM0, nusiz0, enam0 && !resmp0);
    missile_mask(M.m1, posM1, nusiz1, enam1 && !resmp1);
#pragma unroll
    for (int k = 0; k < 5; ++k) M.bl[k] = 0;
    if (vdelbl ? enblo : enbln) place(M.bl, (1u << (1u << ((ctrlpf >> 4) & 3))) - 1u, posBL);
    // playfield: 20 cells per half (PF0 D4-D7, PF1 D7-D0, PF2 D0-D7), each 4 pixels wide
    uint32_t left = ((pf0 >> 4) & 0xF) | (rev8(pf1) << 4) | ((pf2 & 0xFF) << 12);
    uint32_t right = (ctrlpf & 1) ? (__brev(left) >> 12) : left;
    uint64_t cells = (uint64_t)left | ((uint64_t)right << 20);
#pragma unroll
    for (int k = 0; k < 5; ++k) M.pf[k] = spread4((uint32_t)(cells >> (8 * k)));
  }

  // collision latches for visible pixels [xa, xb) (bit layout DESIGN.md §3)
  __device__ __forceinline__ void collide(const Masks& M, uint32_t xa, uint32_t xb) {
    uint32_t a01 = 0, a02 = 0, a03 = 0, a04 = 0, a05 = 0, a06 = 0, a07 = 0, a08 = 0, a09 = 0,
             a10 = 0, a11 = 0, a12 = 0, a14 = 0, a15 = 0, a00 = 0;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      uint32_t lo = 32u * k;
      uint32_t s = xa > lo ? min(xa - lo, 32u) : 0u, e = xb > lo ? min(xb - lo, 32u) : 0u;
      uint32_t r = (e > s) ? ((e - s == 32u ? 0xFFFFFFFFu : ((1u << (e - s)) - 1u)) << s) : 0u;
      uint32_t p0 = M.p0[k] & r, p1 = M.p1[k] & r, m0 = M.m0[k] & r, m1 = M.m1[k] & r,
               bl = M.bl[k] & r, pf = M.pf[k] & r;
      a00 |= m0 & p1; a01 |= m0 & p0; a02 |= m1 & p0; a03 |= m1 & p1;
      a04 |= p0 & pf; a05 |= p0 & bl; a06 |= p1 & pf; a07 |= p1 & bl;
      a08 |= m0 & pf; a09 |= m0 & bl; a10 |= m1 & pf; a11 |= m1 & bl;
      a12 |= bl & pf; a14 |= p0 & p1; a15 |= m0 & m1;
    }
    coll |= (a00 ? 1u : 0u) | (a01 ? 2u : 0u) | (a02 ? 4u : 0u) | (a03 ? 8u : 0u) |
            (a04 ? 0x10u : 0u) | (a05 ? 0x20u : 0u) | (a06 ? 0x40u : 0u) | (a07 ? 0x80u : 0u) |
            (a08 ? 0x100u : 0u) | (a09 ? 0x200u : 0u) | (a10 ? 0x400u : 0u) |
            (a11 ? 0x800u : 0u) | (a12 ? 0x1000u : 0u) | (a14 ? 0x4000u : 0u) |
            (a15 ? 0x8000u : 0u);
  }

  __device__ __forceinline__ uint32_t shade(uint32_t colu, bool gray) const {
    uint32_t idx = (colu >> 1) & 0x7F;
    return (gray ? (uint32_t)sm->gray[idx] : idx) * 0x01010101u;
  }

  // pixels [xa, xb) of window row `row`
  __device__ void render_span(const Masks& M, uint32_t line, uint32_t row, uint32_t xa,
                              uint32_t xb, bool gray) {
    uint32_t cbk = shade(colubk, gray), c0 = shade(colup0, gray), c1 = shade(colup1, gray),
             cbl = shade(colupf, gray);
    uint32_t cpl = (ctrlpf & 2) ? c0 : cbl, cpr = (ctrlpf & 2) ? c1 : cbl;
    bool pfp = ctrlpf & 4;
    bool comb = (int32_t)line == comb_line;
    uint32_t base_g = row * (kFrameW / 4);
    for (uint32_t g = xa >> 2; g <= (xb - 1) >> 2; ++g) {
      uint32_t k = g >> 3, sh = (g & 7) * 4;
      uint32_t np0 = ((M.p0[k] | M.m0[k]) >> sh) & 0xF;
      uint32_t np1 = ((M.p1[k] | M.m1[k]) >> sh) & 0xF;
      uint32_t nbl = (M.bl[k] >> sh) & 0xF;
      uint32_t npf = (M.pf[k] >> sh) & 0xF;
      uint32_t e0, e1, eb, ep;
      if (!pfp) {
        e0 = np0; e1 = np1 & ~e0; eb = nbl & ~(e0 | e1); ep = npf & ~(e0 | e1 | nbl);
      } else {
        eb = nbl; ep = npf & ~nbl; e0 = np0 & ~(nbl | npf); e1 = np1 & ~(nbl | npf | np0);
      }
      uint32_t B0 = nib_bytes(e0), B1 = nib_bytes(e1), Bb = nib_bytes(eb), Bp = nib_bytes(ep);
      uint32_t cp = g < 20 ? cpl : cpr;
      uint32_t px = (c0 & B0) | (c1 & B1) | (cbl & Bb) | (cp & Bp) | (cbk & ~(B0 | B1 | Bb | Bp));
      if (comb && g < 2) px = pw.fill;
      uint32_t x0 = g * 4;
      uint32_t lo = xa > x0 ? xa - x0 : 0u, hi = xb < x0 + 4 ? xb - x0 : 4u;
      uint32_t bm = (0xFFFFFFFFu >> (32 - 8 * (hi - lo))) << (8 * lo);
      pw.put(base_g + g, px, bm);
    }
  }
  __device__ __forceinline__ void render_black(uint32_t row, uint32_t xa, uint32_t xb) {
    uint32_t base_g = row * (kFrameW / 4);
    for (uint32_t g = xa >> 2; g <= (xb - 1) >> 2; ++g) {
      uint32_t x0 = g * 4;
      uint32_t lo = xa > x0 ? xa - x0 : 0u, hi = xb < x0 + 4 ? xb - x0 : 4u;
      uint32_t bm = (0xFFFFFFFFu >> (32 - 8 * (hi - lo))) << (8 * lo);
      pw.put(base_g + g, pw.fill, bm);
    }
  }

  // advance the TIA over colour clocks [t_tia, t_to) with the current register values
  template <bool kGray>
  __device__ void catch_up(uint32_t t_to) {
    uint32_t t0 = t_tia;
    if (t_to <= t0) return;
    t_tia = t_to;
    uint32_t l0 = t0 / 228u, l1 = (t_to - 1) / 228u;
    bool have_masks = false, full_done = false;
    Masks M;
    for (uint32_t ln = l0; ln <= l1; ++ln) {
      uint32_t h0 = (ln == l0) ? t0 - ln * 228u : 0u;
      uint32_t h1 = (ln == l1) ? t_to - ln * 228u : 228u;
      if (h1 <= 68u) continue;
      uint32_t xa = h0 > 68u ? h0 - 68u : 0u, xb = h1 - 68u;
      bool inwin = render && ln >= ystart && ln < ystart + (uint32_t)kFrameH;
      if (vblank) {
        if (inwin) render_black(ln - ystart, xa, xb);
        continue;
      }
      if (!have_masks) { build_masks(M); have_masks = true; }
      bool full = xa == 0 && xb == 160;
      if (!(full && full_done)) collide(M, xa, xb);
      if (full) full_done = true;
      if (inwin) render_span(M, ln, ln - ystart, xa, xb, kGray);
    }
  }

  __device__ __forceinline__ uint32_t tia_read(uint32_t r) const {
    if (r < 8) return (((coll >> (2 * r)) & 1u) << 7) | (((coll >> (2 * r + 1)) & 1u) << 6);
    if (r == 0x0C) return inpt4;
    if (r == 0x0D) return 0x80;
    return 0;
  }

  __device__ void tia_write(uint32_t r, uint32_t v) {
    uint32_t T = 3u * now;
    uint32_t line = T / 228u, h = T - line * 228u;
    int32_t hp = (int32_t)h - 68;
    switch (r) {
      case 0x00: { uint32_t nv = (v >> 1) & 1; if (!vsync && nv) vsync_rose = 1; vsync = nv; } break;
      case 0x01: vblank = (v >> 1) & 1; break;
      case 0x02: wsync_req = 1; break;
      case 0x04: nusiz0 = v; break;
      case 0x05: nusiz1 = v; break;
      case 0x06: colup0 = v; break;
      case 0x07: colup1 = v; break;
      case 0x08: colupf = v; break;
      case 0x09: colubk = v; break;
      case 0x0A: ctrlpf = v; break;
      case 0x0B: refp0 = (v >> 3) & 1; break;
      case 0x0C: refp1 = (v >> 3) & 1; break;
      case 0x0D: pf0 = v; break;
      case 0x0E: pf1 = v; break;
      case 0x0F: pf2 = v; break;
      case 0x10: case 0x11: case 0x12: case 0x13: case 0x14: {
        uint32_t base = r <= 0x11 ? 5u : 4u;
        uint32_t p = hp < -2 ? base - 2u : (uint32_t)(hp + (int32_t)base) % 160u;
        if (r == 0x10) posP0 = p; else if (r == 0x11) posP1 = p;
        else if (r == 0x12) posM0 = p; else if (r == 0x13) posM1 = p; else posBL = p;
      } break;
      case 0x1B: grp0n = v; grp1o = grp1n; break;
      case 0x1C: grp1n = v; grp0o = grp0n; enblo = enbln; break;
      case 0x1D: enam0 = (v >> 1) & 1; break;
      case 0x1E: enam1 = (v >> 1) & 1; break;
      case 0x1F: enbln = (v >> 1) & 1; break;
      case 0x20: hmp0 = v >> 4; break;
      case 0x21: hmp1 = v >> 4; break;
      case 0x22: hmm0 = v >> 4; break;
      case 0x23: hmm1 = v >> 4; break;
      case 0x24: hmbl = v >> 4; break;
      case 0x25: vdelp0 = v & 1; break;
      case 0x26: vdelp1 = v & 1; break;
      case 0x27: vdelbl = v & 1; break;
      case 0x28: {
        uint32_t nv = (v >> 1) & 1;
        if (resmp0 && !nv) {
          uint32_t md = nusiz0 & 7;
          posM0 = (posP0 + (md == 5 ? 6u : md == 7 ? 10u : 3u)) % 160u;
        }
        resmp0 = nv;
      } break;
      case 0x29: {
        uint32_t nv = (v >> 1) & 1;
        if (resmp1 && !nv) {
          uint32_t md = nusiz1 & 7;
          posM1 = (posP1 + (md == 5 ? 6u : md == 7 ? 10u : 3u)) % 160u;
        }
        resmp1 = nv;
      } break;
      case 0x2A: {
        // signed 4-bit motion, positive = left: pos - sx(HM) mod 160
        auto mv = [](uint32_t p, uint32_t hm) -> uint32_t {
          int32_t d = (int32_t)(hm ^ 8u) - 8;
          int32_t q = (int32_t)p - d;
          return (uint32_t)(q < 0 ? q + 160 : (q >= 160 ? q - 160 : q));
        };
        posP0 = mv(posP0, hmp0); posP1 = mv(posP1, hmp1); posM0 = mv(posM0, hmm0);
        posM1 = mv(posM1, hmm1); posBL = mv(posBL, hmbl);
        if (h < 68u) comb_line = (int32_t)line;
      } break;
      case 0x2B: hmp0 = hmp1 = hmm0 = hmm1 = hmbl = 0; break;
      case 0x2C: coll = 0; break;
      default: break;
    }
  }

  // ------------------------------------------------------------------ RIOT timer (closed form)
  __device__ __forceinline__ uint32_t intim() const {
    int32_t e = (int32_t)now - tW;
    int32_t VI = (int32_t)(tV << tS);
    if (e <= VI) return (tV - (uint32_t)((e + (1 << tS) - 1) >> tS)) & 0xFF;
    return (uint32_t)(0xFF - (e - VI - 1)) & 0xFF;
  }
  __device__ __forceinline__ uint32_t timint() const {
    return ((int32_t)now - tW) > (int32_t)(tV << tS) ? 0x80u : 0u;
  }

  // ------------------------------------------------------------------ bus
  __device__ __forceinline__ uint32_t cart_rd(uint32_t a) {
    if (is_f8 && (a & 0x1FFEu) == 0x1FF8u) bank = a & 1u;
    return sm->rom[rom_off + (bank << 12) + (a & 0xFFFu)];
  }
  template <bool kGray, bool kPhaseA>
  __device__ __forceinline__ uint32_t rd(uint32_t addr) {
    uint32_t a = addr & 0x1FFFu;
    if (a & 0x1000u) return cart_rd(a);
    if ((a & 0x0280u) == 0x0080u) return ram_rd(a & 0x7Fu);
    return rd_slow<kGray, kPhaseA>(a);
  }
  template <bool kGray, bool kPhaseA>
  __device__ __noinline__ uint32_t rd_slow(uint32_t a) {
    if (!(a & 0x80u)) {
      catch_up<kGray>(kPhaseA ? t_phaseA : 3u * now);
      return tia_read(a & 0x0Fu);
    }
    if (!(a & 0x04u)) {
      uint32_t k = a & 3u;
      return k == 0 ? swcha : (k == 2 ? 0x0Bu : 0u);
    }
    return (a & 1u) ? timint() : intim();
  }
  template <bool kGray>
  __device__ __forceinline__ void wr(uint32_t addr, uint32_t v) {
    uint32_t a = addr & 0x1FFFu;
    if ((a & 0x1280u) == 0x0080u) { ram_wr(a & 0x7Fu, v); return; }
    wr_slow<kGray>(a, v & 0xFFu);
  }
  template <bool kGray>
  __device__ __noinline__ void wr_slow(uint32_t a, uint32_t v) {
    if (a & 0x1000u) {
      if (is_f8 && (a & 0x1FFEu) == 0x1FF8u) bank = a & 1u;
      return;
    }
    if (!(a & 0x80u)) {
      catch_up<kGray>(3u * now);
      tia_write(a & 0x3Fu, v);
      return;
    }
    if ((a & 0x14u) == 0x14u) {  // RIOT timer write: interval 1/8/64/1024
      tV = v;
      tS = (0xA630u >> (4 * (a & 3u))) & 0xFu;
      tW = (int32_t)now;
    }
  }
  template <bool kGray>
  __device__ __forceinline__ uint32_t fetch() {
    uint32_t p = PC;
    PC = (PC + 1) & 0xFFFFu;
    if (p & 0x1000u) return cart_rd(p & 0x1FFFu);
    return rd<kGray, true>(p);
  }
  template <bool kGray>
  __device__ __forceinline__ void push(uint32_t v) { wr<kGray>(0x100u | SP, v); SP = (SP - 1) & 0xFFu; }
  template <bool kGray>
  __device__ __forceinline__ uint32_t pull() { SP = (SP + 1) & 0xFFu; return rd<kGray, false>(0x100u | SP); }

  __device__ __forceinline__ uint32_t getP() const {
    return (nreg & 0x80u) | (fV << 6) | 0x20u | (fD << 3) | (fI << 2) | ((zreg & 0xFFu) == 0 ? 2u : 0u) | fC;
  }
  __device__ __forceinline__ void setP(uint32_t p) {
    nreg = p & 0x80u; fV = (p >> 6) & 1; fD = (p >> 3) & 1; fI = (p >> 2) & 1;
    zreg = (p & 2u) ? 0u : 1u; fC = p & 1u;
  }
  __device__ __forceinline__ void nz(uint32_t v) { nreg = v; zreg = v & 0xFFu; }

  __device__ __forceinline__ void adc(uint32_t m) {
    if (!fD) {
      uint32_t t = A + m + fC;
      fV = ((~(A ^ m) & (A ^ t)) >> 7) & 1u;
      fC = t >> 8;
      A = t & 0xFFu;
      nz(A);
    } else {
      uint32_t lo = (A & 0xFu) + (m & 0xFu) + fC;
      if (lo >= 0xAu) lo = ((lo + 6u) & 0xFu) + 0x10u;
      uint32_t s = (A & 0xF0u) + (m & 0xF0u) + lo;
      int32_t sv = (int32_t)(int8_t)(A & 0xF0u) + (int32_t)(int8_t)(m & 0xF0u) + (int32_t)lo;
      zreg = (A + m + fC) & 0xFFu;
      nreg = s;
      fV = (sv < -128 || sv > 127) ? 1u : 0u;
      if (s >= 0xA0u) s += 0x60u;
      fC = s >= 0x100u ? 1u : 0u;
      A = s & 0xFFu;
    }
  }
  __device__ __forceinline__ void sbc(uint32_t m) {
    uint32_t t = A + (m ^ 0xFFu) + fC;
    uint32_t r = t & 0xFFu;
    uint32_t v = ((~(A ^ (m ^ 0xFFu)) & (A ^ t)) >> 7) & 1u;
    if (fD) {
      int32_t lo = (int32_t)(A & 0xFu) - (int32_t)(m & 0xFu) + (int32_t)fC - 1;
      if (lo < 0) lo = ((lo - 6) & 0xF) - 0x10;
      int32_t s = (int32_t)(A & 0xF0u) - (int32_t)(m & 0xF0u) + lo;
      if (s < 0) s -= 0x60;
      A = (uint32_t)s & 0xFFu;
    } else {
      A = r;
    }
    fV = v; fC = t >> 8; nz(r);
  }
  __device__ __forceinline__ void cmp(uint32_t reg, uint32_t m) {
    uint32_t t = reg - m;
    fC = reg >= m ? 1u : 0u;
    nz(t & 0xFFu);
  }
};

}  // namespace cule
