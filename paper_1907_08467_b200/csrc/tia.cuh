// tia.cuh — the video chip (TIA) of one environment, as replayed from its on-chip write log.
//
// The CPU loop never touches TIA registers directly: each TIA write is appended, with its
// colour-clock time T, to a per-environment log in shared memory (the paper's "TIA instruction
// buffer", kept on-chip instead of in global memory).  The log is replayed
// ("flushed") by all lanes of a warp together when any lane's log fills, when a frame ends, and
// — for one lane only — before that lane reads a collision latch.  Replay = for each entry,
// advance the TIA over [t_tia, T) with the old register values (collisions on every frame,
// pixels on rendered frames) and then apply the write (DESIGN.md §2 R#4).
//
// A span of colour clocks with constant registers is handled per scanline with 160-bit
// coverage masks (5 x u32 per object): playfield, both players (copies, scaling, reflection),
// missiles and ball.  Collisions are AND-reductions over the masks; pixels are emitted 4 at a
// time by byte-selecting the priority-resolved class masks, and packed into 16-byte stores.
#pragma once
#include <stdint.h>

// The delayed register effects (R#35, R#36) are a run-time option of the interpreter engines;
// a translated kernel is compiled for one setting (CULE_TIA_DELAYS 0 or 1), and with 0 every
// delay test below folds away.  With the option off no start delay can exist (the reset cache
// has none, cule_set_state rejects a nonzero byte 63).
#if defined(CULE_TIA_DELAYS) && CULE_TIA_DELAYS == 0
#define CULE_DELAYS_ON(d) false
#else
#define CULE_DELAYS_ON(d) ((d) != 0u)
#endif

namespace cule {

constexpr int kFrameW = 160;
constexpr int kFrameH = 210;
constexpr int kFrameBytes = kFrameW * kFrameH;  // 33,600
constexpr int kFrameChunks = kFrameBytes / 16;  // 2,100
constexpr int kObs84 = 84 * 84;                 // 7,056

// per-thread shared-memory words, interleaved [word][blockDim] (bank = lane: conflict-free)
constexpr int kTiaWords = 9;     // TIA registers, positions, collisions, t_tia
constexpr int kPwWords = 9;      // pixel writer
constexpr int kLogCap = 32;      // TIA write-log entries per env
constexpr int kLogMargin = 3;    // an instruction appends at most 3 entries (BRK into TIA space)
constexpr int kThreadWords = kTiaWords + kPwWords + kLogCap;

// log entry: T (18 bits) << 14 | reg (6 bits) << 8 | value (8 bits)
__device__ __forceinline__ uint32_t log_entry(uint32_t T, uint32_t reg, uint32_t v) {
  return (T << 14) | ((reg & 0x3Fu) << 8) | (v & 0xFFu);
}

__device__ __forceinline__ uint32_t rev8(uint32_t v) { return __brev(v) >> 24; }
__device__ __forceinline__ uint32_t spread4(uint32_t b) {  // bit k -> bits 4k..4k+3
  uint32_t x = b & 0xFFu;
  x = (x | (x << 12)) & 0x000F000Fu;
  x = (x | (x << 6)) & 0x03030303u;
  x = (x | (x << 3)) & 0x11111111u;
  return x * 0xFu;
}
__device__ __forceinline__ uint32_t spread2(uint32_t b) {  // bit k -> bits 2k..2k+1
  uint32_t x = b & 0xFFu;
  x = (x | (x << 4)) & 0x0F0Fu;
  x = (x | (x << 2)) & 0x3333u;
  x = (x | (x << 1)) & 0x5555u;
  return x * 3u;
}
__device__ __forceinline__ uint32_t nib_bytes(uint32_t n) {  // nibble -> 0x00/0xFF byte lanes
  return (((n & 0xFu) * 0x00204081u) & 0x01010101u) * 0xFFu;
}

// ---- pixel writer (state in shared memory between flushes) --------------------------------
// fill whole chunks [c0, c1) with one 4-byte pattern (frame start/end only: out of line)
__device__ __noinline__ void fill_chunks(uint8_t* base, int32_t c0, int32_t c1, uint32_t fill) {
  uint4* p = reinterpret_cast<uint4*>(base);
  for (int32_t k = c0; k < c1; ++k) p[k] = make_uint4(fill, fill, fill, fill);
}

struct PixWriter {
  uint8_t* base;
  int32_t chunk;  // chunk being assembled (-1: none yet)
  uint32_t w0, w1, w2, w3, fill;

  __device__ __forceinline__ void advance_to(int32_t c) {
    if (chunk >= 0) reinterpret_cast<uint4*>(base)[chunk] = make_uint4(w0, w1, w2, w3);
    if (c > chunk + 1) fill_chunks(base, chunk + 1, c, fill);
    chunk = c;
    w0 = w1 = w2 = w3 = fill;
  }
  // merge the masked bytes of one 16-pixel chunk (pixels arrive in raster order)
  __device__ __forceinline__ void emit(int32_t c, uint32_t p0, uint32_t p1, uint32_t p2, uint32_t p3,
                                       uint32_t m0, uint32_t m1, uint32_t m2, uint32_t m3) {
    if (c != chunk) advance_to(c);
    w0 = (w0 & ~m0) | (p0 & m0);
    w1 = (w1 & ~m1) | (p1 & m1);
    w2 = (w2 & ~m2) | (p2 & m2);
    w3 = (w3 & ~m3) | (p3 & m3);
  }
  // a chunk whose 16 pixels all lie in the span
  __device__ __forceinline__ void emit_full(int32_t c, uint32_t p0, uint32_t p1, uint32_t p2, uint32_t p3) {
    if (c != chunk) advance_to(c);
    w0 = p0; w1 = p1; w2 = p2; w3 = p3;
  }
  __device__ __forceinline__ void load(const uint32_t* w, uint32_t s) {
    base = reinterpret_cast<uint8_t*>((uint64_t)w[0] | ((uint64_t)w[s] << 32));
    chunk = (int32_t)w[2 * s];
    w0 = w[3 * s]; w1 = w[4 * s]; w2 = w[5 * s]; w3 = w[6 * s];
    fill = w[7 * s];
  }
  __device__ __forceinline__ void save(uint32_t* w, uint32_t s) const {
    w[2 * s] = (uint32_t)chunk;
    w[3 * s] = w0; w[4 * s] = w1; w[5 * s] = w2; w[6 * s] = w3;
  }
};

// byte mask of the pixels of group [xg, xg+4) that lie in [xa, xb)
__device__ __forceinline__ uint32_t group_mask(uint32_t xg, uint32_t xa, uint32_t xb) {
  if (xb <= xg || xa >= xg + 4u) return 0u;
  const uint32_t lo = xa > xg ? xa - xg : 0u, hi = xb < xg + 4u ? xb - xg : 4u;
  return (0xFFFFFFFFu >> (32u - 8u * (hi - lo))) << (8u * lo);
}

// begin rendering a frame: writer state in shared memory (flags bit0 = render)
__device__ __forceinline__ void pw_begin(uint32_t* w, uint32_t s, uint8_t* base, uint32_t fill4) {
  const uint64_t b = reinterpret_cast<uint64_t>(base);
  w[0] = (uint32_t)b; w[s] = (uint32_t)(b >> 32);
  w[2 * s] = 0xFFFFFFFFu;  // chunk -1
  w[3 * s] = w[4 * s] = w[5 * s] = w[6 * s] = fill4;
  w[7 * s] = fill4;
  w[8 * s] = 1u;
}
__device__ __forceinline__ bool pw_rendering(const uint32_t* w, uint32_t s) { return (w[8 * s] & 1u) != 0; }
__device__ __forceinline__ void pw_end(uint32_t* w, uint32_t s) {
  PixWriter pw;
  pw.load(w, s);
  pw.advance_to(kFrameChunks);
  w[8 * s] = 0u;
}
__device__ __forceinline__ void pw_stop(uint32_t* w, uint32_t s) { w[8 * s] = 0u; }

// ---- TIA register file (registers while replaying) ------------------------------------------
struct Tia {
  uint32_t colup0, colup1, colupf, colubk, pf0, pf1, pf2, ctrlpf;
  uint32_t nusiz0, nusiz1, grp0n, grp0o, grp1n, grp1o, hmp0, hmp1, hmm0, hmm1, hmbl;
  uint32_t flags;  // bit 0 vblank, 1 refp0, 2 refp1, 3 enam0, 4 enam1, 5 enbln, 6 enblo,
                   // 7 vdelp0, 8 vdelp1, 9 vdelbl, 10 resmp0, 11 resmp1
  int32_t comb_line;
  uint32_t posP0, posP1, posM0, posM1, posBL;
  uint32_t coll;
  uint32_t t_tia;
  uint32_t rdel;  // RESxx start delay (R#36): bits 0 P0, 1 P1, 2 M0, 3 M1 reset during the visible
                  // part of the line t_tia is on; their first copy is not drawn until it ends

  __device__ __forceinline__ uint32_t f(int b) const { return (flags >> b) & 1u; }
  __device__ __forceinline__ void setf(int b, uint32_t v) { flags = (flags & ~(1u << b)) | ((v & 1u) << b); }

  __device__ __forceinline__ void load(const uint32_t* w, uint32_t s) {
    uint32_t a = w[0], b = w[s], c = w[2 * s], d = w[3 * s], e = w[4 * s], g = w[5 * s], h = w[6 * s],
             k = w[7 * s];
    colup0 = a & 0xFF; colup1 = (a >> 8) & 0xFF; colupf = (a >> 16) & 0xFF; colubk = a >> 24;
    pf0 = b & 0xFF; pf1 = (b >> 8) & 0xFF; pf2 = (b >> 16) & 0xFF; ctrlpf = b >> 24;
    nusiz0 = c & 0xFF; nusiz1 = (c >> 8) & 0xFF; grp0n = (c >> 16) & 0xFF; grp0o = c >> 24;
    grp1n = d & 0xFF; grp1o = (d >> 8) & 0xFF; hmp0 = (d >> 16) & 0xFF; hmp1 = d >> 24;
    hmm0 = e & 0xFF; hmm1 = (e >> 8) & 0xFF; hmbl = (e >> 16) & 0xFF; rdel = e >> 24;
    flags = g & 0xFFFF; comb_line = (int32_t)(int16_t)(g >> 16);
    posP0 = h & 0xFF; posP1 = (h >> 8) & 0xFF; posM0 = (h >> 16) & 0xFF; posM1 = h >> 24;
    posBL = k & 0xFF; coll = k >> 16;
    t_tia = w[8 * s];
    mdirty = 0x3Fu;
  }
  __device__ __forceinline__ void store(uint32_t* w, uint32_t s) const {
    w[0] = colup0 | (colup1 << 8) | (colupf << 16) | (colubk << 24);
    w[s] = pf0 | (pf1 << 8) | (pf2 << 16) | (ctrlpf << 24);
    w[2 * s] = nusiz0 | (nusiz1 << 8) | (grp0n << 16) | (grp0o << 24);
    w[3 * s] = grp1n | (grp1o << 8) | (hmp0 << 16) | (hmp1 << 24);
    w[4 * s] = hmm0 | (hmm1 << 8) | (hmbl << 16) | (rdel << 24);
    w[5 * s] = (flags & 0xFFFF) | ((uint32_t)(comb_line & 0xFFFF) << 16);
    w[6 * s] = posP0 | (posP1 << 8) | (posM0 << 16) | (posM1 << 24);
    w[7 * s] = posBL | (coll << 16);
    w[8 * s] = t_tia;
  }

  // a 160-pixel line as five named 32-bit words (no arrays: everything stays in registers)
  struct W5 {
    uint32_t a, b, c, d, e;
    __device__ __forceinline__ uint32_t operator[](int k) const {
      return k == 0 ? a : k == 1 ? b : k == 2 ? c : k == 3 ? d : e;
    }
    __device__ __forceinline__ void zero() { a = b = c = d = e = 0u; }
    // OR a <=32-bit pattern starting at pixel p (0..159) into the circular line
    __device__ __forceinline__ void place(uint32_t pat, uint32_t p) {
      const uint32_t wi = p >> 5, s = p & 31u;
      const uint32_t lo = pat << s, hi = s ? (pat >> (32u - s)) : 0u;
      a |= (wi == 0 ? lo : 0u) | (wi == 4 ? hi : 0u);
      b |= (wi == 1 ? lo : 0u) | (wi == 0 ? hi : 0u);
      c |= (wi == 2 ? lo : 0u) | (wi == 1 ? hi : 0u);
      d |= (wi == 3 ? lo : 0u) | (wi == 2 ? hi : 0u);
      e |= (wi == 4 ? lo : 0u) | (wi == 3 ? hi : 0u);
    }
  };
  struct Masks { W5 p0, p1, m0, m1, bl, pf; };
  // coverage masks kept across the spans of a replay, rebuilt only for the objects a write
  // changed (mdirty bits 0 P0, 1 P1, 2 M0, 3 M1, 4 BL, 5 PF; all set at load)
  Masks mc;
  uint32_t mdirty;

  // NUSIZ copy set: bit0 +0, bit1 +16, bit2 +32, bit3 +64
  __device__ __forceinline__ static uint32_t copies(uint32_t mode) { return (0x1D197531u >> (4 * mode)) & 0xF; }
  __device__ __forceinline__ static void place_copies(W5& m, uint32_t pat, uint32_t pos, uint32_t cp) {
#pragma unroll 1
    for (int c = 0; c < 4; ++c)
      if (cp & (1u << c)) {
        const uint32_t p = pos + (c == 0 ? 0u : (8u << c));
        m.place(pat, p >= 160u ? p - 160u : p);
      }
  }
  __device__ __forceinline__ static void player_mask(W5& m, uint32_t pos, uint32_t nusiz, uint32_t g, uint32_t refl,
                                                     uint32_t skip_first) {
    m.zero();
    if (g == 0) return;
    const uint32_t mode = nusiz & 7;
    uint32_t pat = refl ? g : rev8(g);  // pixel d shows graphic bit 7-d (bit d when reflected)
    if (mode == 5) pat = spread2(pat);
    else if (mode == 7) pat = spread4(pat);
    place_copies(m, pat, pos, copies(mode) & ~skip_first);
  }
  __device__ __forceinline__ static void missile_mask(W5& m, uint32_t pos, uint32_t nusiz, bool en,
                                                      uint32_t skip_first) {
    m.zero();
    if (!en) return;
    const uint32_t mode = nusiz & 7;
    const uint32_t pat = (1u << (1u << ((nusiz >> 4) & 3))) - 1u;
    place_copies(m, pat, pos, ((mode == 5 || mode == 7) ? 1u : copies(mode)) & ~skip_first);
  }
  __device__ __forceinline__ void refresh_masks() {
#ifdef CULE_TIA_NO_MASK_CACHE
    mdirty = 0x3Fu;
#endif
    if (mdirty & 1u) player_mask(mc.p0, posP0, nusiz0, f(7) ? grp0o : grp0n, f(1), rdel & 1u);
    if (mdirty & 2u) player_mask(mc.p1, posP1, nusiz1, f(8) ? grp1o : grp1n, f(2), (rdel >> 1) & 1u);
    if (mdirty & 4u) missile_mask(mc.m0, posM0, nusiz0, f(3) && !f(10), (rdel >> 2) & 1u);
    if (mdirty & 8u) missile_mask(mc.m1, posM1, nusiz1, f(4) && !f(11), (rdel >> 3) & 1u);
    if (mdirty & 16u) {
      mc.bl.zero();
      if (f(9) ? f(6) : f(5)) mc.bl.place((1u << (1u << ((ctrlpf >> 4) & 3))) - 1u, posBL);
    }
    if (mdirty & 32u) {
      const uint32_t left = ((pf0 >> 4) & 0xF) | (rev8(pf1) << 4) | ((pf2 & 0xFF) << 12);
      const uint32_t right = (ctrlpf & 1) ? (__brev(left) >> 12) : left;
      const uint64_t cells = (uint64_t)left | ((uint64_t)right << 20);
      mc.pf.a = spread4((uint32_t)cells);
      mc.pf.b = spread4((uint32_t)(cells >> 8));
      mc.pf.c = spread4((uint32_t)(cells >> 16));
      mc.pf.d = spread4((uint32_t)(cells >> 24));
      mc.pf.e = spread4((uint32_t)(cells >> 32));
    }
    mdirty = 0u;
  }
  __device__ __forceinline__ void build_masks(Masks& M) const {
    player_mask(M.p0, posP0, nusiz0, f(7) ? grp0o : grp0n, f(1), rdel & 1u);
    player_mask(M.p1, posP1, nusiz1, f(8) ? grp1o : grp1n, f(2), (rdel >> 1) & 1u);
    missile_mask(M.m0, posM0, nusiz0, f(3) && !f(10), (rdel >> 2) & 1u);
    missile_mask(M.m1, posM1, nusiz1, f(4) && !f(11), (rdel >> 3) & 1u);
    M.bl.zero();
    if (f(9) ? f(6) : f(5)) M.bl.place((1u << (1u << ((ctrlpf >> 4) & 3))) - 1u, posBL);
    // playfield: 20 cells per half (PF0 D4-D7, PF1 D7-D0, PF2 D0-D7), each 4 pixels wide
    const uint32_t left = ((pf0 >> 4) & 0xF) | (rev8(pf1) << 4) | ((pf2 & 0xFF) << 12);
    const uint32_t right = (ctrlpf & 1) ? (__brev(left) >> 12) : left;
    const uint64_t cells = (uint64_t)left | ((uint64_t)right << 20);
    M.pf.a = spread4((uint32_t)cells);
    M.pf.b = spread4((uint32_t)(cells >> 8));
    M.pf.c = spread4((uint32_t)(cells >> 16));
    M.pf.d = spread4((uint32_t)(cells >> 24));
    M.pf.e = spread4((uint32_t)(cells >> 32));
  }

  // bits of 32-pixel word [lo, lo+32) inside [xa, xb)
  __device__ __forceinline__ static uint32_t range_word(uint32_t lo, uint32_t xa, uint32_t xb) {
    const uint32_t s = xa > lo ? min(xa - lo, 32u) : 0u, e = xb > lo ? min(xb - lo, 32u) : 0u;
    return e > s ? ((e - s == 32u ? 0xFFFFFFFFu : ((1u << (e - s)) - 1u)) << s) : 0u;
  }
  // OR the collision latches of the visible pixels [a0, b0) U [a1, b1) (bit 2r = d7, 2r+1 = d6 of
  // register r).  A rolled loop over the five 32-pixel words (one copy of the body: the
  // instruction cache, not the ALU, is what the replay runs short of), words outside the
  // ranges skipped.
  __device__ __forceinline__ void collide(const Masks& M, uint32_t a0, uint32_t b0, uint32_t a1, uint32_t b1) {
    uint32_t acc = 0u;
#pragma unroll 1
    for (int k = 0; k < 5; ++k) {
      const uint32_t r = range_word(32u * k, a0, b0) | range_word(32u * k, a1, b1);
      if (!r) continue;
      const uint32_t p0 = M.p0[k] & r, p1 = M.p1[k] & r, m0 = M.m0[k] & r, m1 = M.m1[k] & r,
                     bl = M.bl[k] & r, pf = M.pf[k] & r;
      acc |= ((m0 & p1) ? 1u : 0u) | ((m0 & p0) ? 2u : 0u) | ((m1 & p0) ? 4u : 0u) | ((m1 & p1) ? 8u : 0u) |
             ((p0 & pf) ? 0x10u : 0u) | ((p0 & bl) ? 0x20u : 0u) | ((p1 & pf) ? 0x40u : 0u) |
             ((p1 & bl) ? 0x80u : 0u) | ((m0 & pf) ? 0x100u : 0u) | ((m0 & bl) ? 0x200u : 0u) |
             ((m1 & pf) ? 0x400u : 0u) | ((m1 & bl) ? 0x800u : 0u) | ((bl & pf) ? 0x1000u : 0u) |
             ((p0 & p1) ? 0x4000u : 0u) | ((m0 & m1) ? 0x8000u : 0u);
    }
    coll |= acc;
  }

  __device__ __forceinline__ static uint32_t shade(uint32_t colu, const uint8_t* gray) {
    uint32_t idx = (colu >> 1) & 0x7F;
    return (gray ? (uint32_t)gray[idx] : idx) * 0x01010101u;
  }

  // 4 pixels of group g (x = 4g..4g+3) from the four class masks of its 32-pixel word
  __device__ __forceinline__ static uint32_t group_px(uint32_t q0, uint32_t q1, uint32_t qb, uint32_t qp,
                                                     uint32_t sh, bool pfp, uint32_t c0, uint32_t c1,
                                                     uint32_t cbl, uint32_t cp, uint32_t cbk) {
    const uint32_t np0 = (q0 >> sh) & 0xF, np1 = (q1 >> sh) & 0xF, nbl = (qb >> sh) & 0xF, npf = (qp >> sh) & 0xF;
    uint32_t e0, e1, eb, ep;
    if (!pfp) {
      e0 = np0; e1 = np1 & ~e0; eb = nbl & ~(e0 | e1); ep = npf & ~(e0 | e1 | nbl);
    } else {
      eb = nbl; ep = npf & ~nbl; e0 = np0 & ~(nbl | npf); e1 = np1 & ~(nbl | npf | np0);
    }
    const uint32_t B0 = nib_bytes(e0), B1 = nib_bytes(e1), Bb = nib_bytes(eb), Bp = nib_bytes(ep);
    return (c0 & B0) | (c1 & B1) | (cbl & Bb) | (cp & Bp) | (cbk & ~(B0 | B1 | Bb | Bp));
  }

  // one palette byte (gray value in GRAY84, palette index in RAW)
  __device__ __forceinline__ static uint32_t shade1(uint32_t colu, const uint8_t* gray) {
    const uint32_t idx = (colu >> 1) & 0x7F;
    return gray ? (uint32_t)gray[idx] : idx;
  }
  // bit i of the low byte of x -> bit 4i (byte-permute selector nibbles, one per pixel)
  __device__ __forceinline__ static uint32_t sel_bits(uint32_t x) {
    x &= 0xFFu;
    x = (x | (x << 12)) & 0x000F000Fu;
    x = (x | (x << 6)) & 0x03030303u;
    return (x | (x << 3)) & 0x11111111u;
  }

  // Pixels [xa, xb) of window row `row`.  Per 16-pixel chunk the priority (R#13) is resolved
  // on the chunk's coverage bits into a 3-bit colour index per pixel (0 background, 1 playfield,
  // 2 P0/M0, 3 P1/M1, 4 ball); the index bits become byte-permute selectors and four PRMTs pick
  // the colour bytes.
  __device__ __forceinline__ void render_span(const Masks& M, PixWriter& pw, uint32_t line, uint32_t row,
                                              uint32_t xa, uint32_t xb, const uint8_t* gray) {
    const uint32_t gbk = shade1(colubk, gray), g0 = shade1(colup0, gray), g1 = shade1(colup1, gray),
                   gbl = shade1(colupf, gray);
    const bool score = (ctrlpf & 2) != 0, pfp = (ctrlpf & 4) != 0;
    // permute source bytes: 0 background, 1 playfield (score mode: the player colour of the
    // half), 2 P0/M0, 3 P1/M1, 4 ball (COLUPF)
    const uint32_t hiw = (g0 << 16) | (g1 << 24);
    const uint32_t Xl = gbk | ((score ? g0 : gbl) << 8) | hiw, Xr = gbk | ((score ? g1 : gbl) << 8) | hiw;
    const bool comb = (int32_t)line == comb_line;
    // one chunk per iteration, rolled (code size: see collide)
#pragma unroll 1
    for (uint32_t c = xa >> 4; c <= (xb - 1) >> 4; ++c) {
      const int k = (int)(c >> 1);
      const uint32_t sh = 16u * (c & 1u);
      const uint32_t a = ((M.p0[k] | M.m0[k]) >> sh) & 0xFFFFu, b = ((M.p1[k] | M.m1[k]) >> sh) & 0xFFFFu,
                     l = (M.bl[k] >> sh) & 0xFFFFu, f = (M.pf[k] >> sh) & 0xFFFFu;
      uint32_t e0, e1, eb, ep;
      if (!pfp) {
        e0 = a; e1 = b & ~a; eb = l & ~(a | b); ep = f & ~(a | b | l);
      } else {
        eb = l; ep = f & ~l; e0 = a & ~(l | f); e1 = b & ~(l | f | a);
      }
      const uint32_t i0 = ep | e1, i1 = e0 | e1, i2 = eb;
      uint32_t sa = sel_bits(i0), sb = sel_bits(i0 >> 8u);
      if (i1 | i2) {  // (playfield-only chunks need one index bit)
        sa |= (sel_bits(i1) << 1) | (sel_bits(i2) << 2);
        sb |= (sel_bits(i1 >> 8u) << 1) | (sel_bits(i2 >> 8u) << 2);
      }
      const uint32_t x0 = 16u * c;
      const uint32_t X = x0 < 80u ? Xl : Xr;
      uint32_t p0 = __byte_perm(X, gbl, sa), p1 = __byte_perm(X, gbl, sa >> 16);
      const uint32_t p2 = __byte_perm(X, gbl, sb), p3 = __byte_perm(X, gbl, sb >> 16);
      if (comb && c == 0) { p0 = pw.fill; p1 = pw.fill; }  // HMOVE comb, x < 8 (R#11)
      if (xa <= x0 && xb >= x0 + 16u) {
        pw.emit_full((int32_t)(row * 10u + c), p0, p1, p2, p3);
      } else {
        const uint32_t lo = xa > x0 ? xa - x0 : 0u, hi = xb < x0 + 16u ? xb - x0 : 16u;
        const uint32_t r = ((1u << hi) - 1u) & ~((1u << lo) - 1u);
        pw.emit((int32_t)(row * 10u + c), p0, p1, p2, p3, nib_bytes(r), nib_bytes(r >> 4), nib_bytes(r >> 8),
                nib_bytes(r >> 12));
      }
    }
  }

  __device__ __forceinline__ static void render_black(PixWriter& pw, uint32_t row, uint32_t xa, uint32_t xb) {
    for (uint32_t c = xa >> 4; c <= (xb - 1) >> 4; ++c) {
      const uint32_t x0 = 16u * c;
      pw.emit((int32_t)(row * 10u + c), pw.fill, pw.fill, pw.fill, pw.fill, group_mask(x0, xa, xb),
              group_mask(x0 + 4u, xa, xb), group_mask(x0 + 8u, xa, xb), group_mask(x0 + 12u, xa, xb));
    }
  }

  // collision latches the objects present now could still set (an absent object cannot
  // collide); when they are all set already, a span needs no collision work at all
  __device__ __forceinline__ uint32_t open_pairs() const {
    const uint32_t p0 = (f(7) ? grp0o : grp0n) != 0u, p1 = (f(8) ? grp1o : grp1n) != 0u;
    const uint32_t m0 = f(3) & (f(10) ^ 1u), m1 = f(4) & (f(11) ^ 1u);
    const uint32_t bl = f(9) ? f(6) : f(5);
    const uint32_t pf = ((pf0 & 0xF0u) | pf1 | pf2) != 0u;
    const uint32_t possible = (m0 & p1) | ((m0 & p0) << 1) | ((m1 & p0) << 2) | ((m1 & p1) << 3) |
                              ((p0 & pf) << 4) | ((p0 & bl) << 5) | ((p1 & pf) << 6) | ((p1 & bl) << 7) |
                              ((m0 & pf) << 8) | ((m0 & bl) << 9) | ((m1 & pf) << 10) | ((m1 & bl) << 11) |
                              ((bl & pf) << 12) | ((p0 & p1) << 14) | ((m0 & m1) << 15);
    return possible & ~coll;
  }

  // advance over colour clocks [t_tia, t_to) with the current register values
  __device__ __forceinline__ void catch_up(uint32_t t_to, bool render, PixWriter& pw, uint32_t ystart,
                                           const uint8_t* gray) {
    const uint32_t t0 = t_tia;
    if (t_to <= t0) return;
    t_tia = t_to;
    const uint32_t l0 = t0 / 228u, l1 = (t_to - 1) / 228u;
    // visible x range of the first and last line ([xa0,160) on l0, [0,xb1) on l1)
    const uint32_t h0 = t0 - l0 * 228u, h1 = t_to - l1 * 228u;
    const uint32_t xa0 = h0 > 68u ? h0 - 68u : 0u;
    const uint32_t xb1 = h1 > 68u ? h1 - 68u : 0u;
    // a span inside one line with no visible clock (the writes right after a WSYNC, in HBLANK)
    // neither draws nor collides
    if (l1 == l0 && xb1 <= xa0) return;
    const bool vblank = f(0) != 0u;
    const bool need_coll = !vblank && open_pairs() != 0u;
    const uint32_t w0 = ystart, w1 = ystart + (uint32_t)kFrameH;  // window lines [w0, w1)
    const bool any_win = render && l1 >= w0 && l0 < w1;
    if (!need_coll && !any_win) return;
    if (!vblank && mdirty) refresh_masks();
    const Masks& M = mc;
    if (need_coll) {
      // collisions depend on x only: the union of the span's visible x ranges suffices
      uint32_t a0 = xa0, b0 = 160u, a1 = 0u, b1 = xb1;                           // two partial lines
      if (l1 > l0 + 1u || (l1 == l0 + 1u && xa0 <= xb1)) { a0 = 0u; b1 = 0u; }  // every x
      else if (l1 == l0) { b0 = xb1; b1 = 0u; }                                  // one line
      collide(M, a0, b0, a1, b1);
    }
    if (!any_win) return;
    const uint32_t la = l0 > w0 ? l0 : w0, lb = l1 < w1 - 1u ? l1 : w1 - 1u;
    for (uint32_t ln = la; ln <= lb; ++ln) {
      const uint32_t xa = ln == l0 ? xa0 : 0u, xb = ln == l1 ? xb1 : 160u;
      if (xb <= xa) continue;
      if (vblank) render_black(pw, ln - ystart, xa, xb);
      else render_span(M, pw, ln, ln - ystart, xa, xb, gray);
    }
  }

  // apply a logged write at colour clock T (WSYNC/VSYNC/RSYNC/audio never reach the log)
  __device__ __forceinline__ void apply(uint32_t r, uint32_t v, uint32_t T, uint32_t delays = 0u) {
    uint32_t line = T / 228u, h = T - line * 228u;
    int32_t hp = (int32_t)h - 68;
    switch (r) {
      case 0x01: setf(0, (v >> 1) & 1); break;
      case 0x04: nusiz0 = v; mdirty |= 1u | 4u; break;
      case 0x05: nusiz1 = v; mdirty |= 2u | 8u; break;
      case 0x06: colup0 = v; break;
      case 0x07: colup1 = v; break;
      case 0x08: colupf = v; break;
      case 0x09: colubk = v; break;
      case 0x0A: ctrlpf = v; mdirty |= 16u | 32u; break;
      case 0x0B: setf(1, v >> 3); mdirty |= 1u; break;
      case 0x0C: setf(2, v >> 3); mdirty |= 2u; break;
      case 0x0D: pf0 = v; mdirty |= 32u; break;
      case 0x0E: pf1 = v; mdirty |= 32u; break;
      case 0x0F: pf2 = v; mdirty |= 32u; break;
      case 0x10: case 0x11: case 0x12: case 0x13: case 0x14: {
        uint32_t base = r <= 0x11 ? 5u : 4u;
        uint32_t p = hp < -2 ? base - 2u : (uint32_t)(hp + (int32_t)base) % 160u;
        if (r == 0x10) posP0 = p; else if (r == 0x11) posP1 = p;
        else if (r == 0x12) posM0 = p; else if (r == 0x13) posM1 = p; else posBL = p;
        if (CULE_DELAYS_ON(delays) && hp >= 0 && r != 0x14) rdel |= 1u << (r - 0x10);  // RESxx start delay (R#36)
        mdirty |= 1u << (r - 0x10);  // (bits 0 P0 .. 4 BL follow the register order)
      } break;
      case 0x1B: grp0n = v; grp1o = grp1n; mdirty |= 1u | 2u; break;
      case 0x1C: grp1n = v; grp0o = grp0n; setf(6, f(5)); mdirty |= 1u | 2u | 16u; break;
      case 0x1D: setf(3, v >> 1); mdirty |= 4u; break;
      case 0x1E: setf(4, v >> 1); mdirty |= 8u; break;
      case 0x1F: setf(5, v >> 1); mdirty |= 16u; break;
      case 0x20: hmp0 = v >> 4; break;
      case 0x21: hmp1 = v >> 4; break;
      case 0x22: hmm0 = v >> 4; break;
      case 0x23: hmm1 = v >> 4; break;
      case 0x24: hmbl = v >> 4; break;
      case 0x25: setf(7, v); mdirty |= 1u; break;
      case 0x26: setf(8, v); mdirty |= 2u; break;
      case 0x27: setf(9, v); mdirty |= 16u; break;
      case 0x28: case 0x29: {
        const int b = r == 0x28 ? 10 : 11;
        uint32_t nv = (v >> 1) & 1;
        if (f(b) && !nv) {
          uint32_t md = (r == 0x28 ? nusiz0 : nusiz1) & 7;
          uint32_t c = md == 5 ? 6u : (md == 7 ? 10u : 3u);
          if (r == 0x28) posM0 = (posP0 + c) % 160u; else posM1 = (posP1 + c) % 160u;
        }
        setf(b, nv);
        mdirty |= r == 0x28 ? 4u : 8u;
      } break;
      case 0x2A: {
        auto mv = [](uint32_t p, uint32_t hm) -> uint32_t {
          int32_t q = (int32_t)p - ((int32_t)(hm ^ 8u) - 8);
          return (uint32_t)(q < 0 ? q + 160 : (q >= 160 ? q - 160 : q));
        };
        posP0 = mv(posP0, hmp0); posP1 = mv(posP1, hmp1); posM0 = mv(posM0, hmm0);
        posM1 = mv(posM1, hmm1); posBL = mv(posBL, hmbl);
        if (h < 68u) comb_line = (int32_t)line;
        mdirty |= 31u;
      } break;
      case 0x2B: hmp0 = hmp1 = hmm0 = hmm1 = hmbl = 0; break;
      case 0x2C: coll = 0; break;
      default: break;
    }
  }
};

// Effect clock of a logged write at colour clock T (R#35, opt-in `delays`): a
// playfield register written at visible pixel x lands at the next 4-pixel cell boundary
// 4*ceil(x/4), GRP0/GRP1 one colour clock later; without delays, and for every other register,
// T itself (R#4).  The replay catches the TIA up to the effect clock, then applies the write.
__device__ __forceinline__ uint32_t effect_clock(uint32_t T, uint32_t r, uint32_t delays) {
  if (!CULE_DELAYS_ON(delays)) return T;
  if (r - 0x0Du < 3u) {
    const uint32_t h = T % 228u;
    const uint32_t d = h > 68u ? (h - 68u) & 3u : 0u;
    return d ? T + 4u - d : T;
  }
  return (r - 0x1Bu < 2u) ? T + 1u : T;
}

// Replay n log entries of this lane, then (optionally) advance to t_final.
// tw: this thread's TIA words, pw_w: pixel-writer words, lg: log words (all stride s).
__device__ __forceinline__ void flush_lane(uint32_t* tw, uint32_t* pw_w, const uint32_t* lg, uint32_t s,
                                           uint32_t n, bool final_catch, uint32_t t_final, uint32_t ystart,
                                           const uint8_t* gray, uint32_t delays = 0u) {
  Tia t;
  t.load(tw, s);
  PixWriter pw;
  const bool render = pw_rendering(pw_w, s);
  if (render) pw.load(pw_w, s);
  // entries 0..n-1 (catch up to the write's effect clock, then apply it), then the final
  // catch-up; a RESxx start delay ends with its line: the catch-up stops there first (one
  // catch_up call site keeps the replay code small)
  const uint32_t kend = final_catch ? n + 1u : n;
  for (uint32_t k = 0; k < kend;) {
    const uint32_t e = k < n ? lg[k * s] : 0u;
    const uint32_t T = e >> 14, r = (e >> 8) & 0x3Fu;
    uint32_t to = k < n ? effect_clock(T, r, delays) : t_final;
    bool line_end = false;
    if (CULE_DELAYS_ON(delays) && t.rdel) {
      const uint32_t le = (t.t_tia / 228u + 1u) * 228u;
      if (to >= le) { to = le; line_end = true; }
    }
    t.catch_up(to, render, pw, ystart, gray);
    if (line_end) { t.mdirty |= t.rdel; t.rdel = 0u; continue; }
    if (k == n) break;
    t.apply(r, e & 0xFFu, T, delays);
    ++k;
  }
  t.store(tw, s);
  if (render) pw.save(pw_w, s);
}

}  // namespace cule
