// scalar_tia.cuh — warp-cooperative TIA replay for the scalar engine (one env per warp).
//
// The replay of one env's write log is sequential in time, but within a span of colour clocks
// with constant registers the work is parallel in x ("the TIA kernel may be
// scheduled ... with more than one thread per game, as rendering of diverse rows on the screen
// is indeed a parallel operation").  All 32 lanes of the env's warp replay the log together:
// the TIA registers are warp-uniform and kept PACKED in the nine words of the shared-memory
// layout (tia.cuh Tia::load/store), fields extracted on use, so the replay stays within the
// scalar engine's register budget; lane j < 10 owns 16-pixel chunk j of the row being
// assembled and computes its pixels once per span; even lanes 0..8 own 32-pixel coverage word
// j/2 for collisions, OR-reduced across the warp; a completed row leaves as ten coalesced
// 16-byte stores.  Same written model as tia.cuh (DESIGN.md §2 R#7-R#14), independent code.
#pragma once
#include "tia.cuh"

namespace cule {

__device__ __forceinline__ uint32_t byte_of(uint32_t w, int i) { return (w >> (8 * i)) & 0xFFu; }
__device__ __forceinline__ uint32_t with_byte(uint32_t w, int i, uint32_t v) {
  return (w & ~(0xFFu << (8 * i))) | ((v & 0xFFu) << (8 * i));
}

// TIA registers, packed: the nine shared-memory words
//   w0 COLUP0 COLUP1 COLUPF COLUBK | w1 PF0 PF1 PF2 CTRLPF | w2 NUSIZ0 NUSIZ1 GRP0new GRP0old
//   w3 GRP1new GRP1old HMP0 HMP1   | w4 HMM0 HMM1 HMBL     | w5 flags(16) comb_line(16)
//   w6 posP0 posP1 posM0 posM1     | w7 posBL, collisions(16) << 16 | t = colour clock

// collision pairs two present objects can set, by presence bits (0 P0, 1 P1, 2 M0, 3 M1, 4 BL,
// 5 PF) -> latch bits (bit 2r = D7, 2r+1 = D6 of read register r: CXM0P M0-P1/M0-P0, CXM1P
// M1-P0/M1-P1, CXP0FB P0-PF/P0-BL, CXP1FB P1-PF/P1-BL, CXM0FB M0-PF/M0-BL, CXM1FB M1-PF/M1-BL,
// CXBLPF BL-PF, CXPPMM P0-P1/M0-M1)
struct PairTable {
  uint16_t v[64];
  constexpr PairTable() : v() {
    for (int i = 0; i < 64; ++i) {
      const int p0 = i & 1, p1 = (i >> 1) & 1, m0 = (i >> 2) & 1, m1 = (i >> 3) & 1, bl = (i >> 4) & 1,
                pf = (i >> 5) & 1;
      v[i] = (uint16_t)((m0 & p1) | ((m0 & p0) << 1) | ((m1 & p0) << 2) | ((m1 & p1) << 3) | ((p0 & pf) << 4) |
                        ((p0 & bl) << 5) | ((p1 & pf) << 6) | ((p1 & bl) << 7) | ((m0 & pf) << 8) |
                        ((m0 & bl) << 9) | ((m1 & pf) << 10) | ((m1 & bl) << 11) | ((bl & pf) << 12) |
                        ((p0 & p1) << 14) | ((m0 & m1) << 15));
    }
  }
};
__constant__ PairTable kPairTable = PairTable();

// objects whose coverage words a register write changes (bits 0 P0, 1 P1, 2 M0, 3 M1, 4 BL,
// 5 PF): NUSIZ, CTRLPF, REFP, PF0-2, RESxx, GRP0/1 (and the VDEL copies), ENAx, VDELxx, RESMPx,
// HMOVE.  Colours, VBLANK, HMxx, HMCLR and CXCLR change none.
struct DirtyTable {
  uint8_t v[64];
  constexpr DirtyTable() : v() {
    v[0x04] = 1 | 4; v[0x05] = 2 | 8; v[0x0A] = 16 | 32; v[0x0B] = 1; v[0x0C] = 2;
    v[0x0D] = v[0x0E] = v[0x0F] = 32;
    v[0x10] = 1; v[0x11] = 2; v[0x12] = 4; v[0x13] = 8; v[0x14] = 16;
    v[0x1B] = 1 | 2; v[0x1C] = 1 | 2 | 16; v[0x1D] = 4; v[0x1E] = 8; v[0x1F] = 16;
    v[0x25] = 1; v[0x26] = 2; v[0x27] = 16; v[0x28] = 4; v[0x29] = 8; v[0x2A] = 1 | 2 | 4 | 8 | 16;
  }
};
__constant__ DirtyTable kDirtyTable = DirtyTable();

struct TiaP {
  uint32_t w0, w1, w2, w3, w4, w5, w6, w7, t;
  uint32_t pres;  // presence bits (0 P0, 1 P1, 2 M0, 3 M1, 4 BL, 5 PF), kept current by apply()
                  // (not stored in shared memory: recomputed at load)

  __device__ __forceinline__ uint32_t f(int b) const { return (w5 >> b) & 1u; }
  __device__ __forceinline__ void setf(int b, uint32_t v) { w5 = (w5 & ~(1u << b)) | ((v & 1u) << b); }
  __device__ __forceinline__ uint32_t coll() const { return w7 >> 16; }
  __device__ __forceinline__ int32_t comb_line() const { return (int32_t)(int16_t)(w5 >> 16); }
  // the presence bits travel in w7 byte 1 between replays (bit 15: valid; a state loaded from a
  // snapshot has none and computes them once)
  __device__ __forceinline__ void load(const uint32_t* tw) {
    w0 = tw[0]; w1 = tw[1]; w2 = tw[2]; w3 = tw[3]; w4 = tw[4]; w5 = tw[5]; w6 = tw[6]; w7 = tw[7]; t = tw[8];
    if (w7 & 0x8000u) pres = (w7 >> 8) & 0x3Fu;
    else pres = p0_on() | (p1_on() << 1) | (m0_on() << 2) | (m1_on() << 3) | (ball_on() << 4) | (pf_on() << 5);
  }
  __device__ __forceinline__ void store(uint32_t* tw) const {
    tw[0] = w0; tw[1] = w1; tw[2] = w2; tw[3] = w3; tw[4] = w4; tw[5] = w5; tw[6] = w6;
    tw[7] = (w7 & 0xFFFF00FFu) | 0x8000u | (pres << 8); tw[8] = t;
  }
  __device__ __forceinline__ uint32_t grp0() const { return byte_of(w2, f(7) ? 3 : 2); }
  __device__ __forceinline__ uint32_t grp1() const { return byte_of(w3, f(8) ? 1 : 0); }
  __device__ __forceinline__ uint32_t ball_on() const { return f(9) ? f(6) : f(5); }

  // presence of each object (an absent object cannot collide)
  __device__ __forceinline__ uint32_t p0_on() const { return grp0() != 0u ? 1u : 0u; }
  __device__ __forceinline__ uint32_t p1_on() const { return grp1() != 0u ? 1u : 0u; }
  __device__ __forceinline__ uint32_t m0_on() const { return f(3) & (f(10) ^ 1u); }
  __device__ __forceinline__ uint32_t m1_on() const { return f(4) & (f(11) ^ 1u); }
  __device__ __forceinline__ uint32_t pf_on() const { return (w1 & 0x00FFFFF0u) != 0u ? 1u : 0u; }  // PF0 D4-D7, PF1, PF2
  __device__ __forceinline__ void set_pres(int b, uint32_t on) { pres = (pres & ~(1u << b)) | (on << b); }
  // collision latches the objects present now could still set
  __device__ __forceinline__ uint32_t open_pairs() const { return kPairTable.v[pres] & ~coll(); }

  // apply a logged write at colour clock T (DESIGN.md §2 R#7-R#12)
  __device__ __forceinline__ void apply(uint32_t r, uint32_t v, uint32_t T, uint32_t delays) {
    switch (r) {
      case 0x01: setf(0, v >> 1); break;
      case 0x04: w2 = with_byte(w2, 0, v); break;
      case 0x05: w2 = with_byte(w2, 1, v); break;
      case 0x06: case 0x07: case 0x08: case 0x09: w0 = with_byte(w0, (int)(r - 6u), v); break;
      case 0x0A: w1 = with_byte(w1, 3, v); break;
      case 0x0B: setf(1, v >> 3); break;
      case 0x0C: setf(2, v >> 3); break;
      case 0x0D: case 0x0E: case 0x0F: w1 = with_byte(w1, (int)(r - 0x0Du), v); set_pres(5, pf_on()); break;
      case 0x10: case 0x11: case 0x12: case 0x13: case 0x14: {  // RESP0/1, RESM0/1, RESBL
        const int32_t hp = (int32_t)(T % 228u) - 68;
        const uint32_t base = r <= 0x11u ? 5u : 4u;
        const uint32_t p = hp < -2 ? base - 2u : (uint32_t)(hp + (int32_t)base) % 160u;
        if (r == 0x14u) w7 = with_byte(w7, 0, p);
        else w6 = with_byte(w6, (int)(r - 0x10u), p);
        // RESxx start delay (R#36): w4 byte 3, bits 0 P0 .. 3 M1, for the rest of this line
        if (CULE_DELAYS_ON(delays) && hp >= 0 && r != 0x14u) w4 |= 1u << (24u + (r - 0x10u));
      } break;
      case 0x1B:  // GRP0; GRP1 old <- new
        w2 = with_byte(w2, 2, v); w3 = with_byte(w3, 1, byte_of(w3, 0));
        set_pres(0, p0_on()); set_pres(1, p1_on());
        break;
      case 0x1C:  // GRP1; GRP0 old <- new; ENABL old <- new
        w3 = with_byte(w3, 0, v);
        w2 = with_byte(w2, 3, byte_of(w2, 2));
        setf(6, f(5));
        set_pres(0, p0_on()); set_pres(1, p1_on()); set_pres(4, ball_on());
        break;
      case 0x1D: setf(3, v >> 1); set_pres(2, m0_on()); break;
      case 0x1E: setf(4, v >> 1); set_pres(3, m1_on()); break;
      case 0x1F: setf(5, v >> 1); set_pres(4, ball_on()); break;
      case 0x20: w3 = with_byte(w3, 2, v >> 4); break;
      case 0x21: w3 = with_byte(w3, 3, v >> 4); break;
      case 0x22: case 0x23: case 0x24: w4 = with_byte(w4, (int)(r - 0x22u), v >> 4); break;
      case 0x25: setf(7, v); set_pres(0, p0_on()); break;
      case 0x26: setf(8, v); set_pres(1, p1_on()); break;
      case 0x27: setf(9, v); set_pres(4, ball_on()); break;
      case 0x28: case 0x29: {  // RESMP: the missile locks to its player's centre on release
        const int b = r == 0x28u ? 10 : 11;
        const uint32_t nv = (v >> 1) & 1u;
        if (f(b) && !nv) {
          const uint32_t md = byte_of(w2, r == 0x28u ? 0 : 1) & 7u;
          const uint32_t c = md == 5u ? 6u : (md == 7u ? 10u : 3u);
          const uint32_t pp = byte_of(w6, r == 0x28u ? 0 : 1);
          w6 = with_byte(w6, r == 0x28u ? 2 : 3, (pp + c) % 160u);
        }
        setf(b, nv);
        set_pres(2, m0_on()); set_pres(3, m1_on());
      } break;
      case 0x2A: {  // HMOVE
        auto mv = [](uint32_t p, uint32_t hm) -> uint32_t {
          const int32_t q = (int32_t)p - ((int32_t)(hm ^ 8u) - 8);
          return (uint32_t)(q < 0 ? q + 160 : (q >= 160 ? q - 160 : q));
        };
        const uint32_t p0 = mv(byte_of(w6, 0), byte_of(w3, 2)), p1 = mv(byte_of(w6, 1), byte_of(w3, 3));
        const uint32_t m0 = mv(byte_of(w6, 2), byte_of(w4, 0)), m1 = mv(byte_of(w6, 3), byte_of(w4, 1));
        w6 = p0 | (p1 << 8) | (m0 << 16) | (m1 << 24);
        w7 = with_byte(w7, 0, mv(byte_of(w7, 0), byte_of(w4, 2)));
        const uint32_t line = T / 228u, h = T - line * 228u;
        if (h < 68u) w5 = (w5 & 0xFFFFu) | ((line & 0xFFFFu) << 16);
      } break;
      case 0x2B: w3 &= 0x0000FFFFu; w4 &= 0xFF000000u; break;  // HMCLR (byte 3: RESxx start delay, R#36)
      case 0x2C: w7 &= 0xFFFFu; break;               // CXCLR
      default: break;
    }
  }
};

// word k (pixels 32k..32k+31) of a <=32-bit pattern placed at pos + copy offsets (circular 160)
__device__ __forceinline__ uint32_t obj_word(uint32_t k, uint32_t pat, uint32_t pos, uint32_t cps) {
  uint32_t w = 0u;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (!((cps >> c) & 1u)) continue;
    uint32_t p = pos + (c == 0 ? 0u : (8u << c));
    if (p >= 160u) p -= 160u;
    int32_t d = (int32_t)p - (int32_t)(32u * k);
    if (d < 0) d += 160;
    if (d < 32) w |= pat << d;
    if (d > 128) w |= pat >> (160 - d);
  }
  return w;
}

// coverage of the six objects in word k
struct Words { uint32_t p0, p1, m0, m1, bl, pf; };

// coverage words of the six objects in the lane's word k, recomputed only for the objects
// flagged in `dirty`; playfield: 20 cells per half (PF0 D4-D7, PF1 D7-D0, PF2 D0-D7), 4 px each.
// One obj_word call site in a (warp-uniform) loop over the five movable objects keeps the hot
// replay code small (the SM's instruction cache holds ~32 KB).
__device__ __forceinline__ void update_words(const TiaP& t, uint32_t k, Words& w, uint32_t dirty) {
  uint32_t todo = dirty & 31u;
#pragma unroll 1
  while (todo) {
    const uint32_t o = (uint32_t)__ffs(todo) - 1u;
    todo &= todo - 1u;
    const uint32_t idx = o & 1u;                       // P0/M0: 0, P1/M1: 1
    const uint32_t nusiz = byte_of(t.w2, (int)idx), mode = nusiz & 7u;
    uint32_t pat, pos, cps;
    if (o < 2u) {        // players: graphic (VDEL copy, reflection), scaled in modes 5/7
      const uint32_t g = idx ? t.grp1() : t.grp0();
      uint32_t q = t.f(1 + (int)idx) ? g : rev8(g);   // pixel d shows graphic bit 7-d (bit d reflected)
      q = mode == 5u ? spread2(q) : (mode == 7u ? spread4(q) : q);
      pat = g ? q : 0u;
      pos = byte_of(t.w6, (int)idx);
      cps = Tia::copies(mode) & ~((t.w4 >> (24u + o)) & 1u);  // RESxx start delay (R#36)
    } else if (o < 4u) { // missiles: enabled and not locked to the player; one copy in modes 5/7
      const bool en = t.f(3 + (int)idx) && !t.f(10 + (int)idx);
      pat = en ? (1u << (1u << ((nusiz >> 4) & 3u))) - 1u : 0u;
      pos = byte_of(t.w6, 2 + (int)idx);
      cps = ((mode == 5u || mode == 7u) ? 1u : Tia::copies(mode)) & ~((t.w4 >> (24u + o)) & 1u);
    } else {             // ball
      pat = t.ball_on() ? (1u << (1u << ((byte_of(t.w1, 3) >> 4) & 3u))) - 1u : 0u;
      pos = byte_of(t.w7, 0);
      cps = 1u;
    }
    const uint32_t v = pat ? obj_word(k, pat, pos, cps) : 0u;
    if (o == 0u) w.p0 = v;
    else if (o == 1u) w.p1 = v;
    else if (o == 2u) w.m0 = v;
    else if (o == 3u) w.m1 = v;
    else w.bl = v;
  }
  if (dirty & 32u) {
    const uint32_t left = ((byte_of(t.w1, 0) >> 4) & 0xFu) | (rev8(byte_of(t.w1, 1)) << 4) | (byte_of(t.w1, 2) << 12);
    const uint32_t right = (t.w1 & 0x01000000u) ? (__brev(left) >> 12) : left;
    const uint64_t cells = (uint64_t)left | ((uint64_t)right << 20);
    w.pf = spread4((uint32_t)(cells >> (8u * k)));
  }
}

// the row being assembled: lane j < 10 holds chunk j (pixels 16j..16j+15)
struct RowBuf {
  uint32_t r0, r1, r2, r3;
  uint32_t row;       // warp-uniform: window row held (rows before it are stored)
  uint32_t fill;      // black, replicated (palette 0 or gray[0])
  uint8_t* frame;     // 33,600-byte frame of this env (stored rows)
  bool render;
  // fused observation (GRAY84, last frame of the step): completed rows are not stored; each is
  // max-pooled with the same row of frame fs-1 (`prev`, staged in HBM; null for fs = 1) into a
  // 3-row ring in shared memory, and every 2.5 rows an 84-pixel output row is reduced from it
  uint8_t* obs84;     // u8[84][84] observation of this env, or null (store rows to `frame`)
  const uint8_t* prev;
  uint32_t ring_s;    // shared address of the 3 x 160-byte ring (per warp)
  uint32_t cols_s;    // shared address of the 84 packed column weights (per block, area84_col)
};

// column weights of output column j (0..83) of the exact area average, packed c0 | wc0 << 8 |
// wc1 << 16 | wc2 << 24: input columns c0..c0+2 with weights summing to 40 (40/21 per output
// column; kernels.cuh warp_area84 computes the same inline)
__device__ __forceinline__ uint32_t area84_col(uint32_t j) {
  const uint32_t a = 40u * j, b = a + 40u;
  const uint32_t c0 = a / 21u;
  const uint32_t wc0 = min(b, 21u * (c0 + 1)) - a;
  const uint32_t wc1 = min(b, 21u * (c0 + 2)) - 21u * (c0 + 1);
  const uint32_t wc2 = b > 21u * (c0 + 2) ? b - 21u * (c0 + 2) : 0u;
  return c0 | (wc0 << 8) | (wc1 << 16) | (wc2 << 24);
}

__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}

// shaded colour cache: 4 words (COLUP0, COLUP1, COLUPF, COLUBK) right after the warp's ring;
// every lane writes the same word, followed by a warp barrier before the next reads
constexpr uint32_t kShadeOff = 480;
__device__ __forceinline__ void shade_store(uint32_t a, uint32_t colu, const uint8_t* gray) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(Tia::shade(colu, gray)) : "memory");
}
__device__ __forceinline__ void shade_init(uint32_t shade_s, uint32_t w0, const uint8_t* gray) {
  for (uint32_t k = 0; k < 4; ++k) shade_store(shade_s + 4u * k, (w0 >> (8 * k)) & 0xFFu, gray);
}

// output row i (0..83) of the exact area average from input rows r0, r0+1, r0+2 of the ring
// (rows weighted 2:2:1 for even i, 1:2:2 for odd i; total weight 200, round half to even, R#17)
__device__ __noinline__ void area84_row(uint32_t ring_s, uint32_t cols_s, uint32_t r0, uint32_t i, uint8_t* out,
                                           uint32_t lane) {
  const uint32_t q0 = ring_s + (r0 % 3u) * 160u;
  const uint32_t q1 = ring_s + ((r0 + 1u) % 3u) * 160u;
  const uint32_t q2 = ring_s + ((r0 + 2u) % 3u) * 160u;
  const uint32_t w0 = (i & 1u) ? 1u : 2u, w2 = (i & 1u) ? 2u : 1u;
  uint8_t* orow = out + i * 84u;
  for (uint32_t j = lane; j < 84u; j += 32u) {
    uint32_t cw;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cw) : "r"(cols_s + 4u * j) : "memory");
    // the three weighted input columns c0..c0+2 of each row: two aligned words, a funnel shift
    // to bring byte c0 to the bottom, one dp4a with the packed weights wc0 | wc1 << 8 | wc2 << 16
    // (byte 3 weight 0; a zero-weight byte past the row end reads the next ring row or the
    // shaded-colour cache, both inside the warp's area)
    const uint32_t c0 = cw & 0xFFu, wpk = cw >> 8, a4 = c0 & ~3u, sh = 8u * (c0 & 3u);
    auto rowsum = [&](uint32_t q) {
      uint32_t lo, hi;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(lo) : "r"(q + a4) : "memory");
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(hi) : "r"(q + a4 + 4u) : "memory");
      return __dp4a(__funnelshift_r(lo, hi, sh), wpk, 0u);
    };
    const uint32_t s0 = rowsum(q0), s1 = rowsum(q1), s2 = rowsum(q2);
    const uint32_t S = w0 * s0 + 2u * s1 + w2 * s2;
    uint32_t q = S / 200u;
    const uint32_t r = S - 200u * q;
    q += (r > 100u || (r == 100u && (q & 1u))) ? 1u : 0u;
    orow[j] = (uint8_t)q;
  }
}

// a completed row of the fused frame: max with frame fs-1 into the ring; rows 5k+2 and 5k+4
// close output rows 2k and 2k+1 (rows 5k..5k+2 and 5k+2..5k+4)
__device__ __forceinline__ void fused_row(const RowBuf& rb, uint32_t lane) {
  const uint32_t r = rb.row;
  const uint32_t slot = r % 3u;
  if (lane < 10u) {
    uint4 m = make_uint4(rb.r0, rb.r1, rb.r2, rb.r3);
    if (rb.prev) {
      const uint4 q = reinterpret_cast<const uint4*>(rb.prev + r * 160u)[lane];
      // frame fs-1 streams from L2/HBM one row per completed row: prefetch four rows ahead into
      // L1 so the next rows' loads do not stall the replay
      if (r + 4u < (uint32_t)kFrameH)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(rb.prev + (r + 4u) * 160u + 16u * lane));
      m.x = __vmaxu4(m.x, q.x); m.y = __vmaxu4(m.y, q.y); m.z = __vmaxu4(m.z, q.z); m.w = __vmaxu4(m.w, q.w);
    }
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(rb.ring_s + slot * 160u + 16u * lane), "r"(m.x),
                 "r"(m.y), "r"(m.z), "r"(m.w) : "memory");
  }
  __syncwarp();
  const uint32_t k = r % 5u;
  if (k == 2u || k == 4u) {
    area84_row(rb.ring_s, rb.cols_s, r - 2u, 2u * (r / 5u) + (k == 4u ? 1u : 0u), rb.obs84, lane);
    __syncwarp();
  }
}

// collision bits of the visible pixels [a0, b0) U [a1, b1), reduced over the warp (even lanes
// 0..8 hold 32-pixel word lane/2)
__device__ __forceinline__ uint32_t range_bits(uint32_t lo, uint32_t xa, uint32_t xb) {
  const uint32_t s = xa > lo ? min(xa - lo, 32u) : 0u, e = xb > lo ? min(xb - lo, 32u) : 0u;
  return e > s ? ((e - s == 32u ? 0xFFFFFFFFu : ((1u << (e - s)) - 1u)) << s) : 0u;
}
__device__ __forceinline__ uint32_t collide_coop(const Words& w, uint32_t lane, uint32_t a0, uint32_t b0, uint32_t a1,
                                                 uint32_t b1) {
  uint32_t bits = 0u;
  if (lane < 10u && !(lane & 1u)) {
    const uint32_t lo = 16u * lane;
    const uint32_t r = range_bits(lo, a0, b0) | range_bits(lo, a1, b1);
    const uint32_t p0 = w.p0 & r, p1 = w.p1 & r, m0 = w.m0 & r, m1 = w.m1 & r, bl = w.bl & r, pf = w.pf & r;
    bits = ((m0 & p1) ? 1u : 0u) | ((m0 & p0) ? 2u : 0u) | ((m1 & p0) ? 4u : 0u) | ((m1 & p1) ? 8u : 0u) |
           ((p0 & pf) ? 0x10u : 0u) | ((p0 & bl) ? 0x20u : 0u) | ((p1 & pf) ? 0x40u : 0u) |
           ((p1 & bl) ? 0x80u : 0u) | ((m0 & pf) ? 0x100u : 0u) | ((m0 & bl) ? 0x200u : 0u) |
           ((m1 & pf) ? 0x400u : 0u) | ((m1 & bl) ? 0x800u : 0u) | ((bl & pf) ? 0x1000u : 0u) |
           ((p0 & p1) ? 0x4000u : 0u) | ((m0 & m1) ? 0x8000u : 0u);
  }
  return __reduce_or_sync(0xFFFFFFFFu, bits);
}

// the 16 pixels of the lane's chunk (4 words of 4 bytes) with the registers of the current span:
// priority (R#13) resolved on the chunk's 16-bit coverage masks into a 3-bit colour index per
// pixel, turned into byte-permute selectors (tia.cuh render_span does the same per lane)
__device__ __forceinline__ void chunk_px(const TiaP& t, const Words& w, uint32_t lane, uint32_t shade_s,
                                         uint32_t& x0w, uint32_t& x1w, uint32_t& x2w, uint32_t& x3w) {
  // the four shaded colour words (COLUP0, COLUP1, COLUPF, COLUBK), kept current by flush_coop
  uint32_t c0, c1, cbl, cbk;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(c0), "=r"(c1), "=r"(cbl), "=r"(cbk) : "r"(shade_s) : "memory");
  const uint32_t ctrlpf = byte_of(t.w1, 3);
  const uint32_t cp = (ctrlpf & 2u) ? (lane < 5u ? c0 : c1) : cbl;  // score mode: P0/P1 colour per half
  // permute source bytes: 0 background, 1 playfield, 2 P0/M0, 3 P1/M1, 4 ball (COLUPF)
  const uint32_t X = __byte_perm(__byte_perm(cbk, cp, 0x0040u), __byte_perm(c0, c1, 0x0040u), 0x5410u);
  const uint32_t hs = 16u * (lane & 1u);
  const uint32_t a = (w.p0 | w.m0) >> hs, b = (w.p1 | w.m1) >> hs, l = w.bl >> hs, f = w.pf >> hs;
  uint32_t e0, e1, eb, ep;
  if (!(ctrlpf & 4u)) {
    e0 = a; e1 = b & ~a; eb = l & ~(a | b); ep = f & ~(a | b | l);
  } else {
    eb = l; ep = f & ~l; e0 = a & ~(l | f); e1 = b & ~(l | f | a);
  }
  const uint32_t i0 = ep | e1, i1 = e0 | e1, i2 = eb;
  uint32_t sa = Tia::sel_bits(i0), sb = Tia::sel_bits(i0 >> 8);
  if ((i1 | i2) & 0xFFFFu) {  // (playfield-only chunks, the common case, need one index bit)
    sa |= (Tia::sel_bits(i1) << 1) | (Tia::sel_bits(i2) << 2);
    sb |= (Tia::sel_bits(i1 >> 8) << 1) | (Tia::sel_bits(i2 >> 8) << 2);
  }
  x0w = __byte_perm(X, cbl, sa);
  x1w = __byte_perm(X, cbl, sa >> 16);
  x2w = __byte_perm(X, cbl, sb);
  x3w = __byte_perm(X, cbl, sb >> 16);
}

// store the completed row and start the next
__device__ __forceinline__ void row_done(RowBuf& rb, uint32_t lane) {
  if (rb.obs84) fused_row(rb, lane);
  else if (lane < 10u) reinterpret_cast<uint4*>(rb.frame + rb.row * 160u)[lane] = make_uint4(rb.r0, rb.r1, rb.r2, rb.r3);
  rb.r0 = rb.r1 = rb.r2 = rb.r3 = rb.fill;
  ++rb.row;
}

// advance the warp-uniform TIA over colour clocks [t.t, t_to)
__device__ __forceinline__ void catch_up_coop(TiaP& t, uint32_t t_to, RowBuf& rb, uint32_t lane, uint32_t ystart,
                                              const uint8_t* gray, Words& w, uint32_t& dirty) {
  const uint32_t t0 = t.t;
  if (t_to <= t0) return;
  t.t = t_to;
  const bool vblank = t.f(0) != 0u;
  // frames that are not rendered only need collisions: nothing to do under VBLANK or when no
  // pair that is still unlatched can collide (cached until a presence register changes)
  if (!rb.render && (vblank || t.open_pairs() == 0u)) return;
  const uint32_t l0 = t0 / 228u, l1 = (t_to - 1) / 228u;
  const uint32_t h0 = t0 - l0 * 228u, h1 = t_to - l1 * 228u;
  const uint32_t xa0 = h0 > 68u ? h0 - 68u : 0u;
  const uint32_t xb1 = h1 > 68u ? h1 - 68u : 0u;
  // a span inside one line with no visible clock (e.g. writes right after WSYNC, in HBLANK)
  // neither collides nor draws, and cannot complete a row (that needs xb1 = 160 > xa0)
  if (l1 == l0 && xb1 <= xa0) return;
  const uint32_t w0 = ystart, w1 = ystart + (uint32_t)kFrameH;
  const bool any_win = rb.render && l1 >= w0 && l0 < w1;
  const bool need_coll = !vblank && t.open_pairs() != 0u;
  if (!need_coll && !any_win) return;
  // coverage words of the lane's 32-pixel word, recomputed only for objects whose registers
  // changed since (under VBLANK no object is drawn and no pair collides: the words are unused)
  if (!vblank && dirty) {
    update_words(t, lane < 10u ? (lane >> 1) : 0u, w, dirty);
    dirty = 0u;
  }
  if (need_coll) {  // collisions depend on x only: the union of the span's visible x ranges
    uint32_t a0 = xa0, b0 = 160u, a1 = 0u, b1 = xb1;   // two partial lines (l1 == l0 + 1)
    if (l1 > l0 + 1u || (l1 == l0 + 1u && xa0 <= xb1)) { a0 = 0u; b1 = 0u; }  // every x
    else if (l1 == l0) { b0 = xb1; b1 = 0u; }                                  // one line
    t.w7 |= collide_coop(w, lane, a0, b0, a1, b1) << 16;
  }
  if (!any_win) return;
  uint32_t x0w = rb.fill, x1w = rb.fill, x2w = rb.fill, x3w = rb.fill;
  if (!vblank && lane < 10u) chunk_px(t, w, lane, rb.ring_s + kShadeOff, x0w, x1w, x2w, x3w);
  const int32_t comb = vblank ? -1 : t.comb_line();
  const uint32_t la = l0 > w0 ? l0 : w0, lb = l1 < w1 - 1u ? l1 : w1 - 1u;
  const uint32_t cx = 16u * lane;
  for (uint32_t ln = la; ln <= lb; ++ln) {
    const uint32_t xa = ln == l0 ? xa0 : 0u, xb = ln == l1 ? xb1 : 160u;
    if (xb <= xa) continue;
    if (xa == 0u && xb == 160u && (int32_t)ln != comb) {
      // the whole line in one span (the common case once writes that change nothing are
      // dropped, R#37): every pixel of the chunk (lanes >= 10 hold the fill either way)
      rb.r0 = x0w; rb.r1 = x1w; rb.r2 = x2w; rb.r3 = x3w;
    } else {
      // pixels [xa, xb) of this lane's chunk [cx, cx+16) as a 16-bit mask (0 for lanes >= 10),
      // merged branch-free: bit k of the mask <-> byte k % 4 of word k / 4
      const uint32_t a = xa > cx ? min(xa - cx, 16u) : 0u, b = xb > cx ? min(xb - cx, 16u) : 0u;
      const uint32_t pm = b > a ? (0xFFFFu >> (16u - (b - a))) << a : 0u;
      const bool cb = (int32_t)ln == comb && lane == 0u;  // HMOVE comb: x < 8 black (R#11)
      const uint32_t p0 = cb ? rb.fill : x0w, p1 = cb ? rb.fill : x1w;
      const uint32_t m0 = nib_bytes(pm), m1 = nib_bytes(pm >> 4), m2 = nib_bytes(pm >> 8), m3 = nib_bytes(pm >> 12);
      rb.r0 = (rb.r0 & ~m0) | (p0 & m0);
      rb.r1 = (rb.r1 & ~m1) | (p1 & m1);
      rb.r2 = (rb.r2 & ~m2) | (x2w & m2);
      rb.r3 = (rb.r3 & ~m3) | (x3w & m3);
    }
    if (xb == 160u) row_done(rb, lane);
  }
}

// replay n entries of the warp's log, then (optionally) advance to t_final; returns collisions
__device__ __forceinline__ uint32_t flush_coop(uint32_t* tw, const uint32_t* lg, uint32_t n, bool fin,
                                               uint32_t t_final, RowBuf& rb, uint32_t lane, uint32_t ystart,
                                               const uint8_t* gray, uint32_t delays) {
  TiaP t;
  t.load(tw);
  Words w{0u, 0u, 0u, 0u, 0u, 0u};
  uint32_t dirty = 0x3Fu;
  // entries 0..n-1 (catch up to the write's effect clock, then apply it), then (fin) the final
  // catch-up to t_final; a RESxx start delay ends with its line: the catch-up stops there first
  // (one catch_up_coop call site)
  const uint32_t kend = fin ? n + 1u : n;
  for (uint32_t k = 0; k < kend;) {
    const uint32_t e = k < n ? lg[k] : (t_final << 14);
    const uint32_t T = e >> 14, r = (e >> 8) & 0x3Fu;
    uint32_t to = k < n ? effect_clock(T, r, delays) : T;
    bool line_end = false;
    if (CULE_DELAYS_ON(delays) && (t.w4 >> 24)) {
      const uint32_t le = (t.t / 228u + 1u) * 228u;
      if (to >= le) { to = le; line_end = true; }
    }
    catch_up_coop(t, to, rb, lane, ystart, gray, w, dirty);
    if (line_end) {  // the delayed first copies show again from the next line
      dirty |= t.w4 >> 24;
      t.w4 &= 0x00FFFFFFu;
      continue;
    }
    if (k == n) break;
    __syncwarp();  // reconverge: the register update is warp-uniform work, issued once
    t.apply(r, e & 0xFFu, T, delays);
    if (r - 6u < 4u) {  // COLUxx: refresh the shaded colour, ordered before any lane's next read
      shade_store(rb.ring_s + kShadeOff + 4u * (r - 6u), e & 0xFFu, gray);
      __syncwarp();
    }
    dirty |= kDirtyTable.v[r];
    ++k;
  }
  __syncwarp();
  if (lane == 0u) t.store(tw);
  __syncwarp();
  return t.coll();
}

// after the frame's last catch-up: store the partial row and black out the rows never reached
__device__ __noinline__ void finish_frame_coop(RowBuf& rb, uint32_t lane) {
  if (!rb.render) return;
  if (rb.obs84) {  // the partial row, then black rows, through the fused reduction
    while (rb.row < (uint32_t)kFrameH) row_done(rb, lane);
  } else if (rb.row < (uint32_t)kFrameH) {
    if (lane < 10u) reinterpret_cast<uint4*>(rb.frame + rb.row * 160u)[lane] = make_uint4(rb.r0, rb.r1, rb.r2, rb.r3);
    const uint32_t first = (rb.row + 1u) * 10u;
    uint4* p = reinterpret_cast<uint4*>(rb.frame);
    for (uint32_t q = first + lane; q < (uint32_t)kFrameChunks; q += 32u) p[q] = make_uint4(rb.fill, rb.fill, rb.fill, rb.fill);
  }
  rb.render = false;
}

}  // namespace cule
