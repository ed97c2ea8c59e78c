/*
 * cule_oracle.c — plain, slow, single-threaded CPU oracle for the CuLE hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Nothing in the product path may link or call it.
 *
 * It is the plain definition of "what the console does" under the written model of
 * SURVEY.md §8(c) (the paper, fixes none of the hardware details):
 *   - one instruction at a time, a big switch with every opcode's cycle count written out
 *     (SURVEY.md Appendix A);
 *   - all bus effects of an instruction at its end, T = 3(fc+n) colour clocks (§8(c).4);
 *   - the TIA advanced one colour clock at a time (§8(c).8), with every object's coverage
 *     evaluated from its definition at every visible clock;
 *   - the RIOT timer evaluated from its closed form (§8(c).5);
 *   - frames, steps, reward/done, reset cache and preprocessing exactly as §8(c).9-12.
 * No blocking, no caching of derived state, no bit tricks.  Where the paper or the survey is
 * silent the reading is listed in DESIGN.md §2 and cited here as [R#n].
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------ */
/* Machine state (§8(c).1)                                                                     */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
  /* CPU */
  uint8_t A, X, Y, SP, P;
  uint16_t PC;
  uint32_t fc; /* CPU cycles since frame-relative scanline 0 */
  uint8_t ram[128];
  /* TIA */
  uint8_t vsync, vblank, nusiz0, nusiz1, colup0, colup1, colupf, colubk, ctrlpf;
  uint8_t refp0, refp1, pf0, pf1, pf2, grp0new, grp0old, grp1new, grp1old;
  uint8_t enam0, enam1, enablnew, enablold, hmp0, hmp1, hmm0, hmm1, hmbl;
  uint8_t vdelp0, vdelp1, vdelbl, resmp0, resmp1;
  uint8_t posP0, posP1, posM0, posM1, posBL;
  uint16_t coll;
  int16_t comb_line;
  /* RIOT */
  uint8_t timer_v, timer_s;
  int32_t timer_w;
  uint8_t swcha, inpt4;
  /* cartridge */
  uint8_t bank;
  /* bookkeeping */
  uint8_t rom_id, fault;
  uint32_t episode_frames, episode_index;
  uint16_t prev_score;
  int32_t episode_return;
  /* transient (not in the snapshot) */
  uint32_t t_tia;      /* TIA position in colour clocks                                  */
  uint32_t now;        /* CPU cycle at which bus accesses currently sample                */
  int wsync_req;       /* WSYNC strobed during the current instruction                    */
  int vsync_rose;      /* VSYNC 0->1 during the current instruction                       */
  const uint8_t* rom;  /* cartridge image                                                 */
  size_t rom_len;
  int render;          /* write pixels during catch-up                                    */
  int ystart;
  uint8_t* fb;         /* 160x210 palette indices                                        */
  uint32_t last_lines; /* scanlines of the last completed frame (diagnostic)              */
  int tia_delays;      /* delayed register effects [R#35] (opt-in; 0 = every write at T)   */
  uint8_t res_delay;   /* [R#36] objects reset during the visible part of line res_line (bits
                          0 P0, 1 P1, 2 M0, 3 M1): their first copy is not drawn on that line */
  int res_line;
} Machine;

/* ---- snapshot layout --------------------------------------------------------- */
static void put16(uint8_t* p, uint32_t v) { p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); }
static void put32(uint8_t* p, uint32_t v) {
  p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); p[2] = (uint8_t)(v >> 16); p[3] = (uint8_t)(v >> 24);
}
static uint32_t get16(const uint8_t* p) { return (uint32_t)p[0] | ((uint32_t)p[1] << 8); }
static uint32_t get32(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

static void save_state(const Machine* m, uint8_t* s) {
  memset(s, 0, ORC_STATE_BYTES);
  s[0] = m->A; s[1] = m->X; s[2] = m->Y; s[3] = m->SP; s[4] = m->P; s[5] = m->bank;
  put16(s + 6, m->PC);
  put32(s + 8, m->fc);
  put32(s + 12, (uint32_t)m->timer_w);
  s[16] = m->timer_v; s[17] = m->timer_s; s[18] = m->swcha; s[19] = m->inpt4;
  put16(s + 20, m->coll);
  put16(s + 22, (uint16_t)m->comb_line);
  s[24] = m->vsync; s[25] = m->vblank; s[26] = m->nusiz0; s[27] = m->nusiz1;
  s[28] = m->colup0; s[29] = m->colup1; s[30] = m->colupf; s[31] = m->colubk;
  s[32] = m->ctrlpf; s[33] = m->refp0; s[34] = m->refp1; s[35] = m->pf0;
  s[36] = m->pf1; s[37] = m->pf2; s[38] = m->grp0new; s[39] = m->grp0old;
  s[40] = m->grp1new; s[41] = m->grp1old; s[42] = m->enam0; s[43] = m->enam1;
  s[44] = m->enablnew; s[45] = m->enablold; s[46] = m->hmp0; s[47] = m->hmp1;
  s[48] = m->hmm0; s[49] = m->hmm1; s[50] = m->hmbl; s[51] = m->vdelp0;
  s[52] = m->vdelp1; s[53] = m->vdelbl; s[54] = m->resmp0; s[55] = m->resmp1;
  s[56] = m->posP0; s[57] = m->posP1; s[58] = m->posM0; s[59] = m->posM1; s[60] = m->posBL;
  s[61] = m->rom_id; s[62] = m->fault;
  /* [R#36] byte 63: the start-delay bits, when they apply to the line the TIA is on */
  s[63] = (m->res_delay && m->res_line == (int)(m->t_tia / 228)) ? m->res_delay : 0;
  memcpy(s + 64, m->ram, 128);
  put32(s + 192, m->episode_frames);
  put32(s + 196, m->episode_index);
  put32(s + 200, (uint32_t)m->episode_return);
  put16(s + 204, m->prev_score);
}

static void load_state(Machine* m, const uint8_t* s) {
  m->A = s[0]; m->X = s[1]; m->Y = s[2]; m->SP = s[3]; m->P = s[4]; m->bank = s[5];
  m->PC = (uint16_t)get16(s + 6);
  m->fc = get32(s + 8);
  m->timer_w = (int32_t)get32(s + 12);
  m->timer_v = s[16]; m->timer_s = s[17]; m->swcha = s[18]; m->inpt4 = s[19];
  m->coll = (uint16_t)get16(s + 20);
  m->comb_line = (int16_t)get16(s + 22);
  m->vsync = s[24]; m->vblank = s[25]; m->nusiz0 = s[26]; m->nusiz1 = s[27];
  m->colup0 = s[28]; m->colup1 = s[29]; m->colupf = s[30]; m->colubk = s[31];
  m->ctrlpf = s[32]; m->refp0 = s[33]; m->refp1 = s[34]; m->pf0 = s[35];
  m->pf1 = s[36]; m->pf2 = s[37]; m->grp0new = s[38]; m->grp0old = s[39];
  m->grp1new = s[40]; m->grp1old = s[41]; m->enam0 = s[42]; m->enam1 = s[43];
  m->enablnew = s[44]; m->enablold = s[45]; m->hmp0 = s[46]; m->hmp1 = s[47];
  m->hmm0 = s[48]; m->hmm1 = s[49]; m->hmbl = s[50]; m->vdelp0 = s[51];
  m->vdelp1 = s[52]; m->vdelbl = s[53]; m->resmp0 = s[54]; m->resmp1 = s[55];
  m->posP0 = s[56]; m->posP1 = s[57]; m->posM0 = s[58]; m->posM1 = s[59]; m->posBL = s[60];
  m->rom_id = s[61]; m->fault = s[62];
  memcpy(m->ram, s + 64, 128);
  m->episode_frames = get32(s + 192);
  m->episode_index = get32(s + 196);
  m->episode_return = (int32_t)get32(s + 200);
  m->prev_score = (uint16_t)get16(s + 204);
  /* at every frame boundary the TIA has caught up with the CPU (§8(c).1) */
  m->t_tia = 3u * m->fc;
  m->now = m->fc;
  m->wsync_req = 0;
  m->vsync_rose = 0;
  m->res_delay = s[63] & 0x0F;
  m->res_line = (int)(m->t_tia / 228);
}

/* ------------------------------------------------------------------------------------------ */
/* TIA (§8(c).8)                                                                               */
/* ------------------------------------------------------------------------------------------ */
static int mod160(int v) { return ((v % 160) + 160) % 160; }

/* playfield bit at visible pixel x */
static int cover_pf(const Machine* m, int x) {
  int i;
  if (x < 80) i = x / 4;
  else if (m->ctrlpf & 1) i = 19 - (x - 80) / 4;  /* REF: mirrored right half */
  else i = (x - 80) / 4;
  if (i < 4) return (m->pf0 >> (4 + i)) & 1;
  if (i < 12) return (m->pf1 >> (11 - i)) & 1;
  return (m->pf2 >> (i - 12)) & 1;
}

/* NUSIZ modes: copy offsets and scale (§8(c).8 table) */
static int nusiz_offsets(int mode, int* off) {
  switch (mode) {
    case 0: off[0] = 0; return 1;
    case 1: off[0] = 0; off[1] = 16; return 2;
    case 2: off[0] = 0; off[1] = 32; return 2;
    case 3: off[0] = 0; off[1] = 16; off[2] = 32; return 3;
    case 4: off[0] = 0; off[1] = 64; return 2;
    case 5: off[0] = 0; return 1;
    case 6: off[0] = 0; off[1] = 32; off[2] = 64; return 3;
    default: off[0] = 0; return 1;
  }
}
static int nusiz_scale(int mode) { return mode == 5 ? 2 : (mode == 7 ? 4 : 1); }

static uint8_t reverse8(uint8_t g) {
  uint8_t r = 0;
  for (int b = 0; b < 8; b++)
    if (g & (1 << b)) r |= (uint8_t)(1 << (7 - b));
  return r;
}

static int cover_player(int x, uint8_t pos, uint8_t nusiz, uint8_t grp_new, uint8_t grp_old,
                        uint8_t vdel, uint8_t refl, int skip_first) {
  uint8_t g = vdel ? grp_old : grp_new;
  if (refl) g = reverse8(g);
  int mode = nusiz & 7, off[3];
  int n = nusiz_offsets(mode, off);
  int scale = nusiz_scale(mode);
  for (int k = skip_first ? 1 : 0; k < n; k++) {
    int d = mod160(x - pos - off[k]);
    if (d < 8 * scale && ((g >> (7 - d / scale)) & 1)) return 1;
  }
  return 0;
}

static int cover_missile(int x, uint8_t pos, uint8_t nusiz, uint8_t enam, uint8_t resmp, int skip_first) {
  if (!enam || resmp) return 0;
  int width = 1 << ((nusiz >> 4) & 3);
  int mode = nusiz & 7, off[3], n;
  if (mode == 5 || mode == 7) { off[0] = 0; n = 1; }
  else n = nusiz_offsets(mode, off);
  for (int k = skip_first ? 1 : 0; k < n; k++)
    if (mod160(x - pos - off[k]) < width) return 1;
  return 0;
}

static int cover_ball(const Machine* m, int x) {
  int en = m->vdelbl ? m->enablold : m->enablnew;
  if (!en) return 0;
  int width = 1 << ((m->ctrlpf >> 4) & 3);
  return mod160(x - m->posBL) < width;
}

/* one visible colour clock at pixel x on frame-relative line `line` */
static void tia_clock(Machine* m, int line, int x) {
  int in_window = m->render && line >= m->ystart && line < m->ystart + ORC_FB_H;
  if (m->vblank) {
    if (in_window) m->fb[(line - m->ystart) * ORC_FB_W + x] = 0;
    return; /* no collisions under VBLANK [R#12] */
  }
  /* [R#36] the first copy of an object reset during the visible part of this line is not drawn */
  int rd = (m->res_delay && line == m->res_line) ? m->res_delay : 0;
  int p0 = cover_player(x, m->posP0, m->nusiz0, m->grp0new, m->grp0old, m->vdelp0, m->refp0, rd & 1);
  int p1 = cover_player(x, m->posP1, m->nusiz1, m->grp1new, m->grp1old, m->vdelp1, m->refp1, rd & 2);
  int m0 = cover_missile(x, m->posM0, m->nusiz0, m->enam0, m->resmp0, rd & 4);
  int m1 = cover_missile(x, m->posM1, m->nusiz1, m->enam1, m->resmp1, rd & 8);
  int bl = cover_ball(m, x);
  int pf = cover_pf(m, x);
  /* collision latches, bit 2r = d7 and bit 2r+1 = d6 of read register r */
  if (m0 && p1) m->coll |= 1u << 0;
  if (m0 && p0) m->coll |= 1u << 1;
  if (m1 && p0) m->coll |= 1u << 2;
  if (m1 && p1) m->coll |= 1u << 3;
  if (p0 && pf) m->coll |= 1u << 4;
  if (p0 && bl) m->coll |= 1u << 5;
  if (p1 && pf) m->coll |= 1u << 6;
  if (p1 && bl) m->coll |= 1u << 7;
  if (m0 && pf) m->coll |= 1u << 8;
  if (m0 && bl) m->coll |= 1u << 9;
  if (m1 && pf) m->coll |= 1u << 10;
  if (m1 && bl) m->coll |= 1u << 11;
  if (bl && pf) m->coll |= 1u << 12;
  if (p0 && p1) m->coll |= 1u << 14;
  if (m0 && m1) m->coll |= 1u << 15;
  if (!in_window) return;
  uint8_t color;
  if (line == m->comb_line && x < 8) {
    color = 0; /* HMOVE comb [R#11] */
  } else {
    uint8_t pfc = (m->ctrlpf & 2) ? (x < 80 ? m->colup0 : m->colup1) : m->colupf;
    if (m->ctrlpf & 4) { /* PFP: playfield and ball above players */
      if (bl) color = m->colupf;
      else if (pf) color = pfc;
      else if (p0 || m0) color = m->colup0;
      else if (p1 || m1) color = m->colup1;
      else color = m->colubk;
    } else {
      if (p0 || m0) color = m->colup0;
      else if (p1 || m1) color = m->colup1;
      else if (bl) color = m->colupf;
      else if (pf) color = pfc;
      else color = m->colubk;
    }
    color = (uint8_t)(color >> 1);
  }
  m->fb[(line - m->ystart) * ORC_FB_W + x] = color;
}

/* advance the TIA over colour clocks [t_tia, t_to) with the current register values */
static void tia_catch_up(Machine* m, uint32_t t_to) {
  for (uint32_t t = m->t_tia; t < t_to; t++) {
    int line = (int)(t / 228);
    int h = (int)(t % 228);
    if (h >= 68) tia_clock(m, line, h - 68);
  }
  if (t_to > m->t_tia) m->t_tia = t_to;
}

static uint8_t tia_read(const Machine* m, int r) {
  if (r < 8)
    return (uint8_t)((((m->coll >> (2 * r)) & 1) << 7) | (((m->coll >> (2 * r + 1)) & 1) << 6));
  if (r == 0x0C) return m->inpt4;
  if (r == 0x0D) return 0x80;
  return 0; /* INPT0-3 and unused: 0, no open bus [R#14] */
}

static void tia_write(Machine* m, int r, uint8_t v) {
  uint32_t T = 3u * m->now;
  int line = (int)(T / 228);
  int h = (int)(T % 228);
  int hp = h - 68;
  if (m->tia_delays) {
    /* [R#35] a playfield register written at visible pixel x = h - 68 takes effect at the next
     * 4-pixel playfield cell boundary, 4*ceil(x/4); GRP0/GRP1 one colour clock after the
     * write; the TIA runs on with the old value until then (the clocks in between are drawn
     * and collide with it), then the write lands */
    if ((r == 0x0D || r == 0x0E || r == 0x0F) && hp > 0 && hp % 4 != 0)
      tia_catch_up(m, T + (uint32_t)(4 - hp % 4));
    else if (r == 0x1B || r == 0x1C)
      tia_catch_up(m, T + 1u);
  }
  switch (r) {
    case 0x00: { uint8_t nv = (v >> 1) & 1; if (!m->vsync && nv) m->vsync_rose = 1; m->vsync = nv; } break;
    case 0x01: m->vblank = (v >> 1) & 1; break;
    case 0x02: m->wsync_req = 1; break;
    case 0x03: break; /* RSYNC ignored [R#10] */
    case 0x04: m->nusiz0 = v; break;
    case 0x05: m->nusiz1 = v; break;
    case 0x06: m->colup0 = v; break;
    case 0x07: m->colup1 = v; break;
    case 0x08: m->colupf = v; break;
    case 0x09: m->colubk = v; break;
    case 0x0A: m->ctrlpf = v; break;
    case 0x0B: m->refp0 = (v >> 3) & 1; break;
    case 0x0C: m->refp1 = (v >> 3) & 1; break;
    case 0x0D: m->pf0 = v; break;
    case 0x0E: m->pf1 = v; break;
    case 0x0F: m->pf2 = v; break;
    case 0x10: m->posP0 = (uint8_t)(hp < -2 ? 3 : (hp + 5) % 160); break;
    case 0x11: m->posP1 = (uint8_t)(hp < -2 ? 3 : (hp + 5) % 160); break;
    case 0x12: m->posM0 = (uint8_t)(hp < -2 ? 2 : (hp + 4) % 160); break;
    case 0x13: m->posM1 = (uint8_t)(hp < -2 ? 2 : (hp + 4) % 160); break;
    case 0x14: m->posBL = (uint8_t)(hp < -2 ? 2 : (hp + 4) % 160); break;
    case 0x1B: m->grp0new = v; m->grp1old = m->grp1new; break;
    case 0x1C: m->grp1new = v; m->grp0old = m->grp0new; m->enablold = m->enablnew; break;
    case 0x1D: m->enam0 = (v >> 1) & 1; break;
    case 0x1E: m->enam1 = (v >> 1) & 1; break;
    case 0x1F: m->enablnew = (v >> 1) & 1; break;
    case 0x20: m->hmp0 = v >> 4; break;
    case 0x21: m->hmp1 = v >> 4; break;
    case 0x22: m->hmm0 = v >> 4; break;
    case 0x23: m->hmm1 = v >> 4; break;
    case 0x24: m->hmbl = v >> 4; break;
    case 0x25: m->vdelp0 = v & 1; break;
    case 0x26: m->vdelp1 = v & 1; break;
    case 0x27: m->vdelbl = v & 1; break;
    case 0x28: case 0x29: {
      uint8_t nv = (v >> 1) & 1;
      uint8_t* resmp = r == 0x28 ? &m->resmp0 : &m->resmp1;
      if (*resmp == 1 && nv == 0) {
        int mode = (r == 0x28 ? m->nusiz0 : m->nusiz1) & 7;
        int c = mode == 5 ? 6 : (mode == 7 ? 10 : 3);
        if (r == 0x28) m->posM0 = (uint8_t)((m->posP0 + c) % 160);
        else m->posM1 = (uint8_t)((m->posP1 + c) % 160);
      }
      *resmp = nv;
    } break;
    case 0x2A: { /* HMOVE: pos -= signed(HM) (a positive value moves left) */
      int d;
      d = m->hmp0 >= 8 ? m->hmp0 - 16 : m->hmp0; m->posP0 = (uint8_t)mod160(m->posP0 - d);
      d = m->hmp1 >= 8 ? m->hmp1 - 16 : m->hmp1; m->posP1 = (uint8_t)mod160(m->posP1 - d);
      d = m->hmm0 >= 8 ? m->hmm0 - 16 : m->hmm0; m->posM0 = (uint8_t)mod160(m->posM0 - d);
      d = m->hmm1 >= 8 ? m->hmm1 - 16 : m->hmm1; m->posM1 = (uint8_t)mod160(m->posM1 - d);
      d = m->hmbl >= 8 ? m->hmbl - 16 : m->hmbl; m->posBL = (uint8_t)mod160(m->posBL - d);
      if (h < 68) m->comb_line = (int16_t)line;
    } break;
    case 0x2B: m->hmp0 = m->hmp1 = m->hmm0 = m->hmm1 = m->hmbl = 0; break;
    case 0x2C: m->coll = 0; break;
    default: break; /* audio and $2D-$3F ignored */
  }
  if (m->tia_delays && r >= 0x10 && r <= 0x13 && hp >= 0) { /* [R#36] RESxx start delay */
    if (m->res_line != line) m->res_delay = 0;
    m->res_delay |= (uint8_t)(1u << (r - 0x10));
    m->res_line = line;
  }
}

/* ------------------------------------------------------------------------------------------ */
/* RIOT timer (§8(c).5): closed form from the write stamp, never ticked                       */
/* ------------------------------------------------------------------------------------------ */
static uint8_t timer_intim(const Machine* m) {
  int64_t e = (int64_t)m->now - (int64_t)m->timer_w;
  int64_t I = (int64_t)1 << m->timer_s;
  int64_t VI = (int64_t)m->timer_v * I;
  if (e <= VI) {
    int64_t dec = (e + I - 1) / I; /* ceil(e / I) */
    return (uint8_t)(m->timer_v - dec);
  }
  return (uint8_t)((0xFF - (e - VI - 1)) & 0xFF);
}
static uint8_t timer_timint(const Machine* m) {
  int64_t e = (int64_t)m->now - (int64_t)m->timer_w;
  int64_t VI = (int64_t)m->timer_v << m->timer_s;
  return e > VI ? 0x80 : 0x00;
}

/* ------------------------------------------------------------------------------------------ */
/* Bus (§8(c).3, cartridge §8(c).6)                                                           */
/* ------------------------------------------------------------------------------------------ */
/* Bank switching (Atari standard schemes; SURVEY.md §8(f) NEXT-4 widens the paper's 4K/F8):
 * F8 (8 KB, 2 banks): an access to $1FF8 / $1FF9 selects bank 0 / 1;
 * F6 (16 KB, 4 banks): $1FF6 .. $1FF9 select banks 0 .. 3;
 * F4 (32 KB, 8 banks): $1FF4 .. $1FFB select banks 0 .. 7.
 * 2K and 4K cartridges have no hotspots. */
static void cart_hotspot(Machine* m, uint16_t a) {
  switch (m->rom_len) {
    case 8192: if (a >= 0x1FF8 && a <= 0x1FF9) m->bank = (uint8_t)(a - 0x1FF8); break;
    case 16384: if (a >= 0x1FF6 && a <= 0x1FF9) m->bank = (uint8_t)(a - 0x1FF6); break;
    case 32768: if (a >= 0x1FF4 && a <= 0x1FFB) m->bank = (uint8_t)(a - 0x1FF4); break;
    default: break;
  }
}

static uint8_t rd(Machine* m, uint16_t addr) {
  uint16_t a = addr & 0x1FFF;
  if (a & 0x1000) {
    cart_hotspot(m, a);
    if (m->rom_len == 2048) return m->rom[a & 0x07FF]; /* 2K: mirrored twice in the window */
    return m->rom[(size_t)m->bank * 4096 + (a & 0x0FFF)];
  }
  if (!(a & 0x0080)) return tia_read(m, a & 0x0F);
  if (!(a & 0x0200)) return m->ram[a & 0x7F];
  if (!(a & 0x0004)) {
    switch (a & 3) {
      case 0: return m->swcha;
      case 1: return 0x00; /* SWACNT */
      case 2: return 0x0B; /* SWCHB: colour, reset/select released */
      default: return 0x00; /* SWBCNT */
    }
  }
  return (a & 1) ? timer_timint(m) : timer_intim(m);
}

static void wr(Machine* m, uint16_t addr, uint8_t v) {
  uint16_t a = addr & 0x1FFF;
  if (a & 0x1000) { cart_hotspot(m, a); return; }
  if (!(a & 0x0080)) { tia_write(m, a & 0x3F, v); return; }
  if (!(a & 0x0200)) { m->ram[a & 0x7F] = v; return; }
  if ((a & 0x0004) && (a & 0x0010)) {
    static const uint8_t shifts[4] = {0, 3, 6, 10};
    m->timer_v = v;
    m->timer_s = shifts[a & 3];
    m->timer_w = (int32_t)m->now;
  }
}

/* ------------------------------------------------------------------------------------------ */
/* 6502 (§8(c).4)                                                                              */
/* ------------------------------------------------------------------------------------------ */
enum { FC = 0x01, FZ = 0x02, FI = 0x04, FD = 0x08, FB = 0x10, FU = 0x20, FV = 0x40, FN = 0x80 };

static void setf(Machine* m, uint8_t f, int on) {
  if (on) m->P |= f; else m->P &= (uint8_t)~f;
}
static void setnz(Machine* m, uint8_t v) { setf(m, FZ, v == 0); setf(m, FN, v & 0x80); }

static uint8_t fetch(Machine* m) { uint8_t b = rd(m, m->PC); m->PC = (uint16_t)(m->PC + 1); return b; }

/* addressing modes (phase A: operand fetches and pointer reads) */
static uint16_t am_zp(Machine* m) { return fetch(m); }
static uint16_t am_zpx(Machine* m) { return (uint8_t)(fetch(m) + m->X); }
static uint16_t am_zpy(Machine* m) { return (uint8_t)(fetch(m) + m->Y); }
static uint16_t am_abs(Machine* m) { uint16_t lo = fetch(m); uint16_t hi = fetch(m); return (uint16_t)(lo | (hi << 8)); }
static uint16_t am_absx(Machine* m, int* cross) {
  uint16_t base = am_abs(m);
  uint16_t ea = (uint16_t)(base + m->X);
  *cross = (base & 0xFF00) != (ea & 0xFF00);
  return ea;
}
static uint16_t am_absy(Machine* m, int* cross) {
  uint16_t base = am_abs(m);
  uint16_t ea = (uint16_t)(base + m->Y);
  *cross = (base & 0xFF00) != (ea & 0xFF00);
  return ea;
}
static uint16_t am_indx(Machine* m) {
  uint8_t p = (uint8_t)(fetch(m) + m->X);
  uint16_t lo = rd(m, p);
  uint16_t hi = rd(m, (uint8_t)(p + 1));
  return (uint16_t)(lo | (hi << 8));
}
static uint16_t am_indy(Machine* m, int* cross) {
  uint8_t p = fetch(m);
  uint16_t lo = rd(m, p);
  uint16_t hi = rd(m, (uint8_t)(p + 1));
  uint16_t base = (uint16_t)(lo | (hi << 8));
  uint16_t ea = (uint16_t)(base + m->Y);
  *cross = (base & 0xFF00) != (ea & 0xFF00);
  return ea;
}

/* phase B: the instruction takes n cycles; catch the TIA up to its end, where accesses sample */
static void begin(Machine* m, int n) {
  m->now = m->fc + (uint32_t)n;
  tia_catch_up(m, 3u * m->now);
}

static void push(Machine* m, uint8_t v) { wr(m, (uint16_t)(0x0100 | m->SP), v); m->SP = (uint8_t)(m->SP - 1); }
static uint8_t pull(Machine* m) { m->SP = (uint8_t)(m->SP + 1); return rd(m, (uint16_t)(0x0100 | m->SP)); }

/* ALU */
static void op_adc(Machine* m, uint8_t v) {
  int c = m->P & FC;
  if (m->P & FD) {
    /* NMOS decimal ADC (Bruce Clark's sequences 1 and 2) [R#2] */
    int lo = (m->A & 0x0F) + (v & 0x0F) + c;
    if (lo >= 0x0A) lo = ((lo + 0x06) & 0x0F) + 0x10;
    int s = (m->A & 0xF0) + (v & 0xF0) + lo;
    int sa = (int)(int8_t)(m->A & 0xF0) + (int)(int8_t)(v & 0xF0) + lo;
    uint8_t bin = (uint8_t)(m->A + v + c);
    setf(m, FN, s & 0x80);
    setf(m, FV, sa < -128 || sa > 127);
    if (s >= 0xA0) s += 0x60;
    setf(m, FZ, bin == 0);
    setf(m, FC, s >= 0x100);
    m->A = (uint8_t)s;
  } else {
    int t = m->A + v + c;
    uint8_t r = (uint8_t)t;
    setf(m, FV, (~(m->A ^ v)) & (m->A ^ r) & 0x80);
    setf(m, FC, t > 0xFF);
    m->A = r;
    setnz(m, r);
  }
}
static void op_sbc(Machine* m, uint8_t v) {
  int c = m->P & FC;
  if (m->P & FD) {
    /* flags as in binary SBC; accumulator by Bruce Clark's sequence 3 [R#2] */
    int lo = (m->A & 0x0F) - (v & 0x0F) + c - 1;
    if (lo < 0) lo = ((lo - 0x06) & 0x0F) - 0x10;
    int s = (m->A & 0xF0) - (v & 0xF0) + lo;
    if (s < 0) s -= 0x60;
    int t = m->A + (v ^ 0xFF) + c;
    uint8_t r = (uint8_t)t;
    setf(m, FV, (~(m->A ^ (v ^ 0xFF))) & (m->A ^ r) & 0x80);
    setf(m, FC, t > 0xFF);
    setnz(m, r);
    m->A = (uint8_t)s;
  } else {
    op_adc(m, (uint8_t)(v ^ 0xFF));
  }
}
static void op_cmp(Machine* m, uint8_t reg, uint8_t v) {
  setf(m, FC, reg >= v);
  setf(m, FZ, reg == v);
  setf(m, FN, ((uint8_t)(reg - v)) & 0x80);
}
static void op_bit(Machine* m, uint8_t v) {
  setf(m, FN, v & 0x80);
  setf(m, FV, v & 0x40);
  setf(m, FZ, (m->A & v) == 0);
}
static uint8_t op_asl(Machine* m, uint8_t v) { setf(m, FC, v & 0x80); v = (uint8_t)(v << 1); setnz(m, v); return v; }
static uint8_t op_lsr(Machine* m, uint8_t v) { setf(m, FC, v & 0x01); v = (uint8_t)(v >> 1); setnz(m, v); return v; }
static uint8_t op_rol(Machine* m, uint8_t v) {
  int c = m->P & FC;
  setf(m, FC, v & 0x80);
  v = (uint8_t)((v << 1) | c);
  setnz(m, v);
  return v;
}
static uint8_t op_ror(Machine* m, uint8_t v) {
  int c = m->P & FC;
  setf(m, FC, v & 0x01);
  v = (uint8_t)((v >> 1) | (c << 7));
  setnz(m, v);
  return v;
}

static void branch(Machine* m, int cond) {
  int8_t off = (int8_t)fetch(m);
  int n = 2;
  uint16_t target = (uint16_t)(m->PC + off);
  if (cond) {
    n += 1;
    if ((target & 0xFF00) != (m->PC & 0xFF00)) n += 1;
  }
  begin(m, n);
  if (cond) m->PC = target;
}

/* read-class helper macros: phase A address, phase B timing (+page penalty), phase C read */
#define RD_ZP(N, BODY)   { uint16_t ea = am_zp(m); begin(m, N); uint8_t v = rd(m, ea); BODY; } break
#define RD_ZPX(N, BODY)  { uint16_t ea = am_zpx(m); begin(m, N); uint8_t v = rd(m, ea); BODY; } break
#define RD_ZPY(N, BODY)  { uint16_t ea = am_zpy(m); begin(m, N); uint8_t v = rd(m, ea); BODY; } break
#define RD_ABS(N, BODY)  { uint16_t ea = am_abs(m); begin(m, N); uint8_t v = rd(m, ea); BODY; } break
#define RD_ABSX(N, BODY) { int x_; uint16_t ea = am_absx(m, &x_); begin(m, N + x_); uint8_t v = rd(m, ea); BODY; } break
#define RD_ABSY(N, BODY) { int x_; uint16_t ea = am_absy(m, &x_); begin(m, N + x_); uint8_t v = rd(m, ea); BODY; } break
#define RD_INDX(N, BODY) { uint16_t ea = am_indx(m); begin(m, N); uint8_t v = rd(m, ea); BODY; } break
#define RD_INDY(N, BODY) { int x_; uint16_t ea = am_indy(m, &x_); begin(m, N + x_); uint8_t v = rd(m, ea); BODY; } break
#define RD_IMM(N, BODY)  { uint8_t v = fetch(m); begin(m, N); BODY; } break
/* fixed-count variants (no page penalty): stores, RMW, undocumented RMW */
#define FX_ABSX(N) { int x_; ea = am_absx(m, &x_); (void)x_; begin(m, N); }
#define FX_ABSY(N) { int x_; ea = am_absy(m, &x_); (void)x_; begin(m, N); }
#define FX_INDY(N) { int x_; ea = am_indy(m, &x_); (void)x_; begin(m, N); }

/* read-modify-write bodies: v = rd(ea); v = f(v); wr(ea, v) */
#define RMW(F)  { uint8_t v = rd(m, ea); v = F(m, v); wr(m, ea, v); } break
static uint8_t f_inc(Machine* m, uint8_t v) { v = (uint8_t)(v + 1); setnz(m, v); return v; }
static uint8_t f_dec(Machine* m, uint8_t v) { v = (uint8_t)(v - 1); setnz(m, v); return v; }
/* undocumented combined RMW ops (§8(c).4 table) */
static uint8_t f_slo(Machine* m, uint8_t v) { v = op_asl(m, v); m->A |= v; setnz(m, m->A); return v; }
static uint8_t f_rla(Machine* m, uint8_t v) { v = op_rol(m, v); m->A &= v; setnz(m, m->A); return v; }
static uint8_t f_sre(Machine* m, uint8_t v) { v = op_lsr(m, v); m->A ^= v; setnz(m, m->A); return v; }
static uint8_t f_rra(Machine* m, uint8_t v) { v = op_ror(m, v); op_adc(m, v); return v; }
static uint8_t f_dcp(Machine* m, uint8_t v) { v = (uint8_t)(v - 1); op_cmp(m, m->A, v); return v; }
static uint8_t f_isb(Machine* m, uint8_t v) { v = (uint8_t)(v + 1); op_sbc(m, v); return v; }

/* Execute one instruction.  Returns 0, or 1 for a JAM / unstable opcode (fault 1). */
static int exec_one(Machine* m) {
  m->now = m->fc;
  m->wsync_req = 0;
  m->vsync_rose = 0;
  uint8_t op = fetch(m);
  uint16_t ea;
  switch (op) {
    /* ---------------- loads ---------------- */
    case 0xA9: RD_IMM(2, m->A = v; setnz(m, v));
    case 0xA5: RD_ZP(3, m->A = v; setnz(m, v));
    case 0xB5: RD_ZPX(4, m->A = v; setnz(m, v));
    case 0xAD: RD_ABS(4, m->A = v; setnz(m, v));
    case 0xBD: RD_ABSX(4, m->A = v; setnz(m, v));
    case 0xB9: RD_ABSY(4, m->A = v; setnz(m, v));
    case 0xA1: RD_INDX(6, m->A = v; setnz(m, v));
    case 0xB1: RD_INDY(5, m->A = v; setnz(m, v));
    case 0xA2: RD_IMM(2, m->X = v; setnz(m, v));
    case 0xA6: RD_ZP(3, m->X = v; setnz(m, v));
    case 0xB6: RD_ZPY(4, m->X = v; setnz(m, v));
    case 0xAE: RD_ABS(4, m->X = v; setnz(m, v));
    case 0xBE: RD_ABSY(4, m->X = v; setnz(m, v));
    case 0xA0: RD_IMM(2, m->Y = v; setnz(m, v));
    case 0xA4: RD_ZP(3, m->Y = v; setnz(m, v));
    case 0xB4: RD_ZPX(4, m->Y = v; setnz(m, v));
    case 0xAC: RD_ABS(4, m->Y = v; setnz(m, v));
    case 0xBC: RD_ABSX(4, m->Y = v; setnz(m, v));
    /* LAX (undocumented) */
    case 0xA7: RD_ZP(3, m->A = m->X = v; setnz(m, v));
    case 0xB7: RD_ZPY(4, m->A = m->X = v; setnz(m, v));
    case 0xAF: RD_ABS(4, m->A = m->X = v; setnz(m, v));
    case 0xBF: RD_ABSY(4, m->A = m->X = v; setnz(m, v));
    case 0xA3: RD_INDX(6, m->A = m->X = v; setnz(m, v));
    case 0xB3: RD_INDY(5, m->A = m->X = v; setnz(m, v));
    /* ---------------- stores ---------------- */
    case 0x85: ea = am_zp(m); begin(m, 3); wr(m, ea, m->A); break;
    case 0x95: ea = am_zpx(m); begin(m, 4); wr(m, ea, m->A); break;
    case 0x8D: ea = am_abs(m); begin(m, 4); wr(m, ea, m->A); break;
    case 0x9D: FX_ABSX(5); wr(m, ea, m->A); break;
    case 0x99: FX_ABSY(5); wr(m, ea, m->A); break;
    case 0x81: ea = am_indx(m); begin(m, 6); wr(m, ea, m->A); break;
    case 0x91: FX_INDY(6); wr(m, ea, m->A); break;
    case 0x86: ea = am_zp(m); begin(m, 3); wr(m, ea, m->X); break;
    case 0x96: ea = am_zpy(m); begin(m, 4); wr(m, ea, m->X); break;
    case 0x8E: ea = am_abs(m); begin(m, 4); wr(m, ea, m->X); break;
    case 0x84: ea = am_zp(m); begin(m, 3); wr(m, ea, m->Y); break;
    case 0x94: ea = am_zpx(m); begin(m, 4); wr(m, ea, m->Y); break;
    case 0x8C: ea = am_abs(m); begin(m, 4); wr(m, ea, m->Y); break;
    /* SAX (undocumented): M = A & X */
    case 0x87: ea = am_zp(m); begin(m, 3); wr(m, ea, m->A & m->X); break;
    case 0x97: ea = am_zpy(m); begin(m, 4); wr(m, ea, m->A & m->X); break;
    case 0x8F: ea = am_abs(m); begin(m, 4); wr(m, ea, m->A & m->X); break;
    case 0x83: ea = am_indx(m); begin(m, 6); wr(m, ea, m->A & m->X); break;
    /* ---------------- logic / arithmetic ---------------- */
#define ALU_GROUP(B, BODY)                 \
    case (B) + 0x09: RD_IMM(2, BODY);      \
    case (B) + 0x05: RD_ZP(3, BODY);       \
    case (B) + 0x15: RD_ZPX(4, BODY);      \
    case (B) + 0x0D: RD_ABS(4, BODY);      \
    case (B) + 0x1D: RD_ABSX(4, BODY);     \
    case (B) + 0x19: RD_ABSY(4, BODY);     \
    case (B) + 0x01: RD_INDX(6, BODY);     \
    case (B) + 0x11: RD_INDY(5, BODY);
    ALU_GROUP(0x00, m->A |= v; setnz(m, m->A))
    ALU_GROUP(0x20, m->A &= v; setnz(m, m->A))
    ALU_GROUP(0x40, m->A ^= v; setnz(m, m->A))
    ALU_GROUP(0x60, op_adc(m, v))
    ALU_GROUP(0xC0, op_cmp(m, m->A, v))
    ALU_GROUP(0xE0, op_sbc(m, v))
#undef ALU_GROUP
    case 0xEB: RD_IMM(2, op_sbc(m, v)); /* undocumented SBC # */
    case 0xE0: RD_IMM(2, op_cmp(m, m->X, v));
    case 0xE4: RD_ZP(3, op_cmp(m, m->X, v));
    case 0xEC: RD_ABS(4, op_cmp(m, m->X, v));
    case 0xC0: RD_IMM(2, op_cmp(m, m->Y, v));
    case 0xC4: RD_ZP(3, op_cmp(m, m->Y, v));
    case 0xCC: RD_ABS(4, op_cmp(m, m->Y, v));
    case 0x24: RD_ZP(3, op_bit(m, v));
    case 0x2C: RD_ABS(4, op_bit(m, v));
    /* immediate-only undocumented */
    case 0x0B: case 0x2B: RD_IMM(2, m->A &= v; setnz(m, m->A); setf(m, FC, m->A & 0x80)); /* ANC */
    case 0x4B: RD_IMM(2, { uint8_t t = m->A & v; setf(m, FC, t & 1); m->A = (uint8_t)(t >> 1); setnz(m, m->A); }); /* ALR */
    case 0x6B: RD_IMM(2, { /* ARR, binary semantics even when D=1 [R#28] */
      uint8_t t = m->A & v;
      m->A = (uint8_t)((t >> 1) | ((m->P & FC) << 7));
      setnz(m, m->A);
      setf(m, FC, m->A & 0x40);
      setf(m, FV, ((m->A >> 6) ^ (m->A >> 5)) & 1);
    });
    case 0xCB: RD_IMM(2, { /* SBX: X = (A & X) - imm */
      uint8_t t = m->A & m->X;
      setf(m, FC, t >= v);
      m->X = (uint8_t)(t - v);
      setnz(m, m->X);
    });
    /* ---------------- shifts / rotates / inc / dec ---------------- */
    case 0x0A: begin(m, 2); m->A = op_asl(m, m->A); break;
    case 0x4A: begin(m, 2); m->A = op_lsr(m, m->A); break;
    case 0x2A: begin(m, 2); m->A = op_rol(m, m->A); break;
    case 0x6A: begin(m, 2); m->A = op_ror(m, m->A); break;
#define RMW_GROUP(B, F)                                            \
    case (B) + 0x06: ea = am_zp(m); begin(m, 5); RMW(F);           \
    case (B) + 0x16: ea = am_zpx(m); begin(m, 6); RMW(F);          \
    case (B) + 0x0E: ea = am_abs(m); begin(m, 6); RMW(F);          \
    case (B) + 0x1E: FX_ABSX(7); RMW(F);
    RMW_GROUP(0x00, op_asl)
    RMW_GROUP(0x40, op_lsr)
    RMW_GROUP(0x20, op_rol)
    RMW_GROUP(0x60, op_ror)
    RMW_GROUP(0xC0, f_dec)
    RMW_GROUP(0xE0, f_inc)
#undef RMW_GROUP
    /* undocumented RMW groups: zp 5, zp,X 6, abs 6, abs,X 7, abs,Y 7, (zp,X) 8, (zp),Y 8 */
#define URMW_GROUP(B, F)                                           \
    case (B) + 0x07: ea = am_zp(m); begin(m, 5); RMW(F);           \
    case (B) + 0x17: ea = am_zpx(m); begin(m, 6); RMW(F);          \
    case (B) + 0x0F: ea = am_abs(m); begin(m, 6); RMW(F);          \
    case (B) + 0x1F: FX_ABSX(7); RMW(F);                           \
    case (B) + 0x1B: FX_ABSY(7); RMW(F);                           \
    case (B) + 0x03: ea = am_indx(m); begin(m, 8); RMW(F);         \
    case (B) + 0x13: FX_INDY(8); RMW(F);
    URMW_GROUP(0x00, f_slo)
    URMW_GROUP(0x20, f_rla)
    URMW_GROUP(0x40, f_sre)
    URMW_GROUP(0x60, f_rra)
    URMW_GROUP(0xC0, f_dcp)
    URMW_GROUP(0xE0, f_isb)
#undef URMW_GROUP
    /* ---------------- register ops ---------------- */
    case 0xE8: begin(m, 2); m->X++; setnz(m, m->X); break;
    case 0xCA: begin(m, 2); m->X--; setnz(m, m->X); break;
    case 0xC8: begin(m, 2); m->Y++; setnz(m, m->Y); break;
    case 0x88: begin(m, 2); m->Y--; setnz(m, m->Y); break;
    case 0xAA: begin(m, 2); m->X = m->A; setnz(m, m->X); break;
    case 0xA8: begin(m, 2); m->Y = m->A; setnz(m, m->Y); break;
    case 0x8A: begin(m, 2); m->A = m->X; setnz(m, m->A); break;
    case 0x98: begin(m, 2); m->A = m->Y; setnz(m, m->A); break;
    case 0xBA: begin(m, 2); m->X = m->SP; setnz(m, m->X); break;
    case 0x9A: begin(m, 2); m->SP = m->X; break;
    case 0x18: begin(m, 2); setf(m, FC, 0); break;
    case 0x38: begin(m, 2); setf(m, FC, 1); break;
    case 0x58: begin(m, 2); setf(m, FI, 0); break;
    case 0x78: begin(m, 2); setf(m, FI, 1); break;
    case 0xB8: begin(m, 2); setf(m, FV, 0); break;
    case 0xD8: begin(m, 2); setf(m, FD, 0); break;
    case 0xF8: begin(m, 2); setf(m, FD, 1); break;
    /* ---------------- NOPs ---------------- */
    case 0xEA: case 0x1A: case 0x3A: case 0x5A: case 0x7A: case 0xDA: case 0xFA:
      begin(m, 2); break;
    case 0x80: case 0x82: case 0x89: case 0xC2: case 0xE2: RD_IMM(2, (void)v);
    case 0x04: case 0x44: case 0x64: RD_ZP(3, (void)v);
    case 0x14: case 0x34: case 0x54: case 0x74: case 0xD4: case 0xF4: RD_ZPX(4, (void)v);
    case 0x0C: RD_ABS(4, (void)v);
    case 0x1C: case 0x3C: case 0x5C: case 0x7C: case 0xDC: case 0xFC: RD_ABSX(4, (void)v);
    /* ---------------- stack ---------------- */
    case 0x48: begin(m, 3); push(m, m->A); break;
    case 0x08: begin(m, 3); push(m, (uint8_t)(m->P | FB | FU)); break;
    case 0x68: begin(m, 4); m->A = pull(m); setnz(m, m->A); break;
    case 0x28: begin(m, 4); m->P = (uint8_t)((pull(m) & ~(FB | FU)) | FU); break;
    /* ---------------- control flow ---------------- */
    case 0x4C: { uint16_t t = am_abs(m); begin(m, 3); m->PC = t; } break;
    case 0x6C: {
      uint16_t ptr = am_abs(m);
      uint16_t lo = rd(m, ptr);
      uint16_t hi = rd(m, (uint16_t)((ptr & 0xFF00) | ((ptr + 1) & 0x00FF))); /* page-wrap bug */
      begin(m, 5);
      m->PC = (uint16_t)(lo | (hi << 8));
    } break;
    case 0x20: {
      uint16_t lo = fetch(m);
      /* JSR pushes the address of its last byte (PC+2 from the opcode) */
      uint16_t ret = m->PC;
      uint16_t hi = fetch(m);
      begin(m, 6);
      push(m, (uint8_t)(ret >> 8));
      push(m, (uint8_t)ret);
      m->PC = (uint16_t)(lo | (hi << 8));
    } break;
    case 0x60: {
      begin(m, 6);
      uint16_t lo = pull(m);
      uint16_t hi = pull(m);
      m->PC = (uint16_t)((lo | (hi << 8)) + 1);
    } break;
    case 0x40: {
      begin(m, 6);
      m->P = (uint8_t)((pull(m) & ~(FB | FU)) | FU);
      uint16_t lo = pull(m);
      uint16_t hi = pull(m);
      m->PC = (uint16_t)(lo | (hi << 8));
    } break;
    case 0x00: {
      uint16_t ret = (uint16_t)(m->PC + 1); /* BRK pushes PC+2 from the opcode */
      begin(m, 7);
      push(m, (uint8_t)(ret >> 8));
      push(m, (uint8_t)ret);
      push(m, (uint8_t)(m->P | FB | FU));
      setf(m, FI, 1);
      uint16_t lo = rd(m, 0x1FFE);
      uint16_t hi = rd(m, 0x1FFF);
      m->PC = (uint16_t)(lo | (hi << 8));
    } break;
    case 0x10: branch(m, !(m->P & FN)); break;
    case 0x30: branch(m, m->P & FN); break;
    case 0x50: branch(m, !(m->P & FV)); break;
    case 0x70: branch(m, m->P & FV); break;
    case 0x90: branch(m, !(m->P & FC)); break;
    case 0xB0: branch(m, m->P & FC); break;
    case 0xD0: branch(m, !(m->P & FZ)); break;
    case 0xF0: branch(m, m->P & FZ); break;
    /* ---------------- faults: 12 JAM + 8 unstable (§8(c).4, [R#1]) ---------------- */
    default:
      return 1;
  }
  m->fc = m->now;
  if (m->wsync_req) m->fc = ((m->fc + 75) / 76) * 76; /* stall to the next line start [R#5] */
  m->now = m->fc;
  return 0;
}

/* end the frame at the VSYNC edge: catch the TIA up, rebase clocks to the VSYNC line (§8(c).9) */
static void end_frame(Machine* m) {
  tia_catch_up(m, 3u * m->fc);
  uint32_t L = m->fc / 76;
  m->last_lines = L;
  m->fc -= 76 * L;
  m->timer_w -= (int32_t)(76 * L);
  m->t_tia -= 228 * L;
  m->res_line -= (int)L;
  int cl = (int)m->comb_line - (int)L;
  m->comb_line = (int16_t)(cl < 0 ? -1 : cl);
  /* canonical timer stamp (§8(c).5) */
  int64_t e = (int64_t)m->fc - (int64_t)m->timer_w;
  int64_t VI = (int64_t)m->timer_v << m->timer_s;
  if (e > VI) {
    int64_t d = (e - VI - 1) % 256;
    m->timer_w = (int32_t)((int64_t)m->fc - (VI + 1 + d));
  }
  m->now = m->fc;
}

/* Run instructions until the frame ends, a fault, or max_instr (<0: unlimited).
 * Returns 0 (budget), 1 (JAM), 2 (runaway), 3 (frame ended). */
static int run(Machine* m, int line_cap, long max_instr, int64_t* icount) {
  long n = 0;
  for (;;) {
    if (max_instr >= 0 && n >= max_instr) {
      tia_catch_up(m, 3u * m->fc);
      return 0;
    }
    int f = exec_one(m);
    /* on a fault the TIA is still caught up to the CPU clock (R#26) */
    if (f) { m->fault = 1; tia_catch_up(m, 3u * m->fc); if (icount) *icount += n; return 1; }
    n++;
    if ((int)(m->fc / 76) >= line_cap) {
      m->fault = 2; tia_catch_up(m, 3u * m->fc); if (icount) *icount += n; return 2;
    }
    if (m->vsync_rose) { end_frame(m); if (icount) *icount += n; return 3; }
  }
}

static void bind(Machine* m, const uint8_t* rom, size_t rom_len) { m->rom = rom; m->rom_len = rom_len; }

static void power_on(Machine* m, const uint8_t* rom, size_t rom_len) {
  memset(m, 0, sizeof(*m));
  bind(m, rom, rom_len);
  m->SP = 0xFD;
  m->P = 0x24;
  m->bank = (uint8_t)(rom_len > 4096 ? rom_len / 4096 - 1 : 0); /* last bank [R#23] */
  m->timer_s = 10;
  m->timer_v = 0;
  m->timer_w = 0;
  m->swcha = 0xFF;
  m->inpt4 = 0x80;
  m->comb_line = -1;
  uint16_t lo = rd(m, 0x1FFC);
  uint16_t hi = rd(m, 0x1FFD);
  m->PC = (uint16_t)(lo | (hi << 8));
}

/* action -> input latches (§8(c).7, ALE action order) */
static void latch_inputs(Machine* m, int action) {
  int up = 0, down = 0, left = 0, right = 0, fire = 0;
  switch (action) {
    case 1: fire = 1; break;
    case 2: up = 1; break;
    case 3: right = 1; break;
    case 4: left = 1; break;
    case 5: down = 1; break;
    case 6: up = right = 1; break;
    case 7: up = left = 1; break;
    case 8: down = right = 1; break;
    case 9: down = left = 1; break;
    case 10: up = fire = 1; break;
    case 11: right = fire = 1; break;
    case 12: left = fire = 1; break;
    case 13: down = fire = 1; break;
    case 14: up = right = fire = 1; break;
    case 15: up = left = fire = 1; break;
    case 16: down = right = fire = 1; break;
    case 17: down = left = fire = 1; break;
    default: break; /* 0 NOOP, >= 18 treated as NOOP */
  }
  uint8_t sw = 0xFF;
  if (right) sw &= 0x7F;
  if (left) sw &= 0xBF;
  if (down) sw &= 0xDF;
  if (up) sw &= 0xEF;
  m->swcha = sw;
  m->inpt4 = fire ? 0x00 : 0x80;
}

static int valid_rom_len(size_t n) { return n == 2048 || n == 4096 || n == 8192 || n == 16384 || n == 32768; }

/* ------------------------------------------------------------------------------------------ */
/* machine-level C-ABI                                                                         */
/* ------------------------------------------------------------------------------------------ */
int orc_power_on(const uint8_t* rom, size_t rom_len, uint8_t* state) {
  if (!valid_rom_len(rom_len)) return -1;
  Machine m;
  power_on(&m, rom, rom_len);
  save_state(&m, state);
  return 0;
}

int orc_exec(const uint8_t* rom, size_t rom_len, uint8_t* state, int n_instr, int line_cap,
             int64_t* cycles_out) {
  if (!valid_rom_len(rom_len)) return -1;
  Machine m;
  memset(&m, 0, sizeof m);
  load_state(&m, state);
  bind(&m, rom, rom_len);
  uint32_t fc0 = m.fc;
  int r = run(&m, line_cap, n_instr, NULL);
  if (cycles_out) *cycles_out = (int64_t)m.fc - (int64_t)fc0;
  save_state(&m, state);
  return r;
}

int orc_run_frame(const uint8_t* rom, size_t rom_len, uint8_t* state, int action, int ystart,
                  int line_cap, uint8_t* fb, int64_t* instr_out, int64_t* lines_out) {
  return orc_run_frame_ex(rom, rom_len, state, action, ystart, line_cap, fb, instr_out, lines_out, 0);
}

int orc_run_frame_ex(const uint8_t* rom, size_t rom_len, uint8_t* state, int action, int ystart,
                     int line_cap, uint8_t* fb, int64_t* instr_out, int64_t* lines_out, int tia_delays) {
  if (!valid_rom_len(rom_len)) return -1;
  Machine m;
  memset(&m, 0, sizeof m);
  load_state(&m, state);
  bind(&m, rom, rom_len);
  m.tia_delays = tia_delays;
  if (action >= 0) latch_inputs(&m, action);
  m.render = fb != NULL;
  m.ystart = ystart;
  m.fb = fb;
  if (fb) memset(fb, 0, ORC_FB_W * ORC_FB_H);
  int64_t ic = 0;
  int r = run(&m, line_cap, -1, &ic);
  if (instr_out) *instr_out = ic;
  if (lines_out) *lines_out = r == 3 ? (int64_t)m.last_lines : -1;
  save_state(&m, state);
  return r == 3 ? 0 : r;
}

/* ------------------------------------------------------------------------------------------ */
/* preprocessing (§8(c).12)                                                                    */
/* ------------------------------------------------------------------------------------------ */
void orc_gray_lut(const uint8_t* rgb, uint8_t* gray) {
  for (int i = 0; i < 128; i++) {
    int r = rgb[3 * i], g = rgb[3 * i + 1], b = rgb[3 * i + 2];
    gray[i] = (uint8_t)((299 * r + 587 * g + 114 * b + 500) / 1000); /* ITU-R 601, half-up */
  }
}

/* length of the overlap of [a0, a1) and [b0, b1) */
static int overlap(int a0, int a1, int b0, int b1) {
  int lo = a0 > b0 ? a0 : b0, hi = a1 < b1 ? a1 : b1;
  return hi > lo ? hi - lo : 0;
}

/* Exact area average 160x210 -> 84x84.  In units where an input row is 2 long and an output row
 * 5 long (210*2 = 84*5), and an input column 21 long and an output column 40 long
 * (160*21 = 84*40), the weight of input (r,c) in output (i,j) is the product of the overlaps;
 * the weights of one output sum to 5*40 = 200.  Round half to even [R#17]. */
void orc_area84(const uint8_t* g, uint8_t* out) {
  for (int i = 0; i < 84; i++) {
    for (int j = 0; j < 84; j++) {
      long S = 0;
      for (int r = (5 * i) / 2; r <= (5 * i + 4) / 2 && r < 210; r++) {
        int wr = overlap(5 * i, 5 * i + 5, 2 * r, 2 * r + 2);
        for (int c = (40 * j) / 21; c <= (40 * j + 39) / 21 && c < 160; c++) {
          int wc = overlap(40 * j, 40 * j + 40, 21 * c, 21 * c + 21);
          S += (long)wr * wc * g[r * 160 + c];
        }
      }
      long q = S / 200, rem = S % 200;
      if (rem > 100 || (rem == 100 && (q & 1))) q++;
      out[i * 84 + j] = (uint8_t)q;
    }
  }
}

/* ------------------------------------------------------------------------------------------ */
/* RNG (§8(c).11)                                                                              */
/* ------------------------------------------------------------------------------------------ */
uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
uint64_t orc_hash2(uint64_t a, uint64_t b) { return orc_splitmix64(a ^ orc_splitmix64(b)); }

/* ------------------------------------------------------------------------------------------ */
/* environment-level C-ABI                                                                     */
/* ------------------------------------------------------------------------------------------ */
struct orc_env {
  orc_config cfg;
  int n_roms, num_envs, fs;
  uint8_t* roms[4];
  size_t rom_lens[4];
  uint8_t gray[128];
  int obs_bytes;
  /* reset cache */
  uint8_t* cache_state;  /* [n_roms*K][256] */
  uint8_t* cache_obs;    /* [n_roms*K][obs_bytes] */
  uint16_t* cache_score; /* [n_roms*K] */
  /* envs */
  uint8_t* states;       /* [N][256] */
  int64_t* gids;
  uint64_t pick_seed;
  int64_t counters[4];
  uint8_t* fbA;
  uint8_t* fbB;
  uint8_t* gbuf;
};

void orc_default_config(orc_config* c) {
  memset(c, 0, sizeof(*c));
  c->obs_mode = 1;
  c->reset_cache_size = 30;
  c->startup_frames = 64;
  c->max_random_frames = 30;
  c->max_episode_frames = 0;
  c->line_cap = 1024;
  c->ystart = 34;
  c->score_addr = 0x80;
  c->term_addr = 0x82;
  c->term_mask = 0x01;
  c->seed = 0;
  c->env_index_base = 0;
}

static int bcd(uint8_t b) { return 10 * (b >> 4) + (b & 0x0F); }
static uint16_t score_of(const orc_config* c, const uint8_t* ram) {
  return (uint16_t)(100 * bcd(ram[c->score_addr & 0x7F]) + bcd(ram[(c->score_addr + 1) & 0x7F]));
}

/* obs from rendered frames: raw = last frame; gray84 = area84(max(gray A, gray B)) */
static void make_obs(orc_env* e, int nframes, uint8_t* obs) {
  if (e->cfg.obs_mode == 0) {
    if (nframes >= 1) memcpy(obs, e->fbB, ORC_FB_W * ORC_FB_H);
    else memset(obs, 0, ORC_FB_W * ORC_FB_H);
    return;
  }
  if (nframes == 0) { memset(obs, 0, 84 * 84); return; }
  for (int p = 0; p < ORC_FB_W * ORC_FB_H; p++) {
    uint8_t b = e->gray[e->fbB[p] & 0x7F];
    if (nframes >= 2) {
      uint8_t a = e->gray[e->fbA[p] & 0x7F];
      if (a > b) b = a;
    }
    e->gbuf[p] = b;
  }
  orc_area84(e->gbuf, obs);
}

/* run `nframes` frames with fixed inputs, rendering the last one (raw) or two (gray84) */
static int run_frames(orc_env* e, Machine* m, int nframes, int* rendered) {
  *rendered = 0;
  for (int f = 1; f <= nframes; f++) {
    int render = e->cfg.obs_mode == 0 ? (f == nframes) : (f >= nframes - 1);
    uint8_t* fb = NULL;
    if (render) {
      fb = (f == nframes) ? e->fbB : e->fbA;
      memset(fb, 0, ORC_FB_W * ORC_FB_H);
      (*rendered)++;
    }
    m->render = render;
    m->ystart = e->cfg.ystart;
    m->fb = fb;
    m->tia_delays = e->cfg.tia_delays;
    m->episode_frames++;
    int r = run(m, e->cfg.line_cap, -1, NULL);
    m->render = 0;
    m->fb = NULL;
    if (r == 1 || r == 2) return r;
  }
  return 0;
}

static void copy_machine_part(uint8_t* dst, const uint8_t* src) {
  memcpy(dst, src, 61);           /* CPU, clock, timer, inputs, TIA, positions */
  dst[63] = src[63];              /* RESxx start-delay bits [R#36] */
  memcpy(dst + 64, src + 64, 128); /* RAM */
}

orc_env* orc_create(const uint8_t* const* roms, const size_t* rom_lens, int n_roms, int num_envs,
                    int frameskip, const orc_config* cfg, const uint8_t* palette_rgb, int* err) {
  *err = 0;
  if (!roms || !rom_lens || !cfg || !palette_rgb || n_roms < 1 || n_roms > 4 || num_envs <= 0 ||
      frameskip < 1 || cfg->reset_cache_size < 1 || cfg->startup_frames < 0 ||
      cfg->max_random_frames < 0 || cfg->line_cap < 1 || cfg->ystart < 0 ||
      cfg->ystart + ORC_FB_H > cfg->line_cap || (cfg->obs_mode != 0 && cfg->obs_mode != 1) ||
      cfg->score_addr < 0x80 || cfg->score_addr == 0xFF || cfg->term_addr < 0x80) {
    *err = -1;
    return NULL;
  }
  for (int r = 0; r < n_roms; r++)
    if (!roms[r] || !valid_rom_len(rom_lens[r])) { *err = -2; return NULL; }
  orc_env* e = (orc_env*)calloc(1, sizeof(orc_env));
  e->cfg = *cfg;
  e->n_roms = n_roms;
  e->num_envs = num_envs;
  e->fs = frameskip;
  for (int r = 0; r < n_roms; r++) {
    e->roms[r] = (uint8_t*)malloc(rom_lens[r]);
    memcpy(e->roms[r], roms[r], rom_lens[r]);
    e->rom_lens[r] = rom_lens[r];
  }
  orc_gray_lut(palette_rgb, e->gray);
  e->obs_bytes = cfg->obs_mode == 0 ? ORC_FB_W * ORC_FB_H : 84 * 84;
  int K = cfg->reset_cache_size;
  e->cache_state = (uint8_t*)calloc((size_t)n_roms * K, ORC_STATE_BYTES);
  e->cache_obs = (uint8_t*)calloc((size_t)n_roms * K, (size_t)e->obs_bytes);
  e->cache_score = (uint16_t*)calloc((size_t)n_roms * K, sizeof(uint16_t));
  e->states = (uint8_t*)calloc((size_t)num_envs, ORC_STATE_BYTES);
  e->gids = (int64_t*)malloc(sizeof(int64_t) * (size_t)num_envs);
  for (int i = 0; i < num_envs; i++) e->gids[i] = cfg->env_index_base + i;
  e->fbA = (uint8_t*)calloc(ORC_FB_W * ORC_FB_H, 1);
  e->fbB = (uint8_t*)calloc(ORC_FB_W * ORC_FB_H, 1);
  e->gbuf = (uint8_t*)calloc(ORC_FB_W * ORC_FB_H, 1);
  /* reset cache: power-on, then startup + u_k NOOP frames (§8(c).11) */
  for (int r = 0; r < n_roms; r++) {
    for (int k = 0; k < K; k++) {
      uint64_t u = orc_hash2(cfg->seed ^ 0x5245534554434143ull, ((uint64_t)r << 32) | (uint64_t)k) %
                   (uint64_t)(cfg->max_random_frames + 1);
      int nframes = cfg->startup_frames + (int)u;
      Machine m;
      power_on(&m, e->roms[r], e->rom_lens[r]);
      latch_inputs(&m, 0);
      int rendered;
      int fr = run_frames(e, &m, nframes, &rendered);
      if (fr) { *err = -3; orc_destroy(e); return NULL; }
      uint8_t snap[ORC_STATE_BYTES];
      save_state(&m, snap);
      size_t idx = (size_t)r * K + k;
      memset(e->cache_state + idx * ORC_STATE_BYTES, 0, ORC_STATE_BYTES);
      copy_machine_part(e->cache_state + idx * ORC_STATE_BYTES, snap);
      make_obs(e, rendered, e->cache_obs + idx * e->obs_bytes);
      e->cache_score[idx] = score_of(cfg, m.ram);
    }
  }
  return e;
}

int orc_set_env_ids(orc_env* e, const int64_t* gids) {
  for (int i = 0; i < e->num_envs; i++) e->gids[i] = gids[i];
  return 0;
}

static int rom_of(const orc_env* e, int64_t g) { return (int)(g % e->n_roms); }
static int pick(const orc_env* e, int64_t g, uint32_t ep) {
  return (int)(orc_hash2(orc_hash2(e->pick_seed, (uint64_t)g), (uint64_t)ep) %
               (uint64_t)e->cfg.reset_cache_size);
}

/* env i <- cache entry; bookkeeping per §8(c).10 step 6 / §8(c).11 */
static void restore_entry(orc_env* e, int i, uint32_t episode_index) {
  int64_t g = e->gids[i];
  int r = rom_of(e, g);
  size_t idx = (size_t)r * e->cfg.reset_cache_size + pick(e, g, episode_index);
  uint8_t* s = e->states + (size_t)i * ORC_STATE_BYTES;
  memset(s, 0, ORC_STATE_BYTES);
  copy_machine_part(s, e->cache_state + idx * ORC_STATE_BYTES);
  s[61] = (uint8_t)r;
  s[62] = 0;
  put32(s + 192, 0);
  put32(s + 196, episode_index);
  put32(s + 200, 0);
  put16(s + 204, e->cache_score[idx]);
}

int orc_reset(orc_env* e, uint64_t seed, uint8_t* obs) {
  e->pick_seed = seed;
  for (int i = 0; i < e->num_envs; i++) {
    restore_entry(e, i, 0);
    if (obs) {
      int64_t g = e->gids[i];
      size_t idx = (size_t)rom_of(e, g) * e->cfg.reset_cache_size + pick(e, g, 0);
      memcpy(obs + (size_t)i * e->obs_bytes, e->cache_obs + idx * e->obs_bytes, (size_t)e->obs_bytes);
    }
  }
  memset(e->counters, 0, sizeof e->counters);
  return 0;
}

int orc_step(orc_env* e, const uint8_t* actions, uint8_t* obs, int32_t* rewards, uint8_t* dones) {
  for (int i = 0; i < e->num_envs; i++) {
    uint8_t* s = e->states + (size_t)i * ORC_STATE_BYTES;
    int r = s[61];
    Machine m;
    memset(&m, 0, sizeof m);
    load_state(&m, s);
    bind(&m, e->roms[r], e->rom_lens[r]);
    latch_inputs(&m, actions[i]);
    int rendered;
    int fr = run_frames(e, &m, e->fs, &rendered);
    int32_t reward = 0;
    uint16_t score = score_of(&e->cfg, m.ram);
    if (!fr) reward = (int32_t)score - (int32_t)m.prev_score;
    m.prev_score = score;
    m.episode_return += reward;
    int done = m.fault != 0 || (m.ram[e->cfg.term_addr & 0x7F] & e->cfg.term_mask) != 0 ||
               (e->cfg.max_episode_frames > 0 && m.episode_frames >= (uint32_t)e->cfg.max_episode_frames);
    uint8_t* o = obs ? obs + (size_t)i * e->obs_bytes : NULL;
    if (o) {
      if (m.fault) memset(o, 0, (size_t)e->obs_bytes);
      else make_obs(e, rendered, o);
    }
    rewards[i] = reward;
    dones[i] = (uint8_t)done;
    e->counters[0] += e->fs;
    save_state(&m, s);
    if (done) {
      e->counters[1] += 1;
      e->counters[2] += m.episode_return;
      if (m.fault) e->counters[3] += 1;
      restore_entry(e, i, m.episode_index + 1);
    }
  }
  return 0;
}

/* Frame stack of the inference path (R#32), GRAY84 only:
 * stack = u8[N][4][84][84], a ring of the last four observations of each env's current
 * episode.  orc_reset_stacked fills all four slots of every env with its reset observation;
 * orc_step_stacked runs one step, then writes each env's observation into slot `slot`, except
 * for an env whose step ended the episode: it was reset from the cache entry picked for its
 * next episode, and all four of its slots get that entry's stored observation. */
int orc_reset_stacked(orc_env* e, uint64_t seed, uint8_t* stack) {
  size_t ob = (size_t)e->obs_bytes;
  uint8_t* obs = (uint8_t*)malloc((size_t)e->num_envs * ob);
  orc_reset(e, seed, obs);
  for (int i = 0; i < e->num_envs; i++)
    for (int k = 0; k < 4; k++) memcpy(stack + ((size_t)i * 4 + k) * ob, obs + (size_t)i * ob, ob);
  free(obs);
  return 0;
}

int orc_step_stacked(orc_env* e, const uint8_t* actions, uint8_t* stack, int slot, int32_t* rewards,
                     uint8_t* dones) {
  size_t ob = (size_t)e->obs_bytes;
  if (slot < 0 || slot > 3) return -1;
  uint8_t* obs = (uint8_t*)malloc((size_t)e->num_envs * ob);
  orc_step(e, actions, obs, rewards, dones);
  for (int i = 0; i < e->num_envs; i++) {
    if (!dones[i]) {
      memcpy(stack + ((size_t)i * 4 + slot) * ob, obs + (size_t)i * ob, ob);
    } else {
      /* the env now holds the cache entry of its next episode (episode index from its state) */
      const uint8_t* s = e->states + (size_t)i * ORC_STATE_BYTES;
      uint32_t ep = (uint32_t)s[196] | ((uint32_t)s[197] << 8) | ((uint32_t)s[198] << 16) | ((uint32_t)s[199] << 24);
      int64_t g = e->gids[i];
      size_t idx = (size_t)rom_of(e, g) * e->cfg.reset_cache_size + pick(e, g, ep);
      for (int k = 0; k < 4; k++) memcpy(stack + ((size_t)i * 4 + k) * ob, e->cache_obs + idx * ob, ob);
    }
  }
  free(obs);
  return 0;
}

int orc_get_state(orc_env* e, uint8_t* states) {
  memcpy(states, e->states, (size_t)e->num_envs * ORC_STATE_BYTES);
  return 0;
}
int orc_set_state(orc_env* e, const uint8_t* states) {
  memcpy(e->states, states, (size_t)e->num_envs * ORC_STATE_BYTES);
  return 0;
}
int orc_counters(orc_env* e, int64_t* c) { memcpy(c, e->counters, sizeof e->counters); return 0; }
int orc_get_cache(orc_env* e, uint8_t* states, uint8_t* obs) {
  size_t n = (size_t)e->n_roms * e->cfg.reset_cache_size;
  if (states) memcpy(states, e->cache_state, n * ORC_STATE_BYTES);
  if (obs) memcpy(obs, e->cache_obs, n * (size_t)e->obs_bytes);
  return 0;
}
void orc_destroy(orc_env* e) {
  if (!e) return;
  for (int r = 0; r < e->n_roms; r++) free(e->roms[r]);
  free(e->cache_state); free(e->cache_obs); free(e->cache_score);
  free(e->states); free(e->gids); free(e->fbA); free(e->fbB); free(e->gbuf);
  free(e);
}
