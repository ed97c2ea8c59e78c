"""Pins for the oracle's TIA and frame loop.

Expected frames are closed forms from the hardware description [HW] and the written readings
[R#n]: literal pixel positions, literal playfield cell tables, colours written by
the program itself.  Nothing is computed by re-running the oracle's own coverage code.
"""
import numpy as np
import pytest

import helpers as H
from paper_1907_08467_b200.inputs import micro

COLUBK, COLUPF, COLUP0, COLUP1 = 0x09, 0x08, 0x06, 0x07
NUSIZ0, NUSIZ1, CTRLPF, REFP0 = 0x04, 0x05, 0x0A, 0x0B
PF0, PF1, PF2 = 0x0D, 0x0E, 0x0F
RESP0, RESP1, RESM0, RESM1, RESBL = 0x10, 0x11, 0x12, 0x13, 0x14
GRP0, GRP1, ENAM0, ENAM1, ENABL = 0x1B, 0x1C, 0x1D, 0x1E, 0x1F
HMP0, HMBL, VDELP0 = 0x20, 0x24, 0x25
RESMP0 = 0x28


def frames(orc, src, n=3, action=0, size=4096):
    rom = micro.build(src, size)
    s = orc.power_on(rom)
    out = []
    for _ in range(n):
        st, fb, ic, lines = orc.run_frame(rom, s, action=action)
        assert st == 0
        out.append((fb.copy(), lines, s.copy()))
    return out


def test_m1_frame262(orc):
    res = frames(orc, micro.m1_frame262(), n=6)
    for fb, lines, s in res[1:]:
        assert lines == 262          # 262 lines x 76 cycles = 19,912 CPU cycles per frame
        assert H.fc(s) == 3          # VSYNC written 3 cycles into the line, every frame


def test_m2_colubk_rows(orc):
    fb, lines, s = frames(orc, micro.m2_colubk_rows(), n=3)[-1]
    assert lines == 262
    for r in range(210):
        # COLUBK = 2*line written in HBLANK of `line`; palette index = COLUBK >> 1; row r = line 34+r
        assert (fb[r] == ((34 + r) & 0x7F)).all(), r


def static(orc, pokes=(), positions=(), **kw):
    fb, lines, s = frames(orc, micro.static_frame(pokes=pokes, positions=positions, **kw), n=3)[-1]
    assert lines == 262
    return fb, s


BK, PFC, C0, C1 = 0x1E, 0x44, 0x86, 0xC8  # palette indices 0x0F, 0x22, 0x43, 0x64


def test_uniform_background(orc):
    fb, _ = static(orc, [(COLUBK, BK)])
    assert (fb == BK >> 1).all()  # S:133 uniform COLUBK frame


# playfield cell of each (register, bit) — 2600 TIA documentation: PF0 D4..D7 are cells 0..3
# (left to right), PF1 D7..D0 cells 4..11, PF2 D0..D7 cells 12..19; a cell is 4 pixels wide.
PF_CELL = {(PF0, 4): 0, (PF0, 5): 1, (PF0, 6): 2, (PF0, 7): 3,
           (PF1, 7): 4, (PF1, 6): 5, (PF1, 5): 6, (PF1, 4): 7, (PF1, 3): 8, (PF1, 2): 9,
           (PF1, 1): 10, (PF1, 0): 11,
           (PF2, 0): 12, (PF2, 1): 13, (PF2, 2): 14, (PF2, 3): 15, (PF2, 4): 16, (PF2, 5): 17,
           (PF2, 6): 18, (PF2, 7): 19}


@pytest.mark.parametrize("reflect", [0, 1])
@pytest.mark.parametrize("reg_bit", sorted(PF_CELL))
def test_m3_playfield_bits(orc, reg_bit, reflect):
    reg, bit = reg_bit
    fb, _ = static(orc, [(COLUBK, BK), (COLUPF, PFC), (CTRLPF, reflect), (reg, 1 << bit)])
    cell = PF_CELL[reg_bit]
    right = (39 - cell) if reflect else (20 + cell)
    want = np.full(160, BK >> 1, np.uint8)
    want[4 * cell: 4 * cell + 4] = PFC >> 1
    want[4 * right: 4 * right + 4] = PFC >> 1
    assert (fb == want[None, :]).all()


def test_s134_full_playfield(orc):
    # PF0=F0 PF1=FF PF2=FF -> left 80 pixels playfield colour, repeated on the right
    fb, _ = static(orc, [(COLUBK, BK), (COLUPF, PFC), (PF0, 0xF0), (PF1, 0xFF), (PF2, 0xFF)])
    assert (fb == PFC >> 1).all()


def resp_x(k, player=True):
    """RESPx strobe at the end of `STA` after k NOPs from a line start: cycle 2k+3, colour clock
    6k+9, hp = 6k-59; players land at max(hp,-2)+5, missiles/ball at max(hp,-2)+4 [R#10]."""
    hp = max(6 * k - 59, -2)
    return (hp + (5 if player else 4)) % 160


@pytest.mark.parametrize("k", [0, 9, 10, 11, 17, 20, 26, 33, 35])
def test_m4_resp0_position(orc, k):
    fb, s = static(orc, [(COLUBK, BK), (COLUP0, C0), (GRP0, 0x80)], positions=[(RESP0, k)])
    x = resp_x(k)
    assert s[H.OFF["posP0"]] == x
    want = np.full(160, BK >> 1, np.uint8)
    want[x] = C0 >> 1
    assert (fb == want[None, :]).all()


@pytest.mark.parametrize("hm,delta", [(0x70, -7), (0x10, -1), (0x00, 0), (0xF0, 1), (0x90, 7), (0x80, 8)])
def test_m5_hmove(orc, hm, delta):
    # HMP0 = $70 then HMOVE moves player 0 by -7 (left); the nibble is signed
    k = 20
    fb, s = static(orc, [(COLUBK, BK), (COLUP0, C0), (GRP0, 0x80), (HMP0, hm)],
                   positions=[(RESP0, k)], hmove=True)
    x = (resp_x(k) + delta) % 160
    assert s[H.OFF["posP0"]] == x
    assert np.nonzero(fb[100] != BK >> 1)[0].tolist() == [x]


def test_hmove_wraps(orc):
    fb, s = static(orc, [(GRP0, 0x80), (COLUP0, C0), (HMP0, 0x70)], positions=[(RESP0, 0)], hmove=True)
    assert s[H.OFF["posP0"]] == (3 - 7) % 160


def test_hmove_comb(orc):
    # HMOVE strobed during HBLANK of row 0 blanks pixels 0..7 of that line only [R#11]
    fb, s = static(orc, [(COLUBK, BK)], hmove_row0=True)
    assert (fb[0, :8] == 0).all() and (fb[0, 8:] == BK >> 1).all()
    assert (fb[1:] == BK >> 1).all()


# NUSIZ copies / sizes (2600 TIA documentation): mode -> (copy offsets, pixel scale)
NUSIZ_DOC = {0: ((0,), 1), 1: ((0, 16), 1), 2: ((0, 32), 1), 3: ((0, 16, 32), 1),
             4: ((0, 64), 1), 5: ((0,), 2), 6: ((0, 32, 64), 1), 7: ((0,), 4)}


@pytest.mark.parametrize("mode", range(8))
@pytest.mark.parametrize("refl", [0, 8])
def test_m6_nusiz_refp(orc, mode, refl):
    grp = 0xC1  # bits 7, 6, 0
    k = 20
    fb, _ = static(orc, [(COLUBK, BK), (COLUP0, C0), (GRP0, grp), (NUSIZ0, mode), (REFP0, refl)],
                   positions=[(RESP0, k)])
    x0 = resp_x(k)
    offs, scale = NUSIZ_DOC[mode]
    # graphic pixel order: D7 first, or D0 first when reflected
    bits = [7, 6, 5, 4, 3, 2, 1, 0] if not refl else [0, 1, 2, 3, 4, 5, 6, 7]
    lit = set()
    for o in offs:
        for i, b in enumerate(bits):
            if grp >> b & 1:
                for sub in range(scale):
                    lit.add((x0 + o + i * scale + sub) % 160)
    got = set(np.nonzero(fb[50] != BK >> 1)[0].tolist())
    assert got == lit


@pytest.mark.parametrize("width_bits,width", [(0, 1), (1, 2), (2, 4), (3, 8)])
def test_missile_and_ball(orc, width_bits, width):
    k = 15
    fb, _ = static(orc, [(COLUBK, BK), (COLUP0, C0), (NUSIZ0, width_bits << 4), (ENAM0, 2)],
                   positions=[(RESM0, k)])
    x = resp_x(k, player=False)
    assert set(np.nonzero(fb[10] != BK >> 1)[0].tolist()) == {(x + i) % 160 for i in range(width)}
    fb, _ = static(orc, [(COLUBK, BK), (COLUPF, PFC), (CTRLPF, width_bits << 4), (ENABL, 2)],
                   positions=[(RESBL, k)])
    assert set(np.nonzero(fb[10] != BK >> 1)[0].tolist()) == {(x + i) % 160 for i in range(width)}
    assert (fb[10][fb[10] != BK >> 1] == PFC >> 1).all()


def test_resmp_locks_missile(orc):
    # RESMP0 set hides M0; clearing it moves M0 to the player's position + 3 [R#10]
    k = 20
    fb, s = static(orc, [(COLUBK, BK), (COLUP0, C0), (ENAM0, 2), (RESMP0, 2), (RESMP0, 0)],
                   positions=[(RESP0, k)])
    # pokes happen before the RESP0 line, so the 1->0 write sees P0 where the previous frame's
    # RESP0 put it (the frame is identical every time)
    x = (resp_x(k) + 3) % 160
    assert s[H.OFF["posM0"]] == x
    assert np.nonzero(fb[20] != BK >> 1)[0].tolist() == [x]
    fb, s = static(orc, [(COLUBK, BK), (ENAM0, 2), (RESMP0, 2)], positions=[(RESP0, k)])
    assert (fb == BK >> 1).all()


def test_priority_and_score(orc):
    k = 20
    x = resp_x(k)
    base = [(COLUBK, BK), (COLUPF, PFC), (COLUP0, C0), (COLUP1, C1), (GRP0, 0xFF),
            (PF0, 0xF0), (PF1, 0xFF), (PF2, 0xFF)]
    fb, _ = static(orc, base + [(CTRLPF, 0)], positions=[(RESP0, k)])
    assert (fb[5, x:x + 8] == C0 >> 1).all() and fb[5, x + 8] == PFC >> 1   # players above PF
    fb, _ = static(orc, base + [(CTRLPF, 4)], positions=[(RESP0, k)])
    assert (fb[5] == PFC >> 1).all()                                           # PFP: PF above
    fb, _ = static(orc, base + [(CTRLPF, 2), (GRP0, 0)], positions=[(RESP0, k)])
    assert (fb[5, :80] == C0 >> 1).all() and (fb[5, 80:] == C1 >> 1).all()    # SCORE mode


def test_vdelp(orc):
    k = 20
    x = resp_x(k)
    # VDELP0: the displayed graphic is the "old" copy, latched from "new" by a GRP1 write
    fb, s = static(orc, [(COLUBK, BK), (COLUP0, C0), (GRP0, 0xFF), (VDELP0, 1), (GRP0, 0x81)],
                   positions=[(RESP0, k)])
    assert (fb[7] == BK >> 1).all()
    fb, s = static(orc, [(COLUBK, BK), (COLUP0, C0), (VDELP0, 1), (GRP0, 0x81), (GRP1, 0x00)],
                   positions=[(RESP0, k)])
    assert set(np.nonzero(fb[7] != BK >> 1)[0].tolist()) == {x, x + 7}


# collision register bits (2600 TIA documentation): register -> (d7 pair, d6 pair)
def test_m8_collisions(orc):
    k = 20
    # P0 and ball overlap, PF elsewhere -> CXP0FB d6 only
    _, s = static(orc, [(GRP0, 0xFF), (ENABL, 2), (CTRLPF, 0x30)], positions=[(RESP0, k), (RESBL, k)],
                  store_collisions=True)
    cx = [H.ram(s, 0xF0 + r) for r in range(8)]
    assert cx[2] == 0x40 and cx[6] == 0 and cx[0] == cx[1] == cx[3] == cx[7] == 0
    assert cx[4] == cx[5] == 0
    # add playfield everywhere -> CXP0FB d7|d6 and CXBLPF d7
    _, s = static(orc, [(GRP0, 0xFF), (ENABL, 2), (CTRLPF, 0x30), (PF1, 0xFF), (PF0, 0xF0), (PF2, 0xFF)],
                  positions=[(RESP0, k), (RESBL, k)], store_collisions=True)
    cx = [H.ram(s, 0xF0 + r) for r in range(8)]
    assert cx[2] == 0xC0 and cx[6] == 0x80 and cx[3] == 0
    # both players overlap -> CXPPMM d7; missiles overlap -> CXPPMM d6
    _, s = static(orc, [(GRP0, 0xFF), (GRP1, 0xFF), (ENAM0, 2), (ENAM1, 2)],
                  positions=[(RESP0, k), (RESP1, k), (RESM0, 30), (RESM1, 30)], store_collisions=True)
    cx = [H.ram(s, 0xF0 + r) for r in range(8)]
    assert cx[7] == 0xC0 and cx[0] == 0 and cx[1] == 0
    # all objects disabled -> no latches
    _, s = static(orc, [], store_collisions=True)
    assert all(H.ram(s, 0xF0 + r) == 0 for r in range(8))
    assert H.coll(s) == 0


def test_collisions_persist_until_cxclr(orc):
    _, s = static(orc, [(GRP0, 0xFF), (ENABL, 2), (CTRLPF, 0x30)], positions=[(RESP0, 20), (RESBL, 20)],
                  store_collisions=True, clear_collisions=False)
    assert H.ram(s, 0xF2) == 0x40 and H.coll(s) == 1 << 5   # latched bit 5 = CXP0FB d6


def test_m12_stack_into_tia(orc):
    # SP=$09: PHA writes $0109 -> TIA COLUBK; SP=$85: PHA writes $0185 -> RAM $85 (mirror)
    fb, lines, s = frames(orc, micro.m12_stack_decode(0x2A), n=3)[-1]
    assert (fb == 0x15).all()
    assert H.ram(s, 0x85) == 0x5C


def test_vblank_blacks_window(orc):
    fb, s = static(orc, [(COLUBK, BK)], kernel_row0="    LDA #2\n    STA VBLANK\n")
    assert (fb == 0).all()
