"""Pins for the opt-in delayed register effects (R#35; SURVEY.md §8(f) NEXT-4 "Stella-level
TIA details"; SPEC.md:144 names the gap): with tia_delays = 1 a playfield register written at
visible pixel x takes effect at the next 4-pixel playfield cell boundary 4*ceil(x/4), and GRP0/GRP1
take effect one colour clock after the write.  Off (the default) every write lands at its colour
clock T = 3 x (end cycle of the instruction) [R#4].

The write clocks are closed forms of the program's cycle count: window row 0 (frame line 34)
starts after `DEX; BNE` (not taken) + `LDA #0; STA VBLANK` = 9 cycles; then k NOPs, `LDA #imm`
and the `STA` ending at cycle 14 + 2k, colour clock 42 + 6k, visible x = 6k - 26.
"""
import numpy as np
import pytest

from paper_1907_08467_b200.inputs import micro

COLUBK, COLUPF, COLUP0, PF1, GRP0, RESP0 = 0x09, 0x08, 0x06, 0x0E, 0x1B, 0x10
BK, PFC, C0 = 0x1E, 0x44, 0x86


def row0_write_x(k):
    return 6 * k - 26


def run(orc, src, delays):
    rom = micro.build(src)
    s = orc.power_on(rom)
    for _ in range(3):
        st, fb, _, lines = orc.run_frame(rom, s, tia_delays=delays)
        assert st == 0
    assert lines == 262  # (the power-on frame is shorter)
    return fb


def pf_src(k):
    row0 = "    NOP\n" * k + "    LDA #$FF\n    STA $0E\n"
    return micro.static_frame(pokes=[(COLUBK, BK), (COLUPF, PFC), (PF1, 0x00)], kernel_row0=row0)


@pytest.mark.parametrize("k", [7, 8, 9, 10, 11, 12])
def test_pf_write_lands_on_cell_boundary(orc, k):
    x = row0_write_x(k)
    assert 16 <= x < 48  # inside PF1's cells 4..11 (pixels 16..47) of the left half
    for delays, x_eff in ((0, x), (1, 4 * ((x + 3) // 4))):
        fb = run(orc, pf_src(k), delays)
        want = np.full(160, BK >> 1, np.uint8)
        want[16:48] = want[96:128] = PFC >> 1
        # rows 1..209: PF1 = $FF everywhere it shows (the write persists; the next frame's row 0
        # starts from PF1 = $00 again: the VBLANK pokes clear it)
        assert (fb[1:] == want[None, :]).all()
        row0 = np.full(160, BK >> 1, np.uint8)
        row0[x_eff:48] = PFC >> 1
        row0[96:128] = PFC >> 1
        assert (fb[0] == row0).all(), (delays, np.nonzero(fb[0] != row0)[0])


def test_pf_delay_is_at_most_three_pixels(orc):
    # x = 6k - 26 covers every residue mod 4 over k = 7..10: the effect moves by (4 - x % 4) % 4
    shifts = {row0_write_x(k) % 4: (4 - row0_write_x(k) % 4) % 4 for k in range(7, 11)}
    assert sorted(shifts) == [0, 2] and max(shifts.values()) <= 3


@pytest.mark.parametrize("k", [12, 13])
def test_grp_write_one_clock_later(orc, k):
    # player 0 = 8 pixels of GRP0 = $FF; row 0 clears GRP0 at a pixel x the player covers.
    # RESP0 after kk NOPs: colour clock 6kk + 9, hp = 6kk - 59, player at p = hp + 5 [R#10];
    # kk = floor((x + 54) / 6) puts x inside [p, p + 8)
    x = row0_write_x(k)
    kk = (x + 54) // 6
    p = 6 * kk - 59 + 5
    assert p <= x < p + 8
    row0 = "    NOP\n" * k + "    LDA #$00\n    STA $1B\n"
    src = micro.static_frame(pokes=[(COLUBK, BK), (COLUP0, C0), (GRP0, 0xFF)], positions=[(RESP0, kk)],
                             kernel_row0=row0)
    for delays in (0, 1):
        fb = run(orc, src, delays)
        row = np.full(160, BK >> 1, np.uint8)
        row[p:x + delays] = C0 >> 1     # pixels before the effect clock show the old graphic
        assert (fb[0] == row).all(), (delays, p, x, np.nonzero(fb[0] != row)[0])
        assert (fb[1:] == BK >> 1).all()  # GRP0 = 0 from then on


def test_delays_off_by_default_is_the_r4_model(orc):
    # the default run_frame (no tia_delays) equals tia_delays = 0
    rom = micro.build(pf_src(8))
    a, b = orc.power_on(rom), orc.power_on(rom)
    for _ in range(3):
        _, fa, _, _ = orc.run_frame(rom, a)
        _, fb, _, _ = orc.run_frame(rom, b, tia_delays=0)
        assert (fa == fb).all() and (a == b).all()


# ---- RESxx start delay [R#36] ----------------------------------------------------------------
def row0_resp_hp(k):
    """`STA RESP0` after k NOPs on window row 0 ends at cycle 9 + 2k + 3: colour clock 36 + 6k,
    hp = 6k - 32 (visible for k >= 6); the player lands at hp + 5 [R#10]."""
    return 6 * k - 32


@pytest.mark.parametrize("nusiz,copies", [(0, [0]), (1, [0, 16]), (3, [0, 16, 32])])
@pytest.mark.parametrize("k", [10, 14])
def test_resp_start_delay(orc, nusiz, copies, k):
    # player 0 (GRP0 = $FF) first placed at p0 = 6 by a VBLANK RESP0 after 10 NOPs (hp = 1);
    # row 0 strobes RESP0 again at visible hp = 6k - 32: the player moves to p1 = hp + 5
    p0, hp = 6, row0_resp_hp(k)
    p1 = hp + 5
    row0 = "    NOP\n" * k + "    STA $10\n"
    src = micro.static_frame(pokes=[(COLUBK, BK), (COLUP0, C0), (GRP0, 0xFF), (0x04, nusiz)],
                             positions=[(RESP0, 10)], kernel_row0=row0)
    for delays in (0, 1):
        fb = run(orc, src, delays)
        want0 = np.full(160, BK >> 1, np.uint8)
        for c in copies:                # before the strobe: the copies at the old position
            a, b = p0 + c, p0 + c + 8
            want0[a:min(b, hp)] = C0 >> 1
        for i, c in enumerate(copies):  # after it: the copies at the new position, except the
            if delays and i == 0:       # first one on this line when the start delay is on
                continue
            a = max(p1 + c, hp)
            want0[a:p1 + c + 8] = C0 >> 1
        assert (fb[0] == want0).all(), (delays, np.nonzero(fb[0] != want0)[0])
        want = np.full(160, BK >> 1, np.uint8)  # rows 1..: every copy at the new position
        for c in copies:
            want[p1 + c:p1 + c + 8] = C0 >> 1
        assert (fb[1:] == want[None, :]).all()


def test_resp_in_hblank_has_no_start_delay(orc):
    # a strobe in HBLANK (the VBLANK positioning line, hp < 0) draws on its own line
    src = micro.static_frame(pokes=[(COLUBK, BK), (COLUP0, C0), (GRP0, 0xFF)], positions=[(RESP0, 3)])
    for delays in (0, 1):
        fb = run(orc, src, delays)
        assert (fb == run(orc, src, 0)).all()


def test_start_delay_pending_at_frame_boundary(orc):
    # M23: player 0 reset to 72 at hp = 67, VSYNC written at pixel 76 of the same line; the new
    # frame's line 0 continues that line: pixels 76..79 of the player, unless the start delay
    # suppresses the first copy, which the snapshot then carries in byte 63 (bit 0 = P0)
    rom = micro.build(micro.m23_resp_at_vsync())
    for delays in (0, 1):
        s = orc.power_on(rom)
        for _ in range(3):
            st, fb, _, _ = orc.run_frame(rom, s, ystart=0, tia_delays=delays)
            assert st == 0
        assert s[63] == delays
        assert s[56] == 72                                    # posP0
        row0 = np.zeros(160, np.uint8)
        if not delays:
            row0[76:80] = C0 >> 1
        assert (fb[0] == row0).all(), (delays, np.nonzero(fb[0])[0])
