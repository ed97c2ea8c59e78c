"""Pins for the premise of the TIA write elision (DESIGN.md §2 R#37) in the written model the
oracle implements: a write of the value a "pure" register already holds changes nothing — not the
frame, not the collision latches — while a different value does (the tests are sensitive), and
GRP0/GRP1 are NOT pure: with a vertical delay pending (the other player's old and new graphics
differ) rewriting a player's own value still moves the other player's new graphics into its old
register, which the picture shows.

Each program sets the registers in VBLANK (micro.static_frame pokes), then on window row 0 spends
k NOPs and either stores the value into the TIA register or, with the same cycle count, into RAM
$80; the oracle runs three frames of each (the last one compared, plus collision latches copied
to RAM $F0-$F7 by the next frame's VBLANK)."""
import pytest

from paper_1907_08467_b200.inputs import micro

# (register, value held, a different value that shows) — pure stores (scalar_predecode.h kTiaPure)
BASE = [(0x09, 0x1E), (0x08, 0x44), (0x06, 0x86), (0x07, 0xC8), (0x1B, 0xF3), (0x1C, 0xC1), (0x04, 0x01),
        (0x05, 0x00), (0x0D, 0x50), (0x0E, 0xF0), (0x0F, 0x0F), (0x0A, 0x01), (0x1D, 0x02), (0x1E, 0x02),
        (0x1F, 0x02), (0x0B, 0x00), (0x0C, 0x08), (0x20, 0x10), (0x22, 0xF0), (0x25, 0x00), (0x27, 0x00),
        (0x28, 0x00), (0x21, 0x20), (0x23, 0x00), (0x24, 0x10), (0x26, 0x00), (0x29, 0x00)]
HELD = dict(BASE)
VISIBLE = {0x09: 0x3A, 0x08: 0x9C, 0x06: 0x24, 0x07: 0x62, 0x04: 0x03, 0x05: 0x06, 0x0D: 0xA0, 0x0E: 0x0F,
           0x0F: 0xF0, 0x0A: 0x05, 0x1D: 0x00, 0x1E: 0x00, 0x1F: 0x00, 0x0B: 0x08, 0x0C: 0x00}
OTHER_PURE = [0x20, 0x21, 0x22, 0x23, 0x24, 0x25, 0x26, 0x27, 0x28, 0x29]  # HMxx, VDELxx, RESMPx
POS = [(0x10, 12), (0x11, 16), (0x12, 20), (0x13, 24), (0x14, 28)]


def program(reg, value, to_tia, pokes=BASE, k=12):
    target = f"${reg:02X}" if to_tia else "$80"
    row0 = "    NOP\n" * k + f"    LDA #${value:02X}\n    STA {target}\n"
    return micro.static_frame(pokes=pokes, positions=POS, kernel_row0=row0, store_collisions=True)


def frame_and_latches(orc, src):
    rom = micro.build(src)
    s = orc.power_on(rom)
    fb = None
    for _ in range(4):
        st, fb, _, _ = orc.run_frame(rom, s)
        assert st == 0
    snap = s.copy()
    return fb.copy(), snap


def ram_bytes(snap, lo, hi):
    # snapshot layout: RAM $80-$FF at bytes 64..191
    return snap[64 + (lo - 0x80):64 + (hi - 0x80) + 1].tobytes()


@pytest.mark.parametrize("reg", sorted(VISIBLE) + OTHER_PURE)
def test_rewriting_a_pure_register_changes_nothing(orc, reg):
    fa, sa = frame_and_latches(orc, program(reg, HELD[reg], True))
    fb, sb = frame_and_latches(orc, program(reg, HELD[reg], False))
    assert (fa == fb).all(), f"register {reg:#x}: frame changed by a write of its own value"
    assert ram_bytes(sa, 0xF0, 0xF7) == ram_bytes(sb, 0xF0, 0xF7), "collision latches changed"


@pytest.mark.parametrize("reg", sorted(VISIBLE))
def test_a_different_value_shows(orc, reg):
    fa, _ = frame_and_latches(orc, program(reg, VISIBLE[reg], True))
    fb, _ = frame_and_latches(orc, program(reg, HELD[reg], False))
    assert (fa != fb).any(), f"register {reg:#x}: the control write is invisible (test not sensitive)"


def vdel_pokes(pending):
    # VDELP1 on; GRP1 = $AA, then GRP0 (copies GRP1 new -> old: old = $AA), then GRP1 new = $55
    # (a delay pending: old $AA shown, new $55 waiting) or $AA again (old = new, nothing pending)
    return [(0x09, 0x1E), (0x06, 0x86), (0x07, 0xC8), (0x26, 0x01), (0x1C, 0xAA), (0x1B, 0xFF),
            (0x1C, 0x55 if pending else 0xAA)]


def test_grp0_rewrite_is_not_pure_with_a_pending_vertical_delay(orc):
    pk = vdel_pokes(True)
    fa, _ = frame_and_latches(orc, program(0x1B, 0xFF, True, pokes=pk))
    fb, _ = frame_and_latches(orc, program(0x1B, 0xFF, False, pokes=pk))
    assert (fa != fb).any(), "GRP0 rewritten with its own value must still copy GRP1 new -> old"


def test_grp0_rewrite_is_pure_without_a_pending_delay(orc):
    pk = vdel_pokes(False)
    fa, _ = frame_and_latches(orc, program(0x1B, 0xFF, True, pokes=pk))
    fb, _ = frame_and_latches(orc, program(0x1B, 0xFF, False, pokes=pk))
    assert (fa == fb).all()


def vdelbl_pokes(pending):
    # VDELBL on; ENABL new = on, GRP1 (copies ENABL new -> old: old = on), then ENABL new = off
    # (pending: the ball shows old = on) or on again (nothing pending)
    return [(0x09, 0x1E), (0x08, 0x44), (0x27, 0x01), (0x1F, 0x02), (0x1C, 0x00), (0x1F, 0x00 if pending else 0x02)]


@pytest.mark.parametrize("pending", [True, False])
def test_grp1_rewrite_and_the_ball_delay(orc, pending):
    """GRP1 also copies ENABL new -> old: a rewrite of GRP1's own value is visible exactly when a
    ball delay is pending (the elision keeps such a write, scalar_cpu.cuh shd_write)."""
    pk = vdelbl_pokes(pending)
    fa, _ = frame_and_latches(orc, program(0x1C, 0x00, True, pokes=pk))
    fb, _ = frame_and_latches(orc, program(0x1C, 0x00, False, pokes=pk))
    assert (fa != fb).any() == pending
