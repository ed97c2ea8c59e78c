"""Pins for the oracle's RIOT timer, inputs, cartridge and address decode
(§8(c).14 rows 9-13, 16, 18-19)."""
import numpy as np
import pytest

import helpers as H
from paper_1907_08467_b200.inputs import micro


def run_until_done(orc, rom, n=4000):
    s = orc.power_on(rom)
    st, _ = orc.exec_instr(rom, s, n)
    assert st == 0
    return s


def ticking_timer(V, I, e):
    """RIOT interval timer as a per-cycle counter [HW]: after a write of V the counter
    decrements on cycles 1, 1+I, 1+2I, ...; the decrement after it reads 0 wraps to $FF, sets
    the interrupt flag, and from then on it decrements every cycle.  Returns (INTIM, TIMINT)."""
    val, expired = V, False
    for c in range(1, e + 1):
        if expired:
            val = (val - 1) & 0xFF
        elif (c - 1) % I == 0:
            if val == 0:
                val, expired = 0xFF, True
            else:
                val -= 1
    return val, 0x80 if expired else 0x00


@pytest.mark.parametrize("V,reg,I", [(10, "TIM64T", 64), (3, "TIM1T", 1), (40, "TIM8T", 8),
                                     (2, "T1024T", 1024), (0, "TIM64T", 64), (255, "TIM1T", 1)])
def test_m9_timer_vs_ticking_model(orc, V, reg, I):
    src, e_list = micro.m9_timer(V, reg)
    rom = micro.build(src)
    s = run_until_done(orc, rom)
    for j in range(len(e_list) // 2):
        e_intim, e_timint = e_list[2 * j], e_list[2 * j + 1]
        assert H.ram(s, 0x80 + j) == ticking_timer(V, I, e_intim)[0], (j, e_intim)
        assert H.ram(s, 0xC0 + j) == ticking_timer(V, I, e_timint)[1], (j, e_timint)


def test_m10_decimal_program(orc):
    cases = [("ADC", 0x09, 0x01, 0), ("ADC", 0x99, 0x01, 0), ("ADC", 0x58, 0x46, 1),
             ("SBC", 0x10, 0x01, 1), ("SBC", 0x00, 0x01, 1), ("SBC", 0x46, 0x12, 0)]
    rom = micro.build(micro.m10_decimal(cases))
    s = run_until_done(orc, rom, 200)
    want = [0x10, 0x00, 0x05, 0x09, 0x99, 0x33]
    carry = [0, 1, 1, 1, 0, 1]
    for j in range(len(cases)):
        assert H.ram(s, 0x80 + 2 * j) == want[j]
        assert H.ram(s, 0x81 + 2 * j) & 1 == carry[j]
        assert H.ram(s, 0x81 + 2 * j) & 0x38 == 0x38  # D set, B and U pushed as 1


def test_m11_f8_bank_switching(orc):
    # a hotspot access switches banks first and a read returns the new bank's byte
    rom = micro.build(micro.m11_f8(), 8192)
    s = orc.power_on(rom)
    assert s[H.OFF["bank"]] == 1 and H.pc(s) == 0xF000   # power-on bank = last bank [R#23]
    st, _ = orc.exec_instr(rom, s, 400)
    assert [H.ram(s, a) for a in (0x80, 0x81, 0x82, 0x83, 0x84)] == [0xB1, 0x08, 0xB0, 0x08, 3]
    assert s[H.OFF["bank"]] == 1


@pytest.mark.parametrize("nbanks", [4, 8])
def test_m22_f6_f4_bank_switching(orc, nbanks):
    # F6 ($1FF6-$1FF9) and F4 ($1FF4-$1FFB): power-on in the last bank; every bank stores its
    # id; an indexed read of hotspot X switches to bank X first and returns that bank's marker
    rom = micro.build(micro.m22_banks(nbanks), 4096 * nbanks)
    s = orc.power_on(rom)
    assert s[H.OFF["bank"]] == nbanks - 1 and H.pc(s) == 0xF000
    orc.exec_instr(rom, s, 400)
    assert [H.ram(s, 0x80 + b) for b in range(nbanks)] == [0xB0 + b for b in range(nbanks)]
    assert [H.ram(s, 0x90 + x) for x in range(nbanks - 1)] == [17 * x for x in range(nbanks - 1)]
    assert s[H.OFF["bank"]] == 0


def test_m22_2k_mirror(orc):
    # a 2 KB cartridge repeats at $1000-$17FF and $1800-$1FFF: code and data through both
    rom = micro.build(micro.m22_2k(), 2048)
    assert len(rom) == 2048
    s = orc.power_on(rom)
    assert s[H.OFF["bank"]] == 0 and H.pc(s) == 0xF800
    orc.exec_instr(rom, s, 100)
    assert [H.ram(s, a) for a in (0x80, 0x81, 0x82)] == [2, 0x5A, 0x5A]


def test_m13_jmp_indirect_page_bug(orc):
    rom = micro.build(micro.m13_jmp_ind())
    s = run_until_done(orc, rom, 50)
    assert H.ram(s, 0x80) == 0x11


# ALE action set: (up, down, left, right, fire)
ACTIONS = {0: "", 1: "F", 2: "U", 3: "R", 4: "L", 5: "D", 6: "UR", 7: "UL", 8: "DR", 9: "DL",
           10: "UF", 11: "RF", 12: "LF", 13: "DF", 14: "URF", 15: "ULF", 16: "DRF", 17: "DLF"}


@pytest.mark.parametrize("action", list(range(18)) + [18, 255])
def test_m16_inputs(orc, action):
    rom = micro.build(micro.m16_inputs())
    s = orc.power_on(rom)
    for _ in range(3):
        orc.run_frame(rom, s, action=action, render=False)
    d = ACTIONS.get(action, "")
    # SWCHA high nibble = P0 joystick, active low: D7 right, D6 left, D5 down, D4 up; P1 released
    sw = 0xFF & ~((0x80 if "R" in d else 0) | (0x40 if "L" in d else 0) |
                  (0x20 if "D" in d else 0) | (0x10 if "U" in d else 0))
    assert H.ram(s, 0x80) == sw
    assert H.ram(s, 0x81) == (0x00 if "F" in d else 0x80)
    assert H.ram(s, 0x82) == 0x0B and H.ram(s, 0x83) == 0x80


def test_m18_exec_from_ram(orc):
    rom = micro.build(micro.m18_ram_exec())
    s = run_until_done(orc, rom, 200)
    assert H.ram(s, 0xC0) == 0x42 and H.ram(s, 0xC1) == 9


def test_m19_alu_programs(orc):
    rng = np.random.default_rng(7)
    data = rng.integers(0, 256, 48).tolist()
    rom = micro.build(micro.m19_alu(data))
    s = run_until_done(orc, rom, 20000)
    assert [H.ram(s, 0x80 + i) for i in range(16)] == sorted(data[:16])
    for j in range(16):
        p = data[16 + j] * data[32 + j]
        assert H.ram(s, 0x90 + j) == p & 0xFF and H.ram(s, 0xA0 + j) == p >> 8
    fib = [0, 1]
    while len(fib) < 16:
        fib.append((fib[-1] + fib[-2]) & 0xFF)
    assert [H.ram(s, 0xB0 + i) for i in range(16)] == fib
    tot = sum(data[:16])
    assert H.ram(s, 0xC0) == tot & 0xFF and H.ram(s, 0xC1) == tot >> 8


def test_address_decode_totality(orc):
    """Every 13-bit address resolves to exactly one device: a write of a marker to each
    RAM mirror lands in RAM; writes to cartridge space leave RAM untouched."""
    for base in (0x0080, 0x0180, 0x0480, 0x0580, 0x0880, 0x0980, 0x0C80, 0x0D80, 0x2080, 0xE180):
        code = [0xA9, 0x5A, 0x8D, (base + 5) & 0xFF, (base + 5) >> 8]
        rom = bytearray([0xEA] * 4096)
        rom[0:len(code)] = bytes(code)
        rom[0xFFC:0x1000] = bytes([0, 0xF0, 0, 0xF0])
        s = orc.power_on(bytes(rom))
        orc.exec_instr(bytes(rom), s, 2)
        assert H.ram(s, 0x85) == 0x5A, hex(base)
    for addr in (0x1085, 0xF085, 0x0285, 0x0005, 0x0205, 0x0305):
        code = [0xA9, 0x5A, 0x8D, addr & 0xFF, addr >> 8]
        rom = bytearray([0xEA] * 4096)
        rom[0:len(code)] = bytes(code)
        rom[0xFFC:0x1000] = bytes([0, 0xF0, 0, 0xF0])
        s = orc.power_on(bytes(rom))
        orc.exec_instr(bytes(rom), s, 2)
        assert H.ram(s, 0x85) == 0, hex(addr)
