"""Pins for the oracle's 6502.

Every expected value here comes from something other than the oracle itself:
  * the published opcode matrix (tests/golden/opcode_matrix.txt) for
    cycle counts, page-cross penalties, branch timing and the fault set;
  * SPEC.md worked examples S:47-49, S:56-58, S:65-66;
  * closed forms of binary/decimal arithmetic brute-forced over all operands.
"""
import os

import numpy as np
import pytest

import helpers as H

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "opcode_matrix.txt")


def parse_matrix():
    rows = [ln for ln in open(GOLDEN) if not ln.startswith("#") and "|" in ln]
    assert len(rows) == 16
    table = {}
    for ln in rows:
        hi = int(ln[0], 16)
        cells = ln.split("|", 1)[1].rstrip("\n")[1:]
        for lo in range(16):
            cell = cells[9 * lo: 9 * lo + 9].strip()
            op = (hi << 4) | lo
            if cell == "JAM" or cell.startswith("("):
                table[op] = dict(fault=True, mn=cell)
                continue
            parts = cell.split()
            mn = parts[0]
            rest = parts[1] if len(parts) > 1 else ""
            plus = rest.endswith("+")
            branch = rest.endswith("*")
            rest = rest.rstrip("+*")
            i = 0
            while i < len(rest) and not rest[i].isdigit():
                i += 1
            mode, base = rest[:i] or "impl", int(rest[i:])
            table[op] = dict(fault=False, mn=mn, mode=mode, base=base, plus=plus, branch=branch)
    return table


MATRIX = parse_matrix()


def test_matrix_counts():
    # 151 documented, 85 stable undocumented, 12 JAM, 8 unstable
    doc = sum(1 for e in MATRIX.values() if not e["fault"] and e["mn"].isupper())
    und = sum(1 for e in MATRIX.values() if not e["fault"] and e["mn"].islower())
    jam = sum(1 for e in MATRIX.values() if e["fault"] and e["mn"] == "JAM")
    uns = sum(1 for e in MATRIX.values() if e["fault"] and e["mn"] != "JAM")
    assert (doc, und, jam, uns) == (151, 85, 12, 8)


# branch conditions (6502 datasheet): opcode -> (flag bit, taken when set)
BRANCH = {0x10: (0x80, False), 0x30: (0x80, True), 0x50: (0x40, False), 0x70: (0x40, True),
          0x90: (0x01, False), 0xB0: (0x01, True), 0xD0: (0x02, False), 0xF0: (0x02, True)}


def _rom_with(code_at: dict, fill=0xEA):
    rom = bytearray([fill] * 4096)
    rom[0xFFC:0x1000] = bytes([0x00, 0xF0, 0x00, 0xF0])
    for addr, bs in code_at.items():
        for i, b in enumerate(bs):
            rom[(addr + i) & 0xFFF] = b
    return bytes(rom)


def _state_for(rom, pcv=0xF000, A=0, X=0, Y=0, P=0x24, ram=None):
    import oracle
    s = oracle.power_on(rom)
    s[0], s[1], s[2], s[4] = A, X, Y, P
    H.set_pc(s, pcv)
    H.set_fc(s, 0)
    # pointer at $80/$81 -> $0090 (RAM) unless overridden
    s[64 + 0] = 0x90
    s[64 + 1] = 0x00
    if ram:
        for a, v in ram.items():
            s[64 + (a & 0x7F)] = v
    return s


def _operands(mode, cross):
    if mode in ("#",):
        return [0x00]
    if mode in ("z", "zx", "zy", "ix", "iy"):
        return [0x80]
    if mode in ("a", "in"):
        return [0x80, 0xF0]
    if mode in ("ax", "ay"):
        return [0xF0, 0xF0] if cross else [0x80, 0xF0]
    if mode == "r":
        return [0x10]
    return []


@pytest.mark.parametrize("op", [o for o in range(256) if not MATRIX[o]["fault"]])
def test_opcode_cycles(orc, op):
    e = MATRIX[op]
    mode = e["mode"]
    if e["branch"]:
        flag, when_set = BRANCH[op]
        not_taken_p = 0x24 | (0 if when_set else flag)
        taken_p = 0x24 | (flag if when_set else 0)
        rom = _rom_with({0xF000: [op, 0x10], 0xF0F0: [op, 0x20]})
        for P, pcv, expect in ((not_taken_p, 0xF000, 2), (taken_p, 0xF000, 3), (taken_p, 0xF0F0, 4)):
            s = _state_for(rom, pcv=pcv, P=P)
            st, cyc = orc.exec_instr(rom, s, 1)
            assert st == 0 and cyc == expect, (hex(op), P, pcv, cyc, expect)
        return
    for cross in (False, True):
        if cross and mode not in ("ax", "ay", "iy"):
            continue
        rom = _rom_with({0xF000: [op] + _operands(mode, cross)})
        X = 0x20 if (cross and mode == "ax") else 0
        Y = 0x20 if (cross and mode in ("ay", "iy")) else 0
        ram = {0x80: 0xF0, 0x81: 0x00} if (cross and mode == "iy") else None
        s = _state_for(rom, X=X, Y=Y, ram=ram)
        st, cyc = orc.exec_instr(rom, s, 1)
        expect = e["base"] + (1 if (cross and e["plus"]) else 0)
        assert st == 0, hex(op)
        assert cyc == expect, (hex(op), e, cross, cyc)


@pytest.mark.parametrize("op", [o for o in range(256) if MATRIX[o]["fault"]])
def test_fault_opcodes(orc, op):
    rom = _rom_with({0xF000: [op, 0x00, 0x00]})
    s = _state_for(rom)
    st, cyc = orc.exec_instr(rom, s, 1)
    assert st == 1 and s[H.OFF["fault"]] == 1 and cyc == 0


def test_spec_examples(orc):
    # S:47-49 NOP 2 cycles, LDA # 2 cycles; S:56 LDA #$00 -> Z=1 N=0 PC+2
    rom = _rom_with({0xF000: [0xA9, 0x00]})
    s = _state_for(rom, A=0x55, P=0xA4)
    st, cyc = orc.exec_instr(rom, s, 1)
    assert (st, cyc, s[0], H.pc(s)) == (0, 2, 0, 0xF002)
    assert s[4] & 0x02 and not (s[4] & 0x80)
    rom = _rom_with({0xF000: [0xEA]})
    s = _state_for(rom)
    assert orc.exec_instr(rom, s, 1) == (0, 2) and H.pc(s) == 0xF001
    # S:57 decimal ADC 0x09 + 0x01 = 0x10
    rom = _rom_with({0xF000: [0x69, 0x01]})
    s = _state_for(rom, A=0x09, P=0x24 | 0x08)
    orc.exec_instr(rom, s, 1)
    assert s[0] == 0x10
    # S:58 LDA $12F0,X with X=$20 -> 5 cycles (page cross)
    rom = _rom_with({0xF000: [0xBD, 0xF0, 0x12]})
    s = _state_for(rom, X=0x20)
    assert orc.exec_instr(rom, s, 1) == (0, 5)
    # S:65-66 reset vector little-endian
    for lo, hi, want in ((0x00, 0xF0, 0xF000), (0x34, 0x12, 0x1234)):
        r = bytearray([0xEA] * 4096)
        r[0xFFC], r[0xFFD] = lo, hi
        s = orc.power_on(bytes(r))
        assert H.pc(s) == want
        assert s[3] == 0xFD and s[4] == 0x24  # S:62 SP=$FD, I set, D cleared


def _sx(v):
    return v - 256 if v & 0x80 else v


def _run_alu(orc, opcode, cases):
    """cases: iterable of (A, M, P) -> list of (A', P') executing `opcode $80` with RAM[$80]=M."""
    rom = _rom_with({0xF000: [opcode, 0x80]})
    base = _state_for(rom)
    out = []
    for A, M, P in cases:
        s = base.copy()
        s[0], s[4] = A, P
        s[64] = M
        orc.exec_instr(rom, s, 1)
        out.append((int(s[0]), int(s[4]), int(s[64])))
    return out


def _cases(decimal):
    for c in (0, 1):
        for A in range(256):
            for M in range(256):
                yield A, M, 0x24 | c | (0x08 if decimal else 0)


def test_adc_binary_bruteforce(orc):
    res = _run_alu(orc, 0x65, _cases(False))
    for (A, M, P), (a2, p2, _) in zip(_cases(False), res):
        c = P & 1
        t = A + M + c
        r = t & 0xFF
        sv = _sx(A) + _sx(M) + c
        assert a2 == r
        assert (p2 & 1) == (t > 255)
        assert bool(p2 & 0x40) == (sv < -128 or sv > 127)
        assert bool(p2 & 0x02) == (r == 0) and bool(p2 & 0x80) == (r >= 128)


def test_sbc_binary_bruteforce(orc):
    res = _run_alu(orc, 0xE5, _cases(False))
    for (A, M, P), (a2, p2, _) in zip(_cases(False), res):
        c = P & 1
        t = A - M - (1 - c)
        r = t & 0xFF
        sv = _sx(A) - _sx(M) - (1 - c)
        assert a2 == r
        assert (p2 & 1) == (t >= 0)
        assert bool(p2 & 0x40) == (sv < -128 or sv > 127)
        assert bool(p2 & 0x02) == (r == 0) and bool(p2 & 0x80) == (r >= 128)


def _valid_bcd(v):
    return (v >> 4) <= 9 and (v & 15) <= 9


def _dec(v):
    return 10 * (v >> 4) + (v & 15)


def _bcd(n):
    return ((n // 10) << 4) | (n % 10)


def test_adc_decimal_bruteforce(orc):
    # valid-BCD subset: closed form (dec(A)+dec(M)+C) mod 100 with carry;
    # Z from the binary sum (NMOS reading [R#2]); all 131072 cases must execute.
    res = _run_alu(orc, 0x65, _cases(True))
    n_valid = 0
    for (A, M, P), (a2, p2, _) in zip(_cases(True), res):
        c = P & 1
        assert bool(p2 & 0x02) == (((A + M + c) & 0xFF) == 0)
        if _valid_bcd(A) and _valid_bcd(M):
            n_valid += 1
            s = _dec(A) + _dec(M) + c
            assert a2 == _bcd(s % 100), (hex(A), hex(M), c, hex(a2))
            assert (p2 & 1) == (s >= 100)
    assert n_valid == 2 * 100 * 100
    # worked examples: 99 + 01 -> 00, C=1, Z=0 (binary sum $9A != 0)
    (a2, p2, _), = _run_alu(orc, 0x65, [(0x99, 0x01, 0x2C)])
    assert a2 == 0x00 and (p2 & 1) == 1 and not (p2 & 0x02)


def test_sbc_decimal_bruteforce(orc):
    # valid BCD: (dec(A) - dec(M) - (1-C)) mod 100; all flags as binary SBC (NMOS reading [R#2])
    res = _run_alu(orc, 0xE5, _cases(True))
    for (A, M, P), (a2, p2, _) in zip(_cases(True), res):
        c = P & 1
        t = A - M - (1 - c)
        r = t & 0xFF
        sv = _sx(A) - _sx(M) - (1 - c)
        assert (p2 & 1) == (t >= 0)
        assert bool(p2 & 0x40) == (sv < -128 or sv > 127)
        assert bool(p2 & 0x02) == (r == 0) and bool(p2 & 0x80) == (r >= 128)
        if _valid_bcd(A) and _valid_bcd(M):
            d = _dec(A) - _dec(M) - (1 - c)
            assert a2 == _bcd(d % 100), (hex(A), hex(M), c, hex(a2))


def test_cmp_bit_bruteforce(orc):
    cases = [(A, M, 0x24) for A in range(256) for M in range(256)]
    for (A, M, _), (a2, p2, _) in zip(cases, _run_alu(orc, 0xC5, cases)):
        assert a2 == A
        assert (p2 & 1) == (A >= M) and bool(p2 & 2) == (A == M)
        assert bool(p2 & 0x80) == bool(((A - M) & 0xFF) & 0x80)
    for (A, M, _), (a2, p2, _) in zip(cases, _run_alu(orc, 0x24, cases)):
        assert bool(p2 & 0x80) == bool(M & 0x80) and bool(p2 & 0x40) == bool(M & 0x40)
        assert bool(p2 & 2) == ((A & M) == 0)


@pytest.mark.parametrize("opcode,name", [(0x06, "ASL"), (0x46, "LSR"), (0x26, "ROL"), (0x66, "ROR"),
                                         (0xE6, "INC"), (0xC6, "DEC")])
def test_rmw_bruteforce(orc, opcode, name):
    cases = [(0x11, M, 0x24 | c) for c in (0, 1) for M in range(256)]
    for (A, M, P), (a2, p2, m2) in zip(cases, _run_alu(orc, opcode, cases)):
        c = P & 1
        if name == "ASL":
            r, cout = (M << 1) & 0xFF, M >> 7
        elif name == "LSR":
            r, cout = M >> 1, M & 1
        elif name == "ROL":
            r, cout = ((M << 1) | c) & 0xFF, M >> 7
        elif name == "ROR":
            r, cout = (M >> 1) | (c << 7), M & 1
        elif name == "INC":
            r, cout = (M + 1) & 0xFF, c
        else:
            r, cout = (M - 1) & 0xFF, c
        assert m2 == r and a2 == A
        assert (p2 & 1) == cout
        assert bool(p2 & 2) == (r == 0) and bool(p2 & 0x80) == (r >= 128)


def test_stack_roundtrip_and_php(orc):
    # push then pull restores the byte and SP; PHP pushes P|$30 and PLP ignores B/U
    rom = _rom_with({0xF000: [0x48, 0xA9, 0x00, 0x68, 0x08, 0x28]})
    for v in (0x00, 0x7F, 0x80, 0xFF):
        s = _state_for(rom, A=v)
        sp0 = int(s[3])
        orc.exec_instr(rom, s, 3)
        assert s[0] == v and s[3] == sp0
        assert bool(s[4] & 2) == (v == 0) and bool(s[4] & 0x80) == (v >= 0x80)
        orc.exec_instr(rom, s, 1)  # PHP
        assert H.ram(s, 0x100 | sp0) == (int(s[4]) | 0x30)
        orc.exec_instr(rom, s, 1)  # PLP
        assert s[3] == sp0 and (s[4] & 0x30) == 0x20


def test_jsr_rts_brk_rti(orc):
    # JSR pushes the address of its last byte; RTS adds 1; BRK pushes PC+2 and P|$30, sets I
    rom = _rom_with({0xF000: [0x20, 0x00, 0xF1], 0xF100: [0x60], 0xF200: [0x00, 0xEA],
                     0xF300: [0x40], 0xFFFE - 0xF000 + 0xF000: [0x00, 0xF3]})
    s = _state_for(rom)
    assert orc.exec_instr(rom, s, 1) == (0, 6)
    assert H.pc(s) == 0xF100 and s[3] == 0xFB
    assert H.ram(s, 0x1FD) == 0xF0 and H.ram(s, 0x1FC) == 0x02
    assert orc.exec_instr(rom, s, 1) == (0, 6)
    assert H.pc(s) == 0xF003 and s[3] == 0xFD
    s = _state_for(rom, pcv=0xF200, P=0x20 | 0x01)
    assert orc.exec_instr(rom, s, 1) == (0, 7)
    assert H.pc(s) == 0xF300 and (s[4] & 0x04)
    assert H.ram(s, 0x1FD) == 0xF2 and H.ram(s, 0x1FC) == 0x02 and H.ram(s, 0x1FB) == 0x31
    assert orc.exec_instr(rom, s, 1) == (0, 6)  # RTI
    assert H.pc(s) == 0xF202 and s[4] == 0x21 and s[3] == 0xFD


def test_undocumented_semantics(orc):
    # SURVEY.md §8(c).4 table, one representative case each (closed forms)
    def run(code, A=0, X=0, Y=0, P=0x24, ram=None):
        rom = _rom_with({0xF000: code})
        s = _state_for(rom, A=A, X=X, Y=Y, P=P, ram=ram)
        orc.exec_instr(rom, s, 1)
        return s
    s = run([0xA7, 0x85], ram={0x85: 0x9C})            # LAX zp
    assert s[0] == 0x9C and s[1] == 0x9C and s[4] & 0x80
    s = run([0x87, 0x85], A=0xF0, X=0x3C)              # SAX zp
    assert H.ram(s, 0x85) == 0x30
    s = run([0xC7, 0x85], A=0x10, ram={0x85: 0x11})    # DCP: M=$10, CMP -> Z=1 C=1
    assert H.ram(s, 0x85) == 0x10 and s[4] & 0x03 == 0x03
    s = run([0xE7, 0x85], A=0x10, P=0x25, ram={0x85: 0x0F})  # ISB: M=$10, A-M = 0
    assert H.ram(s, 0x85) == 0x10 and s[0] == 0x00 and s[4] & 0x01
    s = run([0x07, 0x85], A=0x01, ram={0x85: 0x81})    # SLO: M=$02 C=1, A=$03
    assert H.ram(s, 0x85) == 0x02 and s[0] == 0x03 and s[4] & 1
    s = run([0x27, 0x85], A=0xFF, P=0x25, ram={0x85: 0x40})  # RLA: M=$81, A=$81
    assert H.ram(s, 0x85) == 0x81 and s[0] == 0x81 and not (s[4] & 1)
    s = run([0x47, 0x85], A=0xFF, ram={0x85: 0x03})    # SRE: M=$01 C=1, A=$FE
    assert H.ram(s, 0x85) == 0x01 and s[0] == 0xFE and s[4] & 1
    s = run([0x67, 0x85], A=0x10, P=0x25, ram={0x85: 0x02})  # RRA: M=$81 C=0, A=$91
    assert H.ram(s, 0x85) == 0x81 and s[0] == 0x91
    s = run([0x0B, 0x80], A=0xC0)                      # ANC: A=$80, C=N=1
    assert s[0] == 0x80 and s[4] & 0x81 == 0x81
    s = run([0x4B, 0x03], A=0xFF)                      # ALR: A=$01, C=1
    assert s[0] == 0x01 and s[4] & 1
    s = run([0x6B, 0xFF], A=0xC0, P=0x25)              # ARR: A=$E0, C=bit6=1, V=b6^b5=0
    assert s[0] == 0xE0 and s[4] & 1 and not (s[4] & 0x40)
    s = run([0xCB, 0x10], A=0xF0, X=0x3F)              # SBX: X=(A&X)-imm = $20, C=1
    assert s[1] == 0x20 and s[4] & 1
    s = run([0xEB, 0x01], A=0x05, P=0x25)              # $EB = SBC #
    assert s[0] == 0x04


def test_addressing_wraps(orc):
    # zp,X wraps in page 0; (zp,X) pointer wraps; (zp),Y pointer high byte from (zp+1)&$FF
    def run(code, A=0, X=0, Y=0, ram=None):
        rom = _rom_with({0xF000: code})
        s = _state_for(rom, A=A, X=X, Y=Y, ram=ram)
        orc.exec_instr(rom, s, 1)
        return s
    s = run([0xB5, 0xF0], X=0x20, ram={0x90: 0x5A})        # LDA $F0,X -> $10 ... wraps to $0010?
    # $F0+$20 = $110 -> wraps to $10 = TIA read reg $0 (CXM0P) = 0
    assert s[0] == 0x00
    s = run([0xB5, 0x80], X=0x10, ram={0x90: 0x5A})        # LDA $80,X -> $90
    assert s[0] == 0x5A
    s = run([0xA1, 0xFF], X=0x00, ram={0xFF: 0xA0})        # (zp,X): ptr lo $FF, hi $00 -> $00A0
    assert s[0] == H.ram(s, 0xA0)
    s = run([0xB1, 0xFF], Y=0x01, ram={0xFF: 0x9F, 0xA0: 0x77})  # (zp),Y: ptr=$xx9F (hi from $00 TIA=0)
    assert s[0] == 0x77
