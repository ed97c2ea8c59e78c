"""Micro-programs M1-M19 with closed-form expected results.

Input generators only: each function returns 6502 source (and the ROM bytes via
`build(source)`); the expected values live in tests/, derived from the hardware definition,
not from either implementation.

Conventions shared by the frame-structured programs:
  * every frame is exactly 262 scanlines: the VSYNC 0->1 write happens 3 cycles after the
    start of a line (after `STA WSYNC`), so each frame ends with fc = 3 after rebasing;
  * the 160x210 window starts at frame line 34 (ystart), VBLANK is on for lines 0-33 only.
"""
from __future__ import annotations

from .asm6502 import EQUATES, assemble, assemble_with_symbols

_HEAD = EQUATES + """
    .org $F000
Reset:
    SEI
    CLD
    LDX #$FF
    TXS
"""

_VECTORS = """
    .org $FFFC
    .word Reset
    .word Reset
"""


def build(source: str, size: int = 4096) -> bytes:
    return assemble(source, size)


def build_sym(source: str, size: int = 4096):
    return assemble_with_symbols(source, size)


# ---------------------------------------------------------------------------------------------
# M1 frame262: VSYNC every 262 WSYNC-paced lines
# ---------------------------------------------------------------------------------------------
def m1_frame262() -> str:
    return _HEAD + """
Frame:
    LDA #2
    STA WSYNC
    STA VSYNC
    STA WSYNC
    STA WSYNC
    STA WSYNC
    LDA #0
    STA VSYNC
    LDX #0
L1: STA WSYNC
    DEX
    BNE L1
    LDX #2
L2: STA WSYNC
    DEX
    BNE L2
    JMP Frame
""" + _VECTORS


# ---------------------------------------------------------------------------------------------
# M2 colubk_rows: COLUBK = (2*line) & $FF written in HBLANK of every line
# ---------------------------------------------------------------------------------------------
def m2_colubk_rows() -> str:
    return _HEAD + """
Frame:
    LDA #2
    STA WSYNC
    STA VSYNC
    LDA #0
    STA VSYNC
    LDY #0
Loop1:
    STA WSYNC
    INY
    TYA
    ASL
    STA COLUBK
    CPY #255
    BNE Loop1
    LDY #0
Loop2:
    STA WSYNC
    TYA
    ASL
    STA COLUBK
    INY
    CPY #6
    BNE Loop2
    JMP Frame
""" + _VECTORS


# ---------------------------------------------------------------------------------------------
# Static frame builder (M3-M8, M12): registers poked during VBLANK, objects positioned by RESPx
# strobes after k NOPs, then an idle 262-line frame.
# ---------------------------------------------------------------------------------------------
def static_frame(pokes=(), positions=(), hmove=False, hmove_row0=False, store_collisions=False,
                 clear_collisions=True, extra_vblank="", kernel_row0="") -> str:
    """pokes: [(reg, value)], positions: [(resp_reg, k_nops)] one scanline each.
    hmove: strobe HMOVE at cycle 3 of the line after the positions (comb on that line).
    hmove_row0: strobe HMOVE at the start of window row 0 (frame line 34).
    store_collisions: at frame line 3 copy CXM0P..CXPPMM into RAM $F0-$F7 (previous frame).
    """
    lines = []
    cur = 3  # frame line after the VSYNC block
    grp = []
    if store_collisions:
        rd = []
        for r in range(8):
            rd.append(f"    LDA ${r:02X}\n    STA ${0xF0 + r:02X}")
        if clear_collisions:
            rd.append("    STA CXCLR")
        lines.append("\n".join(rd) + "\n    STA WSYNC")
        cur += 1
    for i, (reg, val) in enumerate(pokes):
        grp.append(f"    LDA #${val & 0xFF:02X}\n    STA ${reg:02X}")
        if len(grp) == 12:
            lines.append("\n".join(grp) + "\n    STA WSYNC")
            cur += 1
            grp = []
    if grp:
        lines.append("\n".join(grp) + "\n    STA WSYNC")
        cur += 1
    if extra_vblank:
        lines.append(extra_vblank + "\n    STA WSYNC")
        cur += 1
    for reg, k in positions:
        if not 0 <= k <= 35:
            raise ValueError("k must be in [0, 35]")
        lines.append("    NOP\n" * k + f"    STA ${reg:02X}\n    STA WSYNC")
        cur += 1
    if hmove:
        lines.append("    STA HMOVE\n    STA WSYNC")
        cur += 1
    if cur >= 34:
        raise ValueError("too many VBLANK lines")
    body = "\n".join(lines)
    row0 = ""
    if hmove_row0:
        row0 += "    STA HMOVE\n"
    row0 += kernel_row0
    return _HEAD + f"""
    JMP Frame
Frame:
    LDA #2
    STA WSYNC
    STA VSYNC
    STA VBLANK
    STA WSYNC
    STA WSYNC
    STA WSYNC
    LDA #0
    STA VSYNC
{body}
    LDX #{34 - cur}
Idle1:
    STA WSYNC
    DEX
    BNE Idle1
    LDA #0
    STA VBLANK
{row0}
    LDX #227
Idle2:
    STA WSYNC
    DEX
    BNE Idle2
    JMP Frame
""" + _VECTORS


# ---------------------------------------------------------------------------------------------
# M9 timer: TIM64T = 10 then INTIM sampled at known cycle offsets into RAM
# ---------------------------------------------------------------------------------------------
def m9_timer(value: int = 10, reg: str = "TIM64T", delays=(0, 5, 31, 60, 300, 318, 330, 700)) -> tuple[str, list[int]]:
    """Returns (source, e_list): sample j is taken by `LDA INTIM` whose bus access is e_j cycles
    after the end of the timer-write instruction.  Delays are in NOP pairs... computed exactly:
    between samples the program burns `d` cycles with a calibrated loop (5*d + 1 cycles)."""
    # Layout (cycle counts are the [HW] opcode cycle counts):
    #   LDA #v (2) ; STA TIMxx (4, abs)         -> stamp w at the end of the STA
    #   for each sample: [LDX #d (2); loop: DEX (2) BNE (3/2)] ; LDA INTIM (4) ; STA $80+j (3)
    #                   (d == 0: no loop)       ; LDA TIMINT (4) ; STA $C0+j (3)
    code = [f"    LDA #{value}", f"    STA {reg}"]
    e_list = []
    t = 0  # cycles since the stamp
    for j, d in enumerate(delays):
        chunk = 0
        while d:
            c = min(d, 255)
            code += [f"    LDX #{c}", f"Dl{j}_{chunk}:", "    DEX", f"    BNE Dl{j}_{chunk}"]
            t += 2 + 5 * c - 1
            d -= c
            chunk += 1
        code += ["    LDA INTIM", f"    STA ${0x80 + j:02X}"]
        t += 4
        e_list.append(t)
        t += 3
        code += ["    LDA TIMINT", f"    STA ${0xC0 + j:02X}"]
        t += 4
        e_list.append(t)
        t += 3
    src = _HEAD + "    JMP Start\n    .align 256\nStart:\n" + "\n".join(code) + "\nDone:\n    JMP Done\n" + _VECTORS
    return src, e_list


# ---------------------------------------------------------------------------------------------
# M10 decimal: SED ADC/SBC results + flags into RAM
# ---------------------------------------------------------------------------------------------
def m10_decimal(cases) -> str:
    """cases: [(op, a, m, carry)] with op in {'ADC','SBC'}; result j -> RAM $80+2j (A), $81+2j (P)."""
    code = []
    for j, (op, a, m, c) in enumerate(cases):
        code += ["    SED", "    SEC" if c else "    CLC", f"    LDA #${a:02X}", f"    {op} #${m:02X}",
                 f"    STA ${0x80 + 2 * j:02X}", "    PHP", "    PLA", f"    STA ${0x81 + 2 * j:02X}"]
    return _HEAD + "\n".join(code) + "\n    CLD\nDone:\n    JMP Done\n" + _VECTORS


# ---------------------------------------------------------------------------------------------
# M11 F8: same-address trampolines, bank-identifying bytes
# ---------------------------------------------------------------------------------------------
def m11_f8() -> str:
    """Bank 1 (power-on) stores its id, switches to bank 0 through a $1FF8 read, bank 0 stores
    its id and the byte read through the hotspot itself, switches back through a $1FF9 write
    (writes also switch), and bank 1 counts round trips in RAM $84."""
    return EQUATES + """
.bank 1
    .org $F000
Reset:
    SEI
    CLD
    LDX #$FF
    TXS
    LDA #0
    STA $84
Main1:
    LDA BankId
    STA $80
    JMP Tramp
Back1:
    INC $84
    LDA $84
    CMP #3
    BNE Main1
Done1:
    JMP Done1
BankId: .byte $B1
    .org $F800
Tramp:
    LDA $1FF8
    STA $81
    JMP Main0
    .org $F810
Tramp2:
    STA $1FF9
    JMP Back1
    .org $FFF8
    .byte $18, $19
    .org $FFFC
    .word Reset
    .word Reset
.bank 0
    .org $F000
Main0:
    LDA BankId0
    STA $82
    LDA $1FF8
    STA $83
    JMP Tramp2
BankId0: .byte $B0
    .org $F800
    LDA $1FF8
    STA $81
    JMP Main0
    .org $F810
    STA $1FF9
    JMP Back1
    .org $FFF8
    .byte $08, $09
    .org $FFFC
    .word Main0
    .word Main0
"""


# ---------------------------------------------------------------------------------------------
# M12 address decode: stack into TIA space, RAM mirror in the stack page
# ---------------------------------------------------------------------------------------------
def m12_stack_decode(colubk: int = 0x2A) -> str:
    extra = f"""    TSX
    STX $F8
    LDX #$09
    TXS
    LDA #${colubk:02X}
    PHA
    LDX #$85
    TXS
    LDA #$5C
    PHA
    LDX $F8
    TXS"""
    return static_frame(extra_vblank=extra)


# ---------------------------------------------------------------------------------------------
# M13 JMP ($xxFF) page-wrap bug
# ---------------------------------------------------------------------------------------------
def m13_jmp_ind() -> str:
    return EQUATES + """
    .org $F000
Reset:
    SEI
    CLD
    LDX #$FF
    TXS
    JMP ($F1FF)
Right:
    LDA #$11
    STA $80
Done:
    JMP Done
Wrong:
    LDA #$22
    STA $80
    JMP Done
    .org $F100
    .byte >Right
    .org $F1FF
    .byte <Right
    .byte >Wrong
    .org $F200
    .byte >Wrong
    .org $FFFC
    .word Reset
    .word Reset
"""


# ---------------------------------------------------------------------------------------------
# M14 JAM, M15 no VSYNC (runaway)
# ---------------------------------------------------------------------------------------------
def m14_jam(after_frames: int = 3) -> str:
    """Runs `after_frames` normal frames (counter in $80), then executes JAM ($02)."""
    return _HEAD + f"""
    LDA #0
    STA $80
Frame:
    LDA #2
    STA WSYNC
    STA VSYNC
    LDA #0
    STA VSYNC
    INC $80
    LDA $80
    CMP #{after_frames + 2}
    BNE Ok
    .byte $02
Ok:
    LDX #0
L1: STA WSYNC
    DEX
    BNE L1
    LDX #5
L2: STA WSYNC
    DEX
    BNE L2
    JMP Frame
""" + _VECTORS


def m15_no_vsync(after_frames: int = 3) -> str:
    return _HEAD + f"""
    LDA #0
    STA $80
Frame:
    LDA #2
    STA WSYNC
    STA VSYNC
    LDA #0
    STA VSYNC
    INC $80
    LDA $80
    CMP #{after_frames + 2}
    BNE Ok
Spin:
    STA WSYNC
    JMP Spin
Ok:
    LDX #0
L1: STA WSYNC
    DEX
    BNE L1
    LDX #5
L2: STA WSYNC
    DEX
    BNE L2
    JMP Frame
""" + _VECTORS


# ---------------------------------------------------------------------------------------------
# M16 inputs: SWCHA/INPT4 copied into RAM every frame
# ---------------------------------------------------------------------------------------------
def m16_inputs() -> str:
    return static_frame(extra_vblank="""    LDA SWCHA
    STA $80
    LDA INPT4
    STA $81
    LDA SWCHB
    STA $82
    LDA INPT5
    STA $83""")


# ---------------------------------------------------------------------------------------------
# M17 reward/done: BCD score +1 per frame while FIRE held; terminal at score >= 150
# ---------------------------------------------------------------------------------------------
def m17_score(terminal_at_hi: int = 0x01, terminal_at_lo: int = 0x50) -> str:
    extra = f"""    LDA INPT4
    BMI NoFire
    SED
    LDA $81
    CLC
    ADC #1
    STA $81
    LDA $80
    ADC #0
    STA $80
    CLD
NoFire:
    LDA $80
    CMP #${terminal_at_hi:02X}
    BCC NotDone
    LDA $81
    CMP #${terminal_at_lo:02X}
    BCC NotDone
    LDA #1
    STA $82
NotDone:"""
    return static_frame(extra_vblank=extra)


# ---------------------------------------------------------------------------------------------
# M18 execute from RAM
# ---------------------------------------------------------------------------------------------
def m18_ram_exec() -> str:
    """Copies `LDA #$42; STA $C0; INX; RTS` to $E0 and JSRs to it twice."""
    return _HEAD + """
    LDX #0
Copy:
    LDA Routine,X
    STA $E0,X
    INX
    CPX #6
    BNE Copy
    LDX #7
    JSR $00E0
    JSR $00E0
    STX $C1
Done:
    JMP Done
Routine:
    LDA #$42
    STA $C0
    INX
    RTS
""" + _VECTORS


# ---------------------------------------------------------------------------------------------
# M19 ALU kernels: multiply table, bubble sort, BCD counter — whole-instruction semantics
# ---------------------------------------------------------------------------------------------
def m19_alu(seed_bytes) -> str:
    """RAM $80-$8F <- sorted(seed_bytes[0:16]) (bubble sort with CMP/BCC/branches);
    RAM $90-$9F <- (a_j * b_j) & $FF, $A0-$AF <- (a_j * b_j) >> 8 with a/b from seed_bytes[16:48];
    RAM $B0.. <- the first 16 Fibonacci numbers mod 256 (ADC chain);
    RAM $C0/$C1 <- 16-bit sum of seed_bytes[0:16] (ADC carry chain)."""
    vals = list(seed_bytes)
    assert len(vals) >= 48
    f = lambda xs: ", ".join(f"${x & 0xFF:02X}" for x in xs)
    return _HEAD + f"""
    ; copy data to RAM $80-$8F
    LDX #15
Cp: LDA Data,X
    STA $80,X
    DEX
    BPL Cp
    ; 16-bit sum
    LDA #0
    STA $C0
    STA $C1
    LDX #15
Sum:
    LDA $C0
    CLC
    ADC $80,X
    STA $C0
    LDA $C1
    ADC #0
    STA $C1
    DEX
    BPL Sum
    ; bubble sort $80-$8F ascending
Outer:
    LDY #0
    LDX #0
Inner:
    LDA $80,X
    CMP $81,X
    BCC NoSwap
    BEQ NoSwap
    PHA
    LDA $81,X
    STA $80,X
    PLA
    STA $81,X
    INY
NoSwap:
    INX
    CPX #15
    BNE Inner
    CPY #0
    BNE Outer
    ; products
    LDY #15
Prod:
    LDA MulA,Y
    STA $D0
    LDA MulB,Y
    STA $D1
    LDA #0
    LDX #8
MLoop:
    LSR $D1
    BCC MNo
    CLC
    ADC $D0
MNo:
    ROR
    ROR $D2
    DEX
    BNE MLoop
    STA $A0,Y
    LDA $D2
    STA $90,Y
    DEY
    BPL Prod
    ; fibonacci
    LDA #0
    STA $B0
    LDA #1
    STA $B1
    LDX #0
Fib:
    LDA $B0,X
    CLC
    ADC $B1,X
    STA $B2,X
    INX
    CPX #14
    BNE Fib
Done:
    JMP Done
Data: .byte {f(vals[0:16])}
MulA: .byte {f(vals[16:32])}
MulB: .byte {f(vals[32:48])}
""" + _VECTORS


# ---------------------------------------------------------------------------------------------
# M20 timer polls: the RIOT polling idioms of Atari kernels (timer read + branch back), with
# timer values that vary per frame and per action, a loop whose branch crosses a page, and
# time-sensitive reads right after each loop (RAM $81-$85).  M21: a TIMINT poll that never
# exits (runaway at the line cap).  Used for engine-vs-oracle parity.
# ---------------------------------------------------------------------------------------------
def m20_timer_polls() -> str:
    return _HEAD + """
Frame:
    LDA #2
    STA WSYNC
    STA VSYNC
    STA WSYNC
    STA WSYNC
    STA WSYNC
    LDA #0
    STA VSYNC
    INC $80
    LDA $80
    AND #$1F
    ORA #1
    STA TIM8T
P1: LDA INTIM
    BNE P1
    LDA INTIM
    STA $81
    LDA $80
    AND #7
    STA TIM64T
P2: BIT TIMINT
    BPL P2
    LDA INTIM
    STA $82
    LDA #3
    STA T1024T
    LDA SWCHA
    AND #3
P3: CMP INTIM
    BNE P3
    LDX INTIM
    STX $83
    LDA $80
    STA TIM1T
P4: LDX INTIM
    BPL P4
    STX $84
    JMP Cross
    .org $F2FC
Cross:
    LDA #20
    STA TIM8T
P5: LDA INTIM
    BNE P5
    LDA INTIM
    STA $85
    LDX #150
L1: STA WSYNC
    DEX
    BNE L1
    JMP Frame
""" + _VECTORS


def m21_timint_spin(after_frames: int = 3) -> str:
    return _HEAD + f"""
    LDA #0
    STA $80
Frame:
    LDA #2
    STA WSYNC
    STA VSYNC
    LDA #0
    STA VSYNC
    INC $80
    LDA $80
    CMP #{after_frames + 2}
    BNE Ok
    LDA #9
    STA TIM8T
W:  BIT TIMINT
    BPL W
Spin:
    BIT TIMINT
    BMI Spin
Ok:
    LDA #40
    STA TIM64T
W2: LDA INTIM
    BNE W2
    LDX #200
L2: STA WSYNC
    DEX
    BNE L2
    JMP Frame
""" + _VECTORS


# ---------------------------------------------------------------------------------------------
# M22 bank-switching schemes beyond F8: F6 (4 banks, $1FF6-$1FF9)
# and F4 (8 banks, $1FF4-$1FFB), plus the mirrored 2K cartridge
# ---------------------------------------------------------------------------------------------
def m22_banks(nbanks: int) -> str:
    """Power-on runs the last bank.  Bank b stores $B0+b at RAM $80+b and switches to bank b-1
    through `LDA HS,X` (X = b-1) in a stub that sits at the same address in every bank; the
    stub's next instruction runs in the new bank and stores the byte the hotspot read returned
    (the new bank's marker 16*(b-1) + (b-1)) at RAM $90+X.  Bank 0 ends in a loop."""
    hs = {4: 0x1FF6, 8: 0x1FF4}[nbanks]
    src = [EQUATES]
    for b in range(nbanks):
        body = [f".bank {b}", "    .org $F000", f"Entry{b}:", "    SEI", "    CLD", "    LDX #$FF", "    TXS",
                f"    LDA #${0xB0 + b:02X}", f"    STA ${0x80 + b:02X}"]
        if b == 0:
            body += ["Done:", "    JMP Done"]
        else:
            body += [f"    LDX #{b - 1}", "    JMP $FF00"]
        body += ["    .org $FF00", f"    LDA ${hs:04X},X", "    STA $90,X", "    JMP $F000",
                 f"    .org ${0xF000 | (hs & 0xFFF):04X}",
                 "    .byte " + ", ".join(f"${16 * b + k:02X}" for k in range(nbanks)),
                 "    .org $FFFC", f"    .word Entry{b}", f"    .word Entry{b}"]
        src.append("\n".join(body))
    return "\n".join(src) + "\n"


def m22_2k() -> str:
    """A 2 KB cartridge answers at $1000-$17FF and again at $1800-$1FFF: the program runs at
    $F800, jumps into the mirror at $F000 + (same offset) and reads a table through both
    mirrors.  RAM $80 counts passes (2), $81/$82 hold the table byte read through $F7xx/$FFxx."""
    return EQUATES + """
    .org $F800
Reset:
    SEI
    CLD
    LDX #$FF
    TXS
    LDA #0
    STA $80
Pass:
    INC $80
    LDA $80
    CMP #2
    BCS Both
    JMP Pass - $800
Both:
    LDA Tab - $800
    STA $81
    LDA Tab
    STA $82
Done:
    JMP Done
Tab: .byte $5A
    .org $FFFC
    .word Reset
    .word Reset
"""


# ---------------------------------------------------------------------------------------------
# M23 resp_at_vsync: a visible RESP0 right before the VSYNC write on the same line, so a RESxx
# start delay (R#36) is pending at the frame boundary.  After `STA WSYNC`: LDA #2 (2),
# 20 NOPs (40), STA RESP0 ends at cycle 45 (hp = 67, player at 72), STA VSYNC at cycle 48
# (colour clock 144, pixel 76): pixels 76..79 of the player fall on the next frame's line 0.
# ---------------------------------------------------------------------------------------------
def m23_resp_at_vsync() -> str:
    return _HEAD + """
Frame:
    LDA #0
    STA VBLANK
    LDA #$FF
    STA GRP0
    LDA #$86
    STA COLUP0
    LDX #200
L1: STA WSYNC
    DEX
    BNE L1
    STA WSYNC
    LDA #2
""" + "    NOP\n" * 20 + """    STA RESP0
    STA VSYNC
    STA WSYNC
    STA WSYNC
    LDA #0
    STA VSYNC
    LDX #58
L2: STA WSYNC
    DEX
    BNE L2
    JMP Frame
""" + _VECTORS
