"""Synthetic game ROMs R1-R4 (SURVEY.md §8(d) "Synthetic inputs").

The paper benchmarks 57 commercial Atari games, which are not
available here.  These programs reproduce the structure that matters for the hot path:
an NTSC frame (3 VSYNC + 37 VBLANK + 192 kernel + 30 overscan lines, timer-polled blanking),
a WSYNC-paced playfield/sprite kernel with mid-line TIA writes, joystick-driven game logic,
a BCD score at fixed RAM ($80/$81, reward), a terminal flag ($82 bit 0) and a game-over loop.

    R1  "playfield"   4 KB   1-line PF + 2 sprites kernel, BCD score on overlap, LFSR hazards
    R2  "f8"          8 KB   R1 logic in bank 1, kernel in bank 0, >= 2 bank switches / frame
    R3  "collide"     4 KB   2 players + 2 missiles + ball, scores from collision latches
    R4  "heavy"       4 KB   R1 plus heavy per-frame logic (8-bit multiply, insertion sort)
                             and a kernel that computes instead of idling in WSYNC

Every ROM is deterministic in its generator seed (table contents, initial LFSR).  The
generator is an input tool: it holds none of the emulator's arithmetic.
"""
from __future__ import annotations

import hashlib
import random

from .asm6502 import EQUATES, assemble_with_symbols

SCORE_ADDR = 0x80
TERM_ADDR = 0x82
TERM_MASK = 0x01

_RAM = """
SCOREH = $80
SCOREL = $81
FLAGS = $82
LIVES = $83
PX = $84
PY = $85
LFSR = $86
EX = $87
EY = $88
SCROLL = $89
FRAME = $8A
TMP = $8B
PCOL = $8C
TMP2 = $8D
HAZ = $8E
ECOL = $8F
SORTBUF = $90
MULA = $98
MULB = $99
PRODL = $9A
PRODH = $9B
CHK = $9C
MX = $9D
MY = $9E
BX = $9F
"""

SPRITE_H = 10


def _tables(rng: random.Random, n: int = 16) -> str:
    """PF0/PF1/PF2/colour tables (16 rows each) and the sprite shapes."""
    pf0 = [rng.randrange(256) & 0xF0 for _ in range(n)]
    pf1 = [rng.randrange(256) for _ in range(n)]
    pf2 = [rng.randrange(256) for _ in range(n)]
    col = [(rng.randrange(16) << 4) | (rng.randrange(4, 8) << 1) for _ in range(n)]
    spr = [0x18, 0x3C, 0x7E, 0xDB, 0xFF, 0xFF, 0x24, 0x5A, 0x81, 0x42]
    ene = [0x81, 0x42, 0x3C, 0x5A, 0xFF, 0xFF, 0x5A, 0x3C, 0x42, 0x81]
    f = lambda xs: ", ".join(f"${x:02X}" for x in xs)
    return f"""
PF0Tab: .byte {f(pf0)}
PF1Tab: .byte {f(pf1)}
PF2Tab: .byte {f(pf2)}
ColTab: .byte {f(col)}
Sprite: .byte {f(spr)}
Enemy:  .byte {f(ene)}
"""


# -- shared assembly fragments -------------------------------------------------------------

def _init(rng: random.Random) -> str:
    lfsr = rng.randrange(1, 256)
    return f"""
Reset:
    SEI
    CLD
    LDX #$FF
    TXS
    LDA #0
    LDX #$7F
ClearRam:
    STA $80,X
    DEX
    BPL ClearRam
    LDA #9
    STA LIVES
    LDA #${lfsr:02X}
    STA LFSR
    LDA #76
    STA PX
    LDA #40
    STA PY
    LDA #20
    STA EX
    LDA #10
    STA EY
    LDA #$1E
    STA PCOL
    LDA #$46
    STA ECOL
"""


# game logic executed during VBLANK; ends with RTS
_LOGIC = f"""
GameLogic:
    INC FRAME
    LDA FLAGS
    AND #1
    BEQ Alive
    ; game over: keep producing frames, cycle the background
    INC SCROLL
    RTS
Alive:
    LDA SWCHA
    ASL
    BCS NoRight
    INC PX
NoRight:
    ASL
    BCS NoLeft
    DEC PX
NoLeft:
    ASL
    BCS NoDown
    INC PY
NoDown:
    ASL
    BCS NoUp
    DEC PY
NoUp:
    ; clamp PX to [8, 150] and PY to [0, 85]
    LDA PX
    CMP #8
    BCS PxLoOk
    LDA #8
PxLoOk:
    CMP #151
    BCC PxHiOk
    LDA #150
PxHiOk:
    STA PX
    LDA PY
    CMP #200
    BCC PyNotNeg
    LDA #0
PyNotNeg:
    CMP #86
    BCC PyOk
    LDA #85
PyOk:
    STA PY
    ; fire scrolls the playfield and stirs the LFSR
    LDA INPT4
    BMI NoFire
    INC SCROLL
    LDA LFSR
    EOR FRAME
    STA LFSR
NoFire:
    ; Galois LFSR step (taps $B8); never let it stick at zero
    LDA LFSR
    LSR
    BCC NoTap
    EOR #$B8
NoTap:
    BNE LfsrOk
    LDA #1
LfsrOk:
    STA LFSR
    ; enemy drifts by (LFSR & 3) - 1 horizontally, 1 line down every 4 frames
    AND #3
    CLC
    ADC EX
    SEC
    SBC #1
    CMP #150
    BCC ExOk
    LDA #20
ExOk:
    STA EX
    LDA FRAME
    AND #3
    BNE NoEy
    INC EY
    LDA EY
    CMP #86
    BCC NoEy
    LDA #0
    STA EY
NoEy:
    ; overlap: |PX - EX| < 8 and |PY - EY| < {SPRITE_H} -> score +1 (BCD), respawn enemy
    LDA PX
    SEC
    SBC EX
    BCS DxPos
    EOR #$FF
    ADC #1
DxPos:
    CMP #8
    BCS NoHit
    LDA PY
    SEC
    SBC EY
    BCS DyPos
    EOR #$FF
    ADC #1
DyPos:
    CMP #{SPRITE_H}
    BCS NoHit
    SED
    LDA SCOREL
    CLC
    ADC #1
    STA SCOREL
    LDA SCOREH
    ADC #0
    STA SCOREH
    CLD
    LDA LFSR
    AND #$7F
    ADC #10
    STA EX
    LDA #0
    STA EY
NoHit:
    ; hazard: LFSR < 3 costs a life; no lives left -> terminal flag
    LDA LFSR
    CMP #3
    BCS NoHaz
    DEC LIVES
    BNE NoHaz
    LDA FLAGS
    ORA #1
    STA FLAGS
NoHaz:
    RTS

; A = x position, X = object (0 = P0, 1 = P1, 2 = M0, 3 = M1, 4 = BL)
PosObject:
    STA WSYNC
    SEC
Div15:
    SBC #15
    BCS Div15
    EOR #7
    ASL
    ASL
    ASL
    ASL
    STA HMP0,X
    STA RESP0,X
    RTS
"""

# VSYNC + start of VBLANK, timer set for the VBLANK period
_VSYNC = """
    LDA #2
    STA WSYNC
    STA VSYNC
    STA VBLANK
    STA WSYNC
    STA WSYNC
    STA WSYNC
    LDA #0
    STA VSYNC
    LDA #43
    STA TIM64T
"""

_POSITION = """
    LDA PX
    LDX #0
    JSR PosObject
    LDA EX
    LDX #1
    JSR PosObject
    STA WSYNC
    STA HMOVE
    LDA PCOL
    STA COLUP0
    LDA ECOL
    STA COLUP1
"""

_WAIT_VBLANK = """
WaitVBlank:
    LDA INTIM
    BNE WaitVBlank
    STA WSYNC
    LDA #0
    STA VBLANK
"""

_WAIT_VBLANK_TIMINT = """
WaitVBlank:
    BIT TIMINT
    BPL WaitVBlank
    STA WSYNC
    LDA #0
    STA VBLANK
"""

# 2-line kernel, 96 iterations = 192 lines: line A playfield from tables, line B sprites
_KERNEL = f"""
    LDX #0
Kernel:
    STA WSYNC
    TXA
    CLC
    ADC SCROLL
    LSR
    LSR
    AND #15
    TAY
    LDA PF0Tab,Y
    STA PF0
    LDA PF1Tab,Y
    STA PF1
    LDA PF2Tab,Y
    STA PF2
    LDA ColTab,Y
    STA COLUPF
    STA WSYNC
    TXA
    SEC
    SBC PY
    CMP #{SPRITE_H}
    BCC DrawP
    LDA #0
    BEQ StoreP
DrawP:
    TAY
    LDA Sprite,Y
StoreP:
    STA GRP0
    TXA
    SEC
    SBC EY
    CMP #{SPRITE_H}
    BCC DrawE
    LDA #0
    BEQ StoreE
DrawE:
    TAY
    LDA Enemy,Y
StoreE:
    STA GRP1
    INX
    CPX #96
    BNE Kernel
"""

_OVERSCAN = """
    STA WSYNC
    LDA #2
    STA VBLANK
    LDA #0
    STA GRP0
    STA GRP1
    STA PF0
    STA PF1
    STA PF2
    LDA #35
    STA TIM64T
WaitOverscan:
    LDA INTIM
    BNE WaitOverscan
"""

_VECTORS = """
    .org $FFFC
    .word Reset
    .word Reset
"""


def _source_r1(seed: int) -> str:
    rng = random.Random(seed)
    tables = _tables(rng)
    return EQUATES + _RAM + "    .org $F000\n" + _init(rng) + "MainLoop:\n" + _VSYNC + \
        "    JSR GameLogic\n" + _POSITION + _WAIT_VBLANK + _KERNEL + _OVERSCAN + \
        "    JMP MainLoop\n" + _LOGIC + tables + _VECTORS


def _source_r2(seed: int) -> str:
    """F8: bank 1 (power-on bank) holds reset + logic, bank 0 holds the kernel.  Trampolines at
    identical addresses in both banks switch through the $1FF8/$1FF9 hotspots."""
    rng = random.Random(seed)
    tables = _tables(rng)
    # trampoline block placed at $FF00 in both banks:
    #   ToBank0: LDA $1FF8 (switch) ; execution continues in bank 0 at the next address
    tramp = """
    .org $FF00
ToKernel:
    NOP $1FF8
    JMP KernelEntry
ToLogic:
    NOP $1FF9
    JMP LogicEntry
"""
    bank1 = ".bank 1\n    .org $F000\n" + _init(rng) + "LogicEntry:\nMainLoop:\n" + _VSYNC + \
        "    JSR GameLogic\n" + _POSITION + "    JMP ToKernel\n" + _LOGIC + tramp + _VECTORS
    bank0 = ".bank 0\n    .org $F000\nKernelEntry:\n" + _WAIT_VBLANK + _KERNEL + _OVERSCAN + \
        "    JMP ToLogic\n" + tables + \
        "\n    .org $FF00\n    NOP $1FF8\n    JMP KernelEntry\n    NOP $1FF9\n    JMP LogicEntry\n" + \
        "    .org $FFFC\n    .word ToLogic\n    .word ToLogic\n"
    return EQUATES + _RAM + bank1 + bank0


def _source_r3(seed: int) -> str:
    """Two players, two missiles and a ball; the score comes from collision latches."""
    rng = random.Random(seed)
    tables = _tables(rng)
    logic3 = """
Logic3:
    ; read last frame's collisions: P0 with BL or PF, M0 with P1
    BIT CXP0FB
    BVC NoBallHit
    SED
    LDA SCOREL
    CLC
    ADC #1
    STA SCOREL
    LDA SCOREH
    ADC #0
    STA SCOREH
    CLD
NoBallHit:
    BIT CXM0P
    BPL NoMisHit
    SED
    LDA SCOREL
    CLC
    ADC #5
    STA SCOREL
    LDA SCOREH
    ADC #0
    STA SCOREH
    CLD
NoMisHit:
    BIT CXP1FB
    BPL NoPfHit
    LDA LFSR
    CMP #40
    BCS NoPfHit
    DEC LIVES
    BNE NoPfHit
    LDA FLAGS
    ORA #1
    STA FLAGS
NoPfHit:
    STA CXCLR
    ; missile and ball motion
    LDA MX
    CLC
    ADC #3
    CMP #155
    BCC MxOk
    LDA PX
MxOk:
    STA MX
    LDA BX
    SEC
    SBC #1
    BCS BxOk
    LDA #150
BxOk:
    STA BX
    LDA #$25
    STA NUSIZ0
    LDA #$13
    STA NUSIZ1
    LDA #$21
    STA CTRLPF
    RTS
"""
    position3 = """
    LDA PX
    LDX #0
    JSR PosObject
    LDA EX
    LDX #1
    JSR PosObject
    LDA MX
    LDX #2
    JSR PosObject
    LDA EX
    LDX #3
    JSR PosObject
    LDA BX
    LDX #4
    JSR PosObject
    STA WSYNC
    STA HMOVE
    LDA PCOL
    STA COLUP0
    LDA ECOL
    STA COLUP1
"""
    kernel3 = f"""
    LDX #0
Kernel:
    STA WSYNC
    TXA
    CLC
    ADC SCROLL
    LSR
    LSR
    LSR
    AND #15
    TAY
    LDA PF1Tab,Y
    AND #$81
    STA PF1
    LDA ColTab,Y
    STA COLUPF
    TXA
    SEC
    SBC MY
    CMP #4
    LDA #0
    ROL
    EOR #1
    ASL
    STA ENAM0
    STA ENAM1
    TXA
    AND #8
    LSR
    LSR
    STA ENABL
    STA WSYNC
    TXA
    SEC
    SBC PY
    CMP #{SPRITE_H}
    BCC DrawP
    LDA #0
    BEQ StoreP
DrawP:
    TAY
    LDA Sprite,Y
StoreP:
    STA GRP0
    TXA
    SEC
    SBC EY
    CMP #{SPRITE_H}
    BCC DrawE
    LDA #0
    BEQ StoreE
DrawE:
    TAY
    LDA Enemy,Y
StoreE:
    STA GRP1
    INX
    CPX #96
    BNE Kernel
"""
    return EQUATES + _RAM + "    .org $F000\n" + _init(rng) + \
        "    LDA #30\n    STA MX\n    LDA #50\n    STA MY\n    LDA #120\n    STA BX\n" + \
        "MainLoop:\n" + _VSYNC + "    JSR GameLogic\n    JSR Logic3\n" + position3 + \
        _WAIT_VBLANK + kernel3 + _OVERSCAN + "    JMP MainLoop\n" + _LOGIC + logic3 + \
        tables + _VECTORS


def _source_r4(seed: int) -> str:
    """Heavy per-frame logic: an 8-bit shift-add multiply and an insertion sort of 8 RAM bytes
    in VBLANK, and a kernel that folds a checksum every line instead of idling in WSYNC."""
    rng = random.Random(seed)
    tables = _tables(rng)
    heavy = """
Heavy:
    ; refill the sort buffer from the LFSR stream
    LDX #7
    LDA LFSR
Fill:
    ASL
    BCC NoT
    EOR #$1D
NoT:
    STA SORTBUF,X
    DEX
    BPL Fill
    ; insertion sort SORTBUF[0..7] ascending
    LDX #1
SortOuter:
    LDA SORTBUF,X
    STA TMP
    TXA
    TAY
SortInner:
    DEY
    BMI SortPlace
    LDA SORTBUF,Y
    CMP TMP
    BCC SortPlace
    BEQ SortPlace
    STA SORTBUF+1,Y
    JMP SortInner
SortPlace:
    LDA TMP
    STA SORTBUF+1,Y
    INX
    CPX #8
    BNE SortOuter
    ; PROD = SORTBUF[7] * SORTBUF[0] (shift-add)
    LDA SORTBUF+7
    STA MULA
    LDA SORTBUF
    STA MULB
    LDA #0
    STA PRODH
    LDX #8
MulLoop:
    LSR MULB
    BCC MulNoAdd
    CLC
    ADC MULA
MulNoAdd:
    ROR
    ROR PRODL
    DEX
    BNE MulLoop
    STA PRODH
    EOR CHK
    STA CHK
    RTS
"""
    kernel4 = f"""
    LDX #0
Kernel:
    STA WSYNC
    TXA
    CLC
    ADC SCROLL
    LSR
    LSR
    AND #15
    TAY
    LDA PF0Tab,Y
    STA PF0
    LDA PF1Tab,Y
    STA PF1
    LDA PF2Tab,Y
    STA PF2
    LDA ColTab,Y
    STA COLUPF
    ; fold a checksum over the line (busy work instead of idling in WSYNC)
    LDA CHK
    ASL
    ADC PF1Tab,Y
    EOR PRODL
    ROL
    ADC #7
    EOR PRODH
    STA CHK
    STA WSYNC
    TXA
    SEC
    SBC PY
    CMP #{SPRITE_H}
    BCC DrawP
    LDA #0
    BEQ StoreP
DrawP:
    TAY
    LDA Sprite,Y
StoreP:
    STA GRP0
    TXA
    SEC
    SBC EY
    CMP #{SPRITE_H}
    BCC DrawE
    LDA #0
    BEQ StoreE
DrawE:
    TAY
    LDA Enemy,Y
StoreE:
    STA GRP1
    LDA CHK
    EOR FRAME
    LSR
    ADC SORTBUF,X
    LDA CHK
    ADC SORTBUF+1
    EOR Sprite,X
    STA CHK
    INX
    CPX #96
    BNE Kernel
"""
    overscan4 = """
    STA WSYNC
    LDA #2
    STA VBLANK
    LDA #0
    STA GRP0
    STA GRP1
    STA PF0
    STA PF1
    STA PF2
    LDA #35
    STA TIM64T
    JSR Heavy
WaitOverscan:
    BIT TIMINT
    BPL WaitOverscan
"""
    return EQUATES + _RAM + "    .org $F000\n" + _init(rng) + "MainLoop:\n" + _VSYNC + \
        "    JSR GameLogic\n    JSR Heavy\n    JSR Heavy\n" + _POSITION + _WAIT_VBLANK_TIMINT + \
        kernel4 + overscan4 + "    JMP MainLoop\n" + _LOGIC + heavy + tables + _VECTORS


_BUILDERS = {"R1": (_source_r1, 4096, 1), "R2": (_source_r2, 8192, 2),
             "R3": (_source_r3, 4096, 3), "R4": (_source_r4, 4096, 4)}


def build_rom(name: str, seed: int | None = None) -> bytes:
    """Assemble game ROM `name` in {R1, R2, R3, R4} (default seeds 1..4)."""
    fn, size, default_seed = _BUILDERS[name]
    img, _ = assemble_with_symbols(fn(default_seed if seed is None else seed), size)
    return img


def rom_meta(name: str, seed: int | None = None) -> dict:
    rom = build_rom(name, seed)
    return {"name": name, "size": len(rom), "sha256": hashlib.sha256(rom).hexdigest(),
            "score_addr": SCORE_ADDR, "term_addr": TERM_ADDR, "term_mask": TERM_MASK}


def game_source(name: str, seed: int | None = None) -> str:
    fn, _, default_seed = _BUILDERS[name]
    return fn(default_seed if seed is None else seed)
