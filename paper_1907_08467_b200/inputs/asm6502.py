"""Two-pass 6502 assembler for the synthetic workloads (input generator only).

The paper's experiments run commercial Atari ROMs; none are
available here, so every input program is 6502 source in this repo assembled by this module
(SURVEY.md §8(d) "Synthetic inputs", BASELINE.json north_star "the inputs are 4 KB and F8
bank-switched 6502 programs that the build generates itself").

This module is an *input generator*: it holds none of the method's arithmetic (no emulation,
no TIA, no preprocessing).  Both the oracle tests and the CUDA path consume its output bytes.

Syntax (one statement per line, ';' starts a comment):
    label:                      define label at the current address
    NAME = expr                 define a constant
    .org expr                   set the current address (must not go backwards within a bank)
    .bank n                     select bank n (F8: n in {0,1}); each bank spans $F000-$FFFF
    .byte e1, e2, ...           emit bytes
    .word e1, e2, ...           emit little-endian words
    .fill count, value          emit `count` copies of `value`
    .align n                    pad with $00 up to a multiple of n
    MNEMONIC operand            an instruction

Operands: `#expr` immediate, `expr` zp/abs (zp chosen when the value is known and < $100 on the
first pass), `expr,X`, `expr,Y`, `(expr,X)`, `(expr),Y`, `(expr)` (JMP only), `A` or nothing
for accumulator/implied.  Force absolute with `a:expr`.
Expressions: decimal, $hex, %binary, 'c' chars, labels, + - * & | ^ >> <<, parentheses are not
supported inside operands (use constants); unary `<` (low byte) and `>` (high byte).
"""
from __future__ import annotations

import re

# (mnemonic, mode) -> opcode.  Modes: imp acc imm zp zpx zpy abs absx absy ind indx indy rel
_OPS: dict[str, dict[str, int]] = {}


def _def(mn: str, **modes: int) -> None:
    _OPS.setdefault(mn, {}).update(modes)


for _mn, _base in (("ORA", 0x00), ("AND", 0x20), ("EOR", 0x40), ("ADC", 0x60),
                   ("LDA", 0xA0), ("CMP", 0xC0), ("SBC", 0xE0)):
    _def(_mn, indx=_base + 0x01, zp=_base + 0x05, imm=_base + 0x09, abs=_base + 0x0D,
         indy=_base + 0x11, zpx=_base + 0x15, absy=_base + 0x19, absx=_base + 0x1D)
_def("STA", indx=0x81, zp=0x85, abs=0x8D, indy=0x91, zpx=0x95, absy=0x99, absx=0x9D)
for _mn, _base in (("ASL", 0x00), ("ROL", 0x20), ("LSR", 0x40), ("ROR", 0x60)):
    _def(_mn, zp=_base + 0x06, acc=_base + 0x0A, abs=_base + 0x0E, zpx=_base + 0x16,
         absx=_base + 0x1E)
_def("DEC", zp=0xC6, abs=0xCE, zpx=0xD6, absx=0xDE)
_def("INC", zp=0xE6, abs=0xEE, zpx=0xF6, absx=0xFE)
_def("LDX", imm=0xA2, zp=0xA6, abs=0xAE, zpy=0xB6, absy=0xBE)
_def("LDY", imm=0xA0, zp=0xA4, abs=0xAC, zpx=0xB4, absx=0xBC)
_def("STX", zp=0x86, abs=0x8E, zpy=0x96)
_def("STY", zp=0x84, abs=0x8C, zpx=0x94)
_def("CPX", imm=0xE0, zp=0xE4, abs=0xEC)
_def("CPY", imm=0xC0, zp=0xC4, abs=0xCC)
_def("BIT", zp=0x24, abs=0x2C)
_def("JMP", abs=0x4C, ind=0x6C)
_def("JSR", abs=0x20)
for _mn, _op in (("BPL", 0x10), ("BMI", 0x30), ("BVC", 0x50), ("BVS", 0x70),
                 ("BCC", 0x90), ("BCS", 0xB0), ("BNE", 0xD0), ("BEQ", 0xF0)):
    _def(_mn, rel=_op)
for _mn, _op in (("BRK", 0x00), ("PHP", 0x08), ("CLC", 0x18), ("PLP", 0x28), ("SEC", 0x38),
                 ("RTI", 0x40), ("PHA", 0x48), ("CLI", 0x58), ("RTS", 0x60), ("PLA", 0x68),
                 ("SEI", 0x78), ("DEY", 0x88), ("TXA", 0x8A), ("TYA", 0x98), ("TXS", 0x9A),
                 ("TAY", 0xA8), ("TAX", 0xAA), ("CLV", 0xB8), ("TSX", 0xBA), ("INY", 0xC8),
                 ("DEX", 0xCA), ("CLD", 0xD8), ("INX", 0xE8), ("NOP", 0xEA), ("SED", 0xF8)):
    _def(_mn, imp=_op)
# stable undocumented opcodes (used by micro-programs only)
for _mn, _base in (("SLO", 0x00), ("RLA", 0x20), ("SRE", 0x40), ("RRA", 0x60),
                   ("DCP", 0xC0), ("ISB", 0xE0)):
    _def(_mn, indx=_base + 0x03, zp=_base + 0x07, abs=_base + 0x0F, indy=_base + 0x13,
         zpx=_base + 0x17, absy=_base + 0x1B, absx=_base + 0x1F)
_def("SAX", indx=0x83, zp=0x87, abs=0x8F, zpy=0x97)
_def("LAX", indx=0xA3, zp=0xA7, abs=0xAF, indy=0xB3, zpy=0xB7, absy=0xBF)
_def("ANC", imm=0x0B)
_def("ALR", imm=0x4B)
_def("ARR", imm=0x6B)
_def("SBX", imm=0xCB)
_def("JAM", imp=0x02)
_def("NOP", imm=0x80, zp=0x04, zpx=0x14, abs=0x0C, absx=0x1C)

_SIZES = {"imp": 1, "acc": 1, "imm": 2, "zp": 2, "zpx": 2, "zpy": 2, "abs": 3, "absx": 3,
          "absy": 3, "ind": 3, "indx": 2, "indy": 2, "rel": 2}


class AsmError(Exception):
    pass


class Assembler:
    """Assemble source text into a ROM image of `size` bytes: 2048 (2K, mirrored in the 4 KB
    window), 4096, or 4096 x banks (8192 F8, 16384 F6, 32768 F4; `.bank N` selects the bank)."""

    def __init__(self, size: int = 4096):
        if size not in (2048, 4096, 8192, 16384, 32768):
            raise AsmError("ROM size must be 2048, 4096, 8192, 16384 or 32768")
        self.size = size
        self.nbanks = max(1, size // 4096)

    # -- expressions -------------------------------------------------------------------
    def _eval(self, expr: str, syms: dict[str, int], strict: bool) -> int | None:
        expr = expr.strip()
        if not expr:
            raise AsmError("empty expression")
        tokens = re.findall(r"\$[0-9A-Fa-f]+|%[01]+|\d+|'.'|[A-Za-z_.][A-Za-z0-9_.]*|>>|<<|[-+*&|^<>~]", expr)
        if "".join(tokens) != expr.replace(" ", ""):
            raise AsmError(f"bad expression {expr!r}")
        vals: list = []
        for t in tokens:
            if t.startswith("$"):
                vals.append(int(t[1:], 16))
            elif t.startswith("%"):
                vals.append(int(t[1:], 2))
            elif t[0].isdigit():
                vals.append(int(t))
            elif t.startswith("'"):
                vals.append(ord(t[1]))
            elif t[0].isalpha() or t[0] in "_.":
                if t in syms:
                    vals.append(syms[t])
                elif strict:
                    raise AsmError(f"undefined symbol {t}")
                else:
                    return None
            else:
                vals.append(t)
        # unary operators then left-to-right binary (no precedence beyond unary)
        out: list = []
        i = 0
        while i < len(vals):
            v = vals[i]
            if isinstance(v, str) and v in "<>~-" and (not out or isinstance(out[-1], str)):
                j = i + 1
                operand = vals[j]
                if isinstance(operand, str):
                    raise AsmError(f"bad unary in {expr!r}")
                if v == "<":
                    operand &= 0xFF
                elif v == ">":
                    operand = (operand >> 8) & 0xFF
                elif v == "~":
                    operand = ~operand
                else:
                    operand = -operand
                out.append(operand)
                i = j + 1
                continue
            out.append(v)
            i += 1
        acc = out[0]
        k = 1
        while k < len(out):
            op, rhs = out[k], out[k + 1]
            if op == "+":
                acc += rhs
            elif op == "-":
                acc -= rhs
            elif op == "*":
                acc *= rhs
            elif op == "&":
                acc &= rhs
            elif op == "|":
                acc |= rhs
            elif op == "^":
                acc ^= rhs
            elif op == ">>":
                acc >>= rhs
            elif op == "<<":
                acc <<= rhs
            else:
                raise AsmError(f"bad operator {op}")
            k += 2
        return acc

    # -- operand parsing -----------------------------------------------------------------
    @staticmethod
    def _split_operand(operand: str):
        s = operand.strip()
        if s == "" or s.upper() == "A":
            return "none", ""
        if s.startswith("#"):
            return "imm", s[1:]
        m = re.fullmatch(r"\((.+),\s*[Xx]\)", s)
        if m:
            return "indx", m.group(1)
        m = re.fullmatch(r"\((.+)\),\s*[Yy]", s)
        if m:
            return "indy", m.group(1)
        m = re.fullmatch(r"\((.+)\)", s)
        if m:
            return "ind", m.group(1)
        m = re.fullmatch(r"(.+),\s*([XxYy])", s)
        if m:
            return ("x" if m.group(2) in "Xx" else "y"), m.group(1)
        return "direct", s

    def _choose(self, mn: str, kind: str, expr: str, syms, strict: bool):
        modes = _OPS[mn]
        force_abs = expr.strip().startswith("a:")
        if force_abs:
            expr = expr.strip()[2:]
        if kind == "none":
            if "imp" in modes:
                return "imp", None
            if "acc" in modes:
                return "acc", None
            raise AsmError(f"{mn} needs an operand")
        if kind == "imm":
            return "imm", expr
        if kind == "indx":
            return "indx", expr
        if kind == "indy":
            return "indy", expr
        if kind == "ind":
            return "ind", expr
        if "rel" in modes:
            return "rel", expr
        val = self._eval(expr, syms, False)
        small = val is not None and 0 <= val < 0x100 and not force_abs
        if kind == "direct":
            if small and "zp" in modes:
                return "zp", expr
            return "abs", expr
        if kind == "x":
            if small and "zpx" in modes:
                return "zpx", expr
            return "absx", expr
        if kind == "y":
            if small and "zpy" in modes:
                return "zpy", expr
            return "absy", expr
        raise AsmError("bad operand")

    # -- assembly --------------------------------------------------------------------------
    def assemble(self, source: str) -> bytes:
        lines = []
        for raw in source.splitlines():
            line = raw.split(";", 1)[0].rstrip()
            if line.strip():
                lines.append(line.strip())
        syms: dict[str, int] = {}
        sizes_pass1: dict[int, str] = {}
        for pass_no in (1, 2):
            strict = pass_no == 2
            image = bytearray([0xFF] * self.size) if strict else None
            bank = self.nbanks - 1
            pc = 0xF000
            for idx, line in enumerate(lines):
                # label definitions (possibly followed by a statement)
                m = re.match(r"^([A-Za-z_.][A-Za-z0-9_.]*):\s*(.*)$", line)
                if m:
                    name = m.group(1)
                    if pass_no == 1 and name in syms:
                        raise AsmError(f"duplicate label {name}")
                    syms[name] = pc
                    line = m.group(2).strip()
                    if not line:
                        continue
                m = re.match(r"^([A-Za-z_][A-Za-z0-9_]*)\s*=\s*(.+)$", line)
                if m:
                    v = self._eval(m.group(2), syms, strict)
                    if v is not None:
                        syms[m.group(1)] = v
                    continue
                parts = line.split(None, 1)
                word = parts[0]
                rest = parts[1] if len(parts) > 1 else ""
                lw = word.lower()
                if lw == ".org":
                    pc = self._eval(rest, syms, True)
                    continue
                if lw == ".bank":
                    bank = self._eval(rest, syms, True)
                    if not 0 <= bank < self.nbanks:
                        raise AsmError(f"bad bank {bank}")
                    pc = 0xF000
                    continue
                if lw in (".byte", ".word", ".fill", ".align"):
                    args = [a for a in rest.split(",")] if rest else []
                    data: list[int] = []
                    if lw == ".byte":
                        for a in args:
                            v = self._eval(a, syms, strict)
                            data.append((v or 0) & 0xFF)
                    elif lw == ".word":
                        for a in args:
                            v = self._eval(a, syms, strict) or 0
                            data += [v & 0xFF, (v >> 8) & 0xFF]
                    elif lw == ".fill":
                        cnt = self._eval(args[0], syms, True)
                        val = self._eval(args[1], syms, True) if len(args) > 1 else 0
                        data = [val & 0xFF] * cnt
                    else:
                        n = self._eval(args[0], syms, True)
                        data = [0] * ((-pc) % n)
                    if strict:
                        self._emit(image, bank, pc, data)
                    pc += len(data)
                    continue
                mn = word.upper()
                if mn not in _OPS:
                    raise AsmError(f"line {idx}: unknown mnemonic {word}")
                kind, expr = self._split_operand(rest)
                if pass_no == 1:
                    mode, expr2 = self._choose(mn, kind, expr, syms, False)
                    sizes_pass1[idx] = mode
                else:
                    mode = sizes_pass1[idx]
                    expr2 = expr[2:] if expr.strip().startswith("a:") else expr
                    if mode in ("imp", "acc"):
                        expr2 = None
                if mode not in _OPS[mn]:
                    raise AsmError(f"line {idx}: {mn} has no mode {mode} ({line})")
                opc = _OPS[mn][mode]
                size = _SIZES[mode]
                if strict:
                    data = [opc]
                    if mode == "rel":
                        tgt = self._eval(expr2, syms, True)
                        off = tgt - (pc + 2)
                        if not -128 <= off <= 127:
                            raise AsmError(f"line {idx}: branch out of range ({line})")
                        data.append(off & 0xFF)
                    elif size == 2:
                        v = self._eval(expr2, syms, True)
                        if mode != "imm" and not 0 <= v < 0x100:
                            raise AsmError(f"line {idx}: zero-page operand out of range ({line})")
                        if mode == "imm" and not -128 <= v < 0x100:
                            raise AsmError(f"line {idx}: immediate out of range ({line})")
                        data.append(v & 0xFF)
                    elif size == 3:
                        v = self._eval(expr2, syms, True)
                        data += [v & 0xFF, (v >> 8) & 0xFF]
                    self._emit(image, bank, pc, data)
                pc += size
        self.symbols = syms
        return bytes(image)

    def _emit(self, image: bytearray, bank: int, pc: int, data: list[int]) -> None:
        for i, b in enumerate(data):
            a = pc + i
            if not 0xF000 <= a <= 0xFFFF:
                raise AsmError(f"address ${a:04X} outside the $F000-$FFFF cartridge window")
            image[(a & 0x7FF) if self.size == 2048 else bank * 4096 + (a & 0xFFF)] = b


def assemble(source: str, size: int = 4096) -> bytes:
    return Assembler(size).assemble(source)


def assemble_with_symbols(source: str, size: int = 4096):
    a = Assembler(size)
    img = a.assemble(source)
    return img, a.symbols


# TIA / RIOT register names (standard 2600 equates, [HW])
EQUATES = """
VSYNC = $00
VBLANK = $01
WSYNC = $02
RSYNC = $03
NUSIZ0 = $04
NUSIZ1 = $05
COLUP0 = $06
COLUP1 = $07
COLUPF = $08
COLUBK = $09
CTRLPF = $0A
REFP0 = $0B
REFP1 = $0C
PF0 = $0D
PF1 = $0E
PF2 = $0F
RESP0 = $10
RESP1 = $11
RESM0 = $12
RESM1 = $13
RESBL = $14
AUDC0 = $15
GRP0 = $1B
GRP1 = $1C
ENAM0 = $1D
ENAM1 = $1E
ENABL = $1F
HMP0 = $20
HMP1 = $21
HMM0 = $22
HMM1 = $23
HMBL = $24
VDELP0 = $25
VDELP1 = $26
VDELBL = $27
RESMP0 = $28
RESMP1 = $29
HMOVE = $2A
HMCLR = $2B
CXCLR = $2C
CXM0P = $00
CXM1P = $01
CXP0FB = $02
CXP1FB = $03
CXM0FB = $04
CXM1FB = $05
CXBLPF = $06
CXPPMM = $07
INPT4 = $0C
INPT5 = $0D
SWCHA = $0280
SWACNT = $0281
SWCHB = $0282
SWBCNT = $0283
INTIM = $0284
TIMINT = $0285
TIM1T = $0294
TIM8T = $0295
TIM64T = $0296
T1024T = $0297
"""
