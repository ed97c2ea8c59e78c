"""Host-side pins for the scalar engine's pre-decoded cartridge records
(paper_1907_08467_b200/csrc/scalar_predecode.h, built on the host at cule_create).

The record builder is compiled here with g++ into a tiny shared library and checked against the
published opcode matrix (tests/golden/opcode_matrix.txt: lengths, base cycles, page-cross
rules), against the bus map (which operands are RAM, cartridge, TIA or the RIOT timer), and
against the window rules that decide what the fast path may take (an instruction that crosses
the end of its 4 KB window or touches an F8 hotspot, a branch that leaves the window, a jump
outside cartridge space, a zero-page read of the TIA: all general path).  The records' run-time
semantics are covered on the GPU by the random-instruction parity tests.
"""
import ctypes
import os
import subprocess
import tempfile

import pytest

from test_oracle_cpu import parse_matrix

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1907_08467_b200", "csrc")

SHIM = r"""
#include "scalar_predecode.h"
extern "C" unsigned long long pd_one(const unsigned char* bank, unsigned o, int nbanks) {
  static uint64_t stab[256];
  static bool init = false;
  if (!init) { cule::build_scalar_table(stab); init = true; }
  return cule::predecode_one(bank, o, (uint32_t)nbanks, stab);
}
extern "C" int pd_class(const char* name) {
  // the class numbering, by name, so the test does not hard-code the enum
  struct { const char* n; int v; } t[] = {
    {"GEN", cule::C_GEN}, {"LD", cule::C_LD}, {"STTIA", cule::C_STTIA}, {"TLD", cule::C_TLD},
    {"TBIT", cule::C_TBIT}, {"TR", cule::C_TR}, {"CMP", cule::C_CMP}, {"FLAG", cule::C_FLAG},
    {"SBC", cule::C_SBC}, {"WSYNC", cule::C_WSYNC}, {"ORA", cule::C_ORA}, {"AND", cule::C_AND},
    {"EOR", cule::C_EOR}, {"ADC", cule::C_ADC}, {"BIT", cule::C_BIT}, {"LDA", cule::C_LDA},
    {"STATIA", cule::C_STATIA},
    {"STRAM", cule::C_STRAM}, {"INC", cule::C_INC}, {"DEC", cule::C_DEC}, {"ASL", cule::C_ASL},
    {"LSR", cule::C_LSR}, {"ROL", cule::C_ROL}, {"ROR", cule::C_ROR}, {"INR", cule::C_INR},
    {"ASLA", cule::C_ASLA}, {"LSRA", cule::C_LSRA}, {"ROLA", cule::C_ROLA}, {"RORA", cule::C_RORA},
    {"NOP", cule::C_NOP}, {"BR", cule::C_BR}, {"JMP", cule::C_JMP}};
  for (auto& e : t) { const char* a = e.n; const char* b = name; while (*a && *a == *b) { ++a; ++b; } if (!*a && !*b) return e.v; }
  return -1;
}
"""


@pytest.fixture(scope="module")
def pd():
    d = tempfile.mkdtemp()
    src, lib = os.path.join(d, "pd.cpp"), os.path.join(d, "libpd.so")
    with open(src, "w") as f:
        f.write(SHIM)
    subprocess.run(["g++", "-O1", "-std=c++17", "-shared", "-fPIC", "-I", CSRC, "-o", lib, src], check=True)
    L = ctypes.CDLL(lib)
    L.pd_one.argtypes = [ctypes.c_char_p, ctypes.c_uint, ctypes.c_int]
    L.pd_one.restype = ctypes.c_ulonglong
    L.pd_class.argtypes = [ctypes.c_char_p]

    class P:
        cls = {n: L.pd_class(n.encode()) for n in
               "GEN LDA STATIA LD STTIA TLD TBIT TR CMP FLAG SBC WSYNC ORA AND EOR ADC BIT STRAM INC DEC ASL LSR ROL "
               "ROR INR ASLA LSRA ROLA RORA NOP BR JMP".split()}

        @staticmethod
        def rec(code, o=0x100, f8=False, size=4096, nbanks=None):
            bank = bytearray(size)
            bank[o:o + len(code)] = bytes(code)
            v = L.pd_one(bytes(bank), o, nbanks if nbanks is not None else (2 if f8 else 1))
            lo, hi = v & 0xFFFFFFFF, v >> 32
            return dict(cls=lo & 31, aux=(lo >> 5) & 7, cyc=(lo >> 8) & 15, nxt=lo >> 20, hi=hi)
    assert all(v >= 0 for v in P.cls.values())
    return P


MODE_LEN = {"impl": 1, "A": 1, "#": 2, "z": 2, "zx": 2, "zy": 2, "r": 2, "ix": 2, "iy": 2,
            "a": 3, "ax": 3, "ay": 3, "in": 3}


def operand_for(mode):
    """Operand bytes that keep every access in RAM / the cartridge (never the TIA or RIOT)."""
    return {"z": [0x90], "zx": [0x90], "zy": [0x90], "#": [0x42], "r": [0x10], "ix": [0x90], "iy": [0x90],
            "a": [0x34, 0xF2], "ax": [0x34, 0xF2], "ay": [0x34, 0xF2], "in": [0x34, 0xF2]}.get(mode, [])


def test_lengths_cycles_and_page_cross_match_the_opcode_matrix(pd):
    m = parse_matrix()
    fast = 0
    for op, e in m.items():
        if e["fault"]:
            assert pd.rec([op])["cls"] == pd.cls["GEN"], hex(op)  # JAM / unstable: general path
            continue
        r = pd.rec([op] + operand_for(e["mode"]))
        if r["cls"] == pd.cls["GEN"]:
            continue
        fast += 1
        assert r["nxt"] == 0x100 + MODE_LEN[e["mode"]], hex(op)
        if e["branch"]:
            assert r["cls"] == pd.cls["BR"]
            assert r["cyc"] == e["base"] + 1  # taken, same page (target 0x112)
            assert r["hi"] & 0xFFF == 0x102 + 0x10
        else:
            assert r["cyc"] == e["base"], (hex(op), r["cyc"], e["base"])
        if r["cls"] not in (pd.cls["BR"], pd.cls["STTIA"], pd.cls["STATIA"], pd.cls["TLD"], pd.cls["TBIT"], pd.cls["TR"],
                            pd.cls["JMP"]):
            pen = bool(r["hi"] & 0x100)
            assert pen == (e["plus"] and e["mode"] in ("ax", "ay")), hex(op)  # (zp),Y is general path
    assert fast >= 120


def test_classes_of_common_instructions(pd):
    c = pd.cls
    assert pd.rec([0xA9, 0x12])["cls"] == c["LDA"]                         # LDA #
    assert pd.rec([0xA5, 0x85])["cls"] == c["LDA"]                         # LDA zp (RAM)
    assert pd.rec([0xA2, 0x12])["cls"] == c["LD"]                          # LDX #
    assert pd.rec([0x04, 0x85])["cls"] == c["GEN"]                         # NOP zp (read): general path
    assert pd.rec([0xA5, 0x05])["cls"] == c["GEN"]                         # LDA zp (TIA read)
    assert pd.rec([0xAD, 0x84, 0x02])["cls"] == c["TLD"]                   # LDA INTIM
    assert pd.rec([0x2C, 0x85, 0x02])["cls"] == c["TBIT"]                  # BIT TIMINT
    assert pd.rec([0xAD, 0x80, 0x02])["cls"] == c["GEN"]                   # LDA SWCHA (RIOT I/O)
    r = pd.rec([0x85, 0x1B])                                               # STA GRP0
    assert r["cls"] == c["STATIA"] and r["hi"] == 0x1B << 8
    assert pd.rec([0x86, 0x1B])["cls"] == c["STTIA"]                       # STX GRP0
    assert pd.rec([0x85, 0x02])["cls"] == c["WSYNC"]                       # STA WSYNC
    assert pd.rec([0x8D, 0x02, 0x01])["cls"] == c["WSYNC"]                 # STA $0102 (mirror)
    assert pd.rec([0x85, 0x00])["cls"] == c["GEN"]                         # STA VSYNC
    assert pd.rec([0x85, 0x15])["cls"] == c["GEN"]                         # STA AUDC0 (no picture effect)
    r = pd.rec([0x85, 0x85])                                               # STA zp RAM
    assert r["cls"] == c["STRAM"] and r["hi"] >> 31 == 1
    r = pd.rec([0xB9, 0xF0, 0x00])                                         # LDA $00F0,Y: RAM-based abs,Y
    assert r["cls"] == c["LDA"] and r["hi"] >> 31 == 1 and (r["hi"] >> 16) & 0xFFF == 0xF0
    r = pd.rec([0xB9, 0x00, 0xF3])                                         # LDA $F300,Y: cartridge table
    assert r["cls"] == c["LDA"] and r["hi"] >> 31 == 0 and (r["hi"] >> 16) & 0xFFF == 0x300
    assert pd.rec([0xB9, 0x80, 0xFF])["cls"] == c["GEN"]                   # abs,Y past the window end
    assert pd.rec([0x4C, 0x00, 0xF0])["cls"] == c["JMP"]                   # JMP $F000
    assert pd.rec([0x4C, 0x80, 0x00])["cls"] == c["GEN"]                   # JMP into RAM
    assert pd.rec([0x6C, 0x00, 0xF0])["cls"] == c["GEN"]                   # JMP (ind)
    assert pd.rec([0x20, 0x00, 0xF0])["cls"] == c["GEN"]                   # JSR
    assert pd.rec([0xE6, 0x90])["cls"] == c["INC"]                         # INC zp RAM
    assert pd.rec([0xE8])["cls"] == c["INR"] and pd.rec([0xAA])["cls"] == c["TR"]


def test_window_rules(pd):
    c = pd.cls
    assert pd.rec([0xAD, 0x84, 0x02], o=0xFFC)["cls"] == c["TLD"]           # next PC 0xFFF: fits
    assert pd.rec([0xAD, 0x84, 0x02], o=0xFFD)["cls"] == c["GEN"]           # next PC leaves the window
    assert pd.rec([0xAD, 0x84], o=0xFFE)["cls"] == c["GEN"]                 # crosses the window end
    r = pd.rec([0xEA], o=0xFFE)
    assert r["cls"] == c["NOP"] and r["nxt"] == 0xFFF
    assert pd.rec([0xEA], o=0xFFF)["cls"] == c["GEN"]                       # falls through to $x000
    assert pd.rec([0xD0, 0x7F], o=0xF80)["cls"] == c["GEN"]                 # branch target past the window
    assert pd.rec([0xD0, 0x80], o=0x010)["cls"] == c["GEN"]                 # branch target before it
    r = pd.rec([0xD0, 0xFB], o=0x105)                                      # BNE back across a page
    assert r["cls"] == c["BR"] and r["hi"] & 0xFFF == 0x102 and r["cyc"] == 3
    r = pd.rec([0xD0, 0xF0], o=0x105)                                      # target 0x0F7: page cross
    assert r["cls"] == c["BR"] and r["hi"] & 0xFFF == 0xF7 and r["cyc"] == 4
    # F8: an instruction whose bytes touch a hotspot, or a read that can reach one
    assert pd.rec([0xEA], o=0xFF8, f8=True)["cls"] == c["GEN"]
    assert pd.rec([0xAD, 0x84, 0x02], o=0xFF6, f8=True)["cls"] == c["GEN"]
    assert pd.rec([0xAD, 0x84, 0x02], o=0xFF6, f8=False)["cls"] == c["TLD"]
    assert pd.rec([0xAD, 0xF8, 0xFF], f8=True)["cls"] == c["GEN"]           # LDA $FFF8 switches banks
    assert pd.rec([0xAD, 0xF8, 0xFF], f8=False)["cls"] == c["LDA"]
    assert pd.rec([0xB9, 0x00, 0xFF], f8=True)["cls"] == c["GEN"]           # abs,Y can reach $FFF8
    # F6 ($FF6-$FF9) and F4 ($FF4-$FFB) hotspot windows
    assert pd.rec([0xEA], o=0xFF6, nbanks=4)["cls"] == c["GEN"]
    assert pd.rec([0xEA], o=0xFF6, nbanks=2)["cls"] == c["NOP"]
    assert pd.rec([0xEA], o=0xFF4, nbanks=8)["cls"] == c["GEN"]
    assert pd.rec([0xEA], o=0xFFB, nbanks=8)["cls"] == c["GEN"]
    assert pd.rec([0xEA], o=0xFFA, nbanks=4)["cls"] == c["NOP"]
    assert pd.rec([0xAD, 0xF6, 0xFF], nbanks=4)["cls"] == c["GEN"]        # LDA $FFF6 switches (F6)
    assert pd.rec([0xAD, 0xF5, 0xFF], nbanks=4)["cls"] == c["LDA"]
    assert pd.rec([0xAD, 0xFB, 0xFF], nbanks=8)["cls"] == c["GEN"]        # LDA $FFFB switches (F4)
    assert pd.rec([0xB9, 0x00, 0xFF], nbanks=8)["cls"] == c["GEN"]        # abs,Y can reach $FFF4
    assert pd.rec([0xB9, 0x00, 0xFF], nbanks=1)["cls"] == c["LDA"]
    assert pd.rec([0xB9, 0xF0, 0xFE], nbanks=8)["cls"] == c["LDA"]        # ends at $FFEF: clear
