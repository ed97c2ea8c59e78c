"""Mutation check for the oracle's pins (VERDICT r01 "Next round" item 1: "mutating any one of the
collision-bit map, decimal N/V, missile copies or the canonical timer stamp turns a CPU test red").

Test infrastructure (not collected by pytest: the file name does not start with test_).  For each
mutation below it copies the repo to a scratch directory, applies one textual edit to
oracle/cule_oracle.c, rebuilds the oracle there and runs the oracle's CPU pin tests.  A mutation
that leaves every test green is a hole in the pins and is reported as SURVIVED.

    python tests/mutation_check.py [-k substring]
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "oracle/cule_oracle.c"
TESTS = ["tests/test_oracle_pins.py", "tests/test_oracle_tia.py", "tests/test_oracle_cpu.py",
         "tests/test_oracle_riot_cart.py"]

# (name, old text, new text): each old text must occur exactly once in the oracle
MUTATIONS = [
    # collision-pair -> read-register bit map (§8(c).8 read table)
    ("cx_M0P_swap", "if (m0 && p1) m->coll |= 1u << 0;\n  if (m0 && p0) m->coll |= 1u << 1;",
     "if (m0 && p1) m->coll |= 1u << 1;\n  if (m0 && p0) m->coll |= 1u << 0;"),
    ("cx_M1P_swap", "if (m1 && p0) m->coll |= 1u << 2;\n  if (m1 && p1) m->coll |= 1u << 3;",
     "if (m1 && p0) m->coll |= 1u << 3;\n  if (m1 && p1) m->coll |= 1u << 2;"),
    ("cx_P0FB_swap", "if (p0 && pf) m->coll |= 1u << 4;\n  if (p0 && bl) m->coll |= 1u << 5;",
     "if (p0 && pf) m->coll |= 1u << 5;\n  if (p0 && bl) m->coll |= 1u << 4;"),
    ("cx_P1FB_swap", "if (p1 && pf) m->coll |= 1u << 6;\n  if (p1 && bl) m->coll |= 1u << 7;",
     "if (p1 && pf) m->coll |= 1u << 7;\n  if (p1 && bl) m->coll |= 1u << 6;"),
    ("cx_M0FB_swap", "if (m0 && pf) m->coll |= 1u << 8;\n  if (m0 && bl) m->coll |= 1u << 9;",
     "if (m0 && pf) m->coll |= 1u << 9;\n  if (m0 && bl) m->coll |= 1u << 8;"),
    ("cx_M1FB_swap", "if (m1 && pf) m->coll |= 1u << 10;\n  if (m1 && bl) m->coll |= 1u << 11;",
     "if (m1 && pf) m->coll |= 1u << 11;\n  if (m1 && bl) m->coll |= 1u << 10;"),
    ("cx_BLPF_bit", "if (bl && pf) m->coll |= 1u << 12;", "if (bl && pf) m->coll |= 1u << 13;"),
    ("cx_PPMM_swap", "if (p0 && p1) m->coll |= 1u << 14;\n  if (m0 && m1) m->coll |= 1u << 15;",
     "if (p0 && p1) m->coll |= 1u << 15;\n  if (m0 && m1) m->coll |= 1u << 14;"),
    ("cx_P1M1_pair", "if (m1 && p1) m->coll |= 1u << 3;", "if (m1 && p0) m->coll |= 1u << 3;"),
    # decimal ADC N / V (NMOS reading R#2)
    ("dec_N_after_adjust", "setf(m, FN, s & 0x80);", "setf(m, FN, (s >= 0xA0 ? s + 0x60 : s) & 0x80);"),
    ("dec_V_binary", "setf(m, FV, sa < -128 || sa > 127);",
     "setf(m, FV, (~(m->A ^ v)) & (m->A ^ bin) & 0x80);"),
    ("dec_V_zero", "setf(m, FV, sa < -128 || sa > 127);", "setf(m, FV, 0);"),
    ("dec_Z_decimal", "setf(m, FZ, bin == 0);", "setf(m, FZ, (uint8_t)s == 0);"),
    # missile copies and width
    # (dropping mode 5 or 7 from the single-copy test is an equivalent mutant: the player's table
    #  already has one copy in those modes)
    ("missile_player_scale", "if (mod160(x - pos - off[k]) < width) return 1;",
     "if (mod160(x - pos - off[k]) < width * nusiz_scale(mode)) return 1;"),
    ("missile_width", "int width = 1 << ((nusiz >> 4) & 3);", "int width = 1 << ((nusiz >> 4) & 1);"),
    ("missile_no_copies", "else n = nusiz_offsets(mode, off);", "else { off[0] = 0; n = 1; }"),
    # canonical timer stamp at the frame end (§8(c).5)
    ("stamp_mod255", "int64_t d = (e - VI - 1) % 256;", "int64_t d = (e - VI - 1) % 255;"),
    ("stamp_off_by_one", "m->timer_w = (int32_t)((int64_t)m->fc - (VI + 1 + d));",
     "m->timer_w = (int32_t)((int64_t)m->fc - (VI + d));"),
    ("stamp_not_canonical", "  if (e > VI) {\n    int64_t d", "  if (0) {\n    int64_t d"),
    ("stamp_no_rebase", "m->timer_w -= (int32_t)(76 * L);", "m->timer_w -= (int32_t)(76 * L - 1);"),
    # HMOVE / VDELBL / RESMP
    ("hmove_m0_uses_m1", "d = m->hmm0 >= 8 ? m->hmm0 - 16 : m->hmm0;", "d = m->hmm1 >= 8 ? m->hmm1 - 16 : m->hmm1;"),
    ("hmove_bl_uses_m1", "d = m->hmbl >= 8 ? m->hmbl - 16 : m->hmbl;", "d = m->hmm1 >= 8 ? m->hmm1 - 16 : m->hmm1;"),
    ("vdelbl_swapped", "int en = m->vdelbl ? m->enablold : m->enablnew;",
     "int en = m->vdelbl ? m->enablnew : m->enablold;"),
    ("resmp_mode5", "int c = mode == 5 ? 6 : (mode == 7 ? 10 : 3);", "int c = mode == 5 ? 3 : (mode == 7 ? 10 : 3);"),
    ("resmp_mode7", "int c = mode == 5 ? 6 : (mode == 7 ? 10 : 3);", "int c = mode == 5 ? 6 : (mode == 7 ? 6 : 3);"),
    # R#4: (zp,X) pointer reads sample at the instruction start
    ("r4_indx_at_end", "#define RD_INDX(N, BODY) { uint16_t ea = am_indx(m); begin(m, N);",
     "#define RD_INDX(N, BODY) { begin(m, N); uint16_t ea = am_indx(m);"),
]


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("-k", default="")
    args = ap.parse_args()
    text = open(os.path.join(ROOT, SRC)).read()
    survived = []
    for name, old, new in MUTATIONS:
        if args.k not in name:
            continue
        if text.count(old) != 1:
            print(f"{name}: pattern found {text.count(old)} times", flush=True)
            survived.append(name)
            continue
        with tempfile.TemporaryDirectory() as tmp:
            dst = os.path.join(tmp, "repo")
            shutil.copytree(ROOT, dst, ignore=shutil.ignore_patterns(
                ".git", "gpurun_out", "*.so", "__pycache__", ".pytest_cache", "profiles"))
            with open(os.path.join(dst, SRC), "w") as f:
                f.write(text.replace(old, new))
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider"]
                               + TESTS, cwd=dst, capture_output=True, text=True)
            killed = r.returncode != 0
            print(f"{name}: {'killed' if killed else 'SURVIVED'}", flush=True)
            if not killed:
                survived.append(name)
    print("survived:", survived)
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
